# round-2 validation: smoke, full GPU suite, bench lines, r08 profiles
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke8.log
timeout 900 python bench.py > gpurun_out/bench8_default.log 2>&1; echo rc=$? >> gpurun_out/bench8_default.log
for c in ns2d_1024 ns2d_4096 ns3d_128; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench8_$c.log 2>&1; echo rc=$? >> gpurun_out/bench8_$c.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench8_ref.log 2>&1; echo rc=$? >> gpurun_out/bench8_ref.log
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest8.log 2>&1; echo rc=$? >> gpurun_out/pytest8.log
timeout 2000 bash tools/profile_round.sh r08 ns3d_512 ns2d_1024 ns2d_4096 > gpurun_out/prof8.log 2>&1
