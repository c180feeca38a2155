# round-2 final validation: smoke, full GPU suite, every bench config, reference arm, r22 profiles of 512^3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke22.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke18.log
timeout 900 python bench.py > gpurun_out/bench22_default.log 2>&1; echo rc=$? >> gpurun_out/bench22_default.log
for c in ns2d_1024 ns2d_4096 ns3d_128; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench22_$c.log 2>&1; echo rc=$? >> gpurun_out/bench22_$c.log
done
timeout 900 python bench.py --config ns3d_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench22_ns3d_1024.log 2>&1; echo rc=$? >> gpurun_out/bench22_ns3d_1024.log
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=12 ) > gpurun_out/pytest22.log 2>&1; echo rc=$? >> gpurun_out/pytest18.log
timeout 2000 bash tools/profile_round.sh r22 ns3d_512 > gpurun_out/prof22.log 2>&1
