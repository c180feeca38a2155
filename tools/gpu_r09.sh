# re-entry validation of HEAD: smoke, full GPU suite with timing, all bench configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke9.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke9.log
( time timeout 1800 python -m pytest tests -m gpu -x -q --durations=20 ) > gpurun_out/pytest9.log 2>&1; echo rc=$? >> gpurun_out/pytest9.log
timeout 900 python bench.py > gpurun_out/bench9_default.log 2>&1; echo rc=$? >> gpurun_out/bench9_default.log
for c in ns2d_1024 ns2d_4096 ns3d_128; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench9_$c.log 2>&1; echo rc=$? >> gpurun_out/bench9_$c.log
done
