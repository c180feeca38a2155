# Round-2 baseline session: smoke, bench (default ns3d_512 + ns2d configs), GPU test suite.
set -x
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc) > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_512.log 2>&1; echo rc=$? >> gpurun_out/bench_512.log
for c in ns2d_4096 ns2d_1024 ns3d_128; do
timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo rc=$? >> gpurun_out/bench_$c.log
done
timeout 1800 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/pytest.log 2>&1; echo rc=$? >> gpurun_out/pytest.log
