# One GPU session: box info, smoke, bench (ours + reference arm), the GPU test suite.
# Outputs under gpurun_out/ (merged back by gpurun).
set -x
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=40 > gpurun_out/pytest.log 2>&1; echo rc=$? >> gpurun_out/pytest.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
