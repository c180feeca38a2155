# pencil: 512^3 real-split test, emulated pencil / slab bench lines on one GPU
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pencil.py -x -q -m gpu --durations=5 > gpurun_out/pytest10.log 2>&1; echo rc=$? >> gpurun_out/pytest10.log
for g in 2x2 2x4 1x8; do
timeout 600 python bench.py --config ns3d_512 --decomp pencil --grid $g --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench10_pencil_$g.log 2>&1; echo rc=$? >> gpurun_out/bench10_pencil_$g.log
done
timeout 600 python bench.py --config ns3d_128 --decomp pencil --grid 2x4 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench10_pencil128_2x4.log 2>&1; echo rc=$? >> gpurun_out/bench10_pencil128_2x4.log
