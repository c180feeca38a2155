# pencil (2x4, all parts on one GPU) with the final kernels
mkdir -p gpurun_out
timeout 600 python bench.py --config ns3d_512 --decomp pencil --grid 2x4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench26_pencil_2x4.log 2>&1; echo rc=$? >> gpurun_out/bench26_pencil_2x4.log
timeout 600 python bench.py --config ns3d_512 --decomp pencil --grid 2x2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench26_pencil_2x2.log 2>&1; echo rc=$? >> gpurun_out/bench26_pencil_2x2.log
