# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py
# on the GPU box; logs under gpurun_out/sanitize/ (summaries copied to profiles/).
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in ns2d_32 ns2d_64 ns2d_64_w2_p2p ns2d_64_w4 ns3d_16 ns3d_32_w2_p2p ns3d_32_w4; do
    timeout 900 $CS --tool $tool --error-exitcode 17 --print-limit 20 \
      python tools/sanitize_case.py $case > gpurun_out/sanitize/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" >> gpurun_out/sanitize/summary.txt
  done
done
