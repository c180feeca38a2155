mkdir -p gpurun_out
out=gpurun_out/ab_ct.log; : > $out
for v in base ct1 ct2 ct4 ct8 base; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 256 512 >> $out 2>&1
done
