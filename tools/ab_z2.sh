mkdir -p gpurun_out
out=gpurun_out/ab_z2.log; : > $out
for v in base zherm zreg zhr base zherm zreg zhr; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 256 512 >> $out 2>&1
done
