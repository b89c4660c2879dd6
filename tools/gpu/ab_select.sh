for sel in default fused c2; do
  if [ $sel = default ]; then unset FREEKV_SELECT; else export FREEKV_SELECT=$sel; fi
  for cfg in c3 c2; do
    timeout 300 python bench.py --config $cfg --steps 64 --warmup 4 > gpurun_out/ab_${sel}_${cfg}.json 2> gpurun_out/ab_${sel}_${cfg}.err
  done
done
