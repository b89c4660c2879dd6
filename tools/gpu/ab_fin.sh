# A/B of the select kernel width (FREEKV_FIN_THREADS) on c3 and c2
for nt in 512 1024; do
  for cfg in c3 c2; do
    FREEKV_FIN_THREADS=$nt timeout 300 python bench.py --config $cfg --steps 64 --warmup 4 > gpurun_out/fin_${nt}_${cfg}.json 2> gpurun_out/fin_${nt}_${cfg}.err
  done
done
