# bench sweep over env settings: SWEEP="NAME=VAL;NAME=VAL ..." (space separated runs), CFGS
for c in ${CFGS:-c2 c3}; do
  for kv in ${SWEEP}; do
    env $(echo $kv | tr ';' ' ') timeout 300 python bench.py --config $c --steps 128 --no-cpu-baseline > gpurun_out/${TAG}_sw_${c}_${kv//[;=]/_}.json 2>/dev/null
  done
done
