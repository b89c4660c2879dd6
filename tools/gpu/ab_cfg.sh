# A/B/C of three builds (libfreekv_{A,B,C}.so) on one box with bench.py on the configs in $CFGS
for r in 1 2; do
  for c in $CFGS; do
    for v in A B C; do
      FREEKV_LIB_SUFFIX=_$v timeout 300 python bench.py --config $c --steps 128 --no-cpu-baseline > gpurun_out/abc_${c}_${v}_$r.json 2>/dev/null
      python -c "import json; d=json.loads(open('gpurun_out/abc_${c}_${v}_$r.json').read().strip().splitlines()[-1]); print('$c $v $r', d['us_per_layer'])"
    done
  done
done
