for c in c2 c3; do for nc in 1 2 4 8; do
  FREEKV_SELECT_NC=$nc timeout 300 python bench.py --config $c --steps 64 --no-cpu-baseline > gpurun_out/${TAG}_nc_${c}_$nc.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_nc_${c}_$nc.json').read().strip().splitlines()[-1]); print('$c nc=$nc', d['us_per_layer'], d['roofline']['us_per_launch'], d['scoring_hbm']['us_per_launch'])"
done; done
