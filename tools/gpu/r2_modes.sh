# bench lines of the step modes (speculative default vs serial) on c2/c3
python -c "import __graft_entry__ as g; g.build()"
for e in "FREEKV_OVERLAP=1" "FREEKV_OVERLAP=0" "FREEKV_OVERLAP=0 FREEKV_SELECT_NC=1"; do for c in c2 c3; do
  env $e timeout 300 python bench.py --config $c --steps 64 --warmup 4 --no-cpu-baseline > gpurun_out/${TAG}_m.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_m.json').read().strip().splitlines()[-1]); print('$e $c', d['us_per_layer'], d['roofline']['us_per_launch'], d['scoring_hbm']['us_per_launch'])"
done; done
