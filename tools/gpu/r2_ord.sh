python -c "import __graft_entry__ as g; g.build()"
for e in "FREEKV_LAYER_ORDER=0" "FREEKV_LAYER_ORDER=1"; do for c in c2 c3; do
  env $e timeout 300 python bench.py --config $c --steps 64 --warmup 4 --no-cpu-baseline > gpurun_out/${TAG}_m.json 2>gpurun_out/${TAG}_m.err
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_m.json').read().strip().splitlines()[-1]); print('$e $c', d['us_per_layer'], d['roofline']['us_per_launch'])" || tail -3 gpurun_out/${TAG}_m.err
done; done
timeout 200 python tools/trace_layer.py c2 > gpurun_out/${TAG}_tl.log 2>&1
