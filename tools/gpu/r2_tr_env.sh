python -c "import __graft_entry__ as g; g.build()"
for e in "FREEKV_SELECT_NC=2" "FREEKV_SELECT_NC=1" "FREEKV_OVERLAP=0" "FREEKV_SELECT_NC=1 FREEKV_OVERLAP=0"; do
  echo "== $e"; env $e timeout 300 python tools/trace_step.py --graph 2>&1 | python -c "
import json,sys; t=json.load(sys.stdin); k=list(t)[-1]
for nm,v in t[k].items(): print('  ',nm,v['first_start_us'],v['last_start_us'],v['end_us'],v['median_stamps_rel_start_us'][:4])"
done
