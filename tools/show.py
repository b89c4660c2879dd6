"""Print the bench lines and the last traced layer of a gpurun tag (local helper)."""
import json, sys, os
tag = sys.argv[1]
d0 = "/root/repo/gpurun_out/"
for c in ("c1", "c2", "c3", "c4", "c5"):
    f = d0 + f"{tag}_bench_{c}.json"
    if not os.path.exists(f):
        continue
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "no line", open(f.replace('.json', '.err')).read()[-800:]); continue
    print(c, d["value"], "us/layer", d["us_per_layer"], "attn", d["roofline"]["us_per_launch"], d["roofline"]["frac"],
          "score", d["scoring_hbm"]["us_per_launch"], d["scoring_hbm"]["frac"], "corr", d["correction_rate"],
          "e2e", d["e2e"]["value"])
f = d0 + f"{tag}_trace.json"
if os.path.exists(f):
    try:
        t = json.load(open(f))
        k = list(t)[-1]
        print(k)
        for nm, v in t[k].items():
            print("  ", nm, v)
    except Exception as e:
        print("trace:", open(f).read()[-500:])
