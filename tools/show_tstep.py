"""Print the last traced layer of trace_step.py output relative to the first pre-CTA start."""
import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    for k, v in list(d.items())[-1:]:
        print(f, k)
        t0 = v["pre"]["first_start_us"] if "pre" in v else min(x["first_start_us"] for x in v.values())
        for nm, x in v.items():
            print(" %-12s n=%4d start %6.1f..%6.1f end %6.1f" % (nm, x["n"], x["first_start_us"] - t0,
                  x["last_start_us"] - t0, x["end_us"] - t0), x["median_stamps_rel_start_us"])
