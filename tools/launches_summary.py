"""Median per-kernel duration from an ncu --csv launch list (gpu__time_duration.sum)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
acc = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x.get("Metric Name") == "gpu__time_duration.sum":
            acc[x["Kernel Name"].split("(")[0][:60]].append(float(x["Metric Value"].replace(",", "")) / 1e3)
for k, v in sorted(acc.items()):
    v = sorted(v)
    print(f"{k:62s} n={len(v):4d} median={v[len(v)//2]:8.2f} us")
