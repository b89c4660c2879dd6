"""Aggregate ncu warp-stall samples per CUDA source line from a report
(`ncu -i R --page source --print-source sass,cuda --csv`)."""
import csv, subprocess, sys, collections

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr = None, None
agg = collections.Counter()
stall = collections.defaultdict(collections.Counter)
src_text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    line = int(r[0])
    key = (cur_file, line)
    src_text[key] = r[1]
    try:
        smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        smp = 0
    agg[key] += smp
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stall[key][h[6:]] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
print(f"total samples {tot:.0f}")
for key, v in agg.most_common(top):
    st = ", ".join(f"{k}:{int(c)}" for k, c in stall[key].most_common(3))
    print(f"{v / tot * 100:5.1f}% {key[0]}:{key[1]:<5} {src_text[key].strip()[:70]:70s} [{st}]")
