"""Summarise an `ncu --set full` report: per kernel launch the duration, DRAM bytes, launch shape
and the warp-stall mix (usage: python tools/ncu_summary.py REPORT.ncu-rep)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
for r in rows[2:]:
    print(r[idx["Kernel Name"]][:90])
    for w in want:
        if w in idx:
            print("    %-55s %s %s" % (w, r[idx[w]], units[idx[w]]))
    sv = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[idx[h]] or 0) for h in stalls}
    tot = sum(sv.values()) or 1.0
    top = sorted(sv.items(), key=lambda x: -x[1])[:8]
    print("    stall mix (% of samples): " + ", ".join("%s %.1f" % (k, 100 * v / tot) for k, v in top))
    print()
