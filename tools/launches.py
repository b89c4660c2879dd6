"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections, csv, statistics, sys

UNIT = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui, mi, ii = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("fkv::", "")
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        per[r[ii]][r[mi]] = v
        per[r[ii]]["name"] = name
    agg = collections.defaultdict(list)
    for d in per.values():
        agg[d["name"]].append((d.get("gpu__time_duration.sum", 0.0),
                               d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)))
    tot = sum(sum(t for t, _ in v) for v in agg.values())
    med_tot = sum(statistics.median(t for t, _ in v) for k, v in agg.items() if k != "fkv_append_kernel")
    lines = [f"{'kernel':30s} {'n':>4s} {'avg_us':>9s} {'median_us':>10s} {'share(total)':>13s} "
             f"{'share(step, medians)':>21s}"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(t for t, _ in x[1])):
        ts = [t for t, _ in v]
        med = statistics.median(ts)
        step_share = f"{med / med_tot * 100:5.1f}%" if k != "fkv_append_kernel" and med_tot else "   --"
        lines.append(f"{k:30s} {len(ts):4d} {sum(ts) / len(ts):9.2f} {med:10.2f} {sum(ts) / tot * 100:12.1f}% "
                     f"{step_share:>21s}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
