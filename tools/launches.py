"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections, csv, sys

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
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':34s} {'n':>4s} {'avg_us':>9s} {'dram_MB/launch':>15s} {'GB/s':>8s} {'share':>6s}"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = a[2] / (a[1] * 1e3) if a[1] else 0.0
        lines.append(f"{k:34s} {a[0]:4d} {a[1] / a[0]:9.2f} {a[2] / a[0] / 1e6:15.2f} {gbs:8.1f} {a[1] / tot * 100:5.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
