"""Aggregate ncu warp-stall samples per CUDA source line (ncu -i X --page source --csv --print-source cuda,sass)."""
import csv, subprocess, sys

def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, agg, tot = None, {}, 0.0
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) < 5 or r[0] in ("Line No", "Function Name") or not r[0]:
            continue
        try:
            v = float(r[4])
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        agg[key] = (agg.get(key, (0.0, r[1]))[0] + v, r[1])
        tot += v
    for (f, ln), (v, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v / tot * 100:5.1f}% {f}:{ln}: {src.strip()[:100]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
