"""Opcode histogram of the hot kernels' SASS (cuobjdump -sass of libfreekv.so): evidence that the
score kernel runs packed FFMA2 on TMA bulk copies (UBLKCP), the attention runs HMMA on 2D TMA
(UTMALDG / UTMASTG) with cluster barriers (UCGABAR) and DSMEM, the recall moves pages with UBLKCP.

    python tools/sass_summary.py > profiles/r2_sass_opcodes.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_13109_b200", "libfreekv.so")
# the instances the default c2 / c3 step launches (G = 4 / 7 -> head-pair template 4 / 7, PPT 4;
# select LPT 1 / GM 4 / one 1024-thread CTA (c2) and LPT 4 / GM 8 / 4-CTA cluster (c3); attention
# 3 stages x cluster 4 (c2) / 8 (c3))
WANT = [
    ("score c2", r"fkv_score_kernelILi4ELi4ELi8ELi4E"),
    ("score c3", r"fkv_score_kernelILi7ELi4ELi4ELi8E"),
    ("select c2", r"fkv_select_kernelILi1ELi4ELi1ELi1024E"),
    ("select c3", r"fkv_select_kernelILi4ELi8ELi4ELi256E"),
    ("attention c2", r"fkv_attn_cluster_kernelILi3ELi4E"),
    ("attention c3", r"fkv_attn_cluster_kernelILi2ELi8E"),
    ("recall", r"fkv_recall_kernel"),
    ("append", r"fkv_append_kernel"),
]
KEY = ["FFMA2", "FFMA", "FMUL", "HMMA", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "UCGABAR", "LDS", "STS", "LDG",
       "STG", "LDSM", "MOVM", "SHFL", "ATOMS", "RED", "BAR", "MUFU", "ELECT", "ACQBULK"]


def main():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            funcs[cur][m.group(2)] += 1
    print(f"# SASS opcode counts (static, cuobjdump -sass {os.path.relpath(LIB, ROOT)}, sm_100a)")
    for label, pat in WANT:
        names = [f for f in funcs if re.search(pat, f)]
        if not names:
            print(f"\n## {label}: no instance matching {pat}")
            continue
        f = names[0]
        c = funcs[f]
        total = sum(c.values())
        print(f"\n## {label}: {f[:110]}  ({total} instructions)")
        agg = {k: sum(v for op, v in c.items() if op == k or op.startswith(k + "_")) for k in KEY}
        print("   " + ", ".join(f"{k} {agg[k]}" for k in KEY if agg[k]))
        print("   top: " + ", ".join(f"{k} {v}" for k, v in c.most_common(12)))


if __name__ == "__main__":
    sys.exit(main())
