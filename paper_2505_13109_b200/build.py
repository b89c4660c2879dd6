"""Build libfreekv.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so lives
next to this file so it travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# A/B builds only: FKV_VARIANT=<name> with FKV_VARIANT_DEFS="-DX=.." builds libfreekv_<name>.so from the same
# sources (loaded with FREEKV_LIB_SUFFIX=_<name>); the default build takes neither
VARIANT = os.environ.get("FKV_VARIANT", "")
VARIANT_DEFS = os.environ.get("FKV_VARIANT_DEFS", "").split() if VARIANT else []
OBJ = os.path.join(HERE, "..", "build", "obj" + ("_" + VARIANT if VARIANT else ""))
LIB = os.path.join(HERE, "libfreekv" + ("_" + VARIANT if VARIANT else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

def _nccl_dir():
    """The NCCL torch loads (nvidia-nccl wheel) -- one libnccl.so.2 per process; system copy otherwise."""
    try:
        import nvidia.nccl as nn
        d = list(nn.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except Exception:  # noqa: BLE001
        pass
    return None


NCCL = _nccl_dir()
NCCL_INC = ["-I" + os.path.join(NCCL, "include")] if NCCL else []
NCCL_LINK = (["-L" + os.path.join(NCCL, "lib"), "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib"),
              "-l:libnccl.so.2"] if NCCL else ["-lnccl"])
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                "-I" + os.path.join(HERE, "..", "include")] + NCCL_INC + VARIANT_DEFS

SOURCES = ["api.cu", "append.cu", "score.cu", "select.cu", "recall.cu", "attn.cu"]
HEADERS = ["fkv_internal.cuh", "append_unit.cuh", "attn_core.cuh", "select_core.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                [_mtime(os.path.join(HERE, "..", "include", "freekv.h"))])
    procs, objs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if ptxas_v else []) + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose or ptxas_v:
            print(out, file=sys.stderr)
    if force or procs or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + NCCL_LINK
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv)
    print(LIB)
