"""Host-side checks of the C-ABI library (no GPU): it builds for sm_100a, loads,
exports every entry point include/freekv.h declares, and validates configs with
the named errors of include/freekv.h (reading A-6/A-7)."""
import os
import re
import subprocess

import pytest
import torch

import paper_2505_13109_b200 as P
from paper_2505_13109_b200 import freekv as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "freekv.h")).read()
    return sorted(set(re.findall(r"\b(freekv_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2505_13109_b200.build import build
    lib = build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (freekv_\w+)", out))
    syms = header_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(syms) == set(F.EXPORTED)
    L = P.load_library()
    for s in syms:
        assert hasattr(L, s)
    assert L.freekv_abi_version() == 3


def test_library_is_sm100a():
    from paper_2505_13109_b200.build import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def cfg(**kw):
    base = dict(n_layers=2, batch=8, n_qo=32, n_kv=8, head_dim=128, page_size=32, budget_tokens=2048,
                sink_tokens=512, window_tokens=512, max_ctx_tokens=33000)
    base.update(kw)
    return P.FreeKVConfig(**base)


def test_query_sizes_c2_shape():
    dev, host = P.query_sizes(cfg(n_layers=32))
    # host pool = layers * batch * n_page * n_kv * 16 KiB (P:318 combined page of 2*p*d bf16)
    n_page = 33000 // 32 + 1
    assert host == 32 * 8 * n_page * 8 * 16384
    assert dev < 6 * 2 ** 30


@pytest.mark.parametrize("kw,status,needle", [
    (dict(n_qo=30), -1, "n_qo % n_kv"),
    (dict(budget_tokens=1000), -1, "budget < sink + window"),
    (dict(sink_tokens=500), -1, "sink_tokens % page_size"),
    (dict(window_tokens=100), -1, "window_tokens % page_size"),
    (dict(budget_tokens=2050), -1, "(budget - sink - window) % page_size"),
    (dict(head_dim=64), -7, "head_dim"),
    (dict(page_size=8, sink_tokens=512, window_tokens=512), -7, "page_size"),
    (dict(n_qo=72), -7, "group size"),
    (dict(mode=5), -1, "mode"),
])
def test_config_validation(kw, status, needle):
    with pytest.raises(P.FreeKVError) as ei:
        P.query_sizes(cfg(**kw))
    assert ei.value.status == status
    assert needle in str(ei.value)


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.FreeKVError):
        P.FreeKV(cfg(n_layers=1, batch=1, max_ctx_tokens=4096))


def test_comm_unique_id_without_gpu():
    """The NCCL id is created through the library (no device needed): 128 bytes, fresh each call."""
    from paper_2505_13109_b200.freekv import FreeKV
    a, b = FreeKV.comm_unique_id(), FreeKV.comm_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
