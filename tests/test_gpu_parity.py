"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): selected page indices, frontier,
correction flags, pooled cosine and fetch lists bit-exact; page summaries
bit-exact; attention outputs within max relative error 2e-3 per (b, h)
(reading A-21: ||o - o_ref||_inf / max(||o_ref||_inf, 1e-6)).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 2e-3


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def rel_err(out, ref):
    """max over (b, h) of ||o - o_ref||_inf / max(||o_ref||_inf, 1e-6)."""
    num = np.abs(out - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-6)
    return float((num / den).max())


def run_parity(G=4, n_kv=2, batch=2, page=32, sink=64, window=64, budget=256, L0=700, steps=6,
               n_layers=2, tau=0.8, mode=O.MODE_SPECULATIVE, event_rate=0.3, seed=11, tie_pages=False,
               check_summaries=True, use_primitives=False, check_fetch=True, pool=0, corr_pool=0, dense0=0,
               sync_mask=None):
    _need_gpu()
    import paper_2505_13109_b200 as P
    d = 128
    n_qo = G * n_kv
    max_ctx = L0 + steps + 3
    cfg = P.FreeKVConfig(n_layers=n_layers, batch=batch, n_qo=n_qo, n_kv=n_kv, head_dim=d, page_size=page,
                         budget_tokens=budget, sink_tokens=sink, window_tokens=window, max_ctx_tokens=max_ctx,
                         tau=tau, mode=mode, pool=pool, corr_pool=corr_pool, first_layer_dense=dense0)
    fkv = P.FreeKV(cfg)
    ocfg = O.OracleConfig(n_layers=n_layers, batch=batch, n_qo=n_qo, n_kv=n_kv, head_dim=d, page_size=page,
                          budget_tokens=budget, sink_tokens=sink, window_tokens=window, max_ctx_tokens=max_ctx,
                          tau=tau, mode=mode, pool=pool, corr_pool=corr_pool, first_layer_dense=bool(dense0))
    eng = O.OracleEngine(ocfg)
    dev = fkv.device
    for layer in range(n_layers):
        k, v = synth.gen_prefill(batch, n_kv, d, page, L0, sink // page, cfg.K, seed, layer)
        if tie_pages:  # exact duplicate pages -> exact score ties -> lowest page id must win
            n_pages = L0 // page
            for j in range(sink // page + 3, n_pages - 1, 3):
                k[:, j * page:(j + 1) * page] = k[:, (j - 1) * page:j * page]
        eng.append(layer, synth.bf16_bits(k), synth.bf16_bits(v))
        with torch.cuda.stream(fkv.stream):
            fkv.append_kv(layer, k.to(dev), v.to(dev))
    qps = [synth.QueryProcess(batch, n_qo, n_kv, d, seed, layer, event_rate=event_rate)
           for layer in range(n_layers)]
    n_flag = n_unflag = 0
    worst = 0.0
    for i in range(steps):
        for layer in range(n_layers):
            q, _ = qps[layer].next()
            kn, vn = synth.gen_decode_kv(batch, n_kv, d, page, L0 + i, seed, layer)
            ref = eng.step(layer, synth.bf16_bits(q), synth.bf16_bits(kn), synth.bf16_bits(vn))
            out = torch.empty(batch, n_qo, d, dtype=torch.float32, device=dev)
            qd, kd, vd = q.to(dev), kn.to(dev), vn.to(dev)
            fkv.stream.wait_stream(torch.cuda.current_stream())
            if use_primitives:
                fkv.append_kv(layer, kd, vd)
                pages_out = torch.full((batch, n_kv, cfg.K), -7, dtype=torch.int32, device=dev)
                corr_out = torch.zeros((batch, n_kv), dtype=torch.uint8, device=dev)
                fkv.select_pages(layer, qd, pages_out, corr_out)
                mask = None
                if sync_mask == "all":
                    mask = torch.ones((batch, n_kv), dtype=torch.uint8, device=dev)
                elif sync_mask == "alternate":
                    mask = (torch.arange(batch * n_kv, device=dev) % 2).to(torch.uint8).view(batch, n_kv)
                fkv.recall_pages(layer, sync_mask=mask)
                fkv.sparse_decode_attn(layer, qd, out)
            else:
                fkv.decode_step(layer, qd, kd, vd, out)
            fkv.synchronize()
            if dense0 and layer == 0:  # O-7: dense attention over [0, Lc), no selection to compare
                e = rel_err(out.cpu().numpy().astype(np.float64), ref["out"])
                worst = max(worst, e)
                assert e <= REL_TOL, (i, layer, e)
                continue
            sel = fkv.get_selection(layer)
            assert np.array_equal(sel["flags"], ref["flags"]), (i, layer, sel["flags"], ref["flags"])
            assert np.array_equal(sel["cbar"].view(np.uint32), ref["cbar"].view(np.uint32)) or i == 0
            assert np.array_equal(sel["frontier"], ref["frontier"])
            assert np.array_equal(sel["pages"], ref["sel"]), (i, layer, sel["pages"], ref["sel"])
            if use_primitives:
                assert np.array_equal(pages_out.cpu().numpy().reshape(-1, cfg.K), ref["sel"])
                assert np.array_equal(corr_out.cpu().numpy().reshape(-1), ref["flags"])
            n_fetch, fetch_pages = fkv.get_fetch(layer)
            for u in range(fkv.U if check_fetch else 0):
                exp = ref["fetch_sync"][u] if ref["flags"][u] else ref["fetch_bg"][u]
                assert list(fetch_pages[u, :n_fetch[u]]) == exp, (i, layer, u)
            st = fkv.get_step_stats(layer)  # freekv_get_step_stats vs the oracle's fetch lists
            assert st["corrected_units"] == int(ref["flags"].sum())
            if check_fetch:
                assert st["sync_pages"] == sum(len(x) for x in ref["fetch_sync"])
                assert st["bg_pages"] == sum(len(x) for x in ref["fetch_bg"])
            assert st["sync_bytes"] == st["sync_pages"] * 2 * page * d * 2
            e = rel_err(out.cpu().numpy().astype(np.float64), ref["out"])
            worst = max(worst, e)
            assert e <= REL_TOL, (i, layer, e)
            n_flag += int(ref["flags"].sum())
            n_unflag += int((1 - ref["flags"]).sum())
    if check_summaries:
        for layer in range(n_layers):
            for u in range(fkv.U):
                n_off = eng.n_off[layer][u]
                got = fkv.get_summaries(layer, u, sink // page, n_off)
                assert np.array_equal(got, eng.summ[layer][u, sink // page:n_off]), (layer, u)
    fkv.close()
    return n_flag, n_unflag, worst


def test_parity_llama_shape_speculative():
    nf, nu, worst = run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=6)
    assert nf > 0 and nu > 0  # both paths (corrected / speculative) exercised


@pytest.mark.parametrize("prims", [False, True])
def test_parity_first_layer_dense(prims):
    """first_layer_dense (O-7): layer 0 attends all Lc tokens from its dense pool (decode_step
    and the primitive API), the other layers run FreeKV unchanged."""
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4, n_layers=2, dense0=1, use_primitives=prims)


@pytest.mark.parametrize("mask", ["all", "alternate"])
def test_parity_recall_sync_mask(mask):
    """freekv_recall_pages with a caller sync_mask (every unit / every other unit synchronous)
    instead of the correction flags: identical selections, fetch lists and outputs (direct mode)."""
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4, use_primitives=True, sync_mask=mask)


def test_parity_primitives():
    run_parity(G=4, n_kv=2, batch=1, page=32, L0=900, steps=4, use_primitives=True)


@pytest.mark.parametrize("G", [1, 2, 7, 8])
def test_parity_group_sizes(G):
    run_parity(G=G, n_kv=2, batch=1, page=32, L0=1100, steps=4)


@pytest.mark.parametrize("page,sink,window,budget", [(16, 32, 48, 160), (64, 64, 128, 512)])
def test_parity_page_sizes(page, sink, window, budget):
    run_parity(G=4, n_kv=2, batch=2, page=page, sink=sink, window=window, budget=budget, L0=1300, steps=4)


@pytest.mark.parametrize("mode,tau", [(O.MODE_ALWAYS, 0.8), (O.MODE_NEVER, 0.8), (O.MODE_SPECULATIVE, 1.0),
                                      (O.MODE_SPECULATIVE, 0.0)])
def test_parity_modes(mode, tau):
    run_parity(mode=mode, tau=tau, L0=800, steps=5)


def test_parity_ties_lowest_id():
    run_parity(tie_pages=True, L0=1200, steps=4, event_rate=0.0)


def test_parity_dense_equivalence():
    """Budget >= context: sparse path == dense attention (north star)."""
    run_parity(budget=4096, L0=600, steps=4)


def test_parity_short_context_ragged():
    """Context inside sink + window, then crossing it; ragged tail (not a page multiple)."""
    run_parity(L0=37, steps=4, sink=64, window=64, budget=256, page=32)
    run_parity(L0=150, steps=40, sink=32, window=32, budget=128, page=32, n_layers=1)


def test_parity_long_context_many_tiles():
    """|J| > 1024 exercises the multi-leaf-per-thread tree and radix select."""
    run_parity(G=4, n_kv=1, batch=1, page=16, sink=64, window=64, budget=640, L0=20000, steps=3, n_layers=1)


@pytest.mark.parametrize("step_mode", ["serial", "spec"])
def test_step_graph_matches_eager(step_mode, monkeypatch):
    """Whole-step CUDA graphs (one graph with forked recall branches) give the same selections and
    bit-identical outputs as the eager per-layer calls, for the serial step (default: score grid,
    select, attention) and the paper-structure speculative step (FREEKV_STEP=spec: attention beside
    the scoring / selection side streams)."""
    _need_gpu()
    monkeypatch.setenv("FREEKV_STEP", step_mode)
    import paper_2505_13109_b200 as P
    nb, n_kv, G, d, p, L0, steps, n_layers = 2, 2, 4, 128, 32, 1200, 6, 3
    n_qo = G * n_kv
    mk = lambda: P.FreeKV(P.FreeKVConfig(n_layers=n_layers, batch=nb, n_qo=n_qo, n_kv=n_kv, budget_tokens=256,
                                         sink_tokens=64, window_tokens=64, max_ctx_tokens=L0 + steps + 2))
    a, b = mk(), mk()
    dev = a.device
    seed = 77
    for layer in range(n_layers):
        k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 2, a.K, seed, layer, device=dev)
        torch.cuda.synchronize()
        a.append_kv(layer, k, v)
        b.append_kv(layer, k, v)
        a.synchronize()
        b.synchronize()
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.3) for l in range(n_layers)]
    Q = torch.empty(steps, n_layers, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    Kn = torch.empty(steps, n_layers, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    Vn = torch.empty_like(Kn)
    for i in range(steps):
        for l in range(n_layers):
            q, _ = qps[l].next()
            kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i, seed, l, device=dev)
            Q[i, l], Kn[i, l], Vn[i, l] = q, kn, vn
    torch.cuda.synchronize()
    qb, kb, vb = torch.empty_like(Q[0]), torch.empty_like(Kn[0]), torch.empty_like(Vn[0])
    ob = torch.empty(n_layers, nb, n_qo, d, dtype=torch.float32, device=dev)
    b.synchronize()
    b.step_graph_capture(qb, kb, vb, ob)
    oa = torch.empty(nb, n_qo, d, dtype=torch.float32, device=dev)
    for i in range(steps):
        with torch.cuda.stream(b.stream):
            qb.copy_(Q[i]); kb.copy_(Kn[i]); vb.copy_(Vn[i])
        b.step_graph_launch()
        b.synchronize()
        for l in range(n_layers):
            a.decode_step(l, Q[i, l], Kn[i, l], Vn[i, l], oa)
            a.synchronize()
            sa, sb = a.get_selection(l), b.get_selection(l)
            assert np.array_equal(sa["pages"], sb["pages"]) and np.array_equal(sa["flags"], sb["flags"]), (i, l)
            assert torch.equal(oa, ob[l]), (i, l)
    a.close()
    b.close()


def test_parity_without_pdl(monkeypatch):
    monkeypatch.setenv("FREEKV_PDL", "0")
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4)


def test_parity_recall_mode(monkeypatch):
    """FREEKV_CORR=recall: synchronous recall of the corrected units before a second
    attention phase (instead of the attention reading their pages from the host pool)."""
    monkeypatch.setenv("FREEKV_CORR", "recall")
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=5)
    run_parity(G=4, n_kv=2, batch=1, page=32, L0=900, steps=4, use_primitives=True)


def test_parity_full_refresh_direct(monkeypatch):
    """Every unit re-fetches all K pages every step (FREEKV_DEBUG_FULL_REFRESH): all pages of
    every unit are read by the attention kernel from the host pool and written back."""
    monkeypatch.setenv("FREEKV_DEBUG_FULL_REFRESH", "1")
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4, mode=O.MODE_ALWAYS, check_fetch=False)


@pytest.mark.parametrize("nc", ["1", "2", "4", "8"])
def test_parity_select_cluster_widths(nc, monkeypatch):
    """The select kernel at every cluster width (CTAs per unit; CFR-6 power-of-two partition of the
    pairwise tree, DSMEM exchange of maxima, subtree sums, histograms, boundary keys and ranks):
    bit-identical pages to the oracle, |J| from 1 to 4 leaves per thread, G = 4 and G = 7."""
    monkeypatch.setenv("FREEKV_SELECT_NC", nc)
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4)
    run_parity(G=7, n_kv=1, batch=2, page=16, sink=64, window=64, budget=640, L0=20000, steps=3, n_layers=1)
    run_parity(G=4, n_kv=1, batch=1, page=16, sink=64, window=64, budget=640, L0=60000, steps=2, n_layers=1,
               tie_pages=True, event_rate=0.0)


def test_parity_step_spec(monkeypatch):
    """FREEKV_STEP=spec (the paper's overlap structure): pre kernel, then the attention of the units
    that pass the correction check beside the corrected units' scoring / selection (high-priority
    stream) and the others' (side stream, committed by the next step's pre kernel)."""
    monkeypatch.setenv("FREEKV_STEP", "spec")
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=5)


@pytest.mark.parametrize("nt", ["256", "512", "1024"])
def test_parity_select_cta_widths(nt, monkeypatch):
    """One select CTA per unit at 256 / 512 / 1024 threads (the CFR-6 tree over more or fewer
    leaves per thread): bit-identical selections."""
    monkeypatch.setenv("FREEKV_SELECT_NC", "1")
    monkeypatch.setenv("FREEKV_SELECT_NT", nt)
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=40000, steps=3, n_layers=1)


def test_parity_attention_waits_for_select(monkeypatch):
    """FREEKV_ATTN_EARLY=0: every unit's attention waits for the select (no early attention of the
    units that pass the correction check)."""
    monkeypatch.setenv("FREEKV_ATTN_EARLY", "0")
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=5)


@pytest.mark.parametrize("env", [("FREEKV_RECALL_FRAG", "256"), ("FREEKV_RECALL_FRAG", "4096"),
                                 ("FREEKV_SERIAL_RECALL", "1")])
def test_parity_recall_ablation_modes(env, monkeypatch):
    """The f2 ablation's recall variants (256-byte / 4 KiB transfers per page, background recall on
    the compute stream) recall the same bytes: same selections and outputs as the oracle."""
    monkeypatch.setenv(*env)
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=6, event_rate=0.3)


def test_parity_window_zero():
    """W = 0: the page completed by this step's token is a candidate at once (append first)."""
    run_parity(G=4, n_kv=2, batch=1, page=32, sink=64, window=0, budget=256, L0=1000, steps=40, n_layers=1)


@pytest.mark.parametrize("pool", [1, 2, 3, 4, 5])
def test_parity_pooling_variants(pool):
    """Group-consistency variants: MaxS, MeanQK, MaxQK, MeanQ, MaxQ --
    bit-exact selections against the oracle, G = 4 and G = 7."""
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=4, pool=pool)
    run_parity(G=7, n_kv=1, batch=1, page=16, sink=64, window=64, budget=640, L0=5000, steps=3, n_layers=1,
               pool=pool)


@pytest.mark.parametrize("step_mode", ["serial", "spec"])
def test_parity_max_pooled_correction(step_mode, monkeypatch):
    """Max-pooled correction (tab:abl-g-corr, reading R-11): corrected when any head's similarity
    is below tau; more units corrected than with mean pooling on the same inputs."""
    monkeypatch.setenv("FREEKV_STEP", step_mode)
    nf_max, _, _ = run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=5, corr_pool=1, event_rate=0.3)
    nf_mean, _, _ = run_parity(G=4, n_kv=2, batch=2, page=32, L0=1500, steps=5, corr_pool=0, event_rate=0.3)
    assert nf_max >= nf_mean


FULL_SIZE = {
    # BASELINE.json configs[1]: Llama-3.1-8B heads, ctx 32K, batch 8, budget 2048 (the bench line)
    "c2": dict(nb=8, n_qo=32, n_kv=8, ctx=32768, tau=0.8),
    # configs[2]: Qwen-2.5-7B heads (G = 7), ctx 128K, batch 4
    "c3": dict(nb=4, n_qo=28, n_kv=4, ctx=131072, tau=0.8),
    # configs[3]: DeepSeek-R1-Distill-Llama-8B heads at the end of 16K prompt + 32K generation,
    # one point of the correction-threshold sweep (tau = 0.95: every unit corrects, measured 1.000)
    "c4": dict(nb=4, n_qo=32, n_kv=8, ctx=49152, tau=0.95),
    # configs[4]: Llama-3.1-70B heads (64q/8kv), ctx 128K, batch 16 -- one GPU's shard at N = 8
    # (one KV head and its 8 q-heads, all 16 sequences; DESIGN.md multi-GPU section)
    "c5_shard8": dict(nb=16, n_qo=8, n_kv=1, ctx=131072, tau=0.8),
}


def _report(rec):
    """Append one parity record (JSON line) to $FKV_PARITY_REPORT when set (profiles/ evidence)."""
    import json
    import os
    path = os.environ.get("FKV_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def elem_rel_err(out, ref):
    """Elementwise relative error max |o - o_ref| / |o_ref| over the elements with |o_ref| >= 1e-3
    (reported beside A-21's per-(b, h) inf-norm figure; tiny reference elements are excluded
    because their relative error is not meaningful for an fp32-accumulated bf16 product)."""
    m = np.abs(ref) >= 1e-3
    return float((np.abs(out - ref)[m] / np.abs(ref)[m]).max())


def inject_near_ties(k, page, n_sink_pages, every=5):
    """Tie structure on keys k (bf16 NHD [b][L][kv][d]): for candidate pages j = n_sink+3, +every, ...
    page j := page j-1 (exact duplicate: equal summaries, an exact pooled-score tie -> the lower id
    wins, CFR-9), and page j+2 := page j+1 with the lowest mantissa bit of one key element flipped
    (summaries one bf16 ulp apart in one channel: pooled scores equal or a few fp32 ulp apart)."""
    n_pages = k.shape[1] // page
    kb = k.view(torch.int16)
    for j in range(n_sink_pages + 3, n_pages - 3, every):
        kb[:, j * page:(j + 1) * page] = kb[:, (j - 1) * page:j * page]
        kb[:, (j + 2) * page:(j + 3) * page] = kb[:, (j + 1) * page:(j + 2) * page]
        kb[:, (j + 2) * page, :, 0] ^= 1
    return k


def run_full_size(name, c, n_layers=2, steps=4, gen="S", ties=False, check_fetch=False, seed=250513119):
    """Full-size parity through the whole-step CUDA graph (the launch configuration bench.py
    times): every unit of every layer and step vs the oracle -- page indices, frontier, flags (and
    fetch lists) bit-exact, outputs within 2e-3 (A-21).  gen "S": GEN-S/GEN-Q as in the bench;
    "X": unstructured i.i.d. keys and queries (alpha = beta = 0, rho = 0: no topic, cosines ~0,
    every unit corrects every step, full churn)."""
    _need_gpu()
    import paper_2505_13109_b200 as P
    nb, n_qo, n_kv, d, p = c["nb"], c["n_qo"], c["n_kv"], 128, 32
    L0 = c["ctx"] - steps                   # the last step attends over exactly ctx tokens
    kw = dict(n_layers=n_layers, batch=nb, n_qo=n_qo, n_kv=n_kv, head_dim=d, page_size=p, budget_tokens=2048,
              sink_tokens=512, window_tokens=512, max_ctx_tokens=L0 + steps + 2, tau=c["tau"],
              mode=O.MODE_SPECULATIVE)
    fkv = P.FreeKV(P.FreeKVConfig(**kw))
    eng = O.OracleEngine(O.OracleConfig(**kw))
    dev = fkv.device
    alpha = 0.0 if gen == "X" else synth.ALPHA
    for layer in range(n_layers):
        k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 512 // p, fkv.K, seed, layer, device=dev, alpha=alpha)
        if ties:
            k = inject_near_ties(k, p, 512 // p)
        torch.cuda.synchronize()
        fkv.append_kv(layer, k, v)
        fkv.synchronize()
        eng.append(layer, synth.bf16_bits(k), synth.bf16_bits(v))
        del k, v
    if gen == "X":
        qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, beta=0.0, rho=0.0, event_rate=0.0)
               for l in range(n_layers)]
    else:
        qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.05) for l in range(n_layers)]
    qb = torch.empty(n_layers, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    kb = torch.empty(n_layers, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    vb = torch.empty_like(kb)
    ob = torch.empty(n_layers, nb, n_qo, d, dtype=torch.float32, device=dev)
    fkv.step_graph_capture(qb, kb, vb, ob)
    n_flag = n_fetch_tot = 0
    worst = worst_el = 0.0
    for i in range(steps):
        for l in range(n_layers):
            q, _ = qps[l].next()
            kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i, seed, l, device=dev, alpha=alpha)
            qb[l].copy_(q); kb[l].copy_(kn); vb[l].copy_(vn)
        torch.cuda.synchronize()
        fkv.step_graph_launch()
        fkv.synchronize()
        for l in range(n_layers):
            ref = eng.step(l, synth.bf16_bits(qb[l]), synth.bf16_bits(kb[l]), synth.bf16_bits(vb[l]))
            sel = fkv.get_selection(l)
            assert np.array_equal(sel["flags"], ref["flags"]), (i, l)
            assert np.array_equal(sel["frontier"], ref["frontier"]), (i, l)
            assert np.array_equal(sel["pages"], ref["sel"]), (i, l)
            if check_fetch:
                n_fetch, fetch_pages = fkv.get_fetch(l)
                for u in range(fkv.U):
                    exp = ref["fetch_sync"][u] if ref["flags"][u] else ref["fetch_bg"][u]
                    assert list(fetch_pages[u, :n_fetch[u]]) == exp, (i, l, u)
                    n_fetch_tot += len(exp)
            o = ob[l].cpu().numpy().astype(np.float64)
            e = rel_err(o, ref["out"])
            worst = max(worst, e)
            worst_el = max(worst_el, elem_rel_err(o, ref["out"]))
            assert e <= REL_TOL, (i, l, e)
            if i > 0:
                n_flag += int(ref["flags"].sum())
    rate = n_flag / max(1, (steps - 1) * n_layers * nb * n_kv)
    _report({"test": name, "gen": gen, "ties": ties, "layers": n_layers, "steps": steps, "units": fkv.U,
             "tau": c["tau"], "nb": nb, "correction_rate": round(rate, 4), "fetched_pages": n_fetch_tot,
             "a21_rel_err_max": worst, "elementwise_rel_err_max": worst_el})
    fkv.close()
    return rate


@pytest.mark.parametrize("name", sorted(FULL_SIZE))
def test_parity_full_size_step_graph(name):
    """BASELINE.json config sizes (d=128, page 32, budget 2048, S = W = 512) in the launch
    configuration bench.py times: the whole-step CUDA graph, default kernels.  Two layers
    (the per-layer path is identical for all of them), every unit compared with the oracle:
    page indices, frontier and flags bit-exact, outputs within 2e-3.  Step 0 is all-flagged
    (synchronous full recall), the later steps are speculative with seeded query dips
    (event rate 0.05 as in the bench)."""
    c = FULL_SIZE[name]
    rate = run_full_size(name, c)
    if c["tau"] <= 0.8:
        assert rate < 1.0   # speculative steps did not all correct


def test_parity_full_size_deep_c2():
    """configs[1] (c2) through the step graph for 8 layers x 16 steps, fetch lists included: the
    delta / slot double-buffering state machine over many speculative steps at full size."""
    run_full_size("c2_deep", FULL_SIZE["c2"], n_layers=8, steps=16, check_fetch=True)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_parity_full_size_unstructured(name):
    """GEN-X at c2 / c3 sizes: i.i.d. keys and queries (no hot pages, no topic), so every unit
    corrects every step and the top-K boundary falls in a dense, nearly flat score region."""
    rate = run_full_size(name + "_genx", FULL_SIZE[name], n_layers=1, steps=3, gen="X", check_fetch=True)
    assert rate == 1.0


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_parity_full_size_near_ties(name):
    """Injected exact and 1-ulp near-duplicate pages at c2 / c3 sizes (CFR-9: equal pooled
    scores -> lower page id; near-equal ones decided by the canonical fp32 recipe on both sides)."""
    run_full_size(name + "_ties", FULL_SIZE[name], n_layers=1, steps=3, ties=True, check_fetch=True)


@pytest.mark.parametrize("tau", [0.0, 0.8, 0.9, 1.0])
def test_parity_full_size_c4_batch8_tau(tau):
    """configs[3] heads and context (32q/8kv, 48K) at batch 8 across the correction threshold:
    tau = 0 never corrects after bootstrap, tau = 1 corrects every unit every step."""
    c = dict(FULL_SIZE["c4"], nb=8, tau=tau)
    rate = run_full_size(f"c4_b8_tau{tau}", c)
    if tau == 0.0:
        assert rate == 0.0
    if tau == 1.0:
        assert rate == 1.0


def test_summarize_pages_matches_oracle():
    """freekv_summarize_pages rebuilds the channel-wise min/max summaries of offloaded pages from
    the host pool; bit-exact against the oracle's page summaries, after the append's own
    summaries were checked (so a rebuild that changed anything would show)."""
    _need_gpu()
    import paper_2505_13109_b200 as P
    G, n_kv, nb, p, L0, n_layers = 4, 2, 2, 32, 3000, 2
    kw = dict(n_layers=n_layers, batch=nb, n_qo=G * n_kv, n_kv=n_kv, head_dim=128, page_size=p,
              budget_tokens=256, sink_tokens=64, window_tokens=64, max_ctx_tokens=L0 + 8)
    fkv = P.FreeKV(P.FreeKVConfig(**kw))
    eng = O.OracleEngine(O.OracleConfig(**kw))
    for layer in range(n_layers):
        k, v = synth.gen_prefill(nb, n_kv, 128, p, L0, 2, fkv.K, 7, layer)
        eng.append(layer, synth.bf16_bits(k), synth.bf16_bits(v))
        fkv.append_kv(layer, k.to(fkv.device), v.to(fkv.device))
    fkv.synchronize()
    for layer in range(n_layers):
        n_off = eng.n_off[layer][0]
        fkv.summarize_pages(layer, 0, n_off)
        fkv.synchronize()
        for u in range(fkv.U):
            got = fkv.get_summaries(layer, u, 2, n_off)
            assert np.array_equal(got, eng.summ[layer][u, 2:n_off]), (layer, u)
        # a sub-range rebuild leaves the rest untouched and is again exact
        fkv.summarize_pages(layer, n_off // 3, n_off // 2)
        fkv.synchronize()
        for u in range(fkv.U):
            assert np.array_equal(fkv.get_summaries(layer, u, 2, n_off), eng.summ[layer][u, 2:n_off])
    fkv.close()


def test_step_graph_layer_cycling_matches_eager():
    """freekv_step_graph_capture_cycle (L_inst cycling, bench c5): 6 virtual layers over 2
    instantiated ones -- the graph gives the selections and bit-identical outputs of the eager
    calls decode_step(v % 2) in the same order, and each replay appends 3 tokens per layer."""
    _need_gpu()
    import paper_2505_13109_b200 as P
    nb, n_kv, G, d, p, L0, steps, n_inst, n_virt = 2, 2, 4, 128, 32, 1200, 4, 2, 6
    n_qo = G * n_kv
    mk = lambda: P.FreeKV(P.FreeKVConfig(n_layers=n_inst, batch=nb, n_qo=n_qo, n_kv=n_kv, budget_tokens=256,
                                         sink_tokens=64, window_tokens=64,
                                         max_ctx_tokens=L0 + steps * (n_virt // n_inst) + 2))
    a, b = mk(), mk()
    dev = a.device
    seed = 78
    for layer in range(n_inst):
        k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 2, a.K, seed, layer, device=dev)
        torch.cuda.synchronize()
        a.append_kv(layer, k, v)
        b.append_kv(layer, k, v)
        a.synchronize()
        b.synchronize()
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.3) for l in range(n_inst)]
    Q = torch.empty(steps, n_virt, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    Kn = torch.empty(steps, n_virt, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    Vn = torch.empty_like(Kn)
    for i in range(steps):
        for vl in range(n_virt):
            li, occ = vl % n_inst, vl // n_inst
            q, _ = qps[li].next()
            kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i * (n_virt // n_inst) + occ, seed, li, device=dev)
            Q[i, vl], Kn[i, vl], Vn[i, vl] = q, kn, vn
    torch.cuda.synchronize()
    qb, kb, vb = torch.empty_like(Q[0]), torch.empty_like(Kn[0]), torch.empty_like(Vn[0])
    ob = torch.empty(n_virt, nb, n_qo, d, dtype=torch.float32, device=dev)
    b.step_graph_capture_cycle(n_virt, qb, kb, vb, ob)
    oa = torch.empty(n_virt, nb, n_qo, d, dtype=torch.float32, device=dev)
    for i in range(steps):
        with torch.cuda.stream(b.stream):
            qb.copy_(Q[i]); kb.copy_(Kn[i]); vb.copy_(Vn[i])
        b.step_graph_launch()
        b.synchronize()
        for vl in range(n_virt):
            a.decode_step(vl % n_inst, Q[i, vl], Kn[i, vl], Vn[i, vl], oa[vl])
        a.synchronize()
        assert torch.equal(oa, ob), i
        for l in range(n_inst):
            sa, sb = a.get_selection(l), b.get_selection(l)
            assert np.array_equal(sa["pages"], sb["pages"]) and np.array_equal(sa["flags"], sb["flags"]), (i, l)
            assert a.context(l) == b.context(l) == L0 + (i + 1) * (n_virt // n_inst)
    a.close()
    b.close()


def test_step_graph_back_to_back_no_host_sync():
    """Step-graph replays issued back to back with no host synchronisation between them (inputs
    staged and outputs saved by stream-ordered copies): the same outputs, bit for bit, and the
    same final selections as synchronised eager steps -- the stream / event ordering alone
    (recall joins, PDL chains) carries every dependency between steps."""
    _need_gpu()
    import paper_2505_13109_b200 as P
    nb, n_kv, G, d, p, L0, steps, n_layers = 2, 2, 4, 128, 32, 1300, 8, 3
    n_qo = G * n_kv
    mk = lambda: P.FreeKV(P.FreeKVConfig(n_layers=n_layers, batch=nb, n_qo=n_qo, n_kv=n_kv, budget_tokens=256,
                                         sink_tokens=64, window_tokens=64, max_ctx_tokens=L0 + steps + 2))
    a, b, c = mk(), mk(), mk()
    dev = a.device
    seed = 91
    for layer in range(n_layers):
        k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 2, a.K, seed, layer, device=dev)
        torch.cuda.synchronize()
        a.append_kv(layer, k, v)
        b.append_kv(layer, k, v)
        c.append_kv(layer, k, v)
    a.synchronize()
    b.synchronize()
    c.synchronize()
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.3) for l in range(n_layers)]
    Q = torch.empty(steps, n_layers, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    Kn = torch.empty(steps, n_layers, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    Vn = torch.empty_like(Kn)
    for i in range(steps):
        for l in range(n_layers):
            q, _ = qps[l].next()
            kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i, seed, l, device=dev)
            Q[i, l], Kn[i, l], Vn[i, l] = q, kn, vn
    torch.cuda.synchronize()
    qb, kb, vb = torch.empty_like(Q[0]), torch.empty_like(Kn[0]), torch.empty_like(Vn[0])
    ob = torch.empty(n_layers, nb, n_qo, d, dtype=torch.float32, device=dev)
    saved = torch.empty(steps, n_layers, nb, n_qo, d, dtype=torch.float32, device=dev)
    b.step_graph_capture(qb, kb, vb, ob)
    for i in range(steps):  # no host sync inside this loop
        with torch.cuda.stream(b.stream):
            qb.copy_(Q[i]); kb.copy_(Kn[i]); vb.copy_(Vn[i])
        b.step_graph_launch()
        with torch.cuda.stream(b.stream):
            saved[i].copy_(ob)
    # eager calls, also without host sync (stream-ordered output saves)
    saved_c = torch.empty_like(saved)
    c.stream.wait_stream(torch.cuda.current_stream())
    for i in range(steps):
        for l in range(n_layers):
            c.decode_step(l, Q[i, l], Kn[i, l], Vn[i, l], saved_c[i, l])
    b.synchronize()
    c.synchronize()
    oa = torch.empty(nb, n_qo, d, dtype=torch.float32, device=dev)
    for i in range(steps):
        for l in range(n_layers):
            a.decode_step(l, Q[i, l], Kn[i, l], Vn[i, l], oa)
            a.synchronize()
            assert torch.equal(oa, saved[i, l]), (i, l)
            assert torch.equal(oa, saved_c[i, l]), (i, l)
    for l in range(n_layers):
        sa, sb, sc = a.get_selection(l), b.get_selection(l), c.get_selection(l)
        assert np.array_equal(sa["pages"], sb["pages"]) and np.array_equal(sa["flags"], sb["flags"]), l
        assert np.array_equal(sa["pages"], sc["pages"]) and np.array_equal(sa["flags"], sc["flags"]), l
    a.close()
    b.close()
    c.close()


@pytest.mark.parametrize("warps", ["4", "8"])
def test_parity_score_cta_warps(warps, monkeypatch):
    """Score CTAs of 4 or 8 warps (512 / 1024 pages per CTA; 8 is the default for >= 64 units):
    bit-identical scores, selections and fetch lists, ragged last item."""
    monkeypatch.setenv("FREEKV_SCORE_WARPS", warps)
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=40000, steps=3, n_layers=1)
    run_parity(G=7, n_kv=1, batch=2, page=32, L0=3000, steps=3, n_layers=1)


def test_select_tree_grows_across_power_of_two():
    """The select's CFR-6 tree is the smallest power of two covering the current candidates
    (chosen per launch; the step graph is re-captured when a context outgrows its tree): contexts
    crossing n_off = 256 pages, eagerly vs the oracle and through the step graph vs eager calls."""
    _need_gpu()
    import paper_2505_13109_b200 as P
    L0 = (256 + 2) * 32 - 3          # n_off = ctx/p - W/p crosses 256 after 3 tokens
    run_parity(G=4, n_kv=2, batch=2, page=32, L0=L0, steps=8, n_layers=1)
    nb, n_kv, G, d, p, steps, n_layers = 2, 2, 4, 128, 32, 8, 2
    n_qo = G * n_kv
    mk = lambda: P.FreeKV(P.FreeKVConfig(n_layers=n_layers, batch=nb, n_qo=n_qo, n_kv=n_kv, budget_tokens=256,
                                         sink_tokens=64, window_tokens=64, max_ctx_tokens=L0 + 4000))
    a, b = mk(), mk()
    dev = a.device
    seed = 93
    for layer in range(n_layers):
        k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 2, a.K, seed, layer, device=dev)
        torch.cuda.synchronize()
        a.append_kv(layer, k, v)
        b.append_kv(layer, k, v)
    a.synchronize()
    b.synchronize()
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.3) for l in range(n_layers)]
    qb = torch.empty(n_layers, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    kb = torch.empty(n_layers, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    vb = torch.empty_like(kb)
    ob = torch.empty(n_layers, nb, n_qo, d, dtype=torch.float32, device=dev)
    b.step_graph_capture(qb, kb, vb, ob)
    oa = torch.empty(nb, n_qo, d, dtype=torch.float32, device=dev)
    for i in range(steps):
        for l in range(n_layers):
            q, _ = qps[l].next()
            kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i, seed, l, device=dev)
            qb[l], kb[l], vb[l] = q, kn, vn
        torch.cuda.synchronize()
        b.step_graph_launch()
        b.synchronize()
        for l in range(n_layers):
            a.decode_step(l, qb[l], kb[l], vb[l], oa)
            a.synchronize()
            sa, sb = a.get_selection(l), b.get_selection(l)
            assert np.array_equal(sa["pages"], sb["pages"]) and np.array_equal(sa["flags"], sb["flags"]), (i, l)
            assert torch.equal(oa, ob[l]), (i, l)
    a.close()
    b.close()


@pytest.mark.parametrize("stages", ["4", "6", "8"])
def test_parity_score_ring_depth(stages, monkeypatch):
    """4-warp score CTAs with a 4-, 6- or 8-deep stage ring per warp (8 is the default when the
    scoring grid fits the GPU at once): bit-identical selections (odd and even G)."""
    monkeypatch.setenv("FREEKV_SCORE_WARPS", "4")
    monkeypatch.setenv("FREEKV_SCORE_STAGES", stages)
    run_parity(G=7, n_kv=1, batch=2, page=32, L0=9000, steps=3, n_layers=1)
    run_parity(G=4, n_kv=2, batch=1, page=32, L0=3000, steps=3, n_layers=1)
