"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage it pins.  None of them retypes the oracle's own
formula: they use printed/hand-worked values (tests/golden/), closed forms,
invariants, brute force, or a library routine (numpy / torch fp64 / Python
sort) for a special case.
"""
import json
import math
import os
import struct

import numpy as np
import pytest
import torch

from oracle import oracle as O


def bits(x):
    return O.f32_to_bf16(np.asarray(x, np.float32))


def f32bits(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


# ------------------------------------------------------------------ CFR-1 bf16
def test_bf16_conversion_matches_torch():
    x = np.random.default_rng(1).standard_normal(10000).astype(np.float32) * 100
    ours = O.f32_to_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(O.bf16_to_f32(ours), torch.from_numpy(x).to(torch.bfloat16).float().numpy())


# ------------------------------------------------- page summary
def test_summary_worked_example():
    mn, mx = O.page_summary(bits([[1, -2], [3, 0]]))
    assert list(O.bf16_to_f32(mn)) == [1, -2]
    assert list(O.bf16_to_f32(mx)) == [3, 0]


def test_summary_single_token_and_numpy():
    rng = np.random.default_rng(2)
    k = bits(rng.standard_normal((1, 128)))
    mn, mx = O.page_summary(k)
    assert np.array_equal(mn, k[0]) and np.array_equal(mx, k[0])
    for _ in range(50):
        keys = bits(rng.standard_normal((32, 128)) * 3)
        mn, mx = O.page_summary(keys)
        kf = O.bf16_to_f32(keys)
        assert np.array_equal(O.bf16_to_f32(mn), kf.min(0))
        assert np.array_equal(O.bf16_to_f32(mx), kf.max(0))


def test_summary_signed_zero_total_order():
    mn, mx = O.page_summary(np.array([[0x0000], [0x8000]], np.uint16))
    assert mn[0] == 0x8000 and mx[0] == 0x0000


# ------------------------------------------------ page bound (A-1)
def test_page_bound_worked_example():
    assert O.page_bound(bits([1, 1]), bits([0, 0]), bits([2, 3])) == 5.0
    # scaled score of the SPEC example is (2+3)/sqrt(2)
    r = float(O.score_scale(2))
    assert abs(5.0 * r / math.log2(math.e) - 5 / math.sqrt(2)) < 1e-6


def test_page_bound_zero_query():
    rng = np.random.default_rng(3)
    mn, mx = O.page_summary(bits(rng.standard_normal((32, 128))))
    assert O.page_bound(np.zeros(128, np.uint16), mn, mx) == 0.0


def test_page_bound_upper_bounds_every_token():
    """Upper-bound property: bound >= q.k for every key in the page."""
    rng = np.random.default_rng(4)
    for _ in range(10000 // 50):
        keys = bits(rng.standard_normal((32, 16)) * rng.uniform(0.1, 5))
        qs = bits(rng.standard_normal((50, 16)))
        mn, mx = O.page_summary(keys)
        kf = O.bf16_to_f32(keys).astype(np.float64)
        for q in qs:
            u = O.page_bound(q, mn, mx)
            qf = O.bf16_to_f32(q).astype(np.float64)
            best = (kf @ qf).max()
            slack = 1e-6 * (np.abs(qf) @ np.abs(kf).max(0) + 1)
            assert u >= best - slack


def test_page_bound_identical_keys_is_dot():
    rng = np.random.default_rng(5)
    k = bits(rng.standard_normal(128))
    q = bits(rng.standard_normal(128))
    mn, mx = O.page_summary(np.stack([k] * 32))
    dot = float(O.bf16_to_f32(q).astype(np.float64) @ O.bf16_to_f32(k).astype(np.float64))
    assert abs(O.page_bound(q, mn, mx) - dot) <= 1e-5 * (1 + abs(dot))


# --------------------------------------------------------- CFR-3 scale, CFR-5
def test_score_scale_constant():
    assert f32bits(O.score_scale(128)) == 0x3E0293EE
    assert f32bits(O.score_scale(128)) == f32bits(np.float32(math.log2(math.e) / math.sqrt(128)))


def test_cexp2_exact_at_integers_and_accurate():
    for n in range(-125, 1):
        assert O.cexp2(float(n)) == np.float32(2.0 ** n)
    assert O.cexp2(-125.5) == 0.0 and O.cexp2(-1000.0) == 0.0
    rng = np.random.default_rng(6)
    xs = np.concatenate([-rng.uniform(0, 125, 20000), -rng.uniform(0, 2, 20000)]).astype(np.float32)
    for x in xs[:4000]:
        got = float(O.cexp2(float(x)))
        ref = 2.0 ** float(x)
        ulp = np.spacing(np.float32(ref))
        assert abs(got - ref) <= 2 * ulp, (x, got, ref)


# --------------------------------------------------------------- CFR-6 tree
def test_tree_sum_is_pairwise():
    e = 2.0 ** -24
    a = [1.0, e, e, e]
    # pairwise: (1 + e) + (e + e) = 1 + 2^-23 ; sequential would give exactly 1
    assert O.tree_sum(a) == np.float32(1 + 2 ** -23)
    assert np.float32(np.float32(np.float32(1 + np.float32(e)) + np.float32(e)) + np.float32(e)) == 1.0
    rng = np.random.default_rng(7)
    v = rng.uniform(0, 1, 1024).astype(np.float32)
    assert abs(float(O.tree_sum(v)) - math.fsum(v.astype(np.float64))) < 1e-4


# ---------------------------------------------- MeanS pooling (A-2..A-4)
def test_pool_matches_scipy_softmax_mean():
    from scipy.special import softmax
    rng = np.random.default_rng(8)
    for G in (1, 2, 4, 7, 8):
        s = (rng.standard_normal((G, 300)) * 3).astype(np.float32)
        jb, je = 17, 300
        pooled = O.pool_means(s, jb, je)
        ref = softmax(s[:, jb:je].astype(np.float64) * math.log(2), axis=1).sum(0)
        assert np.allclose(pooled[jb:je], ref, rtol=2e-6, atol=1e-9)
        assert abs(pooled[jb:je].astype(np.float64).sum() - G) < 1e-5 * G


def test_pool_uniform_and_g1():
    s = np.zeros((1, 10), np.float32)
    pooled = O.pool_means(s, 0, 10)
    assert np.all(pooled == np.float32(0.1))
    s = np.zeros((3, 8), np.float32)
    assert np.all(O.pool_means(s, 0, 8) == np.float32(3 * np.float32(1 / 8)))


def test_pool_tie_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "select_worked_example.json")))["tie_example"]
    pooled = O.pool_means(np.array(g["s"], np.float32), 0, 2)
    assert pooled[0] == pooled[1]
    assert abs(pooled[0] - 1.0) < 1e-6
    assert list(O.topk(pooled, 0, 2, 1)) == g["top1"]


def test_selection_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "select_worked_example.json")))
    q = bits(g["q"])
    summ = bits(g["summaries"])
    for h in range(2):
        for j in range(3):
            assert O.page_bound(q[h], summ[j, 0], summ[j, 1]) == g["u"][h][j]
    sel1, pooled = O.select_unit(q, summ, 0, 3, 1, want_pooled=True)
    assert np.allclose(pooled, g["pooled_sum"], atol=g["tol"])
    assert list(sel1) == g["top1"]
    assert list(O.select_unit(q, summ, 0, 3, 2)) == g["top2"]


def test_scaling_changes_selection(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "select_worked_example.json")))["scaling_example"]
    u = np.array(g["u"], np.float32)
    r = O.score_scale(g["d"])
    ps = O.pool_means((u * r).astype(np.float32), 0, 3)
    pu = O.pool_means((u * np.float32(math.log2(math.e))).astype(np.float32), 0, 3)
    assert np.allclose(ps, g["pooled_scaled"], atol=g["tol"])
    assert np.allclose(pu, g["pooled_unscaled"], atol=g["tol"])
    assert list(O.topk(ps, 0, 3, 1)) == g["top1_scaled"]
    assert list(O.topk(pu, 0, 3, 1)) == g["top1_unscaled"]


# ---------------------------------------------------------- top-K (A-5)
def test_topk_examples():
    assert list(O.topk([0.1, 0.5, 0.4], 0, 3, 2)) == [1, 2]
    assert list(O.topk([0.3] * 4, 0, 4, 2)) == [0, 1]
    assert list(O.topk([0.3, 0.1], 0, 2, 4)) == [0, 1, -1, -1]
    assert list(O.topk([9, 9, 0.1, 0.5, 0.4], 2, 5, 2)) == [3, 4]
    assert list(O.topk([1.0] * 5, 5, 5, 3)) == [-1, -1, -1]


def test_topk_bruteforce_and_monotone_invariance():
    rng = np.random.default_rng(9)
    for trial in range(1000):
        n = int(rng.integers(1, 200))
        K = int(rng.integers(1, 40))
        v = rng.integers(0, 20, n).astype(np.float32) / 7  # many ties
        jb = int(rng.integers(0, n))
        ref = sorted(range(jb, n), key=lambda j: (-v[j], j))[:K]
        got = [j for j in O.topk(v, jb, n, K) if j >= 0]
        assert got == sorted(ref)
        w = (np.exp(v.astype(np.float64)) * 3 + 1).astype(np.float32)  # strictly monotone
        if len(set(v.tolist())) == len(set(w.tolist())):
            assert list(O.topk(w, jb, n, K)) == list(O.topk(v, jb, n, K))


def test_select_unit_small_candidate_sets():
    rng = np.random.default_rng(10)
    q = bits(rng.standard_normal((4, 128)))
    summ = bits(rng.standard_normal((20, 2, 128)))
    assert list(O.select_unit(q, summ, 4, 4, 8)) == [-1] * 8          # J empty
    assert list(O.select_unit(q, summ, 4, 9, 8)) == [4, 5, 6, 7, 8, -1, -1, -1]  # |J| <= K


# ------------------------------------------------- correction
def test_cosine_special_cases():
    rng = np.random.default_rng(11)
    a = bits(rng.standard_normal(128))
    assert abs(O.cosine(a, a) - 1.0) <= 2 ** -22
    neg = a ^ np.uint16(0x8000)
    assert abs(O.cosine(a, neg) + 1.0) <= 2 ** -22
    assert O.cosine(bits([1, 0]), bits([0, 1])) == 0.0
    assert O.cosine(np.zeros(128, np.uint16), a) == 0.0
    b = bits(rng.standard_normal(128))
    af, bf = O.bf16_to_f32(a).astype(np.float64), O.bf16_to_f32(b).astype(np.float64)
    assert abs(O.cosine(a, b) - af @ bf / np.linalg.norm(af) / np.linalg.norm(bf)) < 1e-6


def test_correction_paper_example():
    # P:250 (fig:algo2): KV head with mean similarity 0.75 (< tau = 0.8) is flagged
    f, c = O.pool_correct([0.7, 0.8], 0.8)
    assert f == 1 and abs(c - 0.75) < 1e-7
    f, c = O.pool_correct([0.8, 0.9], 0.8)
    assert f == 0 and abs(c - 0.85) < 1e-7
    # tau edges, P:661-665 (tab:abl-tau) and A-13
    assert O.pool_correct([-1.0, -1.0], 0.0)[0] == 0
    assert O.pool_correct([1.0, 1.0], 1.0)[0] == 1
    assert O.pool_correct([0.1], 0.8, O.MODE_NEVER)[0] == 0
    assert O.pool_correct([0.99], 0.8, O.MODE_ALWAYS)[0] == 1
    q = bits(np.ones((2, 4)))
    assert O.correct_unit(q, q, 0.8, O.MODE_SPECULATIVE, bootstrap=True)[0] == 1
    assert O.correct_unit(q, q, 0.8, O.MODE_SPECULATIVE, bootstrap=False)[0] == 0


# ------------------------------------------------------ attention
def _sdpa64(q, K, V):
    qf = torch.from_numpy(O.bf16_to_f32(q).astype(np.float64))[None, :, None, :]
    Kf = torch.from_numpy(O.bf16_to_f32(K).astype(np.float64))[None, None]
    Vf = torch.from_numpy(O.bf16_to_f32(V).astype(np.float64))[None, None]
    G = q.shape[0]
    o = torch.nn.functional.scaled_dot_product_attention(qf, Kf.expand(1, G, -1, -1), Vf.expand(1, G, -1, -1))
    return o[0, :, 0].numpy()


def test_attention_special_cases():
    rng = np.random.default_rng(12)
    q = bits(rng.standard_normal((4, 128)))
    K = bits(rng.standard_normal((50, 128)))
    V = bits(rng.standard_normal((50, 128)))
    o = O.attn_unit(q, K, V, [7])
    assert np.array_equal(o, np.broadcast_to(O.bf16_to_f32(V[7]).astype(np.float64), o.shape))
    Ks = np.broadcast_to(K[3], K.shape).copy()
    o = O.attn_unit(q, Ks, V, np.arange(50))
    assert np.allclose(o, O.bf16_to_f32(V).astype(np.float64).mean(0), atol=1e-12)
    toks = rng.permutation(50)[:31]
    o1 = O.attn_unit(q, K, V, toks)
    o2 = O.attn_unit(q, K, V, toks[::-1].copy())
    assert np.allclose(o1, o2, atol=1e-12)
    ref = _sdpa64(q, K[toks], V[toks])
    assert np.allclose(o1, ref, atol=1e-12)


# ------------------------------------------- state machine (T1)
def _t1_engine(tau=0.8, mode=O.MODE_SPECULATIVE):
    cfg = O.OracleConfig(n_layers=1, batch=1, n_qo=2, n_kv=1, head_dim=2, page_size=2,
                         budget_tokens=6, sink_tokens=2, window_tokens=2, max_ctx_tokens=16,
                         tau=tau, mode=mode)
    return O.OracleEngine(cfg)


def test_t1_transcript(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "t1_transcript.json")))
    eng = _t1_engine()
    pk = bits(g["prefill_keys"])
    eng.append(0, pk[None, :, None, :], pk[None, :, None, :])
    for i, exp in enumerate(g["expected"]):
        k = bits([g["step_keys"][i]])
        q = bits(g["queries"][i])[None]
        r = eng.step(0, q, k[None, :, None, :], k[None, :, None, :])
        assert eng.Lc[0] == exp["Lc"]
        assert int(r["frontier"][0]) == exp["n_off"]
        assert int(r["flags"][0]) == exp["flag"]
        if exp["cbar"] is not None:
            assert abs(float(r["cbar"][0]) - exp["cbar"]) < g["tol"]
        assert [j for j in r["sel"][0] if j >= 0] == exp["sel"]
        assert r["used_sel"][0] == exp["used_sel"] and r["used_f"][0] == exp["used_f"]
        toks = eng.token_set(0, 0, r["used_sel"][0], r["used_f"][0])
        assert sorted(toks.tolist()) == exp["tokens"]
        assert r["fetch_sync"][0] == exp["fetch_sync"] and r["fetch_bg"][0] == exp["fetch_bg"]
        sel, pooled = O.select_unit(q[0], eng.summ[0][0], 1, exp["n_off"], 1, want_pooled=True)
        for j, v in exp["pooled"].items():
            assert abs(float(pooled[int(j)]) - v) < g["tol"]


def _run_engine(mode, tau, budget, steps=6, G=4, n_kv=2, batch=2, L0=200, event_rate=0.3, seed=5,
                first_layer_dense=False, n_layers=1):
    import synth
    d, page = 128, 16
    cfg = O.OracleConfig(n_layers=n_layers, batch=batch, n_qo=G * n_kv, n_kv=n_kv, head_dim=d,
                         page_size=page, budget_tokens=budget, sink_tokens=32, window_tokens=32,
                         max_ctx_tokens=L0 + steps + 1, tau=tau, mode=mode,
                         first_layer_dense=first_layer_dense)
    eng = O.OracleEngine(cfg)
    hist = []
    for layer in range(n_layers):
        k, v = synth.gen_prefill(batch, n_kv, d, page, L0, 2, cfg.K, seed, layer)
        eng.append(layer, synth.bf16_bits(k), synth.bf16_bits(v))
    qp = [synth.QueryProcess(batch, G * n_kv, n_kv, d, seed, layer, event_rate=event_rate)
          for layer in range(n_layers)]
    for i in range(steps):
        for layer in range(n_layers):
            q, ev = qp[layer].next()
            k, v = synth.gen_decode_kv(batch, n_kv, d, page, L0 + i, seed, layer)
            r = eng.step(layer, synth.bf16_bits(q), synth.bf16_bits(k), synth.bf16_bits(v))
            r["events"] = ev.numpy().reshape(-1)
            r["q"] = synth.bf16_bits(q)
            hist.append((layer, r))
    return eng, hist


@pytest.mark.parametrize("mode,tau", [(O.MODE_SPECULATIVE, 0.8), (O.MODE_ALWAYS, 1.0), (O.MODE_NEVER, 0.0)])
def test_dense_equivalence_all_modes(mode, tau):
    """Budget >= context => sparse attention == dense attention (north star)."""
    eng, hist = _run_engine(mode, tau, budget=4096, steps=4)
    for layer, r in hist:
        Lc = r["Lc"]
        for u in range(eng.U):
            b, m = divmod(u, eng.cfg.n_kv)
            G = eng.cfg.G
            q = r["q"][b, m * G:(m + 1) * G]
            ref = _sdpa64(q, eng.Kc[layer][u, :Lc], eng.Vc[layer][u, :Lc])
            assert np.allclose(r["out"][b, m * G:(m + 1) * G], ref, atol=1e-10)


def test_tau1_is_synchronous_and_tau0_is_lag_one():
    _, h1 = _run_engine(O.MODE_SPECULATIVE, 1.0, budget=128, steps=5)
    for _, r in h1:
        assert all(r["flags"] == 1)
        for u, us in enumerate(r["used_sel"]):
            assert us == [j for j in r["sel"][u] if j >= 0]
    _, h0 = _run_engine(O.MODE_SPECULATIVE, 0.0, budget=128, steps=5)
    for i in range(1, len(h0)):
        prev, cur = h0[i - 1][1], h0[i][1]
        assert all(cur["flags"] == 0)
        for u, us in enumerate(cur["used_sel"]):
            assert us == [j for j in prev["sel"][u] if j >= 0]
            assert cur["used_f"][u] == prev["frontier"][u]


def test_scheduled_dips_fire_exactly():
    """GEN-Q events (cos ~0.05) fire corrections; smooth steps (cos ~0.9) do not."""
    _, hist = _run_engine(O.MODE_SPECULATIVE, 0.8, budget=128, steps=12, event_rate=0.25)
    n_ev = 0
    for i, (_, r) in enumerate(hist):
        if i == 0:
            assert all(r["flags"] == 1)
            continue
        assert np.array_equal(r["flags"].astype(bool), r["events"])
        n_ev += int(r["events"].sum())
    assert n_ev > 0


def test_first_layer_dense():
    eng, hist = _run_engine(O.MODE_SPECULATIVE, 0.8, budget=128, steps=2, n_layers=2,
                            first_layer_dense=True)
    for layer, r in hist:
        if layer != 0:
            continue
        Lc = r["Lc"]
        for u in range(eng.U):
            b, m = divmod(u, eng.cfg.n_kv)
            G = eng.cfg.G
            ref = _sdpa64(r["q"][b, m * G:(m + 1) * G], eng.Kc[0][u, :Lc], eng.Vc[0][u, :Lc])
            assert np.allclose(r["out"][b, m * G:(m + 1) * G], ref, atol=1e-10)


# ---- group-consistency variants (tab:abl-g-cons) ----------
def _rand_unit(rng, G, d, n_pages):
    q = O.f32_to_bf16(rng.standard_normal((G, d)).astype(np.float32))
    summ = O.f32_to_bf16(np.sort(rng.standard_normal((n_pages, 2, d)).astype(np.float32), axis=1))
    return q, summ


def _variant_pooled_fp64(q, summ, n_sink, n_off, pool):
    """The variant's pooled page weights, written from the paper's definitions in fp64 (independent of
    the oracle): Q = pool the query vectors, QK = pool the page scores, S = pool the softmax weights."""
    qf = O.bf16_to_f32(q).astype(np.float64)
    mn = O.bf16_to_f32(summ[:, 0]).astype(np.float64)[n_sink:n_off]
    mx = O.bf16_to_f32(summ[:, 1]).astype(np.float64)[n_sink:n_off]
    d = qf.shape[1]

    def bound(qv):  # Quest upper bound of q.k over the page (A-1)
        return np.maximum(qv[None, :] * mn, qv[None, :] * mx).sum(axis=1) / math.sqrt(d)

    def softmax(x):
        e = np.exp(x - x.max())
        return e / e.sum()

    if pool in (O.POOL_MEAN_Q, O.POOL_MAX_Q):
        qp = qf.mean(axis=0) if pool == O.POOL_MEAN_Q else qf.max(axis=0)
        return softmax(bound(qp))
    s = np.stack([bound(qf[g]) for g in range(qf.shape[0])])  # [G][pages]
    if pool in (O.POOL_MEAN_QK, O.POOL_MAX_QK):
        return softmax(s.mean(axis=0) if pool == O.POOL_MEAN_QK else s.max(axis=0))
    p = np.stack([softmax(s[g]) for g in range(s.shape[0])])
    return p.sum(axis=0) if pool == O.POOL_MEAN_S else p.max(axis=0)


@pytest.mark.parametrize("pool", range(6))
def test_pooling_variants_match_fp64_definitions(pool):
    """Each pooling variant's top-K equals the top-K of its fp64 definition whenever the K-th and
    (K+1)-th pooled weights are well separated (no near-tie for fp32 to flip)."""
    rng = np.random.default_rng(100 + pool)
    checked = 0
    for trial in range(40):
        G = [2, 4, 7, 8][trial % 4]
        n_sink, n_off, K = 2, 200 + 13 * trial, 16
        q, summ = _rand_unit(rng, G, 128, n_off)
        ref = _variant_pooled_fp64(q, summ, n_sink, n_off, pool)
        order = np.argsort(-ref, kind="stable")
        if ref[order[K - 1]] - ref[order[K]] < 1e-5 * ref[order[K - 1]]:
            continue
        want = np.sort(order[:K] + n_sink)
        got = O.select_unit_pool(q, summ, n_sink, n_off, K, pool)
        assert np.array_equal(got, want), (pool, trial)
        checked += 1
    assert checked >= 20


def test_pooling_variants_coincide_for_one_head():
    """With G = 1 every pooling is the identity, so all six variants select MeanS's pages."""
    rng = np.random.default_rng(7)
    for trial in range(10):
        q, summ = _rand_unit(rng, 1, 128, 300)
        base = O.select_unit(q, summ, 2, 300, 24)
        for pool in range(1, 6):
            assert np.array_equal(O.select_unit_pool(q, summ, 2, 300, 24, pool), base), pool


def test_pooling_variants_differ_from_means():
    """The variants are real alternatives: on random units each one disagrees with MeanS somewhere."""
    rng = np.random.default_rng(11)
    units = [_rand_unit(rng, 4, 128, 300) for _ in range(8)]
    for pool in range(1, 6):
        assert any(not np.array_equal(O.select_unit_pool(q, s, 2, 300, 16, pool), O.select_unit(q, s, 2, 300, 16))
                   for q, s in units), pool


def test_correction_pooling_max_reading():
    """Max-pooled correction (tab:abl-g-corr; reading R-11): a unit is corrected when any head's
    similarity is below tau, so it corrects at least as often as mean pooling."""
    rng = np.random.default_rng(5)
    n_mean = n_max = 0
    for _ in range(2000):
        G = int(rng.integers(1, 9))
        C = rng.uniform(0.5, 1.0, G).astype(np.float32)
        f_max, c_max = O.pool_correct_v(C, 0.8, O.MODE_SPECULATIVE, 1)
        f_mean, _ = O.pool_correct_v(C, 0.8, O.MODE_SPECULATIVE, 0)
        assert f_max == int(bool((C < np.float32(0.8)).any()))
        assert c_max == C.min()
        assert f_max >= f_mean
        n_mean += f_mean
        n_max += f_max
    assert n_max > n_mean
