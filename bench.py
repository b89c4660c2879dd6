#!/usr/bin/env python
"""Benchmark of the FreeKV decode-step KV-retrieval path on B200.

A step = one decode step of the whole hot path
for every layer of the configured model shape over one batch of synthetic
inputs.  Default workload: BASELINE.json configs[1] (Llama-3.1-8B shape,
32 layers, 32q/8kv heads, 32K context, batch 8, budget 2048, S = W = 512,
tau = 0.8, 5% scheduled correction events).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0]: parity/latency case (S = W = 128 -> K = 8, reading A-8)
    "c1": dict(workload="llama3.1-8b-heads-1layer-ctx4k-b1", n_layers=1, batch=1, n_qo=32, n_kv=8, ctx=4096,
               budget=2048 // 4, sink=128, window=128, tau=0.8, event_rate=0.05),
    # BASELINE.json configs[1]: the headline (metric is quoted on it)
    "c2": dict(workload="llama3.1-8b-32layers-ctx32k-b8-budget2048", n_layers=32, batch=8, n_qo=32, n_kv=8,
               ctx=32768, budget=2048, sink=512, window=512, tau=0.8, event_rate=0.05),
    # BASELINE.json configs[2]
    "c3": dict(workload="qwen2.5-7b-28layers-ctx128k-b4-budget2048", n_layers=28, batch=4, n_qo=28, n_kv=4,
               ctx=131072, budget=2048, sink=512, window=512, tau=0.8, event_rate=0.05),
    # BASELINE.json configs[3]: DeepSeek-R1-Distill-Llama-8B shape (Llama-3.1-8B heads, 32 layers) at
    # the end of 16K prompt + 32K generated tokens; batch 8 (the paper states none); --tau sweeps
    # the correction threshold
    "c4": dict(workload="r1-distill-llama-8b-32layers-ctx48k-b8-budget2048", n_layers=32, batch=8, n_qo=32,
               n_kv=8, ctx=49152, budget=2048, sink=512, window=512, tau=0.8, event_rate=0.05),
    # BASELINE.json configs[4]: Llama-3.1-70B heads (64q/8kv), 80 layers, ctx 128K, batch 16.  Host KV for
    # 80 layers is 640 GiB at one GPU, so l_inst = 4 layers are instantiated and the step graph cycles
    # through them (virtual layer v runs layer v % 4; SURVEY §7 hard part 9)
    "c5": dict(workload="llama3.1-70b-80layers-ctx128k-b16-budget2048", n_layers=80, batch=16, n_qo=64, n_kv=8,
               ctx=131072, budget=2048, sink=512, window=512, tau=0.8, event_rate=0.05, l_inst=4),
}

METRIC = "decode-step µs/layer and tokens/s at 32K ctx; attn HBM GB/s; recall GB/s vs host link"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--profile-steps", type=int, default=8)
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--tau", type=float, default=None, help="correction threshold (default: the config's)")
    ap.add_argument("--eager", action="store_true", help="per-layer C-ABI calls instead of the whole-step graph")
    ap.add_argument("--gen", default="S", choices=["S", "spec", "X"],
                    help="input generator: S = GEN-S/GEN-Q as tuned (alpha 8, beta 6; the headline), spec = the "
                         "survey's GEN-S parameters (alpha 4, beta 2.5), X = unstructured i.i.d. keys and queries")
    ap.add_argument("--full-refresh", action="store_true",
                    help="every unit re-fetches all K pages every step (recall stress; FREEKV_DEBUG_FULL_REFRESH)")
    ap.add_argument("--n-layers", type=int, default=None, help="override the config's layer count")
    ap.add_argument("--nested", action="store_true",
                    help="sub-measurement run: no isolated-kernel, end-to-end, exposed-recall or CPU passes")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the nested survey-spec GEN-S and GEN-X full-refresh lines")
    return ap.parse_args()


GEN = {  # (alpha, beta, rho, event_rate or None = the config's)
    "S": (None, None, None, None),
    "spec": (4.0, 2.5, None, None),   # SURVEY §8(d) GEN-S as specified
    "X": (0.0, 0.0, 0.0, 0.0),        # GEN-X: no topic, no persistence -> every unit corrects every step
}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every ~2 ms through NVML during
    the timed region (nvidia-smi as a fallback when NVML is unavailable)."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
             "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.active = False
        self.stop_flag = False
        self.err = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"

    def _loop(self):
        N = self.N
        while not self.stop_flag:
            if self.active:
                try:
                    sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((sm, rs))
                except Exception as e:  # noqa: BLE001
                    self.err = str(e)
            time.sleep(0.002)

    def mark(self):
        """Start of the timed region."""
        self.active = True

    def stop(self):
        self.active = False
        self.stop_flag = True
        if self.err and not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err]}
        reasons = set()
        for _, rs in self.samples:
            for name, attr in self.NAMES.items():
                bit = getattr(self.N, attr, 0)
                if bit and (rs & bit):
                    reasons.add(name)
        sm = [x for x, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}


# ----------------------------------------------------------------- workload
def build_handle(P, c, n_kv_loc, n_qo_loc, max_ctx, stream=None):
    cfg = P.FreeKVConfig(n_layers=c["n_layers"], batch=c["batch"], n_qo=n_qo_loc, n_kv=n_kv_loc, head_dim=128,
                         page_size=32, budget_tokens=c["budget"], sink_tokens=c["sink"], window_tokens=c["window"],
                         max_ctx_tokens=max_ctx, tau=c["tau"], mode=P.MODE_SPECULATIVE)
    return cfg, P.FreeKV(cfg, compute_stream=stream)


def host_link_peak(torch, nbytes=256 << 20, reps=6):
    """Pinned H2D cudaMemcpyAsync peak (the recall roofline denominator), measured in this run."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 1e9
    s = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        d.copy_(h, non_blocking=True)
        b.record(s)
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    del h, d
    return nbytes / best / 1e9


def run_ours(args, c, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2505_13109_b200 as P
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    seed = args.seed if args.seed is not None else synth.SEED0 + 1 + list(CONFIGS).index(args.config)
    n_kv, n_qo, nb, d = c["n_kv"], c["n_qo"], c["batch"], 128
    G = n_qo // n_kv
    # KV-head (then batch) sharding, SURVEY §8(e)
    from paper_2505_13109_b200.shard import shard_for
    sh = shard_for(n_kv, nb, world, rank)
    kv_loc, kv0 = sh.n_kv, sh.kv_begin
    b0, b1 = sh.batch_begin, sh.batch_end
    nb_loc = sh.batch
    n_layers = c["n_layers"]                          # virtual layers of the step
    n_inst = min(c.get("l_inst", n_layers), n_layers)  # instantiated layers (handle)
    tok_per_step = (n_layers + n_inst - 1) // n_inst   # tokens each instantiated layer appends per step
    alpha, beta, rho, ev_rate = GEN[args.gen]
    gkw = {} if alpha is None else {"alpha": alpha}
    qkw = {}
    if beta is not None:
        qkw["beta"] = beta
    if rho is not None:
        qkw["rho"] = rho
    event_rate = c["event_rate"] if ev_rate is None else ev_rate
    if args.full_refresh:
        os.environ["FREEKV_DEBUG_FULL_REFRESH"] = "1"
    exp_steps = 0 if (args.nested or world > 1) else min(args.steps, 64)
    # warm, timed, exposed-recall pair, profiled x2, e2e
    total_steps = args.warmup + 1 + args.steps + 2 * (exp_steps + 2) + 2 * args.profile_steps + \
        (0 if args.nested else args.steps)
    # the prefill leaves room for every step of the run, so the context never exceeds the config's
    # (the select tree is sized for max_ctx: P2 = next_pow2(max pages))
    L0 = c["ctx"] - total_steps * tok_per_step
    max_ctx = c["ctx"] + 1
    stream = torch.cuda.Stream(dev, priority=-1)  # compute outranks the background recall stream
    from paper_2505_13109_b200.numa import bind_to_gpu_node
    numa = bind_to_gpu_node(local_rank)  # the pinned host shard below lands on the GPU's NUMA node
    t0 = time.time()
    cfg, fkv = build_handle(P, dict(c, batch=nb_loc, n_layers=n_inst), kv_loc, kv_loc * G, max_ctx, stream)
    t_alloc = time.time() - t0
    K = cfg.K
    p = 32
    # ---- prefill every layer (GEN-S keys, seeded from global ids, identical for any world size)
    t0 = time.time()
    with torch.cuda.stream(stream):
        for layer in range(n_inst):
            k, v = synth.gen_prefill(nb, n_kv, d, p, L0, c["sink"] // p, K, seed, layer, device=dev, **gkw)
            fkv.append_kv(layer, k[b0:b1, :, kv0:kv0 + kv_loc].contiguous(),
                          v[b0:b1, :, kv0:kv0 + kv_loc].contiguous())
            del k, v
    stream.synchronize()
    t_prefill = time.time() - t0
    # ---- pre-generate every step's inputs (GEN-Q / GEN-S) outside the timed regions
    # one query process / token stream per instantiated layer: with layer cycling its successive
    # occurrences are successive decode steps of that layer (the correction statistics of a model
    # whose every layer is stepped once per token)
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, layer, device=dev, event_rate=event_rate, **qkw)
           for layer in range(n_inst)]
    Qs = torch.empty(total_steps, n_layers, nb_loc, kv_loc * G, d, dtype=torch.bfloat16, device=dev)
    Ks = torch.empty(total_steps, n_layers, nb_loc, 1, kv_loc, d, dtype=torch.bfloat16, device=dev)
    Vs = torch.empty_like(Ks)
    with torch.cuda.stream(stream):
        for i in range(total_steps):
            for layer in range(n_layers):
                li, occ = layer % n_inst, layer // n_inst  # instantiated layer, occurrence in the step
                q, _ = qps[li].next()
                kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i * tok_per_step + occ, seed, li, device=dev,
                                             **gkw)
                Qs[i, layer] = q[b0:b1, kv0 * G:(kv0 + kv_loc) * G]
                Ks[i, layer] = kn[b0:b1, :, kv0:kv0 + kv_loc]
                Vs[i, layer] = vn[b0:b1, :, kv0:kv0 + kv_loc]
    out_loc = [torch.empty(nb_loc, kv_loc * G, d, dtype=torch.float32, device=dev) for _ in range(n_layers)]
    comm_info = None
    if world > 1:
        # the library's own NCCL communicator (id from rank 0, broadcast over the torch process
        # group); every layer's step then ends with its all-gather of the head outputs on the
        # compute stream, inside the step graph (the one exchange step)
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.tensor(list(P.FreeKV.comm_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        fkv.comm_init(bytes(uid.cpu().tolist()), world, rank)
        gather_all = torch.empty(n_layers, world, nb_loc, kv_loc * G, d, dtype=torch.float32, device=dev)
        fkv.set_gather_output(gather_all)
        comm_info = {"ranks": world, "collective": "ncclAllGather per layer (library communicator, in the step graph)",
                     "bytes_per_layer_per_rank": nb_loc * kv_loc * G * d * 4}
        print(f"[rank {rank}/{world}] freekv NCCL communicator ready: kv heads [{kv0}, {kv0 + kv_loc}) x batch "
              f"[{b0}, {b1}), all-gather {comm_info['bytes_per_layer_per_rank']} B per layer", file=sys.stderr)
    stream.synchronize()

    def one_step(i):
        for layer in range(n_layers):
            fkv.decode_step(layer % n_inst, Qs[i, layer], Ks[i, layer], Vs[i, layer], out_loc[layer])

    def capture(profile=0):
        if n_inst == n_layers:
            fkv.step_graph_capture(q_buf, k_buf, v_buf, o_buf, profile=profile)
        else:
            fkv.step_graph_capture_cycle(n_layers, q_buf, k_buf, v_buf, o_buf, profile=profile)

    # whole-step graph: fixed input/output buffers, one replay per step
    q_buf, k_buf, v_buf = torch.empty_like(Qs[0]), torch.empty_like(Ks[0]), torch.empty_like(Vs[0])
    o_buf = torch.empty(n_layers, nb_loc, kv_loc * G, d, dtype=torch.float32, device=dev)

    def graph_step(i):
        with torch.cuda.stream(stream):
            q_buf.copy_(Qs[i], non_blocking=True)
            k_buf.copy_(Ks[i], non_blocking=True)
            v_buf.copy_(Vs[i], non_blocking=True)
        fkv.step_graph_launch()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    clocks = ClockSampler(local_rank)
    clocks.start()
    step = 0
    for _ in range(args.warmup):
        one_step(step)
        step += 1
    fkv.synchronize()
    if not args.eager:
        capture()
        graph_step(step)  # first replay (instantiation warm-up) is a warm-up step too
        step += 1
        fkv.synchronize()
    run = one_step if args.eager else graph_step
    # ---- timed region (device time, CUDA events on the compute stream)
    clocks.mark()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        run(step)
        step += 1
    ev1.record(stream)
    fkv.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # ---- exposed recall (the background recall should hide behind compute):
    # the same step graph with and without its background-recall branches, back to back over the
    # same number of steps.  Without recall the selections (from the summaries) are unchanged but
    # the next step's resident pages are stale -- a timing-only pass, never a parity or bench value.
    exposed = None
    if exp_steps and not args.eager:
        def timed_steps(n):
            nonlocal step
            fkv.step_graph_launch()  # one untimed replay of the freshly captured graph
            step += 1
            fkv.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(n):
                graph_step(step)
                step += 1
            b.record(stream)
            b.synchronize()
            return a.elapsed_time(b)
        os.environ["FREEKV_DEBUG_NO_RECALL"] = "1"
        capture()
        ms_nr = timed_steps(exp_steps)
        os.environ.pop("FREEKV_DEBUG_NO_RECALL")
        capture()
        ms_wr = timed_steps(exp_steps)
        exposed = {"exposed_recall_us_per_layer": round((ms_wr - ms_nr) / exp_steps / n_layers * 1e3, 3),
                   "us_per_layer_with_recall": round(ms_wr / exp_steps / n_layers * 1e3, 3),
                   "us_per_layer_without_recall": round(ms_nr / exp_steps / n_layers * 1e3, 3),
                   "steps": exp_steps,
                   "method": "step graph with vs without its background-recall branches (FREEKV_DEBUG_NO_RECALL), "
                             "back to back on the same inputs; selections identical (summaries unchanged)"}
    # ---- profiled passes.  (a) roofline: the step graph re-captured with an event-record
    # node pair around every attention-split kernel only (the dominant kernel; the other
    # kernels keep their PDL edges), so each bracketed interval is that launch's device time
    # on the stream it runs on; (b) per-kernel table: every kernel bracketed (event nodes
    # then break every PDL overlap, so these are per-kernel durations, not the critical
    # path -- that is the timed region above).  Eager mode: the library's event profiler.
    import paper_2505_13109_b200.freekv as FK
    cls = {k: i for i, k in enumerate(FK.KERNEL_CLASSES)}
    fetched = fetched_sync = flagged = units = t_unit_tokens = j_pages = 0
    t_tok_p1 = t_tok_p2 = units_p1 = 0

    def sel_stats():
        nonlocal fetched, fetched_sync, flagged, units, t_unit_tokens, j_pages, t_tok_p1, t_tok_p2, units_p1
        for layer in range(n_inst):
            n_fetch, _ = fkv.get_fetch(layer)
            sel = fkv.get_selection(layer)
            fl = sel["flags"].astype(bool)
            # background recall (rs stream) moves the unflagged units' fetches; a corrected unit's
            # fetched pages are read from the host pool by the attention kernel itself (direct mode)
            fetched += int(n_fetch[~fl].sum())
            fetched_sync += int(n_fetch[fl].sum())
            flagged += int(fl.sum())
            units += fkv.U
            Lc = fkv.context(layer)
            n_off = max(c["sink"] // p, Lc // p - c["window"] // p)
            n_sel = (sel["pages"] >= 0).sum(axis=1)
            # |T| per unit = sink + selected pages + local [f*p, Lc) (A-9); f = this step's frontier
            f_used = sel["frontier"].astype(np.int64)
            tu = min(c["sink"], Lc) + n_sel * p + (Lc - f_used * p)
            t_unit_tokens += int(tu.sum())
            t_tok_p1 += int(tu[~fl].sum())
            t_tok_p2 += int(tu[fl].sum())
            units_p1 += int((~fl).sum())
            j_pages += fkv.U * (n_off - c["sink"] // p)

    def profiled(mask):
        nonlocal step
        acc = {k: [0.0, 0] for k in FK.KERNEL_CLASSES}
        if args.eager:
            fkv.synchronize()
            fkv.profile_begin(args.profile_steps * n_layers * 12 + 64)
        else:
            capture(profile=mask)
        for _ in range(args.profile_steps):
            if args.eager:
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(4_000_000)  # host runs ahead: events bracket kernels, not launch gaps
            run(step)
            fkv.synchronize()
            if not args.eager:
                for kc, (t, n) in fkv.step_graph_profile().items():
                    acc[kc][0] += t
                    acc[kc][1] += n
            if mask != 1:
                sel_stats()
            step += 1
        if args.eager:
            acc = {k: list(v) for k, v in fkv.profile_end().items()}
        return {k: tuple(v) for k, v in acc.items()}

    roof_prof = profiled((1 << cls["attn_split"]) | (1 << cls["attn_split_phase2"]))
    prof = profiled(1)
    # (c) the dominant kernel alone: the last layer's attention (its page lists are the last
    # ones the select wrote; the launch is idempotent) re-launched through the public API
    # after a 256 MB write that evicts L2 (cold KV, as in the step), bracketed by CUDA events
    # on its stream; a device sleep first keeps the host ahead so the events bracket the
    # kernels, not launch gaps
    iso_ms, iso_ms_dirty, iso_score = [], [], None
    if world == 1 and not args.nested:
        fkv.synchronize()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        # the write leaves L2 full of dirty lines whose write-back would be charged to the
        # kernel's reads (the step's L2 holds mostly clean lines: summaries, KV, pages); a read of
        # another 256 MB replaces them with clean lines before each timed launch
        flush_r = torch.ones(64 << 20, dtype=torch.float32, device=dev)
        flush_acc = torch.empty((), dtype=torch.float32, device=dev)
        o_tmp = torch.empty(nb_loc, kv_loc * G, d, dtype=torch.float32, device=dev)
        q_last = Qs[step - 1, n_layers - 1]
        # (a) scoring: select_pages of the last layer (score + select kernels; the page lists of
        # every unit, which the isolated attention launches below read) under the library's event
        # profiler (CUDA events on the launching stream around each kernel), L2 flushed before each
        fkv.profile_begin(64)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(2_000_000)
            for _ in range(8):
                flush.fill_(1)
                torch.sum(flush_r, dim=0, out=flush_acc)
                fkv.select_pages(n_inst - 1, q_last, stream=stream)
        iso_score = fkv.profile_end()
        # (b) the dominant kernel alone: the attention of the last layer over those page lists
        # (idempotent: it commits the same selection), bracketed by CUDA events on its stream
        for clean in (False, True):  # dirty-L2 variant kept for comparison (iso_ms_dirty)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
            with torch.cuda.stream(stream):
                torch.cuda._sleep(2_000_000)
                for ea, eb in evs:
                    flush.fill_(1)
                    if clean:
                        torch.sum(flush_r, dim=0, out=flush_acc)
                    ea.record(stream)
                    fkv.sparse_decode_attn(n_inst - 1, q_last, o_tmp, stream=stream)
                    eb.record(stream)
            stream.synchronize()
            if clean:
                iso_ms = [ea.elapsed_time(eb) for ea, eb in evs]
            else:
                iso_ms_dirty = [ea.elapsed_time(eb) for ea, eb in evs]
        del flush, flush_r
    link = host_link_peak(torch) if rank == 0 else None
    res = dict(ms=ms, ms_e2e=None, prof=prof, roof_prof=roof_prof, iso_ms=iso_ms, iso_ms_dirty=iso_ms_dirty,
               iso_score=iso_score, fetched=fetched, fetched_sync=fetched_sync, flagged=flagged, units=units,
               t_unit_tokens=t_unit_tokens, j_pages=j_pages, t_tok_p1=t_tok_p1, t_tok_p2=t_tok_p2, units_p1=units_p1,
               clocks=clk, link=link, t_alloc=t_alloc, t_prefill=t_prefill, h2d=0, d2h=0, K=K, G=G, kv_loc=kv_loc,
               nb_loc=nb_loc, seed=seed, exposed=exposed, n_layers=n_layers, comm=comm_info, n_inst=n_inst,
               numa=numa)
    if args.nested:
        fkv.close()
        return res
    if not args.eager:  # plain graph again for the end-to-end pass
        capture()
    # ---- end-to-end pass: inputs from pinned host memory, outputs back to host, every step
    Qh = Qs[step:step + args.steps].cpu().pin_memory()
    Kh = Ks[step:step + args.steps].cpu().pin_memory()
    Vh = Vs[step:step + args.steps].cpu().pin_memory()
    host_out = torch.empty(n_layers, nb_loc, kv_loc * G, d, dtype=torch.float32, pin_memory=True)
    h2d = (Qh[0].numel() + Kh[0].numel() + Vh[0].numel()) * 2
    d2h = host_out.numel() * 4
    # pipelined like a serving loop: the H2D of step i+1's inputs (copy stream, into one of two
    # device staging sets) overlaps step i, and the D2H of step i's outputs overlaps step i+1;
    # the compute stream only does the two device-to-device hand-offs.  Every transfer is
    # inside the timed region (the end event waits for the last D2H).
    copy_s = torch.cuda.Stream(dev)
    st_in = [(torch.empty_like(q_buf), torch.empty_like(k_buf), torch.empty_like(v_buf)) for _ in range(2)]
    st_out = [torch.empty_like(o_buf) for _ in range(2)]
    host_outs = [host_out, torch.empty_like(host_out).pin_memory()]
    ev = lambda: torch.cuda.Event()
    in_ready, in_free, out_ready, out_done = [ev(), ev()], [ev(), ev()], [ev(), ev()], [ev(), ev()]
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    copy_s.wait_stream(stream)

    def stage_inputs(i):
        sq, sk, sv = st_in[i % 2]
        with torch.cuda.stream(copy_s):
            if i >= 2:
                copy_s.wait_event(in_free[i % 2])
            sq.copy_(Qh[i], non_blocking=True)
            sk.copy_(Kh[i], non_blocking=True)
            sv.copy_(Vh[i], non_blocking=True)
            in_ready[i % 2].record(copy_s)

    stage_inputs(0)
    for i in range(args.steps):
        if i + 1 < args.steps:
            stage_inputs(i + 1)
        sq, sk, sv = st_in[i % 2]
        with torch.cuda.stream(stream):
            stream.wait_event(in_ready[i % 2])
            q_buf.copy_(sq, non_blocking=True)
            k_buf.copy_(sk, non_blocking=True)
            v_buf.copy_(sv, non_blocking=True)
            in_free[i % 2].record(stream)
        if args.eager:
            for layer in range(n_layers):
                fkv.decode_step(layer % n_inst, q_buf[layer], k_buf[layer], v_buf[layer], o_buf[layer])
        else:
            fkv.step_graph_launch()
        with torch.cuda.stream(stream):
            if i >= 2:
                stream.wait_event(out_done[i % 2])
            st_out[i % 2].copy_(o_buf, non_blocking=True)
            out_ready[i % 2].record(stream)
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(out_ready[i % 2])
            host_outs[i % 2].copy_(st_out[i % 2], non_blocking=True)
            out_done[i % 2].record(copy_s)
        step += 1
    stream.wait_stream(copy_s)
    e1.record(stream)
    fkv.synchronize()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_e2e = float(t.item())
    res.update(ms_e2e=ms_e2e, h2d=h2d, d2h=d2h)
    fkv.close()
    return res


# ------------------------------------------------------------ CPU oracle arm
def run_oracle_sample(c, seconds, seed):
    """Time the CPU oracle on a bounded sample of the workload: one layer, the KV
    heads of batch row 0 (n_kv units), at the full context, decode steps until
    ~`seconds` of CPU work; extrapolate to tokens/s of the full configuration."""
    import numpy as np

    import synth
    from oracle import oracle as O
    n_kv, n_qo, d, p = c["n_kv"], c["n_qo"], 128, 32
    nb = c["batch"]
    steps_max = 256
    ocfg = O.OracleConfig(n_layers=1, batch=nb, n_qo=n_qo, n_kv=n_kv, head_dim=d, page_size=p,
                          budget_tokens=c["budget"], sink_tokens=c["sink"], window_tokens=c["window"],
                          max_ctx_tokens=c["ctx"] + steps_max + 1, tau=c["tau"])
    eng = O.OracleEngine(ocfg)
    K = ocfg.K
    k, v = synth.gen_prefill(nb, n_kv, d, p, c["ctx"], c["sink"] // p, K, seed, 0)
    eng.append(0, synth.bf16_bits(k), synth.bf16_bits(v))
    del k, v
    qp = synth.QueryProcess(nb, n_qo, n_kv, d, seed, 0, event_rate=c["event_rate"])
    t0 = time.perf_counter()
    n = 0
    busy = 0.0
    while n < steps_max and (time.perf_counter() - t0) < seconds:
        q, _ = qp.next()
        kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, c["ctx"] + n, seed, 0)
        a = (synth.bf16_bits(q), synth.bf16_bits(kn), synth.bf16_bits(vn))
        t1 = time.perf_counter()
        eng.step(0, *a)  # O-1..O-6 of one layer for the whole batch
        busy += time.perf_counter() - t1
        n += 1
    full_step = busy / n * c["n_layers"]
    return {"value": nb / full_step, "unit": "tokens/s", "cores": O.num_threads(), "kind": "oracle",
            "sample": f"1 layer x {nb * n_kv} units (whole batch) x {n} decode steps at ctx {c['ctx']}, "
                      f"{busy:.1f}s of oracle time; x{c['n_layers']} layers per token step",
            "us_per_layer": full_step / c["n_layers"] * 1e6}


def spawn_ranks(args):
    """--gpus N outside torchrun: re-launch this command as N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return its exit code; rank 0 prints the line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def nested_line(args, extra):
    """One sub-measurement (own process: own handle and pinned pool) -> its parsed JSON line."""
    cmd = [sys.executable, os.path.abspath(__file__), "--config", args.config, "--nested", "--no-cpu-baseline",
           "--warmup", "4", "--profile-steps", "4"] + extra
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if out.returncode != 0 or not lines:
            return {"error": f"rc={out.returncode}: {out.stderr.strip().splitlines()[-1:]}"}
        return json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


def main():
    args = parse()
    c = dict(CONFIGS[args.config])
    if args.tau is not None:
        c["tau"] = args.tau
    if args.n_layers is not None:
        c["n_layers"] = args.n_layers
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}", file=sys.stderr)
        sys.exit(2)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    seed = args.seed if args.seed is not None else 250513109 + 1 + list(CONFIGS).index(args.config)
    cfg_out = {"workload": c["workload"], "n_layers": c["n_layers"], "batch": c["batch"], "n_qo": c["n_qo"],
               "n_kv": c["n_kv"], "ctx": c["ctx"], "context": "prefill of ctx minus every step of the run "
               "(warm-up, timed, profiled, end to end), so the decode contexts end at ctx",
               "page": 32, "budget": c["budget"], "sink": c["sink"],
               "window": c["window"], "tau": c["tau"], "correction_event_rate": c["event_rate"],
               "parallelism": f"kv-head/batch shard x{args.gpus} + per-layer NCCL all-gather of head outputs", "l2": "inputs larger than L2 (~100 MB per layer, "
               f"{c['n_layers']} layers per step)", "seed": seed}
    if c.get("l_inst", c["n_layers"]) < c["n_layers"]:
        cfg_out["l_inst"] = c["l_inst"]
        cfg_out["layer_cycling"] = f"{c['l_inst']} instantiated layers, virtual layer v runs layer v % {c['l_inst']}"
    if args.impl == "reference":
        if rank != 0:
            return
        ob = run_oracle_sample(c, args.cpu_sample_s, seed)
        line = {"impl": "reference", "metric": METRIC, "value": ob["value"], "unit": "tokens/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": c["batch"] / ob["value"] * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32 select / f64 attention (bf16 inputs)", "data": "synthetic",
                "config": cfg_out, "cpu_baseline": ob,
                "e2e": {"value": ob["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    r = run_ours(args, c, rank, world, local_rank)
    if rank != 0:
        return
    nb, L = c["batch"], c["n_layers"]
    Li = r["n_inst"]  # per-layer selection statistics are sampled on the instantiated layers
    tok_s = nb * args.steps / (r["ms"] / 1e3)
    tok_s_e2e = nb * args.steps / (r["ms_e2e"] / 1e3) if r["ms_e2e"] else None
    import json as _j
    peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    prof = r["prof"]
    d = 128
    G = r["G"]
    units_per_launch = r["nb_loc"] * r["kv_loc"]
    # algorithmic bytes: attention reads |T|*2*d*2 B KV + G*d*2 B q per unit.
    # Dominant kernel: the attention split kernel.  One launch attends every unit (corrected
    # units read their fetched pages from the host pool in the same launch); in the two-phase
    # modes its first launch covers the units with resident pages and phase 2 the others.
    attn_ms, attn_n = r["roof_prof"]["attn_split"]
    p2_ms, p2_n = r["roof_prof"]["attn_split_phase2"]
    two_phase = p2_n > 0
    tok1 = r["t_tok_p1"] if two_phase else r["t_unit_tokens"]
    units1 = r["units_p1"] if two_phase else r["units"]
    # with layer cycling the statistics cover the Li instantiated layers and the launches all L
    cyc = L / Li
    attn_bytes = (tok1 * 2 * d * 2 + units1 * G * d * 2) * cyc
    attn_gbs = attn_bytes / (attn_ms / 1e3) / 1e9 if attn_ms > 0 else 0.0
    p2_bytes = r["t_tok_p2"] * 2 * d * 2 * cyc
    # scoring: algorithmic bytes = |J| * 2 * d * 2 B summaries + G * d * 2 B q per unit; isolated
    # launches (select_pages of the last layer, L2 flushed, library event profiler) when available
    j_per_launch = r["j_pages"] / max(args.profile_steps * Li, 1)
    if r["iso_score"] and r["iso_score"]["score"][1] > 0:
        sc_ms, sc_n = r["iso_score"]["score"]
        sc_timing = "CUDA events around each score launch (select_pages of the last layer through the C ABI), L2 " \
                    "flushed before each of 8 launches; per-launch average"
    else:
        sc_ms, sc_n = prof["score"]
        sc_timing = "event-record graph nodes around each score launch inside the step graph"
    sc_bytes = sc_n * (j_per_launch * 2 * d * 2 + units_per_launch * G * d * 2)
    sc_gbs = sc_bytes / (sc_ms / 1e3) / 1e9 if sc_ms > 0 else 0.0
    # background recall: the unflagged units' fetched pages (the corrected units' fetches are read by
    # the attention kernel from the host pool in direct mode: recall_direct below)
    rec_ms = prof["recall_bg"][0] + prof["recall_sync"][0]
    rec_bytes = r["fetched"] * 2 * 32 * d * 2 * cyc
    rec_gbs = rec_bytes / (rec_ms / 1e3) / 1e9 if rec_ms > 0 else 0.0
    kernels = {k: {"ms_total": round(v[0], 4), "launches": v[1],
                   "us_avg": round(v[0] / v[1] * 1e3, 3) if v[1] else None} for k, v in prof.items()}
    # DRAM bytes per launch of the attention kernel from the committed ncu --set full capture
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tp):
        try:
            tj = _j.load(open(tp))
            if tj.get("workload") == c["workload"]:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    split_attn = os.environ.get("FREEKV_ATTN", "").startswith("s") or os.environ.get("FREEKV_CORR", "").startswith("r")
    kname = ("fkv_attn_split_kernel" + (" phase 1" if two_phase else " (all units)")) if split_attn or two_phase \
        else "fkv_attn_cluster_kernel (all units: attention + DSMEM merge + commit)"
    # the isolated launches attend the last layer of the last profiled step: its bytes are the
    # per-launch average of that step's layers (all layers have the same shapes and budget)
    iso = sorted(r["iso_ms"])
    in_step = {"us_per_launch": round(attn_ms / max(attn_n, 1) * 1e3, 2),
               "achieved": round(attn_gbs, 1), "frac": round(attn_gbs / hbm_peak, 4),
               "timing": "event-record graph nodes around each attention launch inside the step graph "
                         "(brackets the node's launch latency too)"}
    if iso and not two_phase:
        us_iso = iso[len(iso) // 2] * 1e3  # median
        per_launch = attn_bytes / max(attn_n, 1)
        gbs_iso = per_launch / (us_iso / 1e6) / 1e9
        roof = {"kernel": kname, "bound": "hbm", "achieved": round(gbs_iso, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(gbs_iso / hbm_peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": int(per_launch), "us_per_launch": round(us_iso, 2),
                "timing": "CUDA events around the kernel launched through the C ABI on its stream, L2 flushed "
                          "before each of 8 launches (256 MB write, then a 256 MB read so the evicted lines are "
                          "clean; median); peak = MEASURED_PEAKS.json hbm_gbs (copy, burst)",
                "us_per_launch_dirty_l2": round(sorted(r["iso_ms_dirty"])[len(r["iso_ms_dirty"]) // 2] * 1e3, 2)
                if r["iso_ms_dirty"] else None,
                "in_step": in_step}
    else:
        roof = {"kernel": kname, "bound": "hbm", "achieved": in_step["achieved"], "peak": hbm_peak, "unit": "GB/s",
                "frac": in_step["frac"], "traffic": traffic,
                "algorithmic_bytes_per_launch": int(attn_bytes / max(attn_n, 1)),
                "us_per_launch": in_step["us_per_launch"], "timing": in_step["timing"]}
    line = {
        "metric": METRIC, "value": round(tok_s, 2), "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["ms"] / args.steps, 4),
        "us_per_layer": round(r["ms"] / args.steps / L * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16 KV/q, fp32 scores+accumulate, fp32 out",
        "data": "synthetic (GEN-S keys with hot pages, GEN-Q AR(1) queries, seeded)", "config": cfg_out,
        "roofline": roof,
        "attention_phase2": ({"us_per_launch": round(p2_ms / max(p2_n, 1) * 1e3, 2),
                              "algorithmic_bytes_per_launch": int(p2_bytes / max(p2_n, 1))} if two_phase else None),
        "scoring_hbm": {"kernel": "fkv_score_kernel", "achieved": round(sc_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(sc_gbs / hbm_peak, 4), "us_per_launch": round(sc_ms / max(sc_n, 1) * 1e3, 2),
                        "algorithmic_bytes_per_launch": int(sc_bytes / max(sc_n, 1)), "timing": sc_timing},
        "recall": {"achieved_gbs": round(rec_gbs, 2), "host_link_peak_gbs": round(r["link"], 2) if r["link"] else None,
                   "frac": round(rec_gbs / r["link"], 4) if r["link"] and rec_gbs else None,
                   "pages_per_layer_step": round(r["fetched"] / max(args.profile_steps * Li, 1), 2),
                   "sync_pages_per_layer_step": round(r["fetched_sync"] / max(args.profile_steps * Li, 1), 2),
                   "mechanism": "background recall kernel: TMA bulk copies (cp.async.bulk) from the pinned, "
                                "device-mapped host pool into the free slots, on a low-priority stream; bytes = the "
                                "unflagged units' fetched pages"},
        "recall_direct": {"pages_per_layer_step": round(r["fetched_sync"] / max(args.profile_steps * Li, 1), 2),
                          "achieved_gbs": round(r["fetched_sync"] * 2 * 32 * d * 2 * cyc / (attn_ms / 1e3) / 1e9, 2)
                          if attn_ms > 0 and r["fetched_sync"] else None,
                          "host_link_peak_gbs": round(r["link"], 2) if r["link"] else None,
                          "mechanism": "corrected units' fetched pages read by the attention kernel (2D TMA from the "
                                       "device-mapped host pool) and written back to their slots; GB/s over the "
                                       "attention launches' in-step time"},
        "exposed_recall": r["exposed"],
        "correction_rate": round(r["flagged"] / max(r["units"], 1), 4),
        "kernels": kernels,
        "e2e": None if tok_s_e2e is None else {"value": round(tok_s_e2e, 2), "unit": "tokens/s", "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"],
                "note": "public API; per step H2D of q/k/v from pinned memory and D2H of the outputs, "
                        "double-buffered on a copy stream so they overlap the neighbouring steps"},
        "gpu_launches": int(sum(v[1] for v in prof.values()) / max(args.profile_steps, 1) * args.steps),
        "gpu_launches_per_step": int(sum(v[1] for v in prof.values()) / max(args.profile_steps, 1)),
        "execution": "eager per-layer C-ABI calls" if args.eager else "whole-step CUDA graphs (compute + recall)",
        "clocks": r["clocks"],
        "comm": r["comm"],
        "host_pool_numa": r["numa"],
        "setup_s": {"alloc_pin": round(r["t_alloc"], 1), "prefill": round(r["t_prefill"], 1)},
    }
    if args.gen != "S" or args.full_refresh or args.n_layers is not None:
        line["data"] = f"synthetic (generator {args.gen}{', full refresh' if args.full_refresh else ''}" \
                       f"{', %d layers' % L if args.n_layers is not None else ''}; seeded)"
    if not args.nested and not args.no_extras and world == 1 and not args.eager:
        # sensitivity lines (own processes): the survey's GEN-S parameters beside the tuned headline,
        # and the recall stress (GEN-X: every unit corrects; full refresh: all K pages re-fetched)
        sp = nested_line(args, ["--gen", "spec", "--steps", "64"])
        line["survey_spec_gen"] = {k: sp.get(k) for k in ("value", "us_per_layer", "correction_rate", "recall",
                                                            "recall_direct", "error") if k in sp}
        line["survey_spec_gen"]["generator"] = "GEN-S alpha 4, GEN-Q beta 2.5 (SURVEY §8(d) as specified)"
        gx = nested_line(args, ["--gen", "X", "--full-refresh", "--n-layers", "4", "--steps", "32"])
        rd = gx.get("recall_direct") or {}
        pk = rd.get("host_link_peak_gbs")
        line["genx_full_refresh_recall"] = {
            "us_per_layer": gx.get("us_per_layer"), "correction_rate": gx.get("correction_rate"),
            "pages_per_layer_step": rd.get("pages_per_layer_step"), "achieved_gbs": rd.get("achieved_gbs"),
            "host_link_peak_gbs": pk,
            "frac": round(rd["achieved_gbs"] / pk, 4) if rd.get("achieved_gbs") and pk else None,
            "mechanism": rd.get("mechanism"), "error": gx.get("error"),
            "workload": "GEN-X keys/queries, FREEKV_DEBUG_FULL_REFRESH (all K pages of every unit from the host "
                        "pool every step), 4 layers of the config"}
    if not args.no_cpu_baseline and world == 1 and not args.nested:
        line["cpu_baseline"] = run_oracle_sample(c, args.cpu_sample_s, r["seed"])
    print(json.dumps(line))


if __name__ == "__main__":
    main()
