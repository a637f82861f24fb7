#!/usr/bin/env python
"""Benchmark of the Baton hot path on B200 (BASELINE.json metric):

    decode tokens/s of a Baton batch + decode-attention and splice HBM GB/s vs
    the measured peak, 1-8 GPUs.

One "step" = one full Baton iteration of the hot path over the batch: removes +
release, stores (extract) and compaction where the workload has them, inserts
(KV splice), mask update, and for every layer KV append + decode attention --
every §8(a) row the workload exercises.  Model GEMMs are not part of the path
(no weights); q/k/v are synthetic keyed values (SURVEY.md §8(d) generator).

    python bench.py [--config 7b|13b|70b|stress] [--gpus N] [--steps K] [--warmup W]
                    [--windows R] [--impl baton|reference]

Configs (BASELINE.json ``configs``):
  7b      configs[1] (default): 32 layers x 32 heads x d128, 32 slots per GPU, ctx 2048,
          Poisson 0.08/iteration per GPU -- weak scaling
  13b     configs[2]: 40 layers x 40 heads, 64 slots split over the N GPUs, 2 removes +
          2 inserts every iteration -- strong scaling
  70b     configs[3]: 80 layers, 64 q / 8 kv heads (GQA), 16 slots per GPU (128 on 8),
          ctx 4096 -- weak scaling
  stress  configs[4]: 7B shape, 32 slots per GPU, active slots 2 -> 32 per GPU (16 -> 256
          on 8), 25% of the live queries stored and re-inserted every 16 iterations --
          weak scaling

Timing: R windows of K steps each, spread evenly over the
workload's steady state (every active slot live and a backlog waiting; the first
5% of that range is skipped as the transient of the first wave), each opened by a warm start at its first iteration and W untimed warm-up steps, and
timed with CUDA events on the decode stream between a barrier + synchronize on
both sides (max over ranks).  ``value`` is the median window; every window is
listed with its mean live length.  N > 1: torch.distributed.run, one rank per GPU,
one NCCL all-gather of completion flags per iteration.  Rank 0 prints ONE line.
"""
import argparse
import copy
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

INS_AHEAD = 16            # e2e: steps of lookahead for the prefilled K/V H2D of upcoming inserts
INS_PIECE = 8 << 20       # e2e: bytes per insert H2D piece
INS_BUDGET = 48 << 20     # e2e: insert H2D bytes issued per step (PCIe ~97 MB per 1.95 ms step; mean need ~32 MB)
POOL_BYTES = 32 << 30     # prefilled K/V held in HBM for a window (beyond it: recycled buffers)

CONFIG_TEXT = {
    "7b": "Llama-2-7B-shaped attention, 32 layers x 32 heads x d128, bf16 KV, 32 slots/GPU, "
          "ctx<=2048, Poisson 0.08/iter/GPU",
    "13b": "Llama-2-13B-shaped attention, 40 layers x 40 heads x d128, bf16 KV, 64 slots over "
           "the GPUs, ctx<=2048, 2 removes + 2 inserts per iteration",
    "70b": "70B-shaped GQA attention, 80 layers x 64 q / 8 kv heads x d128, bf16 KV, "
           "16 slots/GPU, ctx<=4096, all queries at iteration 0",
    "stress": "7B-shaped attention, 32 slots/GPU, active 2->32 per GPU (doubling every 64 "
              "iterations), 25% of live queries stored + re-inserted every 16 iterations",
}


def _cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None
        self.spans = []

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def span(self, t0, t1):
        """A timed region (host wall clock) whose samples count."""
        self.spans.append((t0, t1))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        import datetime
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if not any(a - 0.05 <= ts <= b + 0.05 for a, b in self.spans):
                    continue
                sm.append(float(f[2]))
                smax.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workloads
def bench_workload(name, world):
    """(workload, scaling) of a bench config at `world` GPUs (module docstring)."""
    from baton_inputs import config_workload
    from baton_inputs.workload import _mix_queries, CLASSES_7B, Workload
    if name == "7b":
        if world == 1:
            return config_workload("7b"), "weak"
        # weak scaling: 32 slots, 512 queries and lambda = 0.08/iteration per GPU
        rng = np.random.default_rng(18701)
        qs = _mix_queries(rng, 512 * world, 32 * world, 0.08 * world, CLASSES_7B, 2048)
        return Workload("7b", qs, layers=32, q_heads=32, kv_heads=32, head_dim=128,
                        slots=32 * world, max_ctx=2048, gpus=world), "weak"
    if name == "13b":
        if 64 % world:
            raise SystemExit("13b: 64 slots must split evenly over the GPUs")
        return config_workload("13b", gpus=world), "strong"
    if name == "70b":
        wl = config_workload("70b", gpus=world, n_queries=64 * world)
        wl.slots = 16 * world
        return wl, "weak"
    if name == "stress":
        wl = config_workload("stress", gpus=world, n_queries=256 * world)
        wl.slots, wl.active = 32 * world, 2 * world
        wl.control.resize = {t: n // 8 * world for t, n in wl.control.resize.items()}
        return wl, "weak"
    raise SystemExit(f"unknown config {name}")


def fast_forward(planner, t0):
    """Advance the (host-only, deterministic) planner to iteration t0."""
    while planner.t < t0:
        flags = None
        if planner.t > 0:
            flags = sum((planner.local_completion_flags(r) for r in range(planner.world)), [])
        planner.plan(flags)


def steady_windows(wl, world, n_windows, span):
    """Start iterations of `n_windows` windows of `span` iterations spread evenly over
    the steady state: iterations at which every active slot decodes and queries are
    waiting (a planner dry run; the same on every rank)."""
    from paper_2410_18701_b200.scheduler import Planner
    p = Planner(wl, world)
    steady = []
    while not p.finished_all():
        if p.t > 0 and p.queue and len(p.decode_plan()) == p.active * world:
            steady.append(p.t)
        fast_forward(p, p.t + 1)
    lo, hi = (steady[0], steady[-1]) if steady else (1, max(1, p.t - 1))
    lo += (hi - lo) // 20          # skip the first 5%: the transient of the first wave
    room = hi + 1 - span - lo
    if room <= 0 or n_windows == 1:
        starts = [lo + max(0, room) // 2]
    else:
        starts = [lo + (room * i) // (n_windows - 1) for i in range(n_windows)]
    return starts, (lo, hi)


def window_plan(planner, n_iters, rank):
    """Decode lists and fresh inserts of the next n_iters iterations (a copy of
    the planner is stepped; the engine's own planner is untouched)."""
    p = copy.deepcopy(planner)
    decodes, inserts = [], []
    for _ in range(n_iters):
        dec = [(p.local(g), q, pos) for g, q, pos in p.decode_plan() if p.rank_of(g) == rank]
        flags = sum((p.local_completion_flags(r) for r in range(p.world)), []) if p.t > 0 else None
        d = p.plan(flags)
        decodes.append(dec)
        for g, q, n, home in d.inserts:
            if p.rank_of(g) == rank and home is None:
                inserts.append((q, n, d.t))
    return decodes, inserts


# ------------------------------------------------------------------ the CUDA arm
class Window:
    """One timed window [t0, t0 + W + K) of a workload on this rank: its inputs are
    generated into HBM before any timing; the passes below each build a fresh
    Engine warm-started at t0."""

    def __init__(self, ctx, t0):
        import torch
        from paper_2410_18701_b200.baton import baton_keygen_tokens, baton_keygen_history
        _release()                   # cached blocks of earlier passes count as free below
        self.ctx, self.t0 = ctx, t0
        wl, dev, rank = ctx.wl, ctx.dev, ctx.rank
        L, Hq, Hkv, D = wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim
        n_iters = ctx.W + ctx.K
        probe = ctx.planner_at(t0)
        self.decodes, self.fresh = window_plan(probe, n_iters, rank)
        B = probe.per_rank
        self.q_all = torch.empty((n_iters, L, B, Hq, D), dtype=torch.bfloat16, device=dev)
        self.k_all = torch.empty((n_iters, L, B, Hkv, D), dtype=torch.bfloat16, device=dev)
        self.v_all = torch.empty_like(self.k_all)
        for i, dec in enumerate(self.decodes):
            qid = np.full(B, -1, np.int32)
            pos = np.zeros(B, np.int32)
            for b, q, p in dec:
                qid[b], pos[b] = q, p
            dq, dp = torch.from_numpy(qid).to(dev), torch.from_numpy(pos).to(dev)
            baton_keygen_tokens(self.q_all[i], dq, dp, L, B, Hq, D, 0, 0, wl.seed, wl.scales[0])
            baton_keygen_tokens(self.k_all[i], dq, dp, L, B, Hkv, D, 1, 0, wl.seed, wl.scales[1])
            baton_keygen_tokens(self.v_all[i], dq, dp, L, B, Hkv, D, 2, 0, wl.seed, wl.scales[2])
        # prefilled K/V of the window's fresh inserts: each query's own keyed history
        # when they all fit in the pool budget; otherwise (13b churn: ~0.9 GB of K/V
        # per iteration) a ring of P buffers sized for the window's longest prompt,
        # buffer i % P serving insert i as a contiguous [L][Hkv][n][D] prefix view: the
        # insert moves the same bytes, the values are keyed rows of an earlier query
        # (finite, the same distribution)
        tok_bytes = 2 * L * Hkv * D * 2
        # room for the pool: what is free now, less the engine's K/V cache (allocated by
        # each pass after this) and a 24 GiB margin (warm-start staging, stash, e2e)
        cap = (wl.max_ctx + 15) // 16 * 16
        cache = 2 * L * B * Hkv * cap * D * 2
        budget = min(POOL_BYTES, max(2 << 30, torch.cuda.mem_get_info(dev)[0] - cache - (24 << 30)))
        self.pref = {}
        self.pool_reused = 0

        def hist(q, n):
            Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
            Vp = torch.empty_like(Kp)
            baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, wl.scales[1])
            baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, wl.scales[2])
            return Kp, Vp

        if sum(n for _, n, _ in self.fresh) * tok_bytes <= budget:
            for q, n, _ in self.fresh:
                self.pref[q] = hist(q, n)
        elif self.fresh:
            nmax = max(n for _, n, _ in self.fresh)
            P = int(max(1, min(len(self.fresh), budget // (nmax * tok_bytes))))
            ring = [hist(q, nmax) for q, _, _ in self.fresh[:P]]
            for i, (q, n, _) in enumerate(self.fresh):
                self.pref[q] = tuple(t.view(-1)[:L * Hkv * n * D].view(L, Hkv, n, D) for t in ring[i % P])
            self.pool_reused = max(0, len(self.fresh) - P)
        torch.cuda.synchronize()

    def token_dev(self, t, dec):
        i = t - self.t0
        return self.q_all[i], self.k_all[i], self.v_all[i]

    def prefill_dev(self, qid, n):
        return self.pref[qid]

    def free(self):
        for name in ("q_all", "k_all", "v_all"):
            if hasattr(self, name):
                delattr(self, name)
        self.pref = {}


class Ctx:
    def __init__(self, args, rank, world, local_rank):
        import torch
        self.args, self.rank, self.world = args, rank, world
        self.dev = torch.device("cuda", local_rank)
        self.wl, self.scaling = bench_workload(args.config, world)
        self.K, self.W = args.steps, args.warmup
        self.group = None
        if world > 1:
            import torch.distributed as dist
            self.group = dist.group.WORLD
        self._ff = None

    def planner_at(self, t0):
        """A planner at iteration t0 (one incremental fast-forward shared by the windows)."""
        from paper_2410_18701_b200.scheduler import Planner
        if self._ff is None or self._ff.t > t0:
            self._ff = Planner(self.wl, self.world)
        fast_forward(self._ff, t0)
        return copy.deepcopy(self._ff)

    def engine(self, t0, token_source, prefill_source):
        """An Engine whose planner is at t0 and whose shard holds the t0 batch: every
        live query embedded with its keyed history through the ABI (S = max lens,
        pad = S - lens: the state after the last release), and every
        stored query waiting for re-insert on this rank stashed."""
        import torch
        from paper_2410_18701_b200.engine import Engine
        from paper_2410_18701_b200.baton import baton_keygen_history
        wl, dev, rank = self.wl, self.dev, self.rank
        L, Hkv, D = wl.layers, wl.kv_heads, wl.head_dim
        _release()                   # whatever the previous pass left cached
        eng = Engine(wl, rank=rank, world=self.world, device=dev, group=self.group,
                     token_source=token_source, prefill_source=prefill_source, use_graph=True)
        eng.planner = self.planner_at(t0)
        pl = eng.planner

        def hist(q, n):
            Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
            Vp = torch.empty_like(Kp)
            baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, wl.scales[1])
            baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, wl.scales[2])
            return Kp, Vp

        live = [(pl.local(g), q, pl.length[g]) for g, q in pl.live() if pl.rank_of(g) == rank]
        for i in range(0, len(live), 16):            # bounded staging memory
            part = live[i:i + 16]
            kv = [hist(q, n) for _, q, n in part]
            eng.shard.baton_insert_many([b for b, _, _ in part], [k for k, _ in kv],
                                        [v for _, v in kv], [n for _, _, n in part])
            del kv
        for e in pl.queue:
            if e.home == rank:
                eng.stash.put(e.qid, *hist(e.qid, e.length))
        if eng.device_flags:
            eng._sync_targets()          # device completion targets of the embedded queries
        torch.cuda.synchronize()
        return eng


def _release(*objs):
    """Drop the references passed in (the caller must not hold others) and return the
    freed blocks to the driver, so the next pass's cache allocation finds room."""
    import torch
    del objs
    gc.collect()
    torch.cuda.empty_cache()


def run_window(ctx, win, clocks):
    """The three passes over one window: value, roofline events, e2e."""
    import torch
    import torch.distributed as dist
    args, world = ctx.args, ctx.world
    wl, dev = ctx.wl, ctx.dev
    L, Hq, Hkv, D = wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim
    K_steps, W, t0 = ctx.K, ctx.W, win.t0
    B = wl.slots // world

    def barrier_sync():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ================= pass 1: `value` -- graph-replayed decode, inputs in HBM
    eng = ctx.engine(t0, win.token_dev, win.prefill_dev)
    for _ in range(W):
        eng.iteration()
    barrier_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.gather_s, eng.gathers = 0.0, 0
    gc.disable()                     # no collector pause inside the timed region
    h0 = time.time()
    e0.record()
    st, marks = [], []
    for _ in range(K_steps):
        st.append(eng.iteration())
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append(ev)
    e1.record()
    barrier_sync()
    gc.enable()
    clocks.span(h0, time.time())
    ms = e0.elapsed_time(e1)
    iter_ms = [a.elapsed_time(b) for a, b in zip([e0] + marks[:-1], marks)]
    gather_us = 1e6 * eng.gather_s / max(1, eng.gathers)
    eng = None
    _release()

    tokens = sum(s.decoded for s in st)
    live_rows = sum(s.live_rows for s in st)      # sum of lens over decoding slots
    # our kernels per step: mask update + one fused append/attention per layer (+ the
    # GQA split-K combine after the last layer), the remove/release mask splice, per
    # stored query an extract copy (+ its remove), the compaction (copy + mask move),
    # the batched KV copy + mask splice of inserts
    gqa = Hq == 8 * Hkv and D == 128
    n_launch = sum(1 + L + (1 if gqa else 0) + (1 if (s.removed or s.released) else 0)
                   + (2 * s.stored if s.stored else 0) + (2 if s.compact_rows else 0)
                   + (2 if s.inserted else 0) for s in st)
    tau = 2 * Hkv * D * 2                          # K+V bytes per token per layer
    attn_bytes = L * (live_rows * tau + tokens * Hq * D * 2 * 2)
    splice_rows = sum(s.insert_rows + s.extract_rows + s.compact_rows for s in st)

    # ================= pass 2: roofline -- the same window, CUDA events around every
    # decode-step graph (mask update + the L PDL-chained attention launches: per-launch
    # events would serialise them and remove the cross-layer overlap) and around every
    # batched KV embed (splice)
    step_ev, splice_ev = [], []
    eng = ctx.engine(t0, win.token_dev, win.prefill_dev)
    sh = eng.shard
    orig, orig_ins = sh.baton_decode_step, sh.baton_insert_many
    timing = {"on": False}

    def timed_step(q, k_new, v_new, out, stream=None):
        if not timing["on"]:
            return orig(q, k_new, v_new, out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig(q, k_new, v_new, out)
        b.record()
        step_ev.append((a, b))
        return out

    def timed_insert(slots, ks, vs, lens, stream=None):
        if not timing["on"]:
            return orig_ins(slots, ks, vs, lens)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig_ins(slots, ks, vs, lens)
        b.record()
        splice_ev.append((a, b, 2 * sum(lens) * L * tau))

    sh.baton_decode_step, sh.baton_insert_many = timed_step, timed_insert
    for _ in range(W):
        eng.iteration()
    torch.cuda.synchronize()
    timing["on"] = True
    gc.disable()
    for _ in range(K_steps):      # the same K iterations as pass 1 (deterministic window)
        eng.iteration()
    torch.cuda.synchronize()
    gc.enable()
    graph_ms = [a.elapsed_time(b) for a, b in step_ev]
    splice_bytes = sum(n for _, _, n in splice_ev)
    splice_s = sum(a.elapsed_time(b) for a, b, _ in splice_ev) / 1e3
    sh.baton_decode_step, sh.baton_insert_many = orig, orig_ins
    del sh, orig, orig_ins, timed_step, timed_insert
    eng = None
    _release()

    res = dict(t0=t0, ms=ms, tokens=tokens, live_rows=live_rows, attn_bytes=attn_bytes,
               attn_time_s=sum(graph_ms) / 1e3, attn_launches=L * len(graph_ms),
               splice_bytes=splice_bytes, splice_s=splice_s, splice_calls=len(splice_ev),
               splice_rows=splice_rows, iter_ms=iter_ms, gather_us=gather_us, n_launch=n_launch,
               stored=sum(s.stored for s in st), inserted=sum(s.inserted for s in st),
               pool_reused=win.pool_reused)
    if not args.no_e2e:
        res["e2e"] = run_e2e(ctx, win, B)
    return res


def run_e2e(ctx, win, B):
    """e2e: the same window through the public API with HOST buffers.  Every step's
    q/k/v are copied H2D from pinned memory (double-buffered staging, one step ahead
    on a high-priority copy stream) and the step's whole result -- all L layers'
    attention outputs -- is read back D2H, inside the timed region.  7b: the prefilled
    K/V of the window's inserts also come from the host, paced on their own copy
    stream.  13b/70b/stress: they stay in HBM (produced by the GPU-side
    prefill; 13b churn alone would need ~0.9 GB of PCIe per 5 ms step)."""
    import torch
    import torch.distributed as dist
    wl, dev, world = ctx.wl, ctx.dev, ctx.world
    L, Hq, Hkv, D = wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim
    K_steps, W, t_base = ctx.K, ctx.W, win.t0
    n_iters = W + K_steps
    ins_h2d = ctx.args.config == "7b"
    q_h = win.q_all.cpu().pin_memory()
    k_h = win.k_all.cpu().pin_memory()
    v_h = win.v_all.cpu().pin_memory()
    pref_h = {}
    if ins_h2d:
        pref_h = {q: (a.cpu().pin_memory(), b.cpu().pin_memory()) for q, (a, b) in win.pref.items()}
    sets = [tuple(torch.empty(shp, dtype=torch.bfloat16, device=dev)
                  for shp in ((L, B, Hq, D), (L, B, Hkv, D), (L, B, Hkv, D))) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    copy_stream = torch.cuda.Stream(priority=-1)
    ins_stream = torch.cuda.Stream()
    d2h_stream = torch.cuda.Stream()
    # the step's result: snapshot D2D on the decode stream (8 MB at 7b: ~3 us), then
    # D2H on its own copy stream while the next step decodes
    res_dev = [torch.empty((L, B, Hq, D), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    res_h = [torch.empty((L, B, Hq, D), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    res_done = [torch.cuda.Event() for _ in range(2)]
    snap = [torch.cuda.Event() for _ in range(2)]
    counters = {"h2d": 0, "d2h": 0}

    def h2d(i):
        slot = i % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(free[slot])          # the decode that last read it
            for dst, src in zip(sets[slot], (q_h[i], k_h[i], v_h[i])):
                dst.copy_(src, non_blocking=True)
                counters["h2d"] += src.numel() * 2
            ready[slot].record(copy_stream)

    def token_host(t, dec):
        slot = (t - t_base) % 2
        torch.cuda.current_stream().wait_event(ready[slot])
        return sets[slot]

    ins_at = {}
    for q, n, t_ins in win.fresh:
        ins_at.setdefault(t_ins - t_base, []).append(q)
    pref_dev = {}
    pending = []          # [qid, [(dst, src) flat views], part index, element offset, event]

    def prefetch_inserts(i):
        if not ins_h2d:
            return
        for q in ins_at.get(i, []):
            a, b = pref_h[q]
            da = torch.empty(a.shape, dtype=a.dtype, device=dev)
            db = torch.empty(b.shape, dtype=b.dtype, device=dev)
            ev = torch.cuda.Event()
            pref_dev[q] = (da, db, ev)
            pending.append([q, [(da.view(-1), a.view(-1)), (db.view(-1), b.view(-1))], 0, 0, ev])

    def pump(budget, until=None, gate=None):
        """Issue queued insert pieces: `budget` bytes, or through query `until`.
        `gate`: a decode-stream event the pieces wait for (the host runs many steps
        ahead of the GPU, so a per-step budget alone paces nothing)."""
        if gate is not None and pending:
            ins_stream.wait_event(gate)
        with torch.cuda.stream(ins_stream):
            while pending and (budget > 0 or until is not None):
                ent = pending[0]
                dst, src = ent[1][ent[2]]
                n = min(src.numel() - ent[3], INS_PIECE // 2)
                dst[ent[3]:ent[3] + n].copy_(src[ent[3]:ent[3] + n], non_blocking=True)
                budget -= 2 * n
                counters["h2d"] += 2 * n
                ent[3] += n
                if ent[3] == src.numel():
                    ent[2], ent[3] = ent[2] + 1, 0
                    if ent[2] == len(ent[1]):
                        ent[4].record(ins_stream)
                        pending.pop(0)
                        if ent[0] == until:
                            return

    def prefill_host(qid, n):
        if not ins_h2d:
            return win.pref[qid]
        if qid not in pref_dev:          # not prefetched (should not happen): copy now
            a, b = pref_h[qid]
            counters["h2d"] += (a.numel() + b.numel()) * 2
            return a.to(dev, non_blocking=True), b.to(dev, non_blocking=True)
        if any(e[0] == qid for e in pending):   # burst: issue the rest of its pieces now
            pump(0, until=qid)
        da, db, ev = pref_dev.pop(qid)
        torch.cuda.current_stream().wait_event(ev)
        da.record_stream(torch.cuda.current_stream())
        db.record_stream(torch.cuda.current_stream())
        return da, db

    step_ev = []             # (step, event at its start on the decode stream, inserts)

    def step(eng2, i, warm):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        step_ev.append((i, ev0, len(ins_at.get(i, []))))
        if i + 1 < n_iters:
            h2d(i + 1)
        prefetch_inserts(i + INS_AHEAD)
        pump(INS_BUDGET, gate=ev0)
        st_ = eng2.iteration()
        free[i % 2].record()
        r = i % 2
        cur = torch.cuda.current_stream()
        cur.wait_event(res_done[r])                   # D2H of step i-2 finished with it
        res_dev[r].copy_(eng2.out, non_blocking=True)
        snap[r].record()
        with torch.cuda.stream(d2h_stream):
            d2h_stream.wait_event(snap[r])
            res_h[r].copy_(res_dev[r], non_blocking=True)
            res_done[r].record(d2h_stream)
        if not warm:
            counters["d2h"] += res_h[r].numel() * 2
        return st_

    eng = ctx.engine(t_base, token_host, prefill_host)
    for st_set in sets:
        eng.register_staging(*st_set)
    for ev in free + res_done:
        ev.record()
    h2d(0)
    for i in range(INS_AHEAD):
        prefetch_inserts(i)
    pump(1 << 62)
    torch.cuda.synchronize()
    for i in range(W):
        step(eng, i, True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    counters["h2d"] = counters["d2h"] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.disable()
    e0.record()
    h0 = time.perf_counter()
    st2 = [step(eng, W + i, False) for i in range(K_steps)]
    host_ms = (time.perf_counter() - h0) * 1e3
    torch.cuda.current_stream().wait_stream(d2h_stream)   # the last results are on the host
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gc.enable()
    ms2 = e0.elapsed_time(e1)
    marks = [x for x in step_ev if x[0] >= W] + [(None, e1, 0)]
    step_ms = [marks[k][1].elapsed_time(marks[k + 1][1]) for k in range(len(marks) - 1)]
    slow = sorted(range(len(step_ms)), key=lambda k: -step_ms[k])[:3]
    out = {"ms": ms2, "host_ms": host_ms, "step_ms": step_ms,
           "tokens": sum(s.decoded for s in st2), "h2d": counters["h2d"] / K_steps,
           "d2h": counters["d2h"] / K_steps, "inserts_h2d": ins_h2d,
           "slowest": [{"ms": step_ms[k], "t": st2[k].t, "inserted": st2[k].inserted,
                        "stored": st2[k].stored, "compact_rows": st2[k].compact_rows,
                        "removed": st2[k].removed} for k in slow]}
    eng = q_h = k_h = v_h = pref_h = sets = res_dev = res_h = None
    _release()
    return out


def run_full(ctx):
    """The whole workload from iteration 0 until it drains (or its iteration limit),
    one GPU: per-step q/k/v and inserted K/V generated on the device (keygen)
    inside the timed region."""
    import torch
    from paper_2410_18701_b200.engine import Engine
    engf = Engine(ctx.wl, rank=0, world=1, device=ctx.dev, use_graph=True)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    st_f = engf.run()
    f1.record()
    torch.cuda.synchronize()
    ms_f = f0.elapsed_time(f1)
    tok_f = sum(s.decoded for s in st_f)
    out = {"value": tok_f / (ms_f / 1e3), "unit": "tokens/s", "iterations": len(st_f),
           "tokens": tok_f, "queries": len(ctx.wl.queries), "ms": ms_f,
           "mean_live_len": sum(s.live_rows for s in st_f) / max(1, tok_f),
           "what": "whole workload from iteration 0 to drain, one GPU; per-step q/k/v and "
                   "inserted K/V generated on the device (keygen) inside the timed region"}
    engf = st_f = None
    _release()
    return out


def run_prefill(ctx, plens):
    """a8: the windows' inserted prompts (the first 64) through the tcgen05 prefill (P&D
    decouples it from the decode loop): one varlen launch per layer over
    them; all layers cost the same, so one layer is graph-timed.  Beside `value`."""
    import torch
    from paper_2410_18701_b200.baton import baton_prefill_attention_varlen
    wl, dev = ctx.wl, ctx.dev
    Hq, Hkv, D = wl.q_heads, wl.kv_heads, wl.head_dim
    T = sum(plens)
    g = torch.Generator(device=dev).manual_seed(18701)
    qp = torch.randn((Hq, T, D), device=dev, generator=g).to(torch.bfloat16)
    kp = torch.randn((Hkv, T, D), device=dev, generator=g).to(torch.bfloat16)
    vp = torch.randn((Hkv, T, D), device=dev, generator=g).to(torch.bfloat16)
    op = torch.empty_like(qp)
    reps = 10
    for _ in range(2):
        baton_prefill_attention_varlen(qp, kp, vp, op, plens, Hq, Hkv, D)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side), torch.cuda.graph(gr, stream=side):
        for _ in range(reps):
            baton_prefill_attention_varlen(qp, kp, vp, op, plens, Hq, Hkv, D)
    gr.replay()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    gr.replay()
    p1.record()
    torch.cuda.synchronize()
    us = p0.elapsed_time(p1) * 1e3 / reps
    flop = sum(4.0 * Hq * D * n * (n + 1) / 2 for n in plens)
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    bf16_peak = json.load(open(pk))["bf16_tflops"] if os.path.exists(pk) else 2250.0
    out = {"what": "baton_prefill_attention_varlen (tcgen05) over the windows' inserted "
                   "prompts (first 64), one layer, graph-timed", "prompts": len(plens), "tokens": T,
           "us_per_layer": us, "tflops": flop / us / 1e6, "peak_tflops": bf16_peak,
           "peak_source": "measured" if os.path.exists(pk) else "nominal",
           "frac": flop / us / 1e6 / bf16_peak}
    qp = kp = vp = op = gr = None
    _release()
    return out


def read_stream_gbs(dev, gib=8):
    """Context for the roofline: a read-only stream over `gib` GiB (torch's fp32 sum
    reduction, best of 5, CUDA events; an int32 sum accumulates in int64 and ran at a
    sixth of the bandwidth).  The peak the line divides by is
    MEASURED_PEAKS.json's copy (read + write) bandwidth; a read-only kernel such as
    the decode attention can run a little above it."""
    import torch
    x = torch.ones((gib << 30) // 4, dtype=torch.float32, device=dev)
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x.sum()
        b.record()
        torch.cuda.synchronize()
        best = max(best, x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9)
    del x
    torch.cuda.empty_cache()
    return best


def run_baton(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    ctx = Ctx(args, rank, world, local_rank)
    starts, steady = steady_windows(ctx.wl, world, args.windows, args.warmup + args.steps)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    wins = []
    for t0 in starts:
        win = Window(ctx, t0)
        wins.append(run_window(ctx, win, clocks))
        wins[-1]["fresh"] = [n for _, n, _ in win.fresh]
        win.free()
        win = None
        _release()
    clk = clocks.stop()
    full_run = run_full(ctx) if (world == 1 and not args.no_full_run) else None
    plens = sum((w["fresh"] for w in wins), [])[:64]
    prefill = run_prefill(ctx, plens) if (rank == 0 and plens) else None
    read_gbs = read_stream_gbs(ctx.dev) if rank == 0 else None
    return dict(wins=wins, steady=steady, clocks=clk, full_run=full_run, prefill=prefill,
                scaling=ctx.scaling, wl=ctx.wl, read_gbs=read_gbs)


# ------------------------------------------------------------------ the oracle arm
def oracle_sample(config, t0, n_slots=8, budget_s=15.0, max_steps=None, warmup=0):
    """Time the fp64 oracle (O-2 Shard.step, as it stands) on a bounded sample of
    the workload: ONE layer of the `config` batch at iteration t0, the ``n_slots``
    live queries at evenly spaced length quantiles (the sample's mean length tracks
    the batch's).  Returns (seconds per step, rows, L, timed steps, live slots,
    mean sampled length)."""
    from baton_inputs import KIND_K, KIND_V, KIND_Q, bf16_bits_to_f64
    from baton_inputs import query_history_bits, query_token_bits
    from oracle import Shard, Simulator
    wl, _ = bench_workload(config, 1)
    sim = Simulator(wl, kv=False)
    while sim.t <= t0:
        sim.iteration()
    osh = sim.shards[0]
    live = [b for b in range(wl.slots) if osh.qid[b] >= 0]
    lens = osh.lens()
    m = min(n_slots, len(live))
    by_len = sorted(live, key=lambda b: lens[b])
    picked = [by_len[int((i + 0.5) * len(by_len) / m)] for i in range(m)]
    # the oracle keeps DENSE [rows][S] tensors, so the sample shard holds exactly the
    # sampled rows (its cost is then linear in them)
    sh = Shard(m, 1, wl.q_heads, wl.kv_heads, wl.head_dim, wl.max_ctx, kv=True)
    for i, b in enumerate(sorted(picked, key=lambda b: -lens[b])):
        q, n = int(osh.qid[b]), int(lens[b])
        K = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_K, 1, q, 0, n, wl.kv_heads, wl.head_dim, 0))
        V = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_V, 1, q, 0, n, wl.kv_heads, wl.head_dim, 0))
        sh.insert(i, q, n, K, V)
    times = []
    warm = warmup
    while True:
        qids = np.zeros(sh.B, np.int64)
        pos = np.zeros(sh.B, np.int64)
        cur = sh.lens()
        for b in range(m):
            qids[b], pos[b] = sh.qid[b], cur[b]
        qv = bf16_bits_to_f64(query_token_bits(wl.seed, KIND_Q, 0, qids, pos, wl.q_heads, wl.head_dim, 0))[None]
        kv = bf16_bits_to_f64(query_token_bits(wl.seed, KIND_K, 0, qids, pos, wl.kv_heads, wl.head_dim, 0))[None]
        vv = bf16_bits_to_f64(query_token_bits(wl.seed, KIND_V, 0, qids, pos, wl.kv_heads, wl.head_dim, 0))[None]
        t1 = time.perf_counter()
        sh.step(qv, kv, vv)
        if warm > 0:
            warm -= 1
            continue
        times.append(time.perf_counter() - t1)
        if (max_steps and len(times) >= max_steps) or (not max_steps and sum(times) >= budget_s):
            break
    return (float(np.mean(times)), m, wl.layers, len(times), len(live),
            float(np.mean([lens[b] for b in picked])))


def oracle_all_cores(config, t0, n_slots, budget_s):
    """The same sample run as one independent oracle replica per affinity core at
    once (the oracle is single-threaded NumPy): the box's whole-host oracle rate.
    Replicas are separate processes (this script with --oracle-replica), capped by
    free host memory (a replica holds ~2-3 GB of dense fp64 K/V at peak); `cores` is
    the number that ran."""
    cores = len(os.sched_getaffinity(0))
    try:
        import psutil
        cores = max(1, min(cores, int(psutil.virtual_memory().available / (3 << 30))))
    except ImportError:
        pass
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    cmd = [sys.executable, os.path.abspath(__file__), "--oracle-replica",
           f"{config},{t0},{n_slots},{budget_s}"]
    procs = [subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, env=env)
             for _ in range(cores)]
    rate, ran = 0.0, 0
    for p in procs:
        try:
            out, _ = p.communicate(timeout=budget_s + 300)
            t, m, L = json.loads(out.decode().strip().splitlines()[-1])
            rate += m / (L * t)
            ran += 1
        except Exception:
            p.kill()
    return rate, ran


def median_window_t0(config, world=1, windows=5, span=220):
    wl, _ = bench_workload(config, world)
    starts, _ = steady_windows(wl, world, windows, span)
    return starts[len(starts) // 2]


def run_reference(args):
    """The reference arm of this tier is the oracle (fp64 CPU), timed as it stands.
    A step = one oracle layer-iteration of an 8-row shard holding the live queries of
    the median window's first iteration at evenly spaced length quantiles; tokens/s
    is extrapolated to all L layers: rows / (L * t_step)."""
    t0 = median_window_t0(args.config, 1, args.windows, args.warmup + args.steps)
    t_step, m, L, n, live, mlen = oracle_sample(args.config, t0, n_slots=8, max_steps=args.steps,
                                                warmup=args.warmup)
    value = m / (L * t_step)
    sample = (f"O-2 Shard.step (fp64 NumPy, 1 thread), per step 1 of {L} layers x {m} of {live} "
              f"live slots (length quantiles, mean {mlen:.0f}) at iteration {t0} of {args.config}; "
              f"{n} timed steps after {args.warmup} warm-up; tokens/s = {m} / ({L} x step time)")
    line = {
        "impl": "reference", "metric": f"decode tokens/s ({args.config} Baton batch)",
        "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": n, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (keyed generator)",
        "config": {"workload": args.config, "t0": t0},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                         "cpu_model": _cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ main
def summarize(args, r, world, red):
    """Rank 0: the JSON line from this rank's results and the cross-rank reductions."""
    peak, peak_kind = _peaks()
    wins, wl = r["wins"], r["wl"]
    L = wl.layers
    vals = [w["tok_all"] / (w["ms_max"] / 1e3) for w in wins]
    order = sorted(range(len(wins)), key=lambda i: vals[i])
    med = order[len(order) // 2]
    wm = wins[med]
    attn_bytes = sum(w["attn_bytes"] for w in wins)
    attn_s = sum(w["attn_time_s"] for w in wins)
    attn_launches = sum(w["attn_launches"] for w in wins)
    splice_bytes = sum(w["splice_bytes"] for w in wins)
    splice_s = sum(w["splice_s"] for w in wins)
    achieved = attn_bytes / attn_s / 1e9 if attn_s else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r02_traffic.json" if args.config == "7b"
                      else f"r02_traffic_{args.config}.json")
    kernel = {"7b": "decode_attention_kernel<128, 4, 2, 3>", "13b": "decode_attention_kernel<128, 4, 2, 3>",
              "stress": "decode_attention_kernel<128, 4, 2, 3>", "70b": "decode_gqa_tc_kernel"}[args.config]
    if os.path.exists(tp):
        traffic = json.load(open(tp))["traffic_bytes"]
    all_iter = sum((w["iter_ms"] for w in wins), [])
    line = {
        "metric": f"decode tokens/s ({args.config}-shape Baton batch)",
        "value": vals[med],
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": wm["ms_max"] / args.steps,
        "iter_ms_p10_p50_p90": [float(x) for x in np.percentile(all_iter, [10, 50, 90])],
        "higher_is_better": True,
        "scaling": r["scaling"],
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (keyed q/k/v generator, paper-style length mix and arrivals)",
        "config": {"workload": f"{args.config}: {CONFIG_TEXT[args.config]}",
                   "slots_per_gpu": wl.slots // world, "parallelism": f"slots/{world} GPU",
                   "windows": [w["t0"] for w in wins], "steady_state": list(r["steady"]),
                   "l2": "inputs larger than L2 (the K/V read per step is GBs; no flush needed)",
                   "mean_live_len": wm["live_rows"] / max(1, wm["tokens"]),
                   "live_slots_per_step": wm["tokens"] / args.steps},
        "windows": [{"t0": w["t0"], "value": vals[i], "ms_per_step": w["ms_max"] / args.steps,
                     "mean_live_len": w["live_rows"] / max(1, w["tokens"]),
                     "live_slots_per_step_rank0": w["tokens"] / args.steps,
                     "inserts": w["inserted"], "stored": w["stored"],
                     "attn_frac": (w["attn_bytes"] / w["attn_time_s"] / 1e9 / peak) if w["attn_time_s"] else None,
                     **({"e2e": w["e2e_all"] / (w["e2e_ms_max"] / 1e3),
                         "e2e_step_ms_p50_max": [statistics.median(w["e2e"]["step_ms"]),
                                                 max(w["e2e"]["step_ms"])]} if "e2e" in w else {})}
                    for i, w in enumerate(wins)],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": (os.path.relpath(tp, ROOT) + " (one ncu --set full launch)")
                     if traffic else None,
                     "kernel": kernel,
                     "bytes_per_launch": attn_bytes / max(1, attn_launches),
                     "peak_source": peak_kind,
                     "avg_launch_us": 1e6 * attn_s / max(1, attn_launches),
                     "timing": "rank 0: CUDA events around each decode-step graph (mask update + L "
                               "PDL-chained attention launches) over every window's K steps; "
                               "avg_launch_us = graph time / (steps * L)",
                     "step_hbm_GBps": attn_bytes / (sum(w["ms"] for w in wins) / 1e3) / 1e9,
                     "read_stream_GBps": r.get("read_gbs"),
                     "read_stream_note": "context: a read-only stream (torch fp32 sum over 8 GiB, best "
                                         "of 5) on this box; `peak` is the measured copy "
                                         "(read+write) bandwidth, which a read-only kernel can "
                                         "slightly exceed"},
        "splice": {"calls": sum(w["splice_calls"] for w in wins), "bytes": splice_bytes,
                   "GBps": (splice_bytes / splice_s / 1e9) if splice_s else None,
                   "frac": (splice_bytes / splice_s / 1e9 / peak) if splice_s else None,
                   "what": "baton_insert_many (batched KV embed + mask splice) in every window, "
                           "algorithmic read+write bytes / event time (rank 0)",
                   "prefilled_pool_reused": sum(w["pool_reused"] for w in wins)},
        "gpu_launches": wm["n_launch"],
        "clocks": r["clocks"],
    }
    if world > 1:
        line["multi_gpu"] = red["multi"]
    if "e2e" in wm:
        e = wm["e2e"]
        line["e2e"] = {"value": wm["e2e_all"] / (wm["e2e_ms_max"] / 1e3), "unit": "tokens/s",
                       "h2d_bytes_per_step": int(e["h2d"]), "d2h_bytes_per_step": int(e["d2h"]),
                       "what": "median window through Engine with pinned-host q/k/v H2D every step"
                               + (" + prefilled K/V H2D of its inserts" if e["inserts_h2d"] else
                                  " (prefilled K/V in HBM)")
                               + " + D2H of all layers' outputs every step, inside the timed region",
                       "host_enqueue_ms_per_step": e["host_ms"] / args.steps,
                       "slowest_steps": e["slowest"],
                       "step_ms_p50_p90_max": [statistics.median(e["step_ms"]),
                                               sorted(e["step_ms"])[int(0.9 * (len(e["step_ms"]) - 1))],
                                               max(e["step_ms"])]}
    if r.get("prefill"):
        line["prefill"] = r["prefill"]
    if r.get("full_run"):
        line["full_run"] = r["full_run"]
    if world == 1 and not args.no_cpu_baseline:
        t0 = wins[len(wins) // 2]["t0"]         # the middle window's start, as --impl reference
        t_step, m, Lw, n, live, mlen = oracle_sample(args.config, t0, n_slots=8, budget_s=15.0)
        cb = {"value": m / (Lw * t_step), "unit": "tokens/s", "cores": 1, "kind": "oracle",
              "cpu_model": _cpu_model(),
              "sample": f"O-2 Shard.step (fp64 NumPy, 1 thread), 1 of {Lw} layers x {m} of {live} live "
                        f"slots (length quantiles, mean {mlen:.0f}) at iteration {t0} (the middle "
                        f"window's start), {n} steps, tokens/s = {m} / ({Lw} x step time) -- the same "
                        f"sample as --impl reference"}
        if not args.no_all_cores:
            rate, cores = oracle_all_cores(args.config, t0, 8, 10.0)
            cb["all_cores"] = {"value": rate, "cores": cores,
                               "what": "one oracle replica of the same sample per affinity core, "
                                       "run at once; value = sum of their rates"}
        line["cpu_baseline"] = cb
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--windows", type=int, default=5)
    ap.add_argument("--config", default="7b", choices=["7b", "13b", "70b", "stress"])
    ap.add_argument("--impl", default="baton", choices=["baton", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-all-cores", action="store_true")
    ap.add_argument("--no-full-run", action="store_true")
    ap.add_argument("--oracle-replica", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.oracle_replica:                 # one replica of oracle_all_cores
        c, t0, m, bud = args.oracle_replica.split(",")
        t, m, L, _, _, _ = oracle_sample(c, int(t0), n_slots=int(m), budget_s=float(bud))
        print(json.dumps([t, m, L]))
        return
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only overrides (tests/test_gpu_bench_multirank.py runs 2 ranks on ONE GPU over
    # gloo to exercise this N>1 path; the driver's N>1 runs use the defaults: nccl, one GPU
    # per rank)
    backend = os.environ.get("BATON_BENCH_BACKEND", "nccl")
    if "BATON_BENCH_DEVICE" in os.environ:
        local_rank = int(os.environ["BATON_BENCH_DEVICE"])

    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group(backend)
    r = run_baton(args, rank, world, local_rank)

    # per window: max over ranks of the device time, tokens summed over ranks
    red = {}
    rdev = "cuda" if (world > 1 and backend == "nccl") else "cpu"
    for w in r["wins"]:
        w["ms_max"], w["tok_all"] = w["ms"], w["tokens"]
        if "e2e" in w:
            w["e2e_ms_max"], w["e2e_all"] = w["e2e"]["ms"], w["e2e"]["tokens"]
        if world > 1:
            t = torch.tensor([w["ms"], w.get("e2e", {}).get("ms", 0.0)], dtype=torch.float64, device=rdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            w["ms_max"], w["e2e_ms_max"] = t.tolist()
            c = torch.tensor([w["tokens"], w.get("e2e", {}).get("tokens", 0)], dtype=torch.float64, device=rdev)
            dist.all_reduce(c)
            w["tok_all"], w["e2e_all"] = [int(x) for x in c.tolist()]
    if world > 1:
        # SURVEY §8(d) for N > 1: the flag all-gather's host-blocking time per iteration
        # (max over ranks) and the per-rank attention-byte imbalance (max / mean)
        g = torch.tensor([max(w["gather_us"] for w in r["wins"])], dtype=torch.float64, device=rdev)
        dist.all_reduce(g, op=dist.ReduceOp.MAX)
        mine = float(sum(w["attn_bytes"] for w in r["wins"]))
        bts = [torch.zeros(1, dtype=torch.float64, device=rdev) for _ in range(world)]
        dist.all_gather(bts, torch.tensor([mine], dtype=torch.float64, device=rdev))
        bts = [float(x.item()) for x in bts]
        red["multi"] = {"allgather_us_per_iter": float(g.item()),
                        "rank_attn_bytes_max_over_mean": max(bts) / (sum(bts) / world) if sum(bts) else None,
                        "rank_attn_bytes": bts,
                        "collective": "all_gather of int32 completion flags per iteration (" + backend + ")"}
    if rank == 0:
        print(json.dumps(summarize(args, r, world, red)))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
