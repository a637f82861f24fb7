#!/usr/bin/env python
"""Benchmark of the Baton hot path on B200 (BASELINE.json metric):

    decode tokens/s of the 7B-shaped Baton batch (configs[1]: 32 heads x d128,
    bf16 KV, batch 32 per GPU, ctx <= 2048, Poisson arrivals) + decode-attention
    and splice HBM GB/s vs the measured peak.

One "step" = one full Baton iteration of the hot path over the batch: removes +
release, inserts (KV splice), mask update, and for all 32 layers KV append +
decode attention -- every §8(a) row that the workload exercises.  Model GEMMs
are not part of the path (no weights); q/k/v are synthetic keyed values.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl baton|reference]

N > 1: launched by torch.distributed.run, one rank per GPU, 32 slots per GPU
(weak scaling), one NCCL all-gather of completion flags per iteration.
Rank 0 prints ONE JSON line.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T0_DEFAULT = 512          # steady-state start iteration of the Poisson workload
INS_AHEAD = 16            # e2e: steps of lookahead for the prefilled K/V H2D of upcoming inserts
INS_PIECE = 8 << 20       # e2e: bytes per insert H2D piece
INS_BUDGET = 48 << 20     # e2e: insert H2D bytes issued per step (PCIe ~97 MB per 1.95 ms step; mean need ~32 MB)


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

    def mark(self, which):
        setattr(self, which, time.time())

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
        t_lo = getattr(self, "t_start", 0.0)
        t_hi = getattr(self, "t_end", 1e30)
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if not (t_lo - 0.05 <= ts <= t_hi + 0.05):
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


# ------------------------------------------------------------------ workload helpers
def bench_workload(world):
    from baton_inputs import config_workload
    from baton_inputs.workload import _mix_queries, CLASSES_7B, Workload
    if world == 1:
        return config_workload("7b")
    # weak scaling: 32 slots, 512 queries and lambda = 0.08/iteration per GPU
    rng = np.random.default_rng(18701)
    qs = _mix_queries(rng, 512 * world, 32 * world, 0.08 * world, CLASSES_7B, 2048)
    return Workload("7b", qs, layers=32, q_heads=32, kv_heads=32, head_dim=128,
                    slots=32 * world, max_ctx=2048, gpus=world)


def fast_forward(planner, t0):
    """Advance the (host-only, deterministic) planner to iteration t0."""
    while planner.t < t0:
        flags = None
        if planner.t > 0:
            flags = sum((planner.local_completion_flags(r) for r in range(planner.world)), [])
        planner.plan(flags)


def window_plan(planner, n_iters, rank):
    """Decode lists and fresh inserts of the next n_iters iterations (a copy of
    the planner is stepped; the engine's own planner is untouched)."""
    import copy
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
def run_baton(args, rank, world, local_rank):
    import gc
    import torch
    import torch.distributed as dist
    from paper_2410_18701_b200.engine import Engine
    from paper_2410_18701_b200.baton import baton_keygen_tokens, baton_keygen_history
    from paper_2410_18701_b200.scheduler import Planner

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = dist.group.WORLD if world > 1 else None
    wl = bench_workload(world)
    L, Hq, Hkv, D = wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim
    K_steps, W = args.steps, args.warmup
    n_iters = W + K_steps

    def make_engine(token_source, prefill_source, use_graph):
        eng = Engine(wl, rank=rank, world=world, device=dev, group=group,
                     token_source=token_source, prefill_source=prefill_source,
                     use_graph=use_graph)
        fast_forward(eng.planner, args.t0)
        return eng

    # ---- warm start: materialise the t0 state through the ABI (insert every live
    # query with its current keyed history: S = max lens, pad = S - lens, exactly
    # the state after the last release)
    def warm_start(eng):
        pl = eng.planner
        slots, ks, vs, lens = [], [], [], []
        for g, q in pl.live():
            if pl.rank_of(g) != rank:
                continue
            n = pl.length[g]
            Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
            Vp = torch.empty_like(Kp)
            baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, wl.scales[1])
            baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, wl.scales[2])
            slots.append(pl.local(g))
            ks.append(Kp)
            vs.append(Vp)
            lens.append(n)
        eng.shard.baton_insert_many(slots, ks, vs, lens)
        torch.cuda.synchronize()

    def release(eng):
        del eng
        gc.collect()
        torch.cuda.empty_cache()

    # ---- inputs of the window, resident in HBM before any timing
    probe = Planner(wl, world)
    fast_forward(probe, args.t0)
    decodes, fresh = window_plan(probe, n_iters, rank)
    B = probe.per_rank
    q_all = torch.empty((n_iters, L, B, Hq, D), dtype=torch.bfloat16, device=dev)
    k_all = torch.empty((n_iters, L, B, Hkv, D), dtype=torch.bfloat16, device=dev)
    v_all = torch.empty_like(k_all)
    for i, dec in enumerate(decodes):
        qid = np.full(B, -1, np.int32)
        pos = np.zeros(B, np.int32)
        for b, q, p in dec:
            qid[b], pos[b] = q, p
        dq, dp = torch.from_numpy(qid).to(dev), torch.from_numpy(pos).to(dev)
        baton_keygen_tokens(q_all[i], dq, dp, L, B, Hq, D, 0, 0, wl.seed, wl.scales[0])
        baton_keygen_tokens(k_all[i], dq, dp, L, B, Hkv, D, 1, 0, wl.seed, wl.scales[1])
        baton_keygen_tokens(v_all[i], dq, dp, L, B, Hkv, D, 2, 0, wl.seed, wl.scales[2])
    pref = {}
    for q, n, _ in fresh:
        Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
        Vp = torch.empty_like(Kp)
        baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, wl.scales[1])
        baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, wl.scales[2])
        pref[q] = (Kp, Vp)
    torch.cuda.synchronize()
    t_base = args.t0

    def token_dev(t, dec):
        i = t - t_base
        return q_all[i], k_all[i], v_all[i]

    def prefill_dev(qid, n):
        return pref[qid]

    def timed_window(eng, per_iter=None):
        for _ in range(W):
            eng.iteration()
            if per_iter:
                per_iter(eng, warm=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        eng.gather_s, eng.gathers = 0.0, 0
        e0.record()
        st = []
        marks = []                 # one event after every iteration: per-iteration ms
        for _ in range(K_steps):
            st.append(eng.iteration())
            if per_iter:
                per_iter(eng, warm=False)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        it_ms = [a.elapsed_time(b) for a, b in zip([e0] + marks[:-1], marks)]
        timed_window.iter_ms = it_ms
        timed_window.gather_us = 1e6 * eng.gather_s / max(1, eng.gathers)
        return e0.elapsed_time(e1), st

    # ================= pass 1: `value` -- graph-replayed decode, inputs in HBM
    eng = make_engine(token_dev, prefill_dev, use_graph=True)
    warm_start(eng)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    clocks.mark("t_start")
    ms, stats = timed_window(eng)
    iter_ms = list(timed_window.iter_ms)
    gather_us = timed_window.gather_us
    clocks.mark("t_end")
    clk = clocks.stop()
    release(eng)

    tokens = sum(s.decoded for s in stats)
    live_rows = sum(s.live_rows for s in stats)   # sum of lens over decoding slots
    splice_rows = sum(s.insert_rows + s.extract_rows + s.compact_rows for s in stats)
    # our kernels per step: mask update + one fused append/attention per layer (+ the
    # splice: remove/release, the batched KV copy + mask splice of inserts)
    n_launch = sum(1 + L + (1 if (s.removed or s.released) else 0) + s.stored
                   + (2 if s.inserted else 0) for s in stats)
    tau = 2 * Hkv * D * 2       # K+V bytes per token per layer
    attn_bytes_total = L * (live_rows * tau + tokens * Hq * D * 2 * 2)

    # ================= pass 2: roofline -- same window, CUDA events around every
    # decode-step graph (mask update + the L attention launches, PDL-chained: per-launch
    # events would serialise the launches and remove the cross-layer overlap) and
    # around every batched KV embed (splice)
    step_ev = []
    eng = make_engine(token_dev, prefill_dev, use_graph=True)
    warm_start(eng)
    sh = eng.shard
    orig = sh.baton_decode_step
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

    sh.baton_decode_step = timed_step
    # splice (a5/a6/a7) K/V copies timed the same way: bytes = read + write of the rows
    splice_ev = []
    orig_ins = sh.baton_insert_many

    def timed_insert(slots, ks, vs, lens, stream=None):
        if not timing["on"]:
            return orig_ins(slots, ks, vs, lens)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig_ins(slots, ks, vs, lens)
        b.record()
        splice_ev.append((a, b, 2 * sum(lens) * L * Hkv * D * 2 * 2))

    sh.baton_insert_many = timed_insert
    for _ in range(W):
        eng.iteration()
    torch.cuda.synchronize()
    timing["on"] = True
    for _ in range(K_steps):      # the same K iterations as pass 1 (deterministic window)
        eng.iteration()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    splice_bytes = sum(n for _, _, n in splice_ev)
    splice_s = sum(a.elapsed_time(b) for a, b, _ in splice_ev) / 1e3
    sh.baton_decode_step = orig
    sh.baton_insert_many = orig_ins
    del sh, orig, timed_step, orig_ins, timed_insert
    release(eng)
    # the whole decode-step graph is charged to the attention kernel (its mask-update
    # launch, ~3 us of ~2 ms, is included: conservative)
    attn_time_s = sum(step_ms) / 1e3
    attn_launches = L * len(step_ms)

    # ================= pass 3: e2e -- host buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        q_h = q_all.cpu().pin_memory()
        k_h = k_all.cpu().pin_memory()
        v_h = v_all.cpu().pin_memory()
        pref_h = {q: (a.cpu().pin_memory(), b.cpu().pin_memory()) for q, (a, b) in pref.items()}
        del q_all, k_all, v_all
        pref.clear()
        gc.collect()
        # (no empty_cache: the freed prefilled-K/V blocks serve the e2e insert buffers)
        # double-buffered device staging, filled by a copy stream one step ahead so
        # the PCIe transfer of step i+1 overlaps the decode of step i
        sets = [tuple(torch.empty(shp, dtype=torch.bfloat16, device=dev)
                      for shp in ((L, B, Hq, D), (L, B, Hkv, D), (L, B, Hkv, D))) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        # two copy streams: a step's q/k/v must not queue behind a prefilled K/V
        # transfer (hundreds of MB for one insert, several decode steps of PCIe time)
        copy_stream = torch.cuda.Stream(priority=-1)
        ins_stream = torch.cuda.Stream()
        res_h = torch.empty((B, Hq, D), dtype=torch.bfloat16).pin_memory()
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

        # prefilled K/V of the queries inserted at window step i arrive on their own
        # copy stream, enqueued INS_AHEAD steps ahead (inserts are known from the window
        # plan) and issued in pieces of at most INS_PIECE bytes, INS_BUDGET bytes per
        # step: one 7B insert of ~550 tokens is ~0.6 GB (~12 ms of PCIe at 50 GB/s), and
        # issued whole it could sit in a copy engine's queue ahead of the next step's q/k/v
        ins_at = {}
        for q, n, t_ins in fresh:
            ins_at.setdefault(t_ins - t_base, []).append(q)
        pref_dev = {}
        pending = []          # [qid, [(dst, src) flat views], part index, element offset, event]

        def prefetch_inserts(i):
            for q in ins_at.get(i, []):
                a, b = pref_h[q]
                # allocated on the decode stream (whose cached blocks from the device pass
                # have these shapes: no cudaMalloc stalling the host mid-window); the copy
                # stream fills them, the decode stream waits on `ev` before the insert
                da = torch.empty(a.shape, dtype=a.dtype, device=dev)
                db = torch.empty(b.shape, dtype=b.dtype, device=dev)
                ev = torch.cuda.Event()
                pref_dev[q] = (da, db, ev)
                pending.append([q, [(da.view(-1), a.view(-1)), (db.view(-1), b.view(-1))], 0, 0, ev])

        def pump(budget, until=None, gate=None):
            """Issue queued insert pieces: `budget` bytes, or through query `until`.
            `gate`: a decode-stream event the pieces wait for.  The host runs many steps
            ahead of the GPU, so without it a per-step budget is no pacing at all: the
            copy engine would take pieces queued for later steps while this step's q/k/v
            copy still waits on its event, and stall the decode behind them."""
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
            res_h.copy_(eng2.out[L - 1], non_blocking=True)   # the step's result to the host
            if not warm:
                counters["d2h"] += res_h.numel() * 2
            return st_

        eng = make_engine(token_host, prefill_host, use_graph=True)
        for st_set in sets:
            eng.register_staging(*st_set)
        warm_start(eng)
        for ev in free:
            ev.record()
        h2d(0)
        # steady state: the prefetch pipeline is full when the window opens (the inserts
        # of the next INS_AHEAD steps have landed); inside the timed region the pieces of
        # the inserts INS_AHEAD steps ahead move, and those are the bytes counted
        for i in range(INS_AHEAD):
            prefetch_inserts(i)
        pump(1 << 62)
        torch.cuda.synchronize()   # pipeline fill done (else it queues ahead of the first steps' tokens)
        for i in range(W):
            step(eng, i, True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        counters["h2d"] = counters["d2h"] = 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        st2 = [step(eng, W + i, False) for i in range(K_steps)]
        host_ms = (time.perf_counter() - h0) * 1e3
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms2 = e0.elapsed_time(e1)
        marks = [x for x in step_ev if x[0] >= W] + [(None, e1, 0)]
        step_ms = [(marks[k][0], marks[k][2], marks[k][1].elapsed_time(marks[k + 1][1]))
                   for k in range(len(marks) - 1)]
        e2e = {"ms": ms2, "host_ms": host_ms, "step_ms": step_ms, "tokens": sum(s.decoded for s in st2), "h2d": counters["h2d"] / K_steps,
               "d2h": counters["d2h"] / K_steps}
        release(eng)

    # ================= full run (steady-state AND full-run tokens/s): the
    # whole 512-query workload from iteration 0 until the batch drains -- fill, the
    # overloaded steady state, the tail with no replenishment.  Every step's q/k/v and
    # every insert's prefilled K/V come from the keyed generator on the device inside
    # the timed region (standing in for the model's projections and the prefill).
    full_run = None
    if world == 1 and not args.no_full_run:
        engf = Engine(wl, rank=0, world=1, device=dev, use_graph=True)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        st_f = engf.run()
        f1.record()
        torch.cuda.synchronize()
        ms_f = f0.elapsed_time(f1)
        tok_f = sum(s.decoded for s in st_f)
        full_run = {"value": tok_f / (ms_f / 1e3), "unit": "tokens/s", "iterations": len(st_f),
                    "tokens": tok_f, "queries": len(wl.queries), "ms": ms_f,
                    "what": "whole workload from iteration 0 to drain, one GPU; per-step q/k/v and "
                            "inserted K/V generated on the device (keygen) inside the timed region"}
        del engf, st_f
        gc.collect()
        torch.cuda.empty_cache()

    # ================= a8: the window's inserted prompts through the tcgen05 prefill
    # (P&D decouples it from the decode loop): one varlen launch per
    # layer over every prompt the window inserts; all layers cost the same, so one
    # layer is graph-timed.  Reported beside the decode numbers, not part of `value`.
    prefill = None
    if rank == 0 and fresh:
        from paper_2410_18701_b200.baton import baton_prefill_attention_varlen
        plens = [n for _, n, _ in fresh][:64]
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
        prefill = {"what": "baton_prefill_attention_varlen (tcgen05) over the window's inserted prompts, "
                           "one layer, graph-timed", "prompts": len(plens), "tokens": T,
                   "us_per_layer": us, "tflops": flop / us / 1e6, "peak_tflops": bf16_peak,
                   "peak_source": "measured" if os.path.exists(pk) else "nominal",
                   "frac": flop / us / 1e6 / bf16_peak}
        del qp, kp, vp, op, gr

    return dict(splice_bytes=splice_bytes, splice_s=splice_s, splice_calls=len(splice_ev), prefill=prefill,
                full_run=full_run,
                ms=ms, tokens=tokens, attn_bytes=attn_bytes_total, attn_time_s=attn_time_s,
                iter_ms=iter_ms,
                attn_launches=attn_launches, splice_rows=splice_rows, tau=tau, L=L,
                n_launch=n_launch, clocks=clk, e2e=e2e, iters=K_steps,
                live_slots=tokens / K_steps, live_rows=live_rows, gather_us=gather_us)


# ------------------------------------------------------------------ the oracle arm
def oracle_sample(budget_s=15.0, t0=T0_DEFAULT, max_steps=None, n_slots=None, warmup=0):
    """Time the fp64 oracle (O-2 Shard.step, as it stands) on a bounded sample of
    the same workload: ONE layer of the 7B batch at iteration t0, all live slots
    (or the ``n_slots`` longest).  ``warmup`` untimed steps first.
    Returns seconds per timed step, the sampled slot count, L, the timed steps and
    the live slot count of the full batch."""
    from baton_inputs import config_workload, KIND_K, KIND_V, KIND_Q, bf16_bits_to_f64
    from baton_inputs import query_history_bits, query_token_bits
    from oracle import Shard, Simulator
    wl = config_workload("7b")
    sim = Simulator(wl, kv=False)
    while sim.t <= t0:
        sim.iteration()
    osh = sim.shards[0]
    live = [b for b in range(wl.slots) if osh.qid[b] >= 0]
    lens = osh.lens()
    if n_slots:   # rows at evenly spaced length quantiles: the sample's mean length ~ the batch's
        by_len = sorted(live, key=lambda b: lens[b])
        picked = [by_len[int((i + 0.5) * len(by_len) / n_slots)] for i in range(n_slots)]
    else:
        picked = live
    # the oracle keeps DENSE [rows][S] tensors, so a sample shard holds exactly the
    # sampled rows (its cost is then linear in them)
    rows = len(picked) if n_slots else wl.slots
    sh = Shard(rows, 1, wl.q_heads, wl.kv_heads, wl.head_dim, wl.max_ctx, kv=True)
    occ = []
    for i, b in enumerate(sorted(picked, key=lambda b: -lens[b])):
        row = i if n_slots else b
        q = int(osh.qid[b])
        n = int(lens[b])
        K = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_K, 1, q, 0, n, wl.kv_heads, wl.head_dim, 0))
        V = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_V, 1, q, 0, n, wl.kv_heads, wl.head_dim, 0))
        sh.insert(row, q, n, K, V)
        occ.append(row)
    times = []
    step = 0
    warm = warmup
    while True:
        qids = np.zeros(sh.B, np.int64)
        pos = np.zeros(sh.B, np.int64)
        cur = sh.lens()
        for b in occ:
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
        step += 1
        if (max_steps and step >= max_steps) or (not max_steps and sum(times) >= budget_s):
            break
    return float(np.mean(times)), len(occ), wl.layers, step, len(live)


def run_reference(args):
    """The reference arm of this tier is the oracle (fp64 CPU).  A step = one oracle
    layer-iteration of a 4-row shard holding the live queries of the t0 batch at the
    12.5/37.5/62.5/87.5% length quantiles (the dense oracle's cost is linear in
    rows; the sample's mean length tracks the batch's), so W + K steps end within
    about a minute; tokens/s is extrapolated to all L layers: m / (L * t_step)."""
    m = 4
    t_step, m, L, n, live = oracle_sample(t0=args.t0, max_steps=args.steps, n_slots=m,
                                          warmup=args.warmup)
    value = m / (L * t_step)
    cores = 1
    line = {
        "impl": "reference", "metric": "decode tokens/s (7B-shape Baton batch)",
        "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": n, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (keyed generator)",
        "config": {"workload": "7b", "t0": args.t0},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
                         "sample": f"O-2 Shard.step (fp64 NumPy), per step 1 of {L} layers x {m} of {live} "
                                   f"live slots (length quantiles) at iteration {args.t0}; {n} timed steps "
                                   f"after {args.warmup} warm-up; tokens/s = {m} / ({L} x step time)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="baton", choices=["baton", "reference"])
    ap.add_argument("--t0", type=int, default=T0_DEFAULT)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-run", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=20.0)
    args = ap.parse_args()
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

    # max over ranks of the device time; tokens summed over ranks
    ms, tokens = r["ms"], r["tokens"]
    e2e_ms = r["e2e"]["ms"] if r["e2e"] else 0.0
    e2e_tok = r["e2e"]["tokens"] if r["e2e"] else 0
    if world > 1:
        rdev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = t.tolist()
        # SURVEY §8(d) for N > 1: the flag all-gather's host-blocking time per iteration
        # (max over ranks) and the per-rank attention-byte imbalance (max / mean)
        g = torch.tensor([r["gather_us"]], dtype=torch.float64, device=rdev)
        dist.all_reduce(g, op=dist.ReduceOp.MAX)
        bts = [torch.zeros(1, dtype=torch.float64, device=rdev) for _ in range(world)]
        dist.all_gather(bts, torch.tensor([float(r["attn_bytes"])], dtype=torch.float64, device=rdev))
        bts = [float(x.item()) for x in bts]
        multi = {"allgather_us_per_iter": float(g.item()),
                 "rank_attn_bytes_max_over_mean": max(bts) / (sum(bts) / world) if sum(bts) else None,
                 "collective": "all_gather of int32 completion flags per iteration (" + backend + ")"}
        c = torch.tensor([tokens, e2e_tok], dtype=torch.float64, device=rdev)
        dist.all_reduce(c)
        tokens, e2e_tok = [int(x) for x in c.tolist()]

    if rank == 0:
        peak, peak_kind = _peaks()
        achieved = r["attn_bytes"] / r["attn_time_s"] / 1e9 if r["attn_time_s"] else 0.0
        per_launch = r["attn_bytes"] / max(1, r["attn_launches"])
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r01_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp))["traffic_bytes"]
        line = {
            "metric": "decode tokens/s (7B-shape Baton batch)",
            "value": tokens / (ms / 1e3),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "iter_ms_p10_p50_p90": [float(x) for x in np.percentile(r["iter_ms"], [10, 50, 90])],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (keyed q/k/v generator, D1-style length mix, Poisson arrivals)",
            "config": {"workload": "7b: Llama-2-7B-shaped attention, 32 layers x 32 heads x d128, "
                                   "bf16 KV, 32 slots/GPU, ctx<=2048, Poisson 0.08/iter",
                       "t0": args.t0, "slots_per_gpu": 32, "parallelism": f"slots/{world} GPU",
                       "l2": "inputs larger than L2 (32 GiB KV cache, ~12 GiB read per step)",
                       "live_slots_per_step": r["live_slots"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "profiles/r01_traffic.json (one ncu --set full launch)",
                         "kernel": "decode_attention_kernel<128, 4, 2, 3>",
                         "bytes_per_launch": per_launch,
                         "peak_source": peak_kind,
                         "avg_launch_us": 1e6 * r["attn_time_s"] / max(1, r["attn_launches"]),
                         "timing": "CUDA events around each decode-step graph (mask update + L "
                                   "PDL-chained attention launches) over the same K-step window; "
                                   "avg_launch_us = graph time / (K * L)",
                         "step_hbm_GBps": r["attn_bytes"] / (ms / 1e3) / 1e9},
            "splice": {"calls": r["splice_calls"], "bytes": r["splice_bytes"],
                       "GBps": (r["splice_bytes"] / r["splice_s"] / 1e9) if r["splice_s"] else None,
                       "frac": (r["splice_bytes"] / r["splice_s"] / 1e9 / peak) if r["splice_s"] else None,
                       "what": "baton_insert_many (batched KV embed + mask splice) in the window, "
                               "algorithmic read+write bytes / event time"},
            "gpu_launches": r["n_launch"],
            "clocks": r["clocks"],
        }
        if world > 1:
            line["multi_gpu"] = multi
        if r["e2e"]:
            line["e2e"] = {"value": e2e_tok / (e2e_ms / 1e3), "unit": "tokens/s",
                           "h2d_bytes_per_step": int(r["e2e"]["h2d"]),
                           "d2h_bytes_per_step": int(r["e2e"]["d2h"]),
                           "host_enqueue_ms_per_step": r["e2e"]["host_ms"] / r["iters"],
                           "step_ms_p50_p90_max": [statistics.median([x[2] for x in r["e2e"]["step_ms"]]),
                                                   sorted(x[2] for x in r["e2e"]["step_ms"])[
                                                       int(0.9 * (len(r["e2e"]["step_ms"]) - 1))],
                                                   max(x[2] for x in r["e2e"]["step_ms"])],
                           "slowest_steps": sorted(((round(x[2], 2), x[0], x[1]) for x in r["e2e"]["step_ms"]),
                                                   reverse=True)[:4]}
        if r.get("prefill"):
            line["prefill"] = r["prefill"]
        if r.get("full_run"):
            line["full_run"] = r["full_run"]
        if world == 1 and not args.no_cpu_baseline:
            t_step, live, L, n, _ = oracle_sample(budget_s=15.0, t0=args.t0)
            line["cpu_baseline"] = {
                "value": live / (L * t_step), "unit": "tokens/s", "cores": 1, "kind": "oracle",
                "cpu_model": _cpu_model(),
                "sample": f"O-2 Shard.step (fp64 NumPy, single thread), 1 of {L} layers, {live} live "
                          f"slots at iteration {args.t0}, {n} steps, extrapolated x{L} layers"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
