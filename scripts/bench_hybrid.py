"""NEXT-3 measured: the stress workload's stored K/V in HBM, in pinned host memory,
or in the prefetchable hybrid store.

    python scripts/bench_hybrid.py [--iters N] [--budget-frac F] [--workloads priority,stress]

Two workloads (shard_workload), run from iteration 0 under each store:

  hbm     every stored query's K/V in HBM (baton_extract HBM -> HBM)
  host    every stored query's K/V in pinned host memory: the extract kernel writes
          over PCIe, the re-insert kernel reads over PCIe, both on the decode stream
  hybrid  HBM up to F x the peak stored bytes of the hbm run, the rest spilled to the
          host and prefetched back to HBM on a copy stream ahead of the re-insert

Reports decode tokens/s of the run (CUDA events, inputs from the keyed generator
on the device as in bench.py's full run) and, per store, the host-spill bandwidth:
bytes extracted to the host / their extract calls' event time, and the prefetch
H2D bytes / the copy stream's busy time, both against the box's pinned cudaMemcpy
bandwidth measured here (the PCIe peak this path can reach).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from baton_inputs import config_workload, Query               # noqa: E402
from paper_2410_18701_b200.engine import Engine               # noqa: E402


def shard_workload(kind):
    """stress: one GPU's shard of configs[4] -- 25% of the live queries stored every 16
    iterations and re-inserted at the queue head, i.e. at once (nothing to prefetch).
    priority: the 7B batch (32 slots, D1 mix, Poisson 0.08/iteration, overloaded) with
    every fifth query urgent (priority 1, reading C25): an urgent arrival that finds no
    free slot stores the newest low-priority query, which then waits behind the urgent
    queue -- stored K/V that sit in the store for a while, the case prefetch is for."""
    if kind == "stress":
        wl = config_workload("stress", gpus=8)
        wl.slots, wl.gpus, wl.active = 32, 1, 2
        wl.control.resize = {t: n // 8 for t, n in wl.control.resize.items()}
        wl.queries = wl.queries[:400]
        return wl
    wl = config_workload("7b")
    wl.queries = [Query(q.qid, q.arrival, q.l_q, q.A, q.kind, 1 if q.qid % 5 == 4 else 0)
                  for q in wl.queries]
    return wl


def pcie_peak():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    for name, (dst, src) in {"h2d": (d, h), "d2h": (h, d)}.items():
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        out[name] = 3 * n / (a.elapsed_time(b) / 1e3) / 1e9
    return out


def run(kind, mode, iters, budget):
    wl = shard_workload(kind)
    wl.iterations = iters
    kw = {"hbm": {}, "host": {"stash_host": True},
          "hybrid": {"stash_host": "hybrid", "stash_hbm_bytes": budget}}[mode]
    eng = Engine(wl, use_graph=True, **kw)
    sh = eng.shard
    ext_ev, pf_ev = [], []
    orig_ext = sh.baton_extract

    def timed_extract(slot, k_out=None, v_out=None, stream=None):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = orig_ext(slot, k_out, v_out)
        b.record()
        ext_ev.append((a, b, r[0].numel() * 4, not r[0].is_cuda))
        return r

    sh.baton_extract = timed_extract
    st_ = eng.stash
    st_.timing = pf_ev           # events around each prefetch's H2D copies (copy stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stats = eng.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tok = sum(s.decoded for s in stats)
    host = [(a.elapsed_time(b), n) for a, b, n, h in ext_ev if h]
    hbm = [(a.elapsed_time(b), n) for a, b, n, h in ext_ev if not h]
    pf = [(a.elapsed_time(b), n) for a, b, n in pf_ev]
    gbps = lambda xs: (sum(n for _, n in xs) / (sum(t for t, _ in xs) / 1e3) / 1e9) if xs else None
    return {"mode": mode, "iterations": len(stats), "ms": ms, "tokens": tok, "tok_per_s": tok / (ms / 1e3),
            "stored": sum(s.stored for s in stats), "store": dict(st_.stats),
            "peak_stored_bytes": st_.peak_stored_bytes,
            "extract_to_host_GBps": gbps(host), "extract_to_host_bytes": sum(n for _, n in host),
            "extract_hbm_GBps": gbps(hbm), "prefetch_h2d_GBps": gbps(pf),
            "prefetch_bytes": sum(n for _, n in pf)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=640)
    ap.add_argument("--budget-frac", type=float, default=0.25)
    ap.add_argument("--workloads", default="priority,stress")
    args = ap.parse_args()
    peak = pcie_peak()
    print(json.dumps({"pcie_cudaMemcpy_GBps": peak}), flush=True)
    for kind in args.workloads.split(","):
        iters = args.iters if kind == "stress" else 3 * args.iters
        base = run(kind, "hbm", iters, None)
        base["workload"] = kind
        print(json.dumps(base), flush=True)
        budget = int(args.budget_frac * base["peak_stored_bytes"])
        for mode in ("host", "hybrid"):
            r = run(kind, mode, iters, budget)
            r["workload"] = kind
            r["hbm_budget_bytes"] = budget if mode == "hybrid" else None
            if r["extract_to_host_GBps"]:
                r["extract_to_host_frac_of_d2h_peak"] = r["extract_to_host_GBps"] / peak["d2h"]
            if r["prefetch_h2d_GBps"]:
                r["prefetch_frac_of_h2d_peak"] = r["prefetch_h2d_GBps"] / peak["h2d"]
            r["tok_per_s_over_hbm"] = r["tok_per_s"] / base["tok_per_s"]
            print(json.dumps(r), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
