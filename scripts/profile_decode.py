"""Time / profile decode attention alone on the cfg2 (7B) batch at iteration t0.

    python scripts/profile_decode.py [--iters N] [--layers L]

Builds one 7B-shaped shard (L layers, default 2), embeds every live query of the
t0 state with its keyed history through baton_insert_many, runs one mask update,
then launches baton_decode_attention N times per layer and reports the per-launch
time (CUDA events) and algorithmic GB/s.  Used under ncu for the profiles/.
Needs an experiment build (python -m paper_2410_18701_b200.build --experiments):
the product library has no debug timelines.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from baton_inputs import config_workload                                   # noqa: E402
from paper_2410_18701_b200.baton import BatonShard, baton_keygen_history   # noqa: E402
from paper_2410_18701_b200.scheduler import Planner                        # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--t0", type=int, default=512)
    ap.add_argument("--config", default="7b")
    ap.add_argument("--trace", default=None, help="GQA only: write the per-CTA timeline here")
    args = ap.parse_args()
    wl = config_workload(args.config)
    if args.config == "70b":
        wl.slots, wl.gpus = 16, 1
    pl = Planner(wl, 1)
    while pl.t < args.t0:
        pl.plan()
    L = args.layers
    sh = BatonShard(L, wl.slots, wl.q_heads, wl.kv_heads, wl.head_dim, wl.max_ctx)
    slots, ks, vs, lens = [], [], [], []
    for g, q in pl.live():
        n = pl.length[g]
        K = torch.empty((L, wl.kv_heads, n, wl.head_dim), dtype=torch.bfloat16, device="cuda")
        V = torch.empty_like(K)
        baton_keygen_history(K, L, wl.kv_heads, wl.head_dim, q, 0, n, 1, wl.seed, 0)
        baton_keygen_history(V, L, wl.kv_heads, wl.head_dim, q, 0, n, 2, wl.seed, 0)
        slots.append(g); ks.append(K); vs.append(V); lens.append(n)
    sh.baton_insert_many(slots, ks, vs, lens)
    del ks, vs
    sh.baton_mask_update()
    torch.cuda.synchronize()
    m = sh.baton_query()
    live = m["lens"]
    q = torch.randn((wl.slots, wl.q_heads, wl.head_dim), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    tau = 2 * wl.kv_heads * wl.head_dim * 2
    nbytes = int(live.sum()) * tau + int((live > 0).sum()) * wl.q_heads * wl.head_dim * 4
    # capture iters x L launches in a CUDA graph: GPU time only, no host launch overhead
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        for l in range(L):
            sh.baton_decode_attention(l, q, out)   # warm (sets kernel attributes)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s_):
            for it in range(args.iters):
                for l in range(L):
                    sh.baton_decode_attention(l, q, out)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us_graph = e0.elapsed_time(e1) * 1e3 / (args.iters * L)
    times = []
    for it in range(3):
        for l in range(L):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sh.baton_decode_attention(l, q, out)
            b.record()
            times.append((a, b))
    torch.cuda.synchronize()
    us_w = [a.elapsed_time(b) * 1e3 for a, b in times][L:]
    print(json.dumps({"config": args.config, "live_slots": int((live > 0).sum()),
                      "sum_lens": int(live.sum()), "bytes_per_launch": nbytes,
                      "us_per_launch_graph": us_graph, "GBps_graph": nbytes / us_graph / 1e3,
                      "us_eager_median": float(np.median(us_w)),
                      "variant": os.environ.get("BATON_GQA_VARIANT" if wl.kv_heads < wl.q_heads
                                                else "BATON_MHA_VARIANT", "0")}))
    if args.trace:
        trace_gqa(sh, q, out, g, args.trace)


def trace_gqa(sh, q, out, graph, path):
    """Per-CTA timeline of one launch (globaltimer ns) from the debug trace of
    decode_gqa.cu: eager single launch, and the last launch of a graph replay."""
    import ctypes
    from paper_2410_18701_b200 import _lib
    lib = _lib._load()
    fn = lib.baton_debug_gqa_trace
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    res = {}
    for mode in ("eager", "graph"):
        assert fn(1, None, 0) == 0
        if mode == "eager":
            sh.baton_decode_attention(0, q, out)
        else:
            graph.replay()
        torch.cuda.synchronize()
        buf = np.zeros((8, 256, 64), np.int64)
        assert fn(0, buf.ctypes.data, buf.nbytes) == 0
        buf = buf[int(np.argmax(buf[:, :, 0].max(axis=1)))]   # the latest launch
        rows = buf[buf[:, 0] > 0]
        t0 = rows[:, 0].min()
        ctas = []
        for r in rows:
            n = int(r[3])
            items = [[int(r[8 + 4 * k]), *(int(x - t0) if x else 0 for x in r[9 + 4 * k:12 + 4 * k])]
                     for k in range(min(n, 8))]
            ctas.append({"smid": int(r[4]), "enter": int(r[0] - t0), "built": int(r[1] - t0),
                         "exit": int(r[2] - t0), "items": items})
        res[mode] = ctas
        span = max(c["exit"] for c in ctas)
        first_ready = [c["items"][0][2] for c in ctas if c["items"]]
        exits = sorted(c["exit"] for c in ctas)
        busy = [c["items"][-1][3] - c["items"][0][2] for c in ctas if c["items"]]
        durs = [it[3] - it[2] for c in ctas for it in c["items"]]
        print(json.dumps({"trace": mode, "ctas": len(ctas), "span_ns": span,
                          "enter_max_ns": max(c["enter"] for c in ctas),
                          "built_median_ns": float(np.median([c["built"] for c in ctas])),
                          "first_ready_median_ns": float(np.median(first_ready)),
                          "first_ready_max_ns": max(first_ready),
                          "exit_p10_ns": exits[len(exits) // 10], "exit_median_ns": exits[len(exits) // 2],
                          "items_per_cta": float(np.mean([len(c["items"]) for c in ctas])),
                          "item_ns_median": float(np.median(durs)), "item_ns_max": max(durs),
                          "busy_frac": float(np.sum(busy) / (span * len(ctas)))}))
    json.dump(res, open(path, "w"))


if __name__ == "__main__":
    main()
