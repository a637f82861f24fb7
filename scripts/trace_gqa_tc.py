"""Per-tile timeline of the tcgen05 GQA decode kernel (BATON_GQA_VARIANT=20) on the
70B shard, K/V resident in L2 (one layer, stateless launches).
Needs an experiment build (python -m paper_2410_18701_b200.build --experiments):
the product library has no debug timelines.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BATON_GQA_VARIANT", "20")
from baton_inputs import config_workload                                   # noqa: E402
from paper_2410_18701_b200.baton import BatonShard, baton_keygen_history   # noqa: E402
from paper_2410_18701_b200.scheduler import Planner                        # noqa: E402
from paper_2410_18701_b200 import _lib                                     # noqa: E402


def main():
    wl = config_workload("70b")
    wl.slots, wl.gpus = 16, 1
    pl = Planner(wl, 1)
    while pl.t < 512:
        pl.plan()
    L = 1
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
    sh.baton_mask_update()
    q = torch.randn((wl.slots, wl.q_heads, wl.head_dim), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    for _ in range(3):
        sh.baton_decode_attention(0, q, out)
    torch.cuda.synchronize()
    lib = _lib._load()
    fn = lib.baton_debug_gqa_tc_trace
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    mode = sys.argv[1] if len(sys.argv) > 1 else "eager"
    if mode == "graph":   # the last of 10 graph-replayed launches (each overwrites the trace)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                for _ in range(10):
                    sh.baton_decode_attention(0, q, out)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert fn(1, None, 0) == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"graph_us_per_launch": e0.elapsed_time(e1) * 100}))
    else:
        assert fn(1, None, 0) == 0
        sh.baton_decode_attention(0, q, out)
        torch.cuda.synchronize()
    buf = np.zeros((160, 68), np.int64)
    assert fn(0, buf.ctypes.data, buf.nbytes) == 0
    rows = buf[buf[:, 0] > 0]
    t0 = rows[:, 0].min()
    span = rows[:, 1].max() - t0
    per = []
    for r in rows:
        for j in range(16):
            ms, ss, pp, mp = r[4 + 4 * j:8 + 4 * j]
            if ms and ss and pp and mp:
                per.append((ss - ms, pp - ss, mp - pp))
    per = np.array(per).reshape(-1, 3)
    gaps = []
    for r in rows:
        prev = None
        for j in range(16):
            ss = r[5 + 4 * j]
            if ss:
                if prev:
                    gaps.append(ss - prev)
                prev = ss
    print(json.dumps({"mode": mode, "ctas": len(rows), "span_ns": int(span),
                      "enter_spread_ns": int(rows[:, 0].max() - t0),
                      "S_issue_to_softmax_start_ns": float(np.median(per[:, 0])),
                      "softmax_ns": float(np.median(per[:, 1])),
                      "P_to_PV_issue_ns": float(np.median(per[:, 2])),
                      "softmax_start_to_next_start_ns": float(np.median(gaps)),
                      "first_S_issue_ns": float(np.median([r[4] - t0 for r in rows if r[4]])),
                      "exit_median_ns": float(np.median(rows[:, 1] - t0))}))


if __name__ == "__main__":
    main()
