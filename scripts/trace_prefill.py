"""Per-tile clock64 timeline of the a8 prefill kernel (experiment build:
python -m paper_2410_18701_b200.build --experiments): one graph-free launch of a
prompt shape with the debug trace on, then per-CTA intervals over its first 16 tiles.

    python scripts/trace_prefill.py [--shape 70b:3400|7b:1800|...] [--out file.json]

Per tile t (cycles, SM clock): S issued -> softmax holds S(t) ('s_wait' counts from
the later of the S issue and the softmax's previous P), softmax (holds S -> published
P), P published -> the MMA thread's wait for it returns, that return -> P.V issued
(the tcgen05.mma issue itself), softmax idle (P(t-1) -> holds S(t)), and the per-tile
period of a CTA (two CTAs share an SM)."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_18701_b200 import _lib                                          # noqa: E402
from paper_2410_18701_b200.baton import baton_prefill_attention                 # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="70b:3400")
    ap.add_argument("--out", default="gpurun_out/prefill_trace.json")
    args = ap.parse_args()
    cfg, n = args.shape.split(":")
    n = int(n)
    Hq, Hkv = {"7b": (32, 32), "13b": (40, 40), "70b": (64, 8)}[cfg]
    lib = _lib.lib
    fn = lib.baton_debug_prefill_trace
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    fn.restype = ctypes.c_int
    g = torch.Generator(device="cuda").manual_seed(1)
    mk = lambda H: (torch.rand((H, n, 128), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q, k, v = mk(Hq), mk(Hkv), mk(Hkv)
    o = torch.empty_like(q)
    for _ in range(3):
        baton_prefill_attention(q, k, v, o, n, Hq, Hkv, 128)
    torch.cuda.synchronize()
    assert fn(1, None, 0) == 0, "needs an experiment build"
    baton_prefill_attention(q, k, v, o, n, Hq, Hkv, 128)
    torch.cuda.synchronize()
    buf = np.zeros((296, 62), np.int64)
    assert fn(0, buf.ctypes.data, buf.nbytes) == 0
    rows = buf[buf[:, 0] > 0]
    T = 12
    S = rows[:, 2:2 + 5 * T:5]      # MMA issued S(t)
    H = rows[:, 3:3 + 5 * T:5]      # softmax holds S(t)
    P = rows[:, 4:4 + 5 * T:5]      # softmax thread 0 published P(t)
    W = rows[:, 5:5 + 5 * T:5]      # MMA thread's wait for P(t) returned
    V = rows[:, 6:6 + 5 * T:5]      # MMA issued P.V(t)
    ok = (S > 0).all(1) & (H > 0).all(1) & (P > 0).all(1) & (W > 0).all(1) & (V > 0).all(1)
    S, H, P, W, V = S[ok], H[ok], P[ok], W[ok], V[ok]
    ts = slice(4, 10)
    prevP = np.concatenate([np.zeros((len(P), 1), np.int64), P[:, :-1]], 1)
    ready = np.maximum(S, prevP)
    med = lambda x: float(np.median(x))
    stats = {
        "ctas": int(ok.sum()),
        "s_wait": med(H[:, ts] - ready[:, ts]),
        "softmax": med(P[:, ts] - H[:, ts]),
        "p_to_mma_wait_return": med(W[:, ts] - P[:, ts]),
        "pv_issue_after_wait": med(V[:, ts] - W[:, ts]),
        "softmax_idle": med(H[:, ts] - prevP[:, ts]),
        "s_issue_to_hold": med(H[:, ts] - S[:, ts]),
        "pv_issue_to_next2_s_issue": med(S[:, 6:12] - V[:, 4:10]),
        "s_issue_to_next_p_wait_return": med(W[:, 4:10] - S[:, 5:11]),
        "period": med(np.diff(H[:, 3:12], axis=1)),
        "cta_cycles_med": med(rows[:, 1] - rows[:, 0]),
    }
    stats = {k_: float(v_) for k_, v_ in stats.items()}
    print(json.dumps({"shape": args.shape, **stats}))
    json.dump({"shape": args.shape, "stats": stats, "raw": rows.tolist()}, open(args.out, "w"))


if __name__ == "__main__":
    main()
