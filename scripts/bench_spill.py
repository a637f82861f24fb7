"""Host spill of the stress config ("moved to the host memory"; SURVEY §8(d)
"host-spill GB/s vs PCIe"): baton_extract of one 7B-shaped query's K/V into pinned
host memory and baton_insert of it back from there (the copy kernel reads/writes
host memory directly over PCIe), against the box's cudaMemcpy H2D/D2H rates.

    python scripts/bench_spill.py [--len 900] [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_18701_b200.baton import BatonShard, baton_keygen_history   # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, default=900)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    L, H, D, n = 32, 32, 128, args.len
    sh = BatonShard(L, 4, H, H, D, 2048)
    K = torch.empty((L, H, n, D), dtype=torch.bfloat16, device="cuda")
    V = torch.empty_like(K)
    baton_keygen_history(K, L, H, D, 7, 0, n, 1, 18701, 0)
    baton_keygen_history(V, L, H, D, 7, 0, n, 2, 18701, 0)
    kh = torch.empty(K.shape, dtype=torch.bfloat16, pin_memory=True)
    vh = torch.empty(V.shape, dtype=torch.bfloat16, pin_memory=True)
    nbytes = 2 * K.numel() * 2
    ev = lambda: torch.cuda.Event(enable_timing=True)
    ext, ins = [], []
    sh.baton_insert(0, K, V, n)
    for _ in range(args.reps):
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        sh.baton_extract(0, kh, vh)        # device cache -> pinned host
        b.record()
        sh.baton_remove([0])
        torch.cuda.synchronize()
        ext.append(nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
        a, b = ev(), ev()
        a.record()
        sh.baton_insert(0, kh, vh, n)      # pinned host -> device cache
        b.record()
        torch.cuda.synchronize()
        ins.append(nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    assert torch.equal(kh.cuda(), K) and torch.equal(vh.cuda(), V)
    # reference: plain cudaMemcpy of the same bytes
    a, b = ev(), ev()
    a.record()
    kh.copy_(K, non_blocking=True)
    vh.copy_(V, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    d2h = nbytes / (a.elapsed_time(b) / 1e3) / 1e9
    a, b = ev(), ev()
    a.record()
    K.copy_(kh, non_blocking=True)
    V.copy_(vh, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    h2d = nbytes / (a.elapsed_time(b) / 1e3) / 1e9
    print(json.dumps({"what": "host spill of one query (32 layers x 32 heads x d128, K+V)", "tokens": n,
                      "bytes": nbytes, "extract_to_host_GBps": max(ext), "insert_from_host_GBps": max(ins),
                      "memcpy_d2h_GBps": d2h, "memcpy_h2d_GBps": h2d}))


if __name__ == "__main__":
    main()
