"""Decode-step throughput of the other BASELINE.json configs on ONE GPU (shards).

    python scripts/bench_configs.py [--steps K] [--warmup W] [--only NAME]

For each config: warm-start the batch at a steady-state iteration t0 through the
ABI (every live query embedded with its keyed history), pre-generate the window's
q/k/v and prefilled K/V in HBM, then time K graph-replayed decode iterations
(with their splices) with CUDA events.  Prints one JSON line per config with
decode tokens/s and the attention bytes per second of the step.

  7b       configs[1] (the bench.py workload; not in the default list)
  13b      configs[2] at G=1: 40 layers x 40 heads, 64 slots, 2 inserts + 2 removes/iter
  70b      one GPU's shard of configs[3]: 80 layers, 64q/8kv (GQA), 16 slots, ctx 4096
  stress   one GPU's shard of configs[4]: 7B shape, 2 -> 32 active slots, 25% preempted
           (extract to an HBM stash + re-insert) every 16 iterations
"""
import argparse
import copy
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from baton_inputs import config_workload                                   # noqa: E402
from paper_2410_18701_b200.engine import Engine                            # noqa: E402
from paper_2410_18701_b200.baton import baton_keygen_tokens, baton_keygen_history  # noqa: E402


def shard_workload(name):
    if name == "7b":            # configs[1], the bench.py workload (for traces / A-B runs)
        return config_workload("7b"), 512
    if name == "13b":
        return config_workload("13b", gpus=1), 256
    if name == "70b":
        wl = config_workload("70b", gpus=1)
        wl.slots = 16
        return wl, 512
    if name == "stress":
        wl = config_workload("stress", gpus=8)
        wl.slots, wl.gpus, wl.active = 32, 1, 2
        wl.control.resize = {t: n // 8 for t, n in wl.control.resize.items()}
        wl.queries = wl.queries[:400]
        wl.iterations = -1
        return wl, 200
    raise KeyError(name)


def run(name, K, W, dev):
    wl, t0 = shard_workload(name)
    L, Hq, Hkv, D = wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim
    eng = Engine(wl, device=dev, use_graph=True)
    pl = eng.planner
    while pl.t < t0:
        pl.plan()
    # warm start
    slots, ks, vs, lens = [], [], [], []
    for g, q in pl.live():
        n = pl.length[g]
        Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
        Vp = torch.empty_like(Kp)
        baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, 0)
        baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, 0)
        slots.append(g)
        ks.append(Kp)
        vs.append(Vp)
        lens.append(n)
    eng.shard.baton_insert_many(slots, ks, vs, lens)
    del ks, vs
    # window inputs
    probe = copy.deepcopy(pl)
    decs, fresh = [], []
    for _ in range(W + K):
        decs.append(probe.decode_plan())
        d = probe.plan()
        fresh += [(q, n) for g, q, n, home in d.inserts if home is None]
    B = pl.per_rank
    qa = torch.empty((W + K, L, B, Hq, D), dtype=torch.bfloat16, device=dev)
    ka = torch.empty((W + K, L, B, Hkv, D), dtype=torch.bfloat16, device=dev)
    va = torch.empty_like(ka)
    for i, dec in enumerate(decs):
        qid = np.full(B, -1, np.int32)
        pos = np.zeros(B, np.int32)
        for g, q, p in dec:
            qid[g], pos[g] = q, p
        dq, dp = torch.from_numpy(qid).to(dev), torch.from_numpy(pos).to(dev)
        baton_keygen_tokens(qa[i], dq, dp, L, B, Hq, D, 0, 0, wl.seed, 0)
        baton_keygen_tokens(ka[i], dq, dp, L, B, Hkv, D, 1, 0, wl.seed, 0)
        baton_keygen_tokens(va[i], dq, dp, L, B, Hkv, D, 2, 0, wl.seed, 0)
    pref = {}
    for q, n in fresh:
        Kp = torch.empty((L, Hkv, n, D), dtype=torch.bfloat16, device=dev)
        Vp = torch.empty_like(Kp)
        baton_keygen_history(Kp, L, Hkv, D, q, 0, n, 1, wl.seed, 0)
        baton_keygen_history(Vp, L, Hkv, D, q, 0, n, 2, wl.seed, 0)
        pref[q] = (Kp, Vp)
    eng.token_source = lambda t, dec: (qa[t - t0], ka[t - t0], va[t - t0])
    eng.prefill_source = lambda q, n: pref[q]
    torch.cuda.synchronize()
    for _ in range(W):
        eng.iteration()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = [eng.iteration() for _ in range(K)]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tokens = sum(s.decoded for s in st)
    tau = 2 * Hkv * D * 2
    attn_bytes = L * sum(s.live_rows * tau + s.decoded * Hq * D * 4 for s in st)
    splice_rows = sum(s.insert_rows + s.extract_rows + s.compact_rows for s in st)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    gbps = attn_bytes / (ms / 1e3) / 1e9
    return {"config": name, "layers": L, "q_heads": Hq, "kv_heads": Hkv, "slots": B, "t0": t0,
            "steps": K, "ms_per_step": ms / K, "decode_tokens_per_s": tokens / (ms / 1e3),
            "live_slots_per_step": tokens / K, "attn_GBps_step": gbps, "frac_of_peak": gbps / peak,
            "inserts": sum(s.inserted for s in st), "stored": sum(s.stored for s in st),
            "splice_rows": splice_rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    for name in ([args.only] if args.only else ["13b", "70b", "stress"]):
        print(json.dumps(run(name, args.steps, args.warmup, dev)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
