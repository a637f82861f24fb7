"""NEXT-4: the paper's four methods on the same libbaton kernels and the Fig. 6-8
traces, B200 edition.

    python scripts/policy_traces.py [--dataset d2|d1] [--batches 2,4,6,8,10] [--out DIR]

Methods:
  benchmark  transformers batch-wise: run-to-completion batches, the batch's prompts
             prefilled together inside it, left-padded to the longest  (Planner "benchmark")
  pd         P&D decoupling: prompts prefilled separately in groups of similar length
             (one varlen a8 launch per group), run-to-completion decode batches (Planner "pd")
  baton      Baton without P&D: relay race, a new query prefilled inside the batch
             (vector shaping, padded survivors)                         (Planner "shape")
  baton_pd   Baton with P&D: relay race, separately prefilled queries embedded  (Planner "baton")
As in the paper, every method returns a query's response as soon as it is done.

For every (method, batch) the engine's per-iteration log (Engine.log_records, CUDA
events after every iteration) is written as JSON lines to DIR/<dataset>_<method>_b<B>.jsonl:
the cumulative completed queries (Fig. 6), cumulative output tokens (Fig. 7) and the
live / dense K/V bytes (Fig. 8) over device time.  One summary line per batch goes to
stdout.  Model GEMMs are excluded (no weights): q/k/v are keyed synthetic values, so
the times are the attention + splice + prefill-attention path only.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from baton_inputs import Workload                                  # noqa: E402
from baton_inputs.workload import _mix_queries, CLASSES_7B, CLASSES_D2  # noqa: E402
from paper_2410_18701_b200.engine import Engine                    # noqa: E402

METHODS = {"benchmark": "benchmark", "pd": "pd", "baton": "shape", "baton_pd": "baton"}


def dataset(name, batch):
    rng = np.random.default_rng(2410)
    if name == "d2":     # 30 short/short queries, dozens to 200 words
        qs = _mix_queries(rng, 30, 30, 0.0, CLASSES_D2, 4096, all_at_zero=True)
    else:                # 120 queries, 1:1:2 long-in/short-out, short-in/long-out, short/short
        qs = _mix_queries(rng, 120, 120, 0.0, CLASSES_7B, 2048, all_at_zero=True)
    # shaping grows every row by each insert's width: a larger capacity
    # keeps it running longer (d1 may still stop with BATON_E_CAPACITY)
    return Workload(name, qs, layers=32, q_heads=32, kv_heads=32, head_dim=128, slots=batch,
                    max_ctx=4096 if name == "d2" else 8192)


def run(name, batch, method, out_dir):
    wl = dataset(name, batch)
    policy = METHODS[method]
    eng = Engine(wl, policy=policy, use_graph=True, prefill_attention=policy in ("pd", "baton"),
                 trace=True)
    eng.run()                                   # warm-up run (graph capture, allocator)
    eng = Engine(wl, policy=policy, use_graph=True, prefill_attention=policy in ("pd", "baton"),
                 trace=True)
    torch.cuda.synchronize()
    st = eng.run()
    recs = eng.log_records(st)
    path = os.path.join(out_dir, f"{name}_{method}_b{batch}.jsonl")
    with open(path, "w") as f:
        cq = ct = 0
        for r in recs:
            cq += r["completed"]
            ct += r["decoded"] - r["idle"]
            r["cum_completed"], r["cum_tokens"] = cq, ct
            f.write(json.dumps(r) + "\n")
    ms = recs[-1]["t_ms"]
    useful = sum(r["decoded"] - r["idle"] for r in recs)
    assert useful == wl.decode_tokens() and cq == len(wl.queries)
    kv = np.array([r["kv_live_bytes"] for r in recs], dtype=np.float64)
    t = np.array([r["t_ms"] for r in recs])
    dt = np.diff(np.concatenate([[0.0], t]))
    return {"ms": ms, "iterations": len(recs), "useful_tok_per_s": useful / (ms / 1e3),
            "idle_tokens": sum(r["idle"] for r in recs),
            "bubble_rows": sum(r["bubble_rows"] for r in recs),
            "kv_live_peak_GB": kv.max() / 1e9, "kv_live_mean_GB": float((kv * dt).sum() / dt.sum()) / 1e9,
            "kv_utilisation": float((kv * dt).sum() / dt.sum() / kv.max()),
            "t_half_queries_ms": float(t[np.searchsorted(np.cumsum([r["completed"] for r in recs]),
                                                          len(wl.queries) / 2)]),
            "trace": os.path.relpath(path, ROOT)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dataset", default="d2")
    ap.add_argument("--batches", default="2,4,6,8,10")
    ap.add_argument("--methods", default="benchmark,pd,baton,baton_pd")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_traces"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    for b in [int(x) for x in args.batches.split(",")]:
        res = {}
        for m in args.methods.split(","):
            try:
                res[m] = run(args.dataset, b, m, args.out)
            except Exception as e:          # the shaping arm outgrowing its capacity
                res[m] = {"error": str(e)[:200]}
            torch.cuda.empty_cache()
        line = {"dataset": args.dataset, "batch": b, **res}
        if "benchmark" in res:
            line["speedup_over_benchmark"] = {m: res["benchmark"]["ms"] / r["ms"] for m, r in res.items()
                                              if "ms" in r and "ms" in res["benchmark"]}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
