"""NEXT-4 / NEXT-1: Baton's policies vs the paper's run-to-completion Benchmark on B200.

    python scripts/policy_compare.py [--dataset d2|d1] [--batches 2,4,6,8,10] [--no-shape]

Runs the whole synthetic dataset through the same libbaton kernels under
  * "rtc"   -- the paper's Benchmark: a finished query keeps decoding idle EOS
               tokens until its whole batch is done;
  * "shape" -- Baton WITHOUT P&D ("Ours"): a new query is prefilled
               inside the batch, every row padded to its prompt length (NEXT-1);
  * "baton" -- Baton WITH P&D decoupling ("Ours-PD"): width-1 decode for
               everybody, the prompt prefilled separately by a8 -- in the decode
               stream, and asynchronously on a side stream ahead of the insert
               (Engine(async_prefill=True));
and reports, per batch size, the completion time of the dataset (device time of
all iterations) and useful decode tokens/s: the B200 counterpart of Tables 2/3
(P:L230-289), with the paper's datasets replaced by the length mixes of P:L212.
Every arm pays its prefill attention (rtc and baton: a8 per fresh insert; shape:
in the shaped iteration).  Model GEMMs are excluded (no weights), so the bubble
of the shape arm costs only its attention here.
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


def dataset(name, batch):
    rng = np.random.default_rng(2410)
    if name == "d2":     # 30 short/short queries, dozens to 200 words
        qs = _mix_queries(rng, 30, 30, 0.0, CLASSES_D2, 4096, all_at_zero=True)
    else:                # 120 queries, 1:1:2 long-in/short-out, short-in/long-out, short/short
        qs = _mix_queries(rng, 120, 120, 0.0, CLASSES_7B, 2048, all_at_zero=True)
    # run-to-completion grows finished queries until the batch ends: 4096 capacity
    return Workload(name, qs, layers=32, q_heads=32, kv_heads=32, head_dim=128, slots=batch,
                    max_ctx=4096)


def run(name, batch, policy, async_prefill=False):
    wl = dataset(name, batch)
    eng = Engine(wl, policy=policy, use_graph=True, prefill_attention=policy != "shape",
                 async_prefill=async_prefill)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = eng.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    useful = sum(s.decoded - s.idle for s in st)
    assert useful == wl.decode_tokens()
    return {"iterations": len(st), "ms": ms, "useful_tokens": useful,
            "idle_tokens": sum(s.idle for s in st), "useful_tok_per_s": useful / (ms / 1e3),
            "shaped_iterations": sum(1 for s in st if s.prefill_rows),
            "bubble_rows": sum(s.bubble_rows for s in st),
            "max_S": max(s.S for s in st)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dataset", default="d2")
    ap.add_argument("--batches", default="2,4,6,8,10")
    ap.add_argument("--no-shape", action="store_true")
    args = ap.parse_args()
    for b in [int(x) for x in args.batches.split(",")]:
        base = run(args.dataset, b, "rtc")
        bat = run(args.dataset, b, "baton")
        asy = run(args.dataset, b, "baton", async_prefill=True)
        line = {"dataset": args.dataset, "batch": b, "benchmark_rtc": base, "baton_pd": bat,
                "baton_pd_async": asy, "completion_speedup": base["ms"] / bat["ms"],
                "async_over_sync_pd": bat["ms"] / asy["ms"]}
        if not args.no_shape:
            try:
                shp = run(args.dataset, b, "shape")
                line["baton_shape"] = shp
                line["pd_over_shape"] = shp["ms"] / bat["ms"]     # Table 2: Ours-PD vs Ours
            except Exception as e:                                 # KV growth (Fig. 8)
                line["baton_shape"] = {"error": str(e)}
        print(json.dumps(line), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
