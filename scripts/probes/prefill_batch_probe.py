"""Engine P&D accounting: a8 for k fresh queries, per query (L launches each) vs
batched (one varlen launch per layer).  Device time with events + host time."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from baton_inputs import config_workload                    # noqa: E402
from paper_2410_18701_b200.engine import Engine             # noqa: E402


def main():
    wl = config_workload("7b")
    eng = Engine(wl, device="cuda", use_graph=True, prefill_attention=True)
    rng = np.random.default_rng(0)
    for k, lo, hi in ((8, 30, 200), (8, 300, 1800), (2, 400, 1200)):
        items = []
        for i in range(k):
            n = int(rng.integers(lo, hi))
            K, V = eng._prefill(1000 + i, n)
            items.append((1000 + i, n, K, V))
        for mode in ("per_query", "batched", "per_query", "batched"):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0 = time.perf_counter()
            e0.record()
            if mode == "batched":
                eng._prefill_attn_batch(items)
            else:
                for it in items:
                    eng._prefill_attn(*it)
            e1.record()
            h1 = time.perf_counter()
            torch.cuda.synchronize()
            print(json.dumps({"k": k, "lens": [n for _, n, _, _ in items], "mode": mode,
                              "device_ms": e0.elapsed_time(e1), "host_ms": (h1 - h0) * 1e3}))


if __name__ == "__main__":
    main()
