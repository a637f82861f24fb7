"""Measure a8 (baton_prefill_attention, tcgen05) on the configs' prompt shapes.

    python scripts/bench_prefill.py [--iters N]

Prints one JSON line per shape: causal FLOPs (4*H*D*sum_i (i+1), the algorithmic
work of the masked product), CUDA-event time per launch (graph of --iters launches) and TFLOP/s as a fraction
of the measured dense bf16 peak (MEASURED_PEAKS.json bf16_tflops, burst)."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_18701_b200.baton import baton_prefill_attention, baton_prefill_attention_varlen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default=None, help="one shape: e.g. 70b:3400 or 7b-mix64")
    ap.add_argument("--batches-only", action="store_true", help="only the varlen batches and mixes")
    args = ap.parse_args()
    peak = 1657.7
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p))["bf16_tflops"]
    shapes = [("7b", 32, 32, 512), ("7b", 32, 32, 1024), ("7b", 32, 32, 1800),
              ("13b", 40, 40, 1024), ("70b", 64, 8, 3400)]
    def graph_us(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # graph-replayed launches: the per-call host work (three tensor-map encodes)
        # would otherwise starve the GPU on the short prompts
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            for _ in range(args.iters):
                fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / args.iters

    # NEXT-2: the prompts of one iteration's inserts in ONE varlen launch vs one
    # launch per prompt (same arithmetic, bit-identical rows)
    batches = [("13b", 40, 40, [600, 550]), ("7b", 32, 32, [1500, 350, 120, 900]),
               ("70b", 64, 8, [3400, 300, 200])]
    # the bench line's prefill leg: 64 prompts of a config's length mix in one launch
    from baton_inputs import config_workload
    for cname, Hq, Hkv in (("7b", 32, 32), ("13b", 40, 40)):
        wl = config_workload(cname)
        batches.append((cname + "-mix64", Hq, Hkv, [q.l_q for q in wl.queries[:64]]))
    wl = config_workload("70b")
    batches.append(("70b-mix18", 64, 8, [q.l_q for q in wl.queries[:18]]))
    if args.only:   # a batch by name (e.g. 7b-mix64) or one single-prompt shape
        batches = [b for b in batches if b[0] == args.only]
        shapes = [s for s in shapes if f"{s[0]}:{s[3]}" == args.only]
    for name, Hq, Hkv, lens in batches:
        D, T = 128, sum(lens)
        q = torch.randn((Hq, T, D), device="cuda").to(torch.bfloat16)
        k = torch.randn((Hkv, T, D), device="cuda").to(torch.bfloat16)
        v = torch.randn((Hkv, T, D), device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        us_v = graph_us(lambda: baton_prefill_attention_varlen(q, k, v, o, lens, Hq, Hkv, D))
        parts = []
        s0 = 0
        for n in lens:
            parts.append((q[:, s0:s0 + n].contiguous(), k[:, s0:s0 + n].contiguous(),
                          v[:, s0:s0 + n].contiguous(), torch.empty((Hq, n, D), dtype=torch.bfloat16,
                                                                    device="cuda"), n))
            s0 += n
        us_s = graph_us(lambda: [baton_prefill_attention(a, b, c, d, n, Hq, Hkv, D) for a, b, c, d, n in parts])
        flops = sum(4.0 * Hq * D * (n * (n + 1) / 2) for n in lens)
        print(json.dumps({"shape": name, "varlen": lens if len(lens) <= 8 else f"{len(lens)} prompts, {sum(lens)} tokens", "q_heads": Hq, "kv_heads": Hkv, "us": us_v,
                          "us_separate": us_s, "tflops": flops / us_v / 1e6,
                          "tflops_separate": flops / us_s / 1e6, "frac": flops / us_v / 1e6 / peak}))

    for name, Hq, Hkv, n in ([] if args.batches_only else shapes):
        D = 128
        q = torch.randn((Hq, n, D), device="cuda").to(torch.bfloat16)
        k = torch.randn((Hkv, n, D), device="cuda").to(torch.bfloat16)
        v = torch.randn((Hkv, n, D), device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        for _ in range(3):
            baton_prefill_attention(q, k, v, o, n, Hq, Hkv, D)
        torch.cuda.synchronize()
        # graph-replayed launches: the per-call host work (three tensor-map encodes)
        # would otherwise starve the GPU on the short prompts
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            for _ in range(args.iters):
                baton_prefill_attention(q, k, v, o, n, Hq, Hkv, D)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.iters
        flops = 4.0 * Hq * D * (n * (n + 1) / 2)
        tf = flops / us / 1e6
        print(json.dumps({"shape": name, "q_heads": Hq, "kv_heads": Hkv, "len": n, "us": us,
                          "causal_flop": flops, "tflops": tf, "peak_tflops": peak,
                          "frac": tf / peak}))


if __name__ == "__main__":
    main()
