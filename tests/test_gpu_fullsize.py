"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times: the 7B-shaped batch (configs[1]), one GPU's shard of the 70B-GQA batch
(configs[3]) and the 13B churn batch (configs[2]) run through the Engine from
iteration 0.  Metadata and mask are compared bit-exactly with the oracle's
metadata state machine after every iteration; live K/V bytes and attention
outputs are compared on sampled slots/layers against the keyed history and O-1
solo attention computed one query at a time."""
import numpy as np
import pytest
import torch

from baton_inputs import (config_workload, KIND_K, KIND_V, KIND_Q, query_history_bits,
                          query_token_bits, bf16_bits_to_f64)
from oracle import Simulator, solo_attention
from gpu_util import ATTN_RTOL, bf16_bits, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _solo_layer(wl, qid, pos, layer):
    K = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_K, layer + 1, qid, 0, pos + 1,
                                            wl.kv_heads, wl.head_dim, wl.scales[1])[layer])
    V = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_V, layer + 1, qid, 0, pos + 1,
                                            wl.kv_heads, wl.head_dim, wl.scales[2])[layer])
    q = bf16_bits_to_f64(query_token_bits(wl.seed, KIND_Q, layer, [qid], [pos], wl.q_heads,
                                          wl.head_dim, wl.scales[0]))[0]
    return solo_attention(q, K, V)


def _run(wl, iters, sample_layers, n_sample_tokens, seed):
    from paper_2410_18701_b200.engine import Engine
    rng = np.random.default_rng(seed)
    eng = Engine(wl, keep_outputs=True, keep_layers=sample_layers)
    sim = Simulator(wl, kv=False)
    worst = 0.0
    for it in range(iters):
        rec = sim.iteration()
        eng.iteration()
        torch.cuda.synchronize()
        sh, osh = eng.shard, sim.shards[0]
        m = sh.baton_query()
        occ = osh.qid >= 0
        assert m["S"] == osh.S and np.array_equal(m["lens"], osh.lens())
        assert np.array_equal(np.where(occ, m["pad"], 0), np.where(occ, osh.pad, 0))
        assert np.array_equal(sh.mask[:, :osh.S].cpu().numpy(), osh.mask)
        assert int(sh.d_S.item()) == osh.S
        # sampled live K/V bytes == the query's keyed history
        occ_slots = np.nonzero(occ)[0]
        for b in rng.choice(occ_slots, size=min(2, len(occ_slots)), replace=False):
            qid = int(osh.qid[b])
            n = int(osh.lens()[b])
            l = int(rng.choice(sample_layers))
            ref = query_history_bits(wl.seed, KIND_K, l + 1, qid, 0, n, wl.kv_heads, wl.head_dim,
                                     wl.scales[1])[l]
            assert np.array_equal(bf16_bits(sh.k_cache[l, b, :, :n]), ref)
            ref = query_history_bits(wl.seed, KIND_V, l + 1, qid, 0, n, wl.kv_heads, wl.head_dim,
                                     wl.scales[2])[l]
            assert np.array_equal(bf16_bits(sh.v_cache[l, b, :, :n]), ref)
        # sampled attention outputs of this iteration's decode
        if rec.decoded:
            picks = rng.choice(len(rec.decoded), size=min(n_sample_tokens, len(rec.decoded)),
                               replace=False)
            for i in picks:
                g, qid, pos = rec.decoded[i]
                got = eng.outputs[(qid, pos)]
                for li, l in enumerate(sample_layers):
                    err = row_rel_err(got[li], _solo_layer(wl, qid, pos, l))
                    worst = max(worst, err)
        eng.outputs.clear()
    assert worst <= ATTN_RTOL, worst
    return worst


def test_7b_shape_full_size():
    """configs[1]: 32 heads x d128, batch 32, ctx up to 2048, Poisson arrivals."""
    require_cuda()
    wl = config_workload("7b")
    _run(wl, iters=4, sample_layers=[0, 31], n_sample_tokens=3, seed=1)


def test_70b_gqa_shard_full_size():
    """One GPU's shard of configs[3]: 64 q heads / 8 kv heads, 16 slots, ctx 4096."""
    require_cuda()
    wl = config_workload("70b", gpus=1, n_queries=64)
    wl.slots = 16
    _run(wl, iters=3, sample_layers=[0, 79], n_sample_tokens=2, seed=2)


def test_13b_churn_full_size():
    """configs[2] at G=1: 40 heads, batch 64, 2 removes + 2 inserts per iteration."""
    require_cuda()
    wl = config_workload("13b", n_queries=200)
    _run(wl, iters=4, sample_layers=[0, 39], n_sample_tokens=2, seed=3)


def test_stress_shard_full_size_with_preemption():
    """One GPU's shard of configs[4] (7B shape): active slots doubling 2 -> 32 and
    25% of live queries stored (extract to an HBM stash) and re-inserted every 16
    iterations.  Runs from iteration 0 through the first preemption rounds."""
    require_cuda()
    wl = config_workload("stress", gpus=8, n_queries=400)
    wl.slots, wl.gpus, wl.active = 32, 1, 8
    wl.control.resize = {24: 16}          # scale up mid-window
    wl.iterations = -1
    sim = Simulator(wl)
    assert sum(len(sim.iteration().preempted) for _ in range(50)) >= 4
    _run(wl, iters=50, sample_layers=[0, 31], n_sample_tokens=1, seed=4)
