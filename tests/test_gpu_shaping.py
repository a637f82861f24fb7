"""GPU parity of the vector-SHAPING path (NEXT-1, ``baton_shape_step``) against the
oracle's shape policy (oracle/schedule.py, pinned in test_oracle_shaping.py).

The oracle run is replayed through the C ABI iteration by iteration: a shaped
iteration where the oracle prefilled raw queries, an ordinary decode elsewhere,
removal + release every iteration.  After EVERY iteration:
  * bit-exact: S, pad, per-slot region length, the mask bytes (with the padding
    holes of P:L105), and the K/V rows of every occupied slot's region (hole rows
    hold the padding tokens' K/V, zero here as in the oracle's fill);
  * every real output row (survivors' decodes, the new queries' prefill rows)
    within 1e-2 row-relative of the oracle (C13)."""
import numpy as np
import pytest
import torch

from baton_inputs import (Query, Workload, w1_workload, KIND_Q, KIND_K, KIND_V,
                          query_token_bits, SCALES_PEAKY)
from oracle import Simulator
from gpu_util import ATTN_RTOL, bf16_bits, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _f64_to_bits(x):
    return (np.asarray(x, np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def _tok_bits(wl, kind, H, qids, pos):
    scale = wl.scales[{KIND_Q: 0, KIND_K: 1, KIND_V: 2}[kind]]
    return np.stack([query_token_bits(wl.seed, kind, l, qids, pos, H, wl.head_dim, scale)
                     for l in range(wl.layers)])           # [L][B][H][D] uint16


def _to_dev(bits):
    return torch.from_numpy(bits.view(np.int16).copy()).cuda().view(torch.bfloat16)


def _replay(wl):
    from paper_2410_18701_b200.baton import BatonShard
    L, B, Hq, Hkv, D = wl.layers, wl.slots, wl.q_heads, wl.kv_heads, wl.head_dim
    sim = Simulator(wl, kv=True, keep_outputs=True, policy="shape")
    sh = BatonShard(L, B, Hq, Hkv, D, wl.max_ctx)
    osh = sim.shards[0]
    worst, n_shaped = 0.0, 0
    while not sim.done():
        pre_lens = osh.lens().copy()
        pre_qid = osh.qid.copy()
        rec = sim.iteration()
        if rec.t > 0:
            if rec.prefilled:
                W = rec.width[0]
                n_shaped += 1
                q = np.zeros((L, B, W, Hq, D), np.uint16)      # token-major (include/baton.h)
                k = np.zeros((L, B, W, Hkv, D), np.uint16)
                v = np.zeros((L, B, W, Hkv, D), np.uint16)
                occ = np.nonzero(pre_qid >= 0)[0]
                if len(occ):
                    qids, pos = np.where(pre_qid >= 0, pre_qid, 0), pre_lens
                    for kind, H, arr in ((KIND_Q, Hq, q), (KIND_K, Hkv, k), (KIND_V, Hkv, v)):
                        tb = _tok_bits(wl, kind, H, qids, pos)
                        for b in occ:
                            arr[:, b, 0] = tb[:, b]
                for g, qid, l in rec.prefilled:
                    for t in range(l):
                        for kind, H, arr in ((KIND_Q, Hq, q), (KIND_K, Hkv, k), (KIND_V, Hkv, v)):
                            arr[:, g, t] = _tok_bits(wl, kind, H, [qid], [t])[:, 0]
                out = torch.empty((L, B, W, Hq, D), dtype=torch.bfloat16, device="cuda")
                sh.baton_shape_step(W, [g for g, _, _ in rec.prefilled], [l for _, _, l in rec.prefilled],
                                    _to_dev(q), _to_dev(k), _to_dev(v), out)
                o = out.float().cpu().numpy()
                for g, qid, pos in rec.decoded:
                    worst = max(worst, row_rel_err(o[:, g, 0], sim.outputs[(qid, pos)]))
                for g, qid, l in rec.prefilled:
                    for t in range(l):
                        worst = max(worst, row_rel_err(o[:, g, t], sim.outputs[(qid, t)]))
            else:
                qids = np.where(pre_qid >= 0, pre_qid, 0)
                q = _to_dev(_tok_bits(wl, KIND_Q, Hq, qids, pre_lens))
                k = _to_dev(_tok_bits(wl, KIND_K, Hkv, qids, pre_lens))
                v = _to_dev(_tok_bits(wl, KIND_V, Hkv, qids, pre_lens))
                out = torch.empty((L, B, Hq, D), dtype=torch.bfloat16, device="cuda")
                sh.baton_mask_update()
                for l in range(L):
                    sh.baton_decode_layer(l, q[l], out[l], k[l], v[l])
                o = out.float().cpu().numpy()
                for g, qid, pos in rec.decoded:
                    worst = max(worst, row_rel_err(o[:, g], sim.outputs[(qid, pos)]))
            sh.baton_remove(rec.removed)
        torch.cuda.synchronize()
        # ---- state after the iteration, bit for bit
        m = sh.baton_query()
        occ = osh.qid >= 0
        assert m["S"] == osh.S
        assert np.array_equal(m["occ"].astype(bool), occ)
        assert np.array_equal(np.where(occ, m["pad"], 0), np.where(occ, osh.pad, 0))
        assert np.array_equal(np.where(occ, m["lens"], 0), np.where(occ, osh.S - osh.pad, 0))
        assert np.array_equal(sh.mask[:, :osh.S].cpu().numpy(), osh.mask)
        assert not sh.mask[:, osh.S:].cpu().numpy().any()
        for b in np.nonzero(occ)[0]:
            p, n = int(osh.pad[b]), osh.S - int(osh.pad[b])
            for cache, ref in ((sh.k_cache, osh.K), (sh.v_cache, osh.V)):
                assert np.array_equal(bf16_bits(cache[:, b, :, :n]), _f64_to_bits(ref[:, b, :, p:])), b
    assert worst <= ATTN_RTOL, worst
    return n_shaped, worst


def _w1_128(hq=2, hkv=2, scales=None):
    wl = w1_workload() if scales is None else w1_workload(scales=scales)
    wl.head_dim, wl.q_heads, wl.kv_heads, wl.layers, wl.max_ctx = 128, hq, hkv, 2, 512
    return wl


def test_w1_shaping_replay():
    require_cuda()
    n, _ = _replay(_w1_128())
    assert n >= 5


def test_w1_shaping_replay_gqa_peaky():
    require_cuda()
    _replay(_w1_128(8, 1, SCALES_PEAKY))


def test_shaping_multi_tile():
    """Query tiles > 128 rows, key tiles with holes wider than a tile (W - 1 > 64),
    several inserts of different lengths in one iteration."""
    require_cuda()
    qs = [Query(0, 0, 300, 40), Query(1, 0, 170, 30), Query(2, 0, 90, 50),
          Query(3, 5, 260, 20), Query(4, 5, 140, 25), Query(5, 12, 333, 10)]
    wl = Workload("shape-tiles", qs, layers=1, q_heads=4, kv_heads=2, head_dim=128, slots=4,
                  max_ctx=2048)
    n, _ = _replay(wl)
    assert n >= 3


def test_shape_step_errors():
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    from paper_2410_18701_b200._lib import BatonError
    sh = BatonShard(1, 2, 2, 2, 128, 64)
    z = lambda *s: torch.zeros(s, dtype=torch.bfloat16, device="cuda")
    q, kv, out = z(1, 2, 4, 2, 128), z(1, 2, 4, 2, 128), z(1, 2, 4, 2, 128)
    sh.baton_shape_step(4, [0], [3], q, kv, kv, out)
    with pytest.raises(BatonError, match="busy"):
        sh.baton_shape_step(4, [0], [2], q, kv, kv, out)
    with pytest.raises(BatonError, match="capacity"):
        sh.baton_shape_step(4, [1], [5], q, kv, kv, out)        # l > W
    big = z(1, 2, 64, 2, 128)
    with pytest.raises(BatonError, match="capacity"):
        sh.baton_shape_step(64, [1], [64], big, big, big, big)   # S + W > max_ctx
    small = BatonShard(1, 2, 2, 2, 16, 64)
    with pytest.raises(BatonError, match="invalid"):
        small.baton_shape_step(1, [0], [1], z(1, 2, 2, 1, 16), z(1, 2, 2, 1, 16),
                               z(1, 2, 2, 1, 16), z(1, 2, 2, 1, 16))


@pytest.mark.parametrize("wl_fn", ["w1", "tiles"])
def test_engine_shape_policy_replay(wl_fn):
    """The product path (Planner + Engine, policy "shape") against the oracle's
    shape policy: state bit-exact after every iteration, every output (decodes
    and prefill rows) within 1e-2."""
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    if wl_fn == "w1":
        wl = _w1_128(4, 2)
    else:
        qs = [Query(0, 0, 300, 40), Query(1, 0, 170, 30), Query(2, 0, 90, 50),
              Query(3, 5, 260, 20), Query(4, 5, 140, 25), Query(5, 12, 333, 10)]
        wl = Workload("shape-tiles", qs, layers=1, q_heads=4, kv_heads=2, head_dim=128, slots=4,
                      max_ctx=2048)
    sim = Simulator(wl, kv=True, keep_outputs=True, policy="shape")
    eng = Engine(wl, keep_outputs=True, policy="shape")
    osh, sh = sim.shards[0], eng.shard
    while not sim.done():
        sim.iteration()
        eng.iteration()
        torch.cuda.synchronize()
        m = sh.baton_query()
        occ = osh.qid >= 0
        assert m["S"] == osh.S
        assert np.array_equal(np.where(occ, m["pad"], 0), np.where(occ, osh.pad, 0))
        assert np.array_equal(sh.mask[:, :osh.S].cpu().numpy(), osh.mask)
        for b in np.nonzero(occ)[0]:
            p, n = int(osh.pad[b]), osh.S - int(osh.pad[b])
            assert int(m["lens"][b]) == n
            for cache, ref in ((sh.k_cache, osh.K), (sh.v_cache, osh.V)):
                assert np.array_equal(bf16_bits(cache[:, b, :, :n]), _f64_to_bits(ref[:, b, :, p:]))
    assert eng.done()
    assert set(eng.outputs) == set(sim.outputs)
    worst = max(row_rel_err(eng.outputs[k], o) for k, o in sim.outputs.items())
    assert worst <= ATTN_RTOL, worst


@pytest.mark.parametrize("cap", [1, 5])
def test_shaping_replay_persistent_walk(cap):
    """The extend attention on a capped persistent grid (baton_debug_prefill_grid): one
    CTA (or five) walks every (slot, head, query tile) item of a shaped iteration,
    empty slots (zero rows) included, and the whole replay still matches the oracle
    bit for bit in state and within C13 in outputs."""
    require_cuda()
    import ctypes
    from paper_2410_18701_b200 import _lib
    lib = _lib.lib
    lib.baton_debug_prefill_grid.restype = ctypes.c_int
    lib.baton_debug_prefill_grid.argtypes = [ctypes.c_int]
    qs = [Query(0, 0, 300, 40), Query(1, 0, 170, 30), Query(2, 0, 90, 50),
          Query(3, 5, 260, 20), Query(4, 5, 140, 25), Query(5, 12, 333, 10)]
    wl = Workload("shape-walk", qs, layers=1, q_heads=4, kv_heads=2, head_dim=128, slots=4,
                  max_ctx=2048)
    lib.baton_debug_prefill_grid(cap)
    try:
        n, _ = _replay(wl)
    finally:
        lib.baton_debug_prefill_grid(0)
    assert n >= 3
