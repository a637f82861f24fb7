"""End-to-end parity of the CUDA path (Engine -> libbaton C ABI) against the
oracle's paper-literal state machine, after EVERY iteration:

* bit-exact: S, pad_start, lens, occupancy/slot indices (host mirror AND device
  copies), the mask bytes [B][S] (P:L96/L105/L124/L137) and the live K/V bytes
  of every occupied slot (P:L137 embedding, P:L144 store/re-insert, P:L147 moves)
* attention outputs of every decoded token within 1e-2 row-relative (C13)

on the W1 trace and on seeded random event streams (preemption, resize)."""
import numpy as np
import pytest
import torch

from baton_inputs import w1_workload, random_stream, SCALES_PEAKY
from oracle import Simulator
from gpu_util import ATTN_RTOL, bf16_bits, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _f64_to_bf16_bits(x):
    x32 = np.asarray(x, dtype=np.float32)          # exact: values are bf16
    return (x32.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def _check_state(eng, sim):
    sh = eng.shard
    osh = sim.shards[0]
    m = sh.baton_query()
    occ = osh.qid >= 0
    assert m["S"] == osh.S
    assert np.array_equal(m["occ"].astype(bool), occ)
    assert np.array_equal(m["lens"], osh.lens())
    assert np.array_equal(np.where(occ, m["pad"], 0), np.where(occ, osh.pad, 0))
    # device copies of the metadata
    assert int(sh.d_S.item()) == osh.S
    assert np.array_equal(sh.d_lens.cpu().numpy(), m["lens"])
    assert np.array_equal(np.where(occ, sh.d_pad.cpu().numpy(), 0), np.where(occ, osh.pad, 0))
    # the paper's mask, bit for bit, and zero beyond S
    dm = sh.mask.cpu().numpy()
    assert np.array_equal(dm[:, :osh.S], osh.mask)
    assert not dm[:, osh.S:].any()
    # live K/V bytes of every occupied slot
    for b in np.nonzero(occ)[0]:
        Ko, Vo = osh.live_kv(b)
        Kd, Vd = sh.live_kv(b)
        assert np.array_equal(bf16_bits(Kd), _f64_to_bf16_bits(Ko)), f"K slot {b}"
        assert np.array_equal(bf16_bits(Vd), _f64_to_bf16_bits(Vo)), f"V slot {b}"


def _replay(wl, check_every=1, use_graph=True, **engine_kwargs):
    from paper_2410_18701_b200.engine import Engine
    eng = Engine(wl, keep_outputs=True, use_graph=use_graph, **engine_kwargs)
    sim = Simulator(wl, kv=True, keep_outputs=True, fill=np.nan)
    n = 0
    while True:
        rec = sim.iteration()
        eng.iteration()
        torch.cuda.synchronize()
        if n % check_every == 0 or sim.done():
            _check_state(eng, sim)
        n += 1
        if sim.done():
            assert eng.done()
            break
    assert set(eng.outputs) == set(sim.outputs)
    worst = 0.0
    for k, o in sim.outputs.items():
        worst = max(worst, row_rel_err(eng.outputs[k], o))
    assert worst <= ATTN_RTOL, worst
    return n, worst


def test_w1_replay():
    require_cuda()
    n, worst = _replay(w1_workload())
    assert n == 19


def test_w1_replay_peaky():
    require_cuda()
    _replay(w1_workload(scales=SCALES_PEAKY))


@pytest.mark.parametrize("seed", list(range(200)))
def test_random_stream_replay(seed):
    """All 200 random event streams of SURVEY §8(c), state checked after every
    iteration."""
    require_cuda()
    _replay(random_stream(seed))


def test_splice_error_codes():
    require_cuda()
    from paper_2410_18701_b200 import _lib
    from paper_2410_18701_b200.baton import BatonShard, BatonError
    sh = BatonShard(2, 4, 2, 2, 16, 64)
    K = torch.zeros((2, 2, 5, 16), dtype=torch.bfloat16, device="cuda")
    sh.baton_insert(1, K, K, 5)
    for call, code in [(lambda: sh.baton_insert(1, K, K, 5), _lib.BATON_E_SLOT_BUSY),
                       (lambda: sh.baton_remove([2]), _lib.BATON_E_SLOT_EMPTY),
                       (lambda: sh.baton_extract(0), _lib.BATON_E_SLOT_EMPTY),
                       (lambda: sh.baton_insert(0, K, K, 65), _lib.BATON_E_CAPACITY),
                       (lambda: sh.baton_insert(0, K, K, 0), _lib.BATON_E_CAPACITY),
                       (lambda: sh.baton_insert(7, K, K, 5), _lib.BATON_E_INVALID),
                       (lambda: sh.baton_remove([1, 1]), _lib.BATON_E_INVALID)]:
        with pytest.raises(BatonError) as e:
            call()
        assert e.value.code == code
    # a failed call changed nothing
    m = sh.baton_query()
    assert m["S"] == 5 and list(m["occ"]) == [0, 1, 0, 0]
    for b in (0, 2, 3):
        sh.baton_insert(b, K, K, 5)
    with pytest.raises(BatonError) as e:
        sh.baton_compact(2)
    assert e.value.code == _lib.BATON_E_CAPACITY


def test_extract_insert_round_trip_bitwise():
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    sh = BatonShard(3, 4, 8, 2, 128, 512)
    g = torch.Generator(device="cuda").manual_seed(3)
    K = torch.randn((3, 2, 300, 128), generator=g, device="cuda").to(torch.bfloat16)
    V = torch.randn((3, 2, 300, 128), generator=g, device="cuda").to(torch.bfloat16)
    sh.baton_insert(2, K, V, 300)
    K2, V2 = sh.baton_extract(2)
    assert torch.equal(K2, K) and torch.equal(V2, V)
    sh.baton_remove([2])
    sh.baton_insert(0, K2, V2, 300)
    Kd, Vd = sh.live_kv(0)
    assert torch.equal(Kd, K) and torch.equal(Vd, V)


def test_graph_step_equals_eager_layers_bitwise():
    """baton_decode_step (captured graph, PDL-chained) == per-layer eager launches."""
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    wl = random_stream(17)
    a = Engine(wl, keep_outputs=True, use_graph=True)
    b = Engine(wl, keep_outputs=True, use_graph=False)
    while not a.done():
        a.iteration()
        b.iteration()
    assert b.done() and a.outputs.keys() == b.outputs.keys()
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k])


@pytest.mark.parametrize("hq,hkv", [(16, 2), (8, 8)])
def test_gqa_graph_step_deferred_merge_equals_eager_and_oracle(hq, hkv):
    """The decode-step graph runs layer l's split-K merge (head_dim 128: GQA and MHA)
    at the start of layer l+1's launch (one combine after the last layer).  Multi-chunk
    queries (lengths past 256 keys, at most 8 chunks): every output of the graph path
    equals the per-layer path (GQA: attention + combine per call; MHA: the in-kernel
    last-arriver merge) bitwise, and the oracle within C13."""
    require_cuda()
    from baton_inputs import Workload, Query
    from paper_2410_18701_b200.engine import Engine
    rng = np.random.default_rng(11)
    qs = [Query(i, int(i // 2), int(rng.integers(200, 1500)), int(rng.integers(2, 7))) for i in range(10)]
    wl = Workload("gqa_defer", qs, layers=3, q_heads=hq, kv_heads=hkv, head_dim=128, slots=4,
                  max_ctx=2048, scales=SCALES_PEAKY)
    a = Engine(wl, keep_outputs=True, use_graph=True)
    b = Engine(wl, keep_outputs=True, use_graph=False)
    while not a.done():
        a.iteration()
        b.iteration()
    assert b.done() and a.outputs.keys() == b.outputs.keys()
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k]), k
    sim = Simulator(wl, kv=True, keep_outputs=True)
    sim.run()
    worst = max(row_rel_err(a.outputs[k], o) for k, o in sim.outputs.items())
    assert worst <= ATTN_RTOL, worst


def test_w1_replay_eager_layers():
    require_cuda()
    _replay(w1_workload(), use_graph=False)


@pytest.mark.parametrize("seed", [3, 11])
def test_random_stream_replay_host_stash(seed):
    """Preempted queries stored in pinned HOST memory and re-inserted from
    there: still bit-exact state and parity."""
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    wl = random_stream(seed)
    eng = Engine(wl, keep_outputs=True, stash_host=True)
    sim = Simulator(wl, kv=True, keep_outputs=True, fill=np.nan)
    stored = 0
    while True:
        rec = sim.iteration()
        eng.iteration()
        torch.cuda.synchronize()
        stored += len(rec.preempted)
        _check_state(eng, sim)
        if sim.done():
            break
    assert stored > 0
    for k, o in sim.outputs.items():
        assert row_rel_err(eng.outputs[k], o) <= ATTN_RTOL


@pytest.mark.parametrize("budget_rows,staging_rows", [(0, 0), (24, 1 << 20), (0, 1 << 20), (64, 40)])
def test_random_stream_replay_hybrid_store(budget_rows, staging_rows):
    """NEXT-3, the prefetchable GPU&CPU hybrid store: stored
    queries stay in HBM up to a budget, spill to pinned host memory beyond it, and
    host entries near the queue head are prefetched back to HBM (staging budget) on a
    copy stream before their re-insert.  State bit-exact after every iteration and
    parity, on several preempting streams; across the cases every path is taken (HBM
    store, host spill, prefetched re-insert, re-insert straight from the host)."""
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    tot = {}
    for seed in (3, 11, 23, 42, 77):
        wl = random_stream(seed)
        tau = 2 * wl.layers * wl.kv_heads * wl.head_dim * 2
        eng = Engine(wl, keep_outputs=True, stash_host="hybrid", stash_hbm_bytes=budget_rows * tau)
        eng.stash.lookahead = 1 + seed % 3
        eng.stash.staging_budget = staging_rows * tau
        sim = Simulator(wl, kv=True, keep_outputs=True, fill=np.nan)
        while True:
            sim.iteration()
            eng.iteration()
            torch.cuda.synchronize()
            _check_state(eng, sim)
            if sim.done():
                break
        for k, o in sim.outputs.items():
            assert row_rel_err(eng.outputs[k], o) <= ATTN_RTOL
        for k, v in eng.stash.stats.items():
            tot[k] = tot.get(k, 0) + v
    if budget_rows == 0:                      # everything spills
        assert tot["stored_hbm"] == 0 and tot["stored_host"] > 0
    if staging_rows == 0:                     # nothing prefetched: re-inserts read the host
        assert tot["prefetched"] == 0 and tot["inserted_from_host"] > 0
    if staging_rows == 1 << 20:               # every host entry near the head is prefetched
        assert tot["prefetched"] > 0
    if budget_rows == 24:
        assert tot["stored_hbm"] > 0 and tot["stored_host"] > 0


def test_extract_to_pinned_host_and_back():
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    sh = BatonShard(2, 3, 4, 4, 64, 256)
    K = torch.randn((2, 4, 100, 64), device="cuda").to(torch.bfloat16)
    V = torch.randn((2, 4, 100, 64), device="cuda").to(torch.bfloat16)
    sh.baton_insert(1, K, V, 100)
    kh = torch.empty((2, 4, 100, 64), dtype=torch.bfloat16, pin_memory=True)
    vh = torch.empty_like(kh).pin_memory()
    sh.baton_extract(1, kh, vh)
    torch.cuda.synchronize()
    assert torch.equal(kh, K.cpu()) and torch.equal(vh, V.cpu())
    sh.baton_remove([1])
    sh.baton_insert(2, kh, vh, 100)
    Kd, Vd = sh.live_kv(2)
    assert torch.equal(Kd, K) and torch.equal(Vd, V)


@pytest.mark.parametrize("hq,hkv", [(32, 32), (64, 8)])
def test_early_prefetch_sees_previous_append(hq, hkv):
    """A decode launch that follows a decode launch prefetches K/V before
    griddepcontrol.wait (DecodeArgs::early).  The previous launch may have just
    written cache row lens-1 (fused append): a second, append-free launch on the
    SAME layer must read that row, and give bit-for-bit the first launch's output
    (which took the row from k_new/v_new)."""
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    torch.manual_seed(0)
    L, B, D, cap = 2, 24, 128, 2048
    sh = BatonShard(L, B, hq, hkv, D, cap)
    lens = [1 + (97 * i) % 1500 for i in range(B)]
    ks = [torch.randn((L, hkv, n, D), device="cuda").to(torch.bfloat16) for n in lens]
    vs = [torch.randn((L, hkv, n, D), device="cuda").to(torch.bfloat16) for n in lens]
    sh.baton_insert_many(list(range(B)), ks, vs, lens)
    for it in range(3):
        sh.baton_mask_update()
        q = torch.randn((B, hq, D), device="cuda").to(torch.bfloat16)
        kn = torch.randn((B, hkv, D), device="cuda").to(torch.bfloat16)
        vn = torch.randn((B, hkv, D), device="cuda").to(torch.bfloat16)
        outs = []
        for l in range(L):
            o1 = torch.empty_like(q)
            sh.baton_decode_layer(l, q, o1, k_new=kn, v_new=vn)   # l > 0: early
            o2 = torch.empty_like(q)
            sh.baton_decode_layer(l, q, o2)                       # early, reads row lens-1
            outs.append((o1, o2))
        torch.cuda.synchronize()
        for l, (o1, o2) in enumerate(outs):
            assert torch.equal(o1, o2), (it, l)
            ref = torch.empty_like(q)
            sh.baton_decode_attention(l, q, ref)                  # stateless, no early
            torch.cuda.synchronize()
            assert torch.equal(o1, ref), (it, l)


@pytest.mark.parametrize("seed", [5, 12])
def test_async_prefill_replay(seed):
    """Asynchronous P&D: queued queries are prefilled (keyed K/V + a8 on
    their prompts) on a side stream ahead of their insert; the state and every
    output stay bit-exact with the oracle."""
    require_cuda()
    wl = random_stream(seed)
    _replay(wl, async_prefill=True, prefill_attention=wl.head_dim == 128, prefill_lookahead=3)


@pytest.mark.parametrize("seed", [1, 3, 8, 45, 61, 69, 85, 93])
def test_policy_stream_replay(seed):
    """§3.3 policies (C25 priority preemption, C26 memory governor): the engine's
    stores and re-inserts keep the state bit-exact and every output within 1e-2.
    Seeds 45-93 store governor / priority victims after a compaction."""
    require_cuda()
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_policies import _policy_stream
    _replay(_policy_stream(seed))


def test_capacity_boundary():
    """A query can fill its slot up to max_ctx exactly: the full slot decodes over
    all max_ctx keys (finite output; the empty slot's row is zero, C6), and the step
    that would write column max_ctx is refused (BATON_E_CAPACITY, C24) and changes
    nothing."""
    require_cuda()
    from paper_2410_18701_b200 import _lib
    from paper_2410_18701_b200.baton import BatonShard, BatonError
    sh = BatonShard(1, 2, 2, 2, 16, 64)
    K = torch.randn((1, 2, 63, 16), device="cuda").to(torch.bfloat16)
    V = torch.randn_like(K)
    sh.baton_insert(0, K, V, 63)
    sh.baton_mask_update()                       # S = 64 = max_ctx, lens[0] = 64
    m = sh.baton_query()
    assert m["S"] == 64 and list(m["lens"])[:1] == [64]
    q = torch.randn((2, 2, 16), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    kn = torch.randn((2, 2, 16), device="cuda").to(torch.bfloat16)
    sh.baton_decode_layer(0, q, out, kn, kn)     # appends row 63 and attends over 64 keys
    torch.cuda.synchronize()
    assert torch.isfinite(out[0].float()).all() and (out[1] == 0).all()
    with pytest.raises(BatonError) as e:
        sh.baton_mask_update()
    assert e.value.code == _lib.BATON_E_CAPACITY
    assert sh.baton_query()["S"] == 64


@pytest.mark.parametrize("hq,hkv,d", [(2, 2, 16), (32, 32, 128), (64, 8, 128)])
def test_all_slots_empty(hq, hkv, d):
    """Degenerate batch: no occupied slot.  The step computes nothing and writes zero
    rows (C6), eager and graph-replayed, for the MHA and the tcgen05 GQA kernels."""
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    sh = BatonShard(2, 4, hq, hkv, d, 64)
    q = torch.randn((2, 4, hq, d), device="cuda").to(torch.bfloat16)
    kn = torch.randn((2, 4, hkv, d), device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, 7.0)
    sh.baton_decode_step(q, kn, kn, out)
    torch.cuda.synchronize()
    assert (out == 0).all()
    out.fill_(7.0)
    sh.baton_mask_update()
    for l in range(2):
        sh.baton_decode_layer(l, q[l], out[l], kn[l], kn[l])
    torch.cuda.synchronize()
    assert (out == 0).all()
    assert sh.baton_query()["S"] == 2
