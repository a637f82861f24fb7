"""Pins of the vector-SHAPING oracle (``Shard.shape_step``, Simulator policy
"shape", NEXT-1) against things other than itself:

* the textbook definition: dense attention over all S+W columns with an additive
  -inf mask (mask 0 or beyond the causal bound), written out independently here;
* solo attention of each query over its own keyed history ("the padding
  ... will not affect the output"), bitwise through O-1 and to 1e-12 through the
  correctly rounded O-1 variant;
* the reduction W = 1, no insert == ``Shard.step`` (bitwise, whole state);
* the P&D policy: every decode output of the shape policy equals the P&D output
  bit for bit (the paper's two paths compute the same tokens);
* the bubble closed form (B-1)(l_q3-1) of a single insert into a full batch
  (reading of P:L128-130);
* the mask/KV shapes of reading C4 (both grow by the input width W)."""
import copy
import math

import numpy as np
import pytest

from baton_inputs import (w1_workload, KIND_Q, KIND_K, KIND_V, query_history_bits,
                          query_token_bits, bf16_bits_to_f64)
from oracle import Simulator, solo_attention, solo_attention_exact
from oracle.batch import Shard, SlotBusy, Capacity

SEED, L, HQ, HKV, D = 7, 2, 4, 2, 16


def _hist(qid, n):
    K = bf16_bits_to_f64(query_history_bits(SEED, KIND_K, L, qid, 0, n, HKV, D, 0))
    V = bf16_bits_to_f64(query_history_bits(SEED, KIND_V, L, qid, 0, n, HKV, D, 0))
    return K, V


def _tok(kind, H, qid, pos):
    return np.stack([bf16_bits_to_f64(query_token_bits(SEED, kind, l, [qid], [pos], H, D, 0))[0]
                     for l in range(L)])


def _shard_with(queries, B=4, S_cap=256, fill=0.0):
    """Shard holding prefilled queries {slot: (qid, length)}."""
    sh = Shard(B, L, HQ, HKV, D, S_cap, fill=fill)
    for slot, (qid, n) in queries.items():
        K, V = _hist(qid, n)
        sh.insert(slot, qid, n, K, V)
    return sh


def _inputs(sh, new, W):
    """Keyed q/k/v of every real input token of a shaped iteration."""
    q = np.zeros((L, sh.B, W, HQ, D))
    k = np.zeros((L, sh.B, W, HKV, D))
    v = np.zeros((L, sh.B, W, HKV, D))
    lens = sh.lens()
    for b in sh.occupied():
        qid, pos = int(sh.qid[b]), int(lens[b])
        q[:, b, 0] = _tok(KIND_Q, HQ, qid, pos)
        k[:, b, 0] = _tok(KIND_K, HKV, qid, pos)
        v[:, b, 0] = _tok(KIND_V, HKV, qid, pos)
    for b, qid, l in new:
        for t in range(l):
            q[:, b, t] = _tok(KIND_Q, HQ, qid, t)
            k[:, b, t] = _tok(KIND_K, HKV, qid, t)
            v[:, b, t] = _tok(KIND_V, HKV, qid, t)
    return q, k, v


def _dense_reference(mask, K, V, q, b, t, S0):
    """softmax(q K^T / sqrt(D) + M) V over ALL columns, M = -inf where the mask is 0
    or the column is after the token's own column S0 + t."""
    S = mask.shape[1]
    allowed = (mask[b] == 1) & (np.arange(S) <= S0 + t)
    out = np.zeros((L, HQ, D))
    for l in range(L):
        for h in range(HQ):
            g = h * HKV // HQ
            s = K[l, b, g] @ q[l, b, t, h] / math.sqrt(D)
            s = np.where(allowed, s, -np.inf)
            e = np.exp(s - s.max())
            out[l, h] = (e[:, None] * np.nan_to_num(V[l, b, g])).sum(0) / e.sum()
    return out


def test_width_one_without_insert_is_a_decode_step():
    a = _shard_with({0: (1, 9), 2: (2, 5), 3: (3, 12)})
    b = copy.deepcopy(a)
    q, k, v = _inputs(a, [], 1)
    oa = a.shape_step([], q, k, v)
    ob = b.step(q[:, :, 0], k[:, :, 0], v[:, :, 0])
    assert a.S == b.S and np.array_equal(a.mask, b.mask) and np.array_equal(a.pad, b.pad)
    assert np.array_equal(a.K, b.K) and np.array_equal(a.V, b.V)
    assert np.array_equal(oa[:, :, 0], ob)


@pytest.mark.parametrize("l_new", [1, 7, 20])
def test_shaped_iteration_equals_solo_and_dense_definition(l_new):
    sh = _shard_with({0: (1, 9), 2: (2, 5), 3: (3, 12)}, fill=np.nan)
    S0 = sh.S
    new = [(1, 9, l_new)]
    W = max(1, l_new)
    q, k, v = _inputs(sh, new, W)
    before = sh.lens()
    o = sh.shape_step(new, q, k, v)
    # survivors: an ordinary decode of their next position
    for b, qid in ((0, 1), (2, 2), (3, 3)):
        n = int(before[b]) + 1
        K, V = _hist(qid, n)
        for l in range(L):
            assert np.array_equal(o[l, b, 0], solo_attention(q[l, b, 0], K[l], V[l]))
            ex = solo_attention_exact(q[l, b, 0], K[l], V[l])
            assert np.max(np.abs(o[l, b, 0] - ex)) <= 1e-12 * np.max(np.abs(ex))
        assert not o[:, b, 1:].any()                       # padding tokens: no output
        dense = _dense_reference(sh.mask, np.nan_to_num(sh.K), sh.V, q, b, 0, S0)
        assert np.allclose(o[:, b, 0], dense, rtol=1e-12, atol=1e-14)
    # the new query: causal prefill over its own prompt, nothing else
    K, V = _hist(9, l_new)
    for t in range(l_new):
        for l in range(L):
            assert np.array_equal(o[l, 1, t], solo_attention(q[l, 1, t], K[l, :, :t + 1], V[l, :, :t + 1]))
        dense = _dense_reference(sh.mask, np.nan_to_num(sh.K), sh.V, q, 1, t, S0)
        assert np.allclose(o[:, 1, t], dense, rtol=1e-12, atol=1e-14)


def test_mask_and_kv_shapes_follow_reading_c4():
    sh = _shard_with({0: (1, 9), 2: (2, 5)})
    S0 = sh.S
    new = [(1, 9, 6), (3, 10, 4)]
    q, k, v = _inputs(sh, new, 6)
    sh.shape_step(new, q, k, v)
    W = 6
    assert sh.S == S0 + W and sh.mask.shape[1] == sh.S and sh.K.shape[3] == sh.S
    assert list(sh.mask[0, S0:]) == [1, 0, 0, 0, 0, 0]        # survivor: token, then padding
    assert list(sh.mask[2, S0:]) == [1, 0, 0, 0, 0, 0]
    assert not sh.mask[1, :S0].any() and list(sh.mask[1, S0:]) == [1] * 6
    assert not sh.mask[3, :S0].any() and list(sh.mask[3, S0:]) == [1, 1, 1, 1, 0, 0]
    assert sh.pad[1] == S0 and sh.pad[3] == S0 and sh.qid[1] == 9 and sh.qid[3] == 10
    # live tokens of the new rows are exactly their prompts
    for b, qid, l in new:
        K, V = _hist(qid, l)
        Kl, Vl = sh.live_kv(b)
        assert np.array_equal(Kl, K) and np.array_equal(Vl, V)


def test_insert_errors():
    sh = _shard_with({0: (1, 9)}, S_cap=20)
    with pytest.raises(SlotBusy):
        sh.shape_step([(0, 5, 3)], *_inputs(sh, [], 3))
    with pytest.raises(Capacity):
        sh.shape_step([(1, 5, 12)], *_inputs(sh, [(1, 5, 12)], 12))   # 9 + 12 > 20


def test_shape_policy_decodes_exactly_the_pd_tokens():
    wl = w1_workload()
    wl.max_ctx = 256
    pd = Simulator(wl, kv=True, keep_outputs=True, policy="pd")
    pd.run()
    sp = Simulator(wl, kv=True, keep_outputs=True, policy="shape")
    recs = sp.run()
    assert set(pd.outputs) <= set(sp.outputs)
    for key, o in pd.outputs.items():
        assert np.array_equal(sp.outputs[key], o), key
    # the shape policy's extra outputs are the prompts' prefill rows
    prompt = {(q.qid, t) for q in wl.queries for t in range(q.l_q)}
    assert set(sp.outputs) - set(pd.outputs) == prompt
    # every query: one prefill iteration, then exactly A decode iterations
    pre = {qid: r.t for r in recs for _, qid, _ in r.prefilled}
    dec = {}
    for r in recs:
        for _, qid, _ in r.decoded:
            dec.setdefault(qid, []).append(r.t)
    for q in wl.queries:
        assert len(dec[q.qid]) == q.A and min(dec[q.qid]) == pre[q.qid] + 1


def test_single_insert_bubble_closed_form():
    """one raw insert of length l into a full batch of B pads the other
    B-1 rows by l-1 tokens each: (B-1)(l-1) bubble rows in that iteration."""
    B, l = 4, 11
    sh = Shard(B, L, HQ, HKV, D, 256, kv=False)      # metadata mode is enough here
    for slot, (qid, n) in {0: (1, 9), 1: (2, 5), 2: (3, 12)}.items():
        sh.insert(slot, qid, n)
    new = [(3, 9, l)]
    sh.shape_step(new)
    rows = sh.mask[:, -l:]
    real = int(rows.sum())
    assert real == (B - 1) + l
    assert B * l - real == (B - 1) * (l - 1)


def test_release_after_shaping_keeps_holes():
    sh = _shard_with({0: (1, 9), 2: (2, 5)})
    new = [(1, 9, 6)]
    sh.shape_step(new, *_inputs(sh, new, 6))
    holes = sh.mask[0].copy()
    sh.remove(2)
    p = sh.release()
    assert p == min(int(sh.pad[b]) + p for b in sh.occupied())
    assert np.array_equal(sh.mask[0], holes[p:])
