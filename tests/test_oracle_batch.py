"""Pins for O-2 (oracle/batch.py) and the serving loop (oracle/schedule.py).

Pinned against: SPEC.md worked examples, the paper's
text formulas, the closed form of the mask (P1), the
W1 hand trace (tests/golden/w1_trace.json), the schedule-independent closed form
of live key reads, solo equivalence (P7: each query's batched outputs equal its
solo decode), placeholder inertness (P5), release transparency (P6) and
extract/insert round trips (P3)."""
import json
import os

import numpy as np
import pytest

from baton_inputs import (Workload, Query, ControlEvents, w1_workload, random_stream,
                          config_workload, SCALES_PEAKY)
from oracle import Shard, Simulator, SlotBusy, SlotEmpty, Capacity
from oracle_checks import (closed_form_failures, run_checked, solo_output, history,
                           live_kv_failures, token_accounting_failures)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _meta_shard(B=4, S_cap=64):
    return Shard(B, 1, 1, 1, 4, S_cap, kv=False)


# ----------------------------------------------------------------- SPEC examples
def test_inserting_prompts_reproduces_left_padded_batch():
    # S:L194 "prompts of lengths [2,4] -> masks [0,0,1,1] and [1,1,1,1]" (P:L63
    # left-padded prefill): embedding them one by one gives the same mask.
    sh = _meta_shard(2)
    sh.insert(0, 0, 2)
    sh.insert(1, 1, 4)
    assert sh.mask.tolist() == [[0, 0, 1, 1], [1, 1, 1, 1]]
    assert sh.pad.tolist() == [2, 0]


def test_embed_end_aligned_case():
    # S:L239 "l_q 3, l_kv 5 -> slot mask [0,0,1,1,1], pad_start 2" (P:L137 case 1)
    sh = _meta_shard(2)
    sh.insert(0, 0, 5)
    sh.insert(1, 1, 3)
    assert sh.S == 5
    assert sh.mask[1].tolist() == [0, 0, 1, 1, 1]
    assert sh.pad[1] == 2
    assert sh.mask[0].tolist() == [1, 1, 1, 1, 1]     # "no other slot changes"


def test_embed_exact_fit():
    # S:L240 "l_q = l_kv -> zero placeholders, pad_start 0"
    sh = _meta_shard(2)
    sh.insert(0, 0, 5)
    sh.insert(1, 1, 5)
    assert sh.pad.tolist() == [0, 0] and sh.S == 5


def test_embed_left_expansion_case():
    # S:L241 "l_q 7, l_kv 5 -> kv_len 7; existing slots gain 2 masked prefix columns"
    sh = _meta_shard(3)
    sh.insert(0, 0, 5)
    sh.insert(1, 1, 3)
    sh.insert(2, 2, 7)
    assert sh.S == 7
    assert sh.mask.tolist() == [[0, 0, 1, 1, 1, 1, 1], [0, 0, 0, 0, 1, 1, 1],
                                [1, 1, 1, 1, 1, 1, 1]]
    assert sh.pad.tolist() == [2, 4, 0]


def test_release_example():
    # S:L249 "pad_start [3,5,4] -> p=3, new pad_start [0,2,1], kv_len -3"
    sh = _meta_shard(3)
    sh.insert(0, 0, 9)       # S = 9
    sh.insert(1, 1, 4)       # pad 5
    sh.insert(2, 2, 5)       # pad 4
    sh.remove(0)
    sh.insert(0, 3, 6)       # pad 3
    assert sh.pad.tolist() == [3, 5, 4]
    p = sh.release()
    assert p == 3 and sh.pad.tolist() == [0, 2, 1] and sh.S == 6


def test_release_noop_when_some_pad_zero():
    sh = _meta_shard(2)
    sh.insert(0, 0, 4)
    sh.insert(1, 1, 2)
    assert sh.release() == 0 and sh.S == 4


def test_release_of_empty_batch_drops_everything():
    sh = _meta_shard(2)
    sh.insert(0, 0, 4)
    sh.step()
    sh.remove(0)
    assert sh.release() == 5 and sh.S == 0


def test_step_appends_one_column():
    # "add a column with the value of all 1"; empty rows get 0 (C6)
    sh = _meta_shard(3)
    sh.insert(0, 0, 2)
    sh.insert(2, 1, 1)
    sh.step()
    assert sh.S == 3
    assert sh.mask[:, -1].tolist() == [1, 0, 1]
    assert sh.lens().tolist() == [3, 0, 2]


def test_remove_zeroes_the_row():
    # "set all the values of the query^2 part ... to 0"
    sh = _meta_shard(2)
    sh.insert(0, 0, 3)
    sh.insert(1, 1, 3)
    sh.remove(1)
    assert sh.mask[1].tolist() == [0, 0, 0]


def test_contract_errors():
    sh = _meta_shard(2, S_cap=8)
    sh.insert(0, 0, 3)
    with pytest.raises(SlotBusy):
        sh.insert(0, 1, 2)
    with pytest.raises(SlotEmpty):
        sh.remove(1)
    with pytest.raises(SlotEmpty):
        sh.extract(1)
    with pytest.raises(Capacity):
        sh.insert(1, 2, 9)
    with pytest.raises(Capacity):
        sh.insert(1, 2, 0)


def test_insert_order_independence():
    # C7: two inserts in one iteration give the same state in either order
    def build(order):
        sh = Shard(4, 1, 2, 2, 4, 64, kv=True)
        rng = np.random.default_rng(0)
        base = [(0, 0, 6), (1, 1, 2)]
        new = {2: (2, 10), 3: (3, 4)}
        for slot, qid, l in base:
            sh.insert(slot, qid, l, np.full((1, 2, l, 4), qid + 1.0), np.full((1, 2, l, 4), -qid - 1.0))
        sh.step(np.zeros((1, 4, 2, 4)), np.ones((1, 4, 2, 4)), np.ones((1, 4, 2, 4)))
        for slot in order:
            qid, l = new[slot]
            sh.insert(slot, qid, l, np.full((1, 2, l, 4), qid + 1.0), np.full((1, 2, l, 4), -qid - 1.0))
        return sh
    a, b = build([2, 3]), build([3, 2])
    assert a.S == b.S == 10
    assert np.array_equal(a.mask, b.mask) and np.array_equal(a.pad, b.pad)
    assert np.array_equal(a.K, b.K) and np.array_equal(a.V, b.V)


# ----------------------------------------------------------------- W1 golden
def test_w1_golden_trace():
    g = json.load(open(os.path.join(GOLDEN, "w1_trace.json")))
    sim = Simulator(w1_workload())
    recs = sim.run()
    assert len(recs) - 1 == g["iterations"]
    assert sum(len(r.decoded) for r in recs) == g["decode_tokens"]
    by_t = {r.t: r for r in recs}
    for row in g["rows"]:
        r = by_t[row["t"]]
        if "lens_after_append" in row:
            lens = [0] * 4
            for gs, qid, pos in r.decoded:
                lens[gs] = pos + 1
            assert lens == row["lens_after_append"], row["t"]
        assert sorted(r.finished) == sorted(row["removed_qids"]), row["t"]
        assert sum(r.released) == row["release_p"], row["t"]
        assert [list(x) for x in r.inserted] == row["inserts"], row["t"]
        assert r.S[0] == row["S"], row["t"]
        assert r.qid[0].tolist() == row["qid"], row["t"]
        for b, p in enumerate(row["pad"]):
            if p is not None:
                assert r.pad[0][b] == p, (row["t"], b)
    live = sum(pos + 1 for r in recs for _, _, pos in r.decoded)
    assert live == g["live_key_columns"]
    # schedule-independent closed form: sum_q A*l_q + A(A+1)/2
    wl = w1_workload()
    assert live == sum(q.A * q.l_q + q.A * (q.A + 1) // 2 for q in wl.queries)
    dense = sum(4 * (recs[i - 1].S[0] + 1) for i in range(1, len(recs)))
    assert dense == g["dense_key_columns"]


def test_w1_closed_form_every_iteration():
    sim, recs, errs = run_checked(w1_workload(), kv=True)
    assert errs == []


# ----------------------------------------------------------------- P7 solo equivalence
@pytest.mark.parametrize("scales", ["flat", "peaky"])
def test_w1_batched_equals_solo_bitwise(scales):
    wl = w1_workload(scales=SCALES_PEAKY) if scales == "peaky" else w1_workload()
    sim = Simulator(wl, kv=True, keep_outputs=True)
    sim.run()
    assert len(sim.outputs) == 71
    for (qid, pos), o in sim.outputs.items():
        assert np.array_equal(o, solo_output(wl, qid, pos)), (qid, pos)


# ----------------------------------------------------------------- P5 inertness
@pytest.mark.parametrize("fill", [np.nan, 1e30, -np.inf])
def test_placeholder_fill_is_inert(fill):
    wl = w1_workload()
    a = Simulator(wl, kv=True, keep_outputs=True, fill=0.0)
    a.run()
    b = Simulator(wl, kv=True, keep_outputs=True, fill=fill)
    b.run()
    assert a.outputs.keys() == b.outputs.keys()
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k])


# ----------------------------------------------------------------- P6 release transparency
def test_release_is_output_transparent():
    wl = w1_workload()
    wl.max_ctx = 4096
    a = Simulator(wl, kv=True, keep_outputs=True, release=True)
    a.run()
    b = Simulator(wl, kv=True, keep_outputs=True, release=False)
    recs = b.run()
    assert max(r.S[0] for r in recs) > 39       # S really kept growing without release
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k])


# ----------------------------------------------------------------- P3 extract round trip
def test_extract_returns_history_and_reinsert_continues():
    wl = Workload("rt", [Query(0, 0, 5, 6), Query(1, 0, 3, 6)], layers=2, q_heads=4,
                  kv_heads=2, head_dim=16, slots=3, max_ctx=32,
                  control=ControlEvents(preempt={2: 1, 4: 1}))
    sim = Simulator(wl, kv=True, keep_outputs=True)
    recs = sim.run()
    assert any(r.preempted for r in recs)
    # each preempted query re-entered and every output still equals solo decode
    for (qid, pos), o in sim.outputs.items():
        assert np.array_equal(o, solo_output(wl, qid, pos))
    sh = Shard(2, 2, 4, 2, 16, 32)
    K, V = history(wl, 7, 9)
    sh.insert(1, 7, 9, K, V)
    K2, V2 = sh.extract(1)
    assert np.array_equal(K2, K) and np.array_equal(V2, V)


def test_compact_moves_to_lowest_free_rows():
    sh = Shard(6, 1, 1, 1, 4, 16, kv=True)
    for slot, l in [(0, 2), (2, 3), (4, 4), (5, 1)]:
        sh.insert(slot, slot + 10, l, np.full((1, 1, l, 4), slot), np.full((1, 1, l, 4), slot))
    mask_before = {int(sh.qid[b]): sh.mask[b].copy() for b in sh.occupied()}
    o2n = sh.compact(4)
    assert o2n == [0, 1, 2, 3, 1, 3]
    assert sh.qid.tolist() == [10, 14, 12, 15, -1, -1]
    for b in sh.occupied():
        assert np.array_equal(sh.mask[b], mask_before[int(sh.qid[b])])
    assert np.all(sh.K[0, 1, 0, -4:] == 4) and np.all(sh.K[0, 3, 0, -1:] == 5)


def test_compact_without_room_raises():
    sh = _meta_shard(3)
    for s in range(3):
        sh.insert(s, s, 2)
    with pytest.raises(Capacity):
        sh.compact(2)


# ----------------------------------------------------------------- random streams
@pytest.mark.parametrize("seed", range(200))
def test_random_stream_metadata(seed):
    wl = random_stream(seed)
    sim, recs, errs = run_checked(wl, kv=False)
    assert errs == []
    assert token_accounting_failures(wl, sim, recs) == []


@pytest.mark.parametrize("seed", [0, 3, 7, 11, 19, 42, 77, 123])
def test_random_stream_kv_and_solo(seed):
    wl = random_stream(seed)
    sim, recs, errs = run_checked(wl, kv=True, fill=np.nan, check_kv_every=3)
    assert errs == []
    keys = sorted(sim.outputs)
    rng = np.random.default_rng(seed)
    for i in rng.choice(len(keys), size=min(25, len(keys)), replace=False):
        qid, pos = keys[i]
        assert np.array_equal(sim.outputs[(qid, pos)], solo_output(wl, qid, pos))


def test_random_streams_cover_both_embedding_cases_and_release():
    exp = emb = rel = pre = res = 0
    for seed in range(40):
        wl = random_stream(seed)
        sim = Simulator(wl)
        prevS = [0]
        for _ in range(100000):
            S_before = [sh.S for sh in sim.shards]
            rec = sim.iteration()
            for g, qid, l in rec.inserted:
                pass
            exp += any(rec.S[0] > s + (1 if rec.t > 0 else 0) for s in S_before)
            emb += len(rec.inserted)
            rel += sum(1 for p in rec.released if p > 0)
            pre += len(rec.preempted)
            res += rec.resized is not None
            if sim.done():
                break
    assert exp > 10 and emb > 100 and rel > 10 and pre > 5 and res > 2


# ----------------------------------------------------------------- full-size configs (metadata)
@pytest.mark.parametrize("name,G", [("7b", 1), ("13b", 1), ("13b", 4), ("70b", 8)])
def test_config_schedules_metadata(name, G):
    wl = config_workload(name, gpus=G, n_queries=200 if name != "13b" else 400)
    sim, recs, errs = run_checked(wl, kv=False)
    assert errs == []
    assert token_accounting_failures(wl, sim, recs) == []
    if name == "13b":
        # "exactly 2 removes + 2 inserts every iteration" while the backlog lasts
        steady = [r for r in recs[1:150]]
        assert all(len(r.removed) == 2 and len(r.inserted) == 2 for r in steady)


def test_stress_schedule_metadata():
    wl = config_workload("stress", n_queries=600)
    wl.iterations = 200
    sim, recs, errs = run_checked(wl, kv=False)
    assert errs == []
    assert token_accounting_failures(wl, sim, recs) == []
    assert sum(len(r.preempted) for r in recs) > 10
    assert recs[64].resized == 32 and recs[128].resized == 64
