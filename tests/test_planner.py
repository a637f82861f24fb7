"""The product planner (paper_2410_18701_b200/scheduler.py) takes exactly the
decisions of the oracle's serving loop (oracle/schedule.py) -- the two are
independent implementations of readings C5-C9, C17-C20b.  Slot indices are
compared bit-exactly after every iteration."""
import numpy as np
import pytest

from baton_inputs import w1_workload, random_stream, config_workload
from oracle import Simulator
from paper_2410_18701_b200.scheduler import Planner


def _compare(wl, G=None, max_iters=100000):
    G = G or wl.gpus
    sim = Simulator(wl, G=G)
    pl = Planner(wl, G)
    n = 0
    while True:
        rec = sim.iteration()
        d = pl.plan()
        assert d.t == rec.t
        assert sorted(d.decode) == sorted(rec.decoded), rec.t
        assert sorted(g for g, _ in d.finished) == sorted(rec.removed), rec.t
        assert [(q, g) for g, q, _ in d.victims] == rec.preempted, rec.t
        if rec.resized is not None:
            assert d.resize * G == rec.resized
        assert [(g, q, l) for g, q, l, _ in d.inserts] == rec.inserted, rec.t
        occ = np.concatenate(rec.qid)
        assert list(occ) == pl.occupant, rec.t
        lens = np.concatenate(rec.lens)
        assert list(lens) == pl.length, rec.t
        n += 1
        if sim.done() or n >= max_iters:
            assert pl.finished_all() == sim.done()
            break
    return n


def test_w1():
    assert _compare(w1_workload()) == 19


@pytest.mark.parametrize("seed", range(200))
def test_random_streams(seed):
    _compare(random_stream(seed))


@pytest.mark.parametrize("name,G", [("7b", 1), ("13b", 1), ("13b", 2), ("13b", 8), ("70b", 8)])
def test_configs(name, G):
    wl = config_workload(name, gpus=G, n_queries=150 if name != "13b" else 300)
    _compare(wl, G)


@pytest.mark.parametrize("G", [1, 2, 8])
def test_stress_with_preemption_and_resize(G):
    wl = config_workload("stress", gpus=G, n_queries=400)
    wl.iterations = 200
    _compare(wl, G)


def test_flags_path_equals_local_bookkeeping():
    wl = config_workload("13b", gpus=4, n_queries=200)
    a, b = Planner(wl, 4), Planner(wl, 4)
    for _ in range(60):
        flags = sum((b.local_completion_flags(r) for r in range(4)), []) if b.t > 0 else None
        da, db = a.plan(), b.plan(flags)
        assert da == db


def test_run_to_completion_policy():
    """NEXT-4 baseline: no slot is refilled before the whole batch has
    finished; finished queries keep decoding (idle tokens) until then."""
    from baton_inputs import Workload, Query
    A = [10, 2, 3, 9, 2, 4, 8, 1, 2]
    qs = [Query(i, 0, 5 + i, A[i]) for i in range(9)]
    wl = Workload("rtc", qs, layers=1, q_heads=2, kv_heads=2, head_dim=16, slots=3, max_ctx=64)
    pl = Planner(wl, 1, policy="rtc")
    useful = idle = 0
    batches = []
    while not pl.finished_all():
        d = pl.plan()
        idle += pl.idle_decodes(d.decode)
        useful += len(d.decode) - pl.idle_decodes(d.decode)
        if d.finished:                      # the whole batch leaves at once
            assert len(d.finished) == 3 or not pl.queue
        if d.inserts:
            live = sorted(q for q in pl.occupant if q >= 0)
            assert live == sorted(i[1] for i in d.inserts)     # only into an empty batch
            batches.append([i[1] for i in d.inserts])
    assert batches == [[0, 1, 2], [3, 4, 5], [6, 7, 8]]
    assert useful == sum(A)
    assert idle == sum(max(A[j] for j in b) * len(b) - sum(A[j] for j in b) for b in batches)
    base = Planner(wl, 1)
    while not base.finished_all():
        base.plan()
    assert base.t < pl.t            # the relay race finishes the same work sooner


@pytest.mark.parametrize("policy", ["benchmark", "pd"])
def test_paper_baseline_policies(policy):
    """NEXT-4, the paper's two comparison methods as planner policies.
    Both run decode batches to completion and only refill an empty batch;
    "benchmark" places the batch's queries raw (prefilled together inside the batch,
    padded to the longest prompt: one shaped iteration with every row new), "pd"
    embeds separately prefilled queries (the same decisions as "rtc").  Every query
    yields exactly its A tokens and is reported complete exactly once (a
    response returns as soon as it is done)."""
    from baton_inputs import Workload, Query
    A = [10, 2, 3, 9, 2, 4, 8, 1, 2]
    qs = [Query(i, 0, 5 + i, A[i]) for i in range(9)]
    wl = Workload("rtc", qs, layers=1, q_heads=2, kv_heads=2, head_dim=16, slots=3, max_ctx=64)
    pl, ref = Planner(wl, 1, policy=policy), Planner(wl, 1, policy="rtc")
    useful, completed, shaped = 0, [], []
    while not pl.finished_all():
        d = pl.plan()
        useful += len(d.decode) - pl.idle_decodes(d.decode)
        completed += [q for _, q in d.completed]
        if d.prefill:
            shaped.append(sorted(q for _, q, _ in d.prefill))
            assert not d.decode                    # every row of the batch is new
        if policy == "pd":
            r = ref.plan()
            assert (d.decode, d.finished, d.inserts) == (r.decode, r.finished, r.inserts)
        else:
            assert not d.inserts
            if d.raw:
                assert len(pl.live()) == len(d.raw)  # only into an empty batch
    assert useful == sum(A) and sorted(completed) == list(range(9))
    if policy == "benchmark":
        assert shaped == [[0, 1, 2], [3, 4, 5], [6, 7, 8]]
    with pytest.raises(ValueError):
        w2 = random_stream(3)                      # preemption events: relay race only
        Planner(w2, 1, policy=policy)


def test_completed_once_per_query_relay():
    wl = random_stream(5)
    pl = Planner(wl, 1)
    done = []
    while not pl.finished_all():
        d = pl.plan()
        done += [q for _, q in d.completed]
    assert len(done) == len(set(done))
    assert set(done) <= {q.qid for q in wl.queries}


def _compare_shape(wl, G=None):
    """Planner policy "shape" (product) == Simulator policy "shape" (oracle)."""
    G = G or wl.gpus
    sim = Simulator(wl, G=G, policy="shape")
    pl = Planner(wl, G, policy="shape")
    n = 0
    while True:
        rec = sim.iteration()
        d = pl.plan()
        assert sorted(d.decode) == sorted(rec.decoded), rec.t
        assert sorted(d.prefill) == sorted(rec.prefilled), rec.t
        assert sorted(g for g, _ in d.finished) == sorted(rec.removed), rec.t
        assert d.raw == rec.inserted and not d.inserts, rec.t
        # a reserved raw slot is still empty in the oracle until its shaped step
        assert list(np.concatenate(rec.qid)) == [-1 if g in pl.raw else q
                                                 for g, q in enumerate(pl.occupant)], rec.t
        # live token counts (the oracle's mask-1 count) of every decoding/prefilled slot
        lens = np.concatenate(rec.lens)
        for g, q in enumerate(pl.occupant):
            if q >= 0 and g not in pl.raw:
                assert pl.length[g] == lens[g], (rec.t, g)
        n += 1
        if sim.done():
            assert pl.finished_all()
            break
    return n


def test_shape_policy_w1():
    wl = w1_workload()
    wl.max_ctx = 256
    assert _compare_shape(wl) > 19          # one extra prefill iteration per insert wave


@pytest.mark.parametrize("seed", [1, 4, 9])
def test_shape_policy_random_streams(seed):
    from baton_inputs import ControlEvents
    wl = random_stream(seed)
    wl.control = ControlEvents()
    wl.max_ctx = 4096
    wl.iterations = -1
    _compare_shape(wl)


def _mirror_replay(wl, G):
    """Apply each rank's splice ops (scheduler.local_splice_ops, the exact call
    order the engine executes) to a host mirror of the library's slot state and
    check every call is legal (extract/remove of an occupied slot holding the
    victim the planner named, insert into an empty slot, no duplicates) and that
    the mirror ends every iteration equal to the planner's occupancy/lengths."""
    from paper_2410_18701_b200.scheduler import local_splice_ops
    pl = Planner(wl, G)
    B = pl.per_rank
    occ = [[-1] * B for _ in range(G)]
    ln = [[0] * B for _ in range(G)]
    stash = {}
    while not pl.finished_all():
        dec = pl.decode_plan() if pl.t > 0 else []
        for g, q, _ in dec:
            r, b = pl.rank_of(g), pl.local(g)
            assert occ[r][b] == q
            ln[r][b] += 1
        d = pl.plan()
        for r in range(G):
            for op in local_splice_ops(pl, d, r):
                if op[0] == "remove":
                    assert len(set(op[1])) == len(op[1]), (d.t, op)
                    for b in op[1]:
                        assert occ[r][b] >= 0, (d.t, op)
                        occ[r][b], ln[r][b] = -1, 0
                elif op[0] == "extract":
                    _, b, q = op
                    assert occ[r][b] == q, (d.t, op, occ[r])      # the victim the planner named
                    stash[q] = (r, ln[r][b])
                elif op[0] == "compact":
                    n = op[1]
                    for b in range(n, B):
                        if occ[r][b] >= 0:
                            f = next(x for x in range(n) if occ[r][x] < 0)
                            occ[r][f], ln[r][f] = occ[r][b], ln[r][b]
                            occ[r][b], ln[r][b] = -1, 0
                else:
                    for b, q, n, home in op[1]:
                        assert occ[r][b] < 0, (d.t, op)
                        if home is not None:
                            assert stash.pop(q) == (r, n) and home == r   # C20b
                        occ[r][b], ln[r][b] = q, n
        assert sum(occ, []) == pl.occupant, d.t
        assert sum(ln, []) == pl.length, d.t
    return pl.t


@pytest.mark.parametrize("seed", range(100))
def test_engine_call_order_on_policy_streams(seed):
    """governor and priority-preemption victims are chosen on the
    compacted batch, so they must be stored after baton_compact (seeds 45, 61, 69,
    85, 93 extracted the wrong/empty slot before the fix)."""
    from test_oracle_policies import _policy_stream
    wl = _policy_stream(seed)
    _mirror_replay(wl, wl.gpus)


@pytest.mark.parametrize("G", [1, 2, 8])
def test_engine_call_order_stress(G):
    wl = config_workload("stress", gpus=G, n_queries=400)
    wl.iterations = 300
    _mirror_replay(wl, G)


def test_shape_policy_rejects_governor_and_priorities():
    import dataclasses
    wl = w1_workload()
    with pytest.raises(ValueError):
        Planner(dataclasses.replace(wl, governor=(0.7, 0.5)), 1, policy="shape")
    qs = [dataclasses.replace(q, priority=1) if q.qid == 3 else q for q in wl.queries]
    with pytest.raises(ValueError):
        Planner(dataclasses.replace(wl, queries=qs), 1, policy="shape")
