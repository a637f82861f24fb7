"""§3.3 policies (NEXT-3): priority preemption (reading C25) and the
memory-threshold batch-size governor (reading C26).

Pins (against things other than the policy code):
* scheduling never changes a token: every decode output equals the plain FCFS run
  bit for bit (both equal solo attention);
* a hand-worked C25 scenario: the exact victim, the urgent query's slot, and the
  victim's re-entry;
* the governor's invariant: live tokens per shard <= hi * T after every iteration,
  and every admitted insert fitted lo * T;
* the product planner takes exactly the oracle's decisions (random workloads)."""
import dataclasses

import numpy as np
import pytest

from baton_inputs import Query, Workload, random_stream, ControlEvents
from oracle import Simulator
from paper_2410_18701_b200.scheduler import Planner


def _wl(queries, slots=2, max_ctx=64, governor=None, layers=1, heads=2, D=16):
    return Workload("policy", queries, layers=layers, q_heads=heads, kv_heads=heads, head_dim=D,
                    slots=slots, max_ctx=max_ctx, governor=governor)


def test_priority_preemption_scenario():
    """Two slots busy with long low-priority queries; an urgent query arrives at
    t=3: the most recently inserted low-priority query (ties: higher qid, C17) is
    stored, the urgent one takes its slot, and the victim re-enters at the head
    when the urgent query finishes."""
    qs = [Query(0, 0, 5, 20), Query(1, 0, 4, 20), Query(2, 3, 3, 2, priority=1),
          Query(3, 1, 2, 3)]
    sim = Simulator(_wl(qs), kv=True, keep_outputs=True)
    recs = sim.run()
    r3 = recs[3]
    assert r3.preempted == [(1, 1)]                    # qid 1 stored from slot 1
    assert (1, 2, 3) in r3.inserted                    # urgent qid 2 -> slot 1
    # qid 3 (priority 0, arrived earlier) waits behind the victim: the victim
    # re-enters first when qid 2 finishes
    back = [(r.t, g, q) for r in recs for g, q, _ in r.inserted if q in (1, 3) and r.t > 3]
    assert back[0][2] == 1
    # the stored K/V came back: qid 1 decodes all of its 20 tokens
    assert sum(1 for r in recs for _, q, _ in r.decoded if q == 1) == 20
    # and the tokens are the FCFS run's, bit for bit
    plain = [dataclasses.replace(q, priority=0) for q in qs]
    ref = Simulator(_wl(plain), kv=True, keep_outputs=True)
    ref.run()
    assert set(ref.outputs) == set(sim.outputs)
    for k, o in ref.outputs.items():
        assert np.array_equal(sim.outputs[k], o), k


def test_no_preemption_of_equal_or_higher_priority():
    qs = [Query(0, 0, 5, 10, priority=1), Query(1, 0, 4, 10, priority=1), Query(2, 2, 3, 2, priority=1)]
    recs = Simulator(_wl(qs)).run()
    assert not any(r.preempted for r in recs)


@pytest.mark.parametrize("gov", [(0.5, 0.35), (0.35, 0.2)])
def test_governor_invariant_and_outputs(gov):
    rng = np.random.default_rng(7)
    qs = [Query(i, int(rng.integers(0, 30)), int(rng.integers(10, 30)), int(rng.integers(30, 90)))
          for i in range(16)]
    qs.sort(key=lambda q: (q.arrival, q.qid))
    qs = [dataclasses.replace(q, qid=i) for i, q in enumerate(qs)]
    wl = _wl(qs, slots=4, max_ctx=128, governor=gov)
    sim = Simulator(wl, kv=True, keep_outputs=True)
    T = wl.slots * wl.max_ctx
    n_stored = 0
    while not sim.done():
        rec = sim.iteration()
        n_stored += len(rec.preempted)
        assert int(sum(rec.lens[0][rec.qid[0] >= 0])) <= gov[0] * T, rec.t
    assert n_stored > 0                                  # the governor did act
    ref = Simulator(dataclasses.replace(wl, governor=None), kv=True, keep_outputs=True)
    ref.run()
    assert set(ref.outputs) == set(sim.outputs)
    for k, o in ref.outputs.items():
        assert np.array_equal(sim.outputs[k], o), k


def _policy_stream(seed):
    wl = random_stream(seed)
    rng = np.random.default_rng(seed + 99)
    qs = [dataclasses.replace(q, priority=int(rng.random() < 0.2)) for q in wl.queries]
    wl.queries = qs
    wl.governor = (0.7, 0.5) if seed % 2 else None
    return wl


@pytest.mark.parametrize("seed", list(range(12)))
def test_planner_mirrors_oracle_with_policies(seed):
    wl = _policy_stream(seed)
    G = wl.gpus
    sim = Simulator(wl, G=G)
    pl = Planner(wl, G)
    while True:
        rec = sim.iteration()
        d = pl.plan()
        assert sorted(d.decode) == sorted(rec.decoded), rec.t
        assert sorted(g for g, _ in d.finished) == sorted(rec.removed), rec.t
        assert [(q, g) for g, q, _ in d.victims] == rec.preempted, rec.t
        assert [(g, q, l) for g, q, l, _ in d.inserts] == rec.inserted, rec.t
        assert list(np.concatenate(rec.qid)) == pl.occupant, rec.t
        assert list(np.concatenate(rec.lens)) == pl.length, rec.t
        if sim.done():
            assert pl.finished_all()
            break
