"""Host-side decisions of the hybrid K/V store (paper_2410_18701_b200/kvstore.py,
NEXT-3) driven by the product planner on a preempting workload, with
the device calls stubbed out (no GPU): placement by the HBM budget, prefetch only of
host entries among the queue head's stored queries within the staging budget, byte
accounting back to zero when the store drains."""
import types

import numpy as np
import pytest
import torch

from baton_inputs import config_workload, Query
from paper_2410_18701_b200 import kvstore
from paper_2410_18701_b200.scheduler import Planner, local_splice_ops


class _Ev:
    def record(self, *a):
        pass

    def query(self):
        return True


class _Ctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class _Shard:
    L, Hkv, D = 1, 1, 8

    def __init__(self):
        self.lensarr = np.zeros(32, np.int64)

    def baton_query(self):
        return {"lens": self.lensarr}

    def baton_extract(self, slot, k=None, v=None):
        n = int(self.lensarr[slot])
        t = torch.zeros((1, 1, n, 8))
        return (k if k is not None else t), (v if v is not None else t.clone())


@pytest.fixture
def stubbed(monkeypatch):
    cuda = kvstore.torch.cuda
    monkeypatch.setattr(cuda, "Event", lambda *a, **k: _Ev())
    monkeypatch.setattr(cuda, "Stream", lambda *a, **k: types.SimpleNamespace(wait_event=lambda e: None))
    monkeypatch.setattr(cuda, "current_stream", lambda *a: types.SimpleNamespace(wait_event=lambda e: None))
    monkeypatch.setattr(cuda, "stream", lambda s: _Ctx())
    real_empty = torch.empty

    def empty(*a, **k):
        k.pop("device", None)
        k.pop("pin_memory", None)
        return real_empty(*a, **k)
    monkeypatch.setattr(kvstore.torch, "empty", empty)
    monkeypatch.setattr(kvstore.torch, "empty_like", lambda t: real_empty(t.shape))


def _run(budget_rows, staging_rows, lookahead=8):
    wl = config_workload("7b")
    wl.queries = [Query(q.qid, q.arrival, q.l_q, q.A, q.kind, 1 if q.qid % 5 == 4 else 0)
                  for q in wl.queries]
    wl.iterations = 1500
    pl = Planner(wl, 1)
    sh = _Shard()
    tau = 2 * 8 * 2
    st = kvstore.HybridKVStore(sh, None, hbm_budget=budget_rows * tau, host=True, prefetch=True,
                               lookahead=lookahead, staging_budget=staging_rows * tau)
    seen_host_waits = 0
    while not pl.finished_all():
        d = pl.plan()
        for op in local_splice_ops(pl, d, 0):
            if op[0] == "extract":
                _, b, q = op
                sh.lensarr[:] = 0
                sh.lensarr[b] = [x for x in d.victims if x[1] == q][0][2]
                st.store(b, q)
                assert st.hbm_used <= budget_rows * tau
            elif op[0] == "insert":
                for b, q, n, home in op[1]:
                    if home is not None:
                        K, V = st.take(q)
                        assert K.shape[2] == n              # the stored rows come back
                st.after_insert()
        order = [pl.queue[i].qid for i in pl._order() if pl.queue[i].home == 0]
        seen_host_waits += sum(1 for q in order if q in st.entries and st.entries[q].where == "host")
        st.prefetch(order)
        assert st.staging_used <= staging_rows * tau
        # only stored queries among the first `lookahead` in service order are prefetched
        for q, e in st.entries.items():
            if e.where == "prefetching":
                assert q in order[:lookahead]
    return st, seen_host_waits


def test_all_hbm_when_budget_unlimited(stubbed):
    st, _ = _run(10 ** 9, 0)
    s = st.stats
    assert s["stored_host"] == 0 and s["prefetched"] == 0 and s["stored_hbm"] > 0
    assert s["inserted_from_hbm"] == s["stored_hbm"]


def test_spill_without_prefetch_reinserts_from_host(stubbed):
    st, waits = _run(0, 0)
    s = st.stats
    assert s["stored_hbm"] == 0 and s["prefetched"] == 0
    assert s["inserted_from_host"] == s["stored_host"] > 0 and waits > 0


def test_spilled_queries_prefetched_before_reinsert(stubbed):
    st, _ = _run(600, 10 ** 6)
    s = st.stats
    assert s["stored_hbm"] > 0 and s["stored_host"] > 0
    # every spilled query waited in the queue long enough to be prefetched
    assert s["prefetched"] == s["stored_host"] and s["inserted_from_host"] == 0
    assert st.stored_bytes == 0 and st.hbm_used == 0 and st.staging_used == 0 and not st.entries
