"""NEXT-4 on the GPU: the paper's comparison methods run through the
same libbaton kernels, and scheduling never changes a token -- every useful output
of the "benchmark" (in-batch padded prefill, run-to-completion), "pd" (P&D with
length-grouped prefill, run-to-completion) and "rtc" arms equals the oracle's, and
the per-iteration log (the Fig. 6-8 traces) adds up."""
import numpy as np
import pytest
import torch

from baton_inputs import Workload, Query, SCALES_PEAKY
from oracle import Simulator
from gpu_util import ATTN_RTOL, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _wl(D=128, Hq=8, Hkv=2):
    rng = np.random.default_rng(7)
    qs = [Query(i, 0, int(rng.integers(3, 150)), int(rng.integers(1, 24))) for i in range(14)]
    return Workload("pol", qs, layers=2, q_heads=Hq, kv_heads=Hkv, head_dim=D, slots=4,
                    max_ctx=2048, scales=SCALES_PEAKY)


@pytest.mark.parametrize("policy", ["benchmark", "pd", "rtc"])
def test_baseline_policy_outputs_equal_oracle(policy):
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    wl = _wl()
    eng = Engine(wl, policy=policy, keep_outputs=True, prefill_attention=policy != "benchmark",
                 trace=True)
    st = eng.run()
    # the oracle's serving loop of the same queries: Baton (shape: prompt positions too)
    sim = Simulator(wl, kv=True, keep_outputs=True, fill=np.nan,
                    policy="shape" if policy == "benchmark" else "pd")
    sim.run()
    useful = {k for k in sim.outputs}
    meta = {q.qid: q for q in wl.queries}
    idle = 0
    for (q, pos), o in eng.outputs.items():
        if (q, pos) in useful:
            assert row_rel_err(o, sim.outputs[(q, pos)]) <= ATTN_RTOL, (q, pos)
        else:                                   # run-to-completion: idle EOS decodes only
            assert pos >= meta[q].l_q + meta[q].A
            idle += 1
    decode_keys = {k for k in useful if k[1] >= meta[k[0]].l_q}
    assert decode_keys <= set(eng.outputs)
    assert idle == sum(s.idle for s in st) > 0
    recs = eng.log_records(st)
    assert sum(r["completed"] for r in recs) == len(wl.queries)
    assert sum(r["decoded"] - r["idle"] for r in recs) == sum(q.A for q in wl.queries)
    t = [r["t_ms"] for r in recs]
    assert all(b >= a for a, b in zip(t, t[1:])) and t[-1] > 0
    if policy == "benchmark":
        assert sum(r["bubble_rows"] for r in recs) > 0      # padded in-batch prefill


def test_relay_race_log_kv_sawtooth_vs_rtc():
    """P:L306-309 (Fig. 8): under run-to-completion the live K/V keeps growing until
    the whole batch ends and drops at once; under Baton it is released per query
    (consistently higher
    utilisation)."""
    require_cuda()
    from paper_2410_18701_b200.engine import Engine
    wl = _wl(D=16, Hq=2, Hkv=2)
    logs = {}
    for policy in ("baton", "rtc"):
        eng = Engine(wl, policy=policy, trace=True)
        logs[policy] = eng.log_records(eng.run())
    rtc = [r["kv_live_rows"] for r in logs["rtc"]]
    drops = sum(1 for a, b in zip(rtc, rtc[1:]) if b < a)
    assert drops <= len(wl.queries) // wl.slots + 1      # one drop per batch
    bat = [r["kv_live_rows"] for r in logs["baton"]]
    assert len(bat) < len(rtc)                           # the relay race finishes sooner
    assert sum(1 for a, b in zip(bat, bat[1:]) if b < a) > drops   # released per query
