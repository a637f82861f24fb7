"""Brute force (P8) and mutation check (P9) for the oracle.

P8: every workload of 3 queries with (l_q, A) in [1..3]x[1..3] on B in {1,2,3}
(2187 schedules) satisfies the closed-form mask/pad/S invariants after every
iteration and decodes every query at exactly positions l_q..l_q+A-1; a seeded
sample also runs with K/V and NaN placeholders and must equal solo decoding
bitwise.

P9 ("inject 'skip mask zeroing', and the suite must fail"): plausible bugs
injected into the oracle are each caught by the checkers above."""
import itertools

import numpy as np
import pytest

import oracle.batch as ob
from baton_inputs import Workload, Query, ControlEvents, w1_workload
from oracle import Simulator
from oracle_checks import run_checked, token_accounting_failures, solo_output


def _tiny(B, spec, preempt=None, H=(2, 1), D=4):
    qs = [Query(i, 0, l, a) for i, (l, a) in enumerate(spec)]
    return Workload("bf", qs, layers=1, q_heads=H[0], kv_heads=H[1], head_dim=D, slots=B,
                    max_ctx=12, control=ControlEvents(preempt=preempt or {}))


def test_bruteforce_metadata_all_small_schedules():
    pairs = list(itertools.product(range(1, 4), range(1, 4)))
    n = 0
    for B in (1, 2, 3):
        for spec in itertools.product(pairs, repeat=3):
            wl = _tiny(B, spec)
            sim, recs, errs = run_checked(wl)
            assert errs == [], (B, spec, errs[:3])
            assert token_accounting_failures(wl, sim, recs) == [], (B, spec)
            n += 1
    assert n == 2187


def test_bruteforce_kv_sample_equals_solo():
    rng = np.random.default_rng(8)
    pairs = list(itertools.product(range(1, 5), range(1, 4)))
    for trial in range(60):
        B = int(rng.integers(1, 4))
        spec = [pairs[i] for i in rng.integers(0, len(pairs), size=int(rng.integers(3, 5)))]
        pre = {int(rng.integers(1, 6)): 1} if rng.random() < 0.5 else None
        wl = _tiny(B, spec, preempt=pre)
        sim, recs, errs = run_checked(wl, kv=True, fill=np.nan)
        assert errs == []
        for (qid, pos), o in sim.outputs.items():
            assert np.array_equal(o, solo_output(wl, qid, pos)), (trial, qid, pos)


# ------------------------------------------------------------------- P9
def _suite_fails(wl):
    """Run the pins on one workload; True if any of them flags a failure."""
    try:
        sim, recs, errs = run_checked(wl, kv=True)
    except Exception:
        return True
    if errs or token_accounting_failures(wl, sim, recs):
        return True
    for (qid, pos), o in sim.outputs.items():
        if not np.array_equal(o, solo_output(wl, qid, pos)):
            return True
    return False


def _w1_with_preempt():
    wl = w1_workload()
    wl.control = ControlEvents(preempt={4: 1, 11: 2})
    return wl


def _idle_slot_workload():
    # a slot stays empty while others decode (reading C6), then a late arrival fills it
    qs = [Query(0, 0, 3, 6), Query(1, 0, 5, 2), Query(2, 4, 2, 3)]
    return Workload("idle", qs, layers=1, q_heads=2, kv_heads=1, head_dim=4, slots=3, max_ctx=16)


def test_unmutated_suite_passes():
    assert not _suite_fails(w1_workload())
    assert not _suite_fails(_w1_with_preempt())
    assert not _suite_fails(_idle_slot_workload())


def _mut_pad_off_by_one(orig):
    def insert(self, slot, qid, l_q, K_pref=None, V_pref=None):
        orig(self, slot, qid, l_q, K_pref, V_pref)
        if self.pad[slot] > 0:
            self.pad[slot] -= 1
    return insert


def _mut_skip_mask_zeroing(orig):
    def remove(self, slot):
        keep = self.mask[slot].copy()
        orig(self, slot)
        self.mask[slot] = keep
    return remove


def _mut_copy_lq_minus_1(orig):
    def insert(self, slot, qid, l_q, K_pref=None, V_pref=None):
        orig(self, slot, qid, l_q, K_pref, V_pref)
        if self.kv:
            self.K[:, slot, :, self.S - l_q, :] = self.fill   # first prefilled token lost
    return insert


def _mut_skip_release(orig):
    def release(self):
        return 0
    return release


def _mut_expansion_keeps_pads(orig):
    def insert(self, slot, qid, l_q, K_pref=None, V_pref=None):
        before = self.pad.copy()
        S = self.S
        orig(self, slot, qid, l_q, K_pref, V_pref)
        if l_q > S:
            for b in self.occupied():
                if b != slot:
                    self.pad[b] = before[b]
    return insert


def _mut_empty_rows_get_ones(orig):
    def step(self, *a):
        out = orig(self, *a)
        self.mask[:, -1] = 1
        return out
    return step


def _mut_release_max(orig):
    def release(self):
        occ = self.occupied()
        if not occ:
            return orig(self)
        p = max(int(self.pad[b]) for b in occ)
        self.mask = self.mask[:, p:]
        if self.kv:
            self.K = self.K[:, :, :, p:, :]
            self.V = self.V[:, :, :, p:, :]
        for b in occ:
            self.pad[b] = max(0, self.pad[b] - p)
        self.S -= p
        return p
    return release


@pytest.mark.parametrize("method,mutator", [
    ("insert", _mut_pad_off_by_one),
    ("remove", _mut_skip_mask_zeroing),
    ("insert", _mut_copy_lq_minus_1),
    ("release", _mut_skip_release),
    ("insert", _mut_expansion_keeps_pads),
    ("step", _mut_empty_rows_get_ones),
    ("release", _mut_release_max),
])
def test_mutation_is_caught(monkeypatch, method, mutator):
    orig = getattr(ob.Shard, method)
    monkeypatch.setattr(ob.Shard, method, mutator(orig))
    assert (_suite_fails(w1_workload()) or _suite_fails(_w1_with_preempt())
            or _suite_fails(_idle_slot_workload()))
