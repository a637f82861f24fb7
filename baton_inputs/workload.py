"""Seeded query streams shaped like the paper's workloads.

The paper evaluates on two synthetic datasets (§4.1
"Dataset"): (1) 120 queries mixing long-input/short-output,
short-input/long-output and short/short in a 1:1:2 ratio, "long" around 4,000
words and "short" a few dozen to 400; (2) 30 short/short queries of a few dozen
to 200 words.  One word is taken as one token and the lengths
are scaled to each configuration's context capacity.

A query is (qid, arrival iteration, l_q = prefilled length, A = answer length).
Reading C9: a query with answer length A occupies exactly A decode iterations;
its live length at removal is l_q + A, which never exceeds the capacity.

Control events (preemption points, batch resizes) are random draws that the
schedulers on both sides take as INPUTS; the policy that turns them into slot
decisions is implemented separately by the oracle and
by the product scheduler.  Nothing here implements Baton's arithmetic.
"""
from dataclasses import dataclass, field
from typing import Optional, Dict, List, Tuple

import numpy as np

from .keygen import SCALES_FLAT, SCALES_PEAKY

SEED_MAIN = 18701
SEED_SECOND = 2410


@dataclass(frozen=True)
class Query:
    qid: int
    arrival: int     # iteration at whose insert phase the query becomes available
    l_q: int         # prefilled length (prompt), >= 1
    A: int           # answer length = number of decode iterations, >= 1
    kind: str = ""
    priority: int = 0  # SLA priority (reading C25): higher preempts lower


@dataclass
class ControlEvents:
    # iteration -> number of live queries to preempt (C17 picks the victims)
    preempt: Dict[int, int] = field(default_factory=dict)
    # iteration -> fraction of live queries to preempt (resolved by the scheduler)
    preempt_frac: Dict[int, float] = field(default_factory=dict)
    # iteration -> "halve" | "double" | int (new global active-slot count)
    resize: Dict[int, object] = field(default_factory=dict)


@dataclass
class Workload:
    name: str
    queries: List[Query]
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    slots: int            # global batch capacity (all GPUs)
    max_ctx: int          # per-slot KV capacity S_cap
    gpus: int = 1
    active: int = -1      # initial active (usable) global slots; -1 = all
    seed: int = SEED_MAIN
    scales: Tuple[int, int, int] = SCALES_FLAT
    control: ControlEvents = field(default_factory=ControlEvents)
    iterations: int = -1  # -1 = until every query finished
    # P:L146-147 batch-size governor (reading C26): (hi, lo) fractions of a shard's
    # token budget active_slots x max_ctx; None = off
    governor: Optional[Tuple[float, float]] = None

    @property
    def slots_per_gpu(self):
        return self.slots // self.gpus

    def initial_active(self):
        return self.slots if self.active < 0 else self.active

    def decode_tokens(self):
        return sum(q.A for q in self.queries)


# --------------------------------------------------------------------------
# configs[0]: the toy W1 trace (SURVEY.md §8(c) "Worked trace W1")
W1_LQ = [4, 3, 36, 39, 19, 11, 35, 14, 10, 19]
W1_A = [10, 18, 1, 6, 9, 11, 3, 4, 5, 4]


def w1_workload(seed=SEED_MAIN, scales=SCALES_FLAT):
    qs = [Query(i, 0, W1_LQ[i], W1_A[i], "w1") for i in range(10)]
    return Workload("toy", qs, layers=1, q_heads=2, kv_heads=2, head_dim=16, slots=4,
                    max_ctx=64, seed=seed, scales=scales)


def _mix_queries(rng, n, first_wave, lam, classes, max_ctx, all_at_zero=False):
    """D1-style 1:1:2 mix with Poisson arrivals."""
    kinds = rng.choice(len(classes), size=n, p=[0.25, 0.25, 0.5])
    arrivals = np.zeros(n, dtype=np.int64)
    if not all_at_zero and n > first_wave:
        gaps = rng.exponential(1.0 / lam, size=n - first_wave)
        arrivals[first_wave:] = np.floor(np.cumsum(gaps)).astype(np.int64)
    qs = []
    for i in range(n):
        name, (plo, phi), (alo, ahi) = classes[kinds[i]]
        l_q = int(rng.integers(plo, phi + 1))
        A = int(rng.integers(alo, ahi + 1))
        A = max(1, min(A, max_ctx - l_q))
        qs.append(Query(i, int(arrivals[i]), l_q, A, name))
    return qs


CLASSES_7B = [("LI-SO", (1200, 1800), (30, 200)),
              ("SI-LO", (30, 400), (1000, 1600)),
              ("SI-SO", (30, 400), (30, 400))]
CLASSES_D2 = [("SI-SO", (30, 200), (30, 200))] * 3
CLASSES_70B = [("LI-SO", (3000, 3800), (30, 200)),
               ("SI-LO", (30, 400), (3000, 3800)),
               ("SI-SO", (30, 400), (30, 400))]


def config_workload(name, seed=SEED_MAIN, gpus=None, n_queries=None, scales=SCALES_FLAT):
    """The five BASELINE.json configs."""
    rng = np.random.default_rng(seed)
    if name == "toy":
        return w1_workload(seed, scales)
    if name in ("7b", "7b-d2"):
        n = n_queries or 512
        cls = CLASSES_7B if name == "7b" else CLASSES_D2
        qs = _mix_queries(rng, n, 32, 0.08, cls, 2048)
        return Workload(name, qs, layers=32, q_heads=32, kv_heads=32, head_dim=128, slots=32,
                        max_ctx=2048, gpus=gpus or 1, seed=seed, scales=scales)
    if name == "13b":
        n = n_queries or 2064
        g = gpus or 1
        qs = []
        for i in range(n):
            l_q = int(rng.integers(128, 1025))
            A = 1 + (i % 32) if i < 64 else 32
            qs.append(Query(i, 0, l_q, A, "churn"))
        return Workload(name, qs, layers=40, q_heads=40, kv_heads=40, head_dim=128, slots=64,
                        max_ctx=2048, gpus=g, seed=seed, scales=scales)
    if name == "70b":
        n = n_queries or 512
        qs = _mix_queries(rng, n, n, 0.0, CLASSES_70B, 4096, all_at_zero=True)
        return Workload(name, qs, layers=80, q_heads=64, kv_heads=8, head_dim=128, slots=128,
                        max_ctx=4096, gpus=gpus or 8, seed=seed, scales=scales)
    if name == "stress":
        n = n_queries or 2048
        g = gpus or 8
        qs = _mix_queries(rng, n, n, 0.0, CLASSES_7B, 2048, all_at_zero=True)
        ctl = ControlEvents()
        for t in range(16, 641, 16):
            ctl.preempt_frac[t] = 0.25
        active = 16
        for t in range(64, 641, 64):
            active = min(256, active * 2)
            ctl.resize[t] = active
        return Workload(name, qs, layers=32, q_heads=32, kv_heads=32, head_dim=128, slots=256,
                        max_ctx=2048, gpus=g, active=16, seed=seed, scales=scales, control=ctl,
                        iterations=640)
    raise KeyError(name)


CONFIGS = ("toy", "7b", "13b", "70b", "stress")


def random_stream(seed):
    """One of the 200 toy-scale random parity streams."""
    rng = np.random.default_rng(1_000_003 + seed)
    B = int(rng.integers(2, 9))
    S_cap = int(rng.integers(8, 65))
    Hq, Hkv = [(2, 2), (4, 2), (8, 1)][int(rng.integers(0, 3))]
    D = [16, 128][int(rng.integers(0, 2))]
    L = int(rng.integers(1, 3))
    scales = SCALES_FLAT if rng.random() < 0.5 else SCALES_PEAKY
    iters = int(rng.integers(40, 121))
    qs = []
    qid = 0
    for t in range(iters):
        if t == 0:
            n_arr = int(rng.integers(1, B + 1))
        else:
            n_arr = int(rng.random() < 0.5)
        for _ in range(n_arr):
            l_q = int(rng.integers(1, S_cap // 2 + 1))
            A = int(rng.integers(1, 13))
            A = max(1, min(A, S_cap - l_q))
            qs.append(Query(qid, t, l_q, A, "rand"))
            qid += 1
    ctl = ControlEvents()
    for t in range(1, iters):
        if rng.random() < 0.1:
            ctl.preempt[t] = 1
        r = rng.random()
        if r < 0.05:
            ctl.resize[t] = "halve" if rng.random() < 0.5 else "double"
    return Workload(f"rand{seed}", qs, layers=L, q_heads=Hq, kv_heads=Hkv, head_dim=D, slots=B,
                    max_ctx=S_cap, seed=SEED_MAIN + seed, scales=scales, control=ctl,
                    iterations=iters)
