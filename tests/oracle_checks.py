"""Invariant checkers used by the oracle pins and by the mutation check (P9).

Each checker returns a list of failure strings (empty = pass), so the mutation
test can assert that an injected bug is caught."""
import numpy as np

from baton_inputs import (KIND_Q, KIND_K, KIND_V, bf16_bits_to_f64, query_history_bits,
                          query_token_bits)
from oracle import Simulator, solo_attention


def closed_form_failures(sim, rec, release=True):
    """P1/P2: mask[b][j] = occ_b and j >= pad_b; popcount = lens; pad = S - lens;
    after release min over occupied pad == 0."""
    errs = []
    for r, sh in enumerate(sim.shards):
        S = sh.S
        if sh.mask.shape[1] != S:
            errs.append(f"t{rec.t} shard{r}: mask width {sh.mask.shape[1]} != S {S}")
            continue
        occ = sh.qid >= 0
        j = np.arange(S)[None, :]
        expect = (occ[:, None] & (j >= sh.pad[:, None])).astype(np.uint8)
        if not np.array_equal(expect, sh.mask):
            errs.append(f"t{rec.t} shard{r}: mask != closed form")
        lens = sh.lens()
        for b in range(sh.B):
            if occ[b] and sh.pad[b] != S - lens[b]:
                errs.append(f"t{rec.t} shard{r} slot{b}: pad {sh.pad[b]} != S-lens")
            if not occ[b] and lens[b] != 0:
                errs.append(f"t{rec.t} shard{r} slot{b}: empty row has live columns")
        if release and occ.any() and min(sh.pad[occ]) != 0:
            errs.append(f"t{rec.t} shard{r}: front not released")
        if release and not occ.any() and S != 0:
            errs.append(f"t{rec.t} shard{r}: empty shard keeps S={S}")
    return errs


def history(wl, qid, n):
    K = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_K, wl.layers, qid, 0, n,
                                            wl.kv_heads, wl.head_dim, wl.scales[1]))
    V = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_V, wl.layers, qid, 0, n,
                                            wl.kv_heads, wl.head_dim, wl.scales[2]))
    return K, V


def solo_output(wl, qid, pos):
    """O-1 on the query's own keyed history [0, pos] (the query decoded alone)."""
    K, V = history(wl, qid, pos + 1)
    out = []
    for l in range(wl.layers):
        q = bf16_bits_to_f64(query_token_bits(wl.seed, KIND_Q, l, [qid], [pos], wl.q_heads,
                                              wl.head_dim, wl.scales[0]))[0]
        out.append(solo_attention(q, K[l], V[l]))
    return np.stack(out)


def live_kv_failures(sim):
    """P3: every live row holds exactly the query's own keyed history."""
    errs = []
    for r, sh in enumerate(sim.shards):
        for b in sh.occupied():
            qid = int(sh.qid[b])
            Kl, Vl = sh.live_kv(b)
            n = Kl.shape[2]
            K, V = history(sim.wl, qid, n)
            if not (np.array_equal(K, Kl) and np.array_equal(V, Vl)):
                errs.append(f"t{sim.t} shard{r} slot{b}: live KV != history of q{qid}")
    return errs


def run_checked(wl, kv=False, fill=0.0, release=True, check_kv_every=1, G=None):
    """Run a simulation, checking P1/P2 after every iteration (and P3 when kv)."""
    sim = Simulator(wl, G=G, kv=kv, fill=fill, release=release, keep_outputs=kv)
    errs = []
    recs = []
    while True:
        rec = sim.iteration()
        recs.append(rec)
        errs += closed_form_failures(sim, rec, release=release)
        if kv and (rec.t % check_kv_every == 0):
            errs += live_kv_failures(sim)
        if sim.done():
            break
        if len(recs) > 100000:
            errs.append("runaway")
            break
    return sim, recs, errs


def token_accounting_failures(wl, sim, recs):
    """Every query decodes exactly A tokens at positions l_q .. l_q+A-1 (C9),
    whatever the interleaving of preemptions and resizes."""
    errs = []
    seen = {}
    for rec in recs:
        for g, qid, pos in rec.decoded:
            seen.setdefault(qid, []).append(pos)
    done_all = wl.iterations < 0
    for q in wl.queries:
        got = seen.get(q.qid, [])
        if done_all and got != list(range(q.l_q, q.l_q + q.A)):
            errs.append(f"q{q.qid}: positions {got[:5]}.. != {q.l_q}..{q.l_q + q.A - 1}")
        elif got and got != list(range(q.l_q, q.l_q + len(got))):
            errs.append(f"q{q.qid}: non-contiguous positions")
    return errs
