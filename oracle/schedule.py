"""Oracle serving loop over G shards (TEST INFRASTRUCTURE ONLY).

Drives ``batch.Shard`` through Baton's relay-race loop ("replenish a new
query as soon as inference of any query is completed, like a relay race") with
P&D decoupling (queries are prefilled separately and embedded, then
everybody decodes width-1).  Per iteration t >= 1, in this order (reading of
P:L101 and P:L124, DESIGN.md §3 C5):

  1. decode   -- ``Shard.step`` on every shard
  2. finish   -- a query with answer length A finishes after its A-th step (C9)
  3. remove   -- finished rows zeroed in ascending slot order, then the
                 front [0:min(index)] released ("before inserting")
  4. preempt  -- control input: store the K/V of the lowest-priority queries and
                 free their rows; victims = most recently inserted, ties
                 by higher qid (C17); they re-enter at the HEAD of the queue
  5. resize   -- control input: change the number of active slots; shrinking moves
                 queries out: victims as in 4 if the remaining rows do
                 not fit, then compaction (C19)
  6. insert   -- arrivals join the FCFS queue; repeatedly the first queue entry
                 that has an eligible free active slot takes the lowest such
                 global slot (C7, C8); global slot g lives on shard floor(g / B_g)
                 (C20).  A stored (preempted) query is eligible only for slots of
                 the shard holding its stored K/V (C20b); a fresh query for any.

Policy ``"shape"`` (the vector-SHAPING path, Baton without P&D, P:L101-113;
NEXT-1): step 6 only reserves the lowest free slot for a RAW query; step 1 of the
next iteration is ``Shard.shape_step``, whose input width is the longest reserved
prompt.  That iteration is the new query's prefill (it yields its first token,
C9), so its A decode iterations follow it; everybody else decodes as usual in the
same padded iteration (the bubble of P:L128).  Control events are not used with
this policy.

Priorities and the memory governor (readings C25/C26; off unless the
workload sets query priorities / ``governor``):
  * the queue is served by (priority desc, then stored victims -- newest batch
    first, in eviction order -- then FCFS arrival order);
  * C25: before any insert of the phase, if the best waiting query has no
    eligible free (and admissible) slot while a live query of LOWER priority sits
    on an eligible shard, that query is stored (victim order: lowest priority, then
    C17) -- at most one such preemption per iteration -- and the urgent query then
    takes the freed slot;
  * C26: after step 5, a shard whose live tokens exceed hi * T (T = active slots x
    max_ctx) stores victims (same order) until it does not; an insert is admitted
    only if live tokens + its length <= lo * T on its shard.

Iteration 0 runs only step 6.  A query's tokens are keyed by (qid, position) so a
decode step of a query with live length n (after the append) handles position
n-1 (C3); its prefilled K/V are positions [0, l_q).
"""
from collections import deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from baton_inputs import (KIND_Q, KIND_K, KIND_V, bf16_bits_to_f64, query_history_bits,
                          query_token_bits)
from .batch import Shard


@dataclass
class IterationRecord:
    t: int
    decoded: List[Tuple[int, int, int]] = field(default_factory=list)   # (gslot, qid, pos)
    finished: List[int] = field(default_factory=list)                    # qids
    removed: List[int] = field(default_factory=list)                     # gslots
    released: List[int] = field(default_factory=list)                    # p per shard
    preempted: List[Tuple[int, int]] = field(default_factory=list)       # (qid, gslot)
    resized: Optional[int] = None
    moved: List[Tuple[int, int]] = field(default_factory=list)           # (old gslot, new gslot)
    inserted: List[Tuple[int, int, int]] = field(default_factory=list)   # (gslot, qid, l_q)
    prefilled: List[Tuple[int, int, int]] = field(default_factory=list)  # (gslot, qid, l_q), shape
    width: List[int] = field(default_factory=list)                       # input width per shard
    S: List[int] = field(default_factory=list)
    pad: List[np.ndarray] = field(default_factory=list)
    qid: List[np.ndarray] = field(default_factory=list)
    lens: List[np.ndarray] = field(default_factory=list)


class Simulator:
    def __init__(self, wl, G=None, kv=False, fill=0.0, release=True, keep_outputs=False,
                 snapshot_masks=False, policy="pd"):
        assert policy in ("pd", "shape")
        self.policy = policy
        self.wl = wl
        self.G = G or wl.gpus
        assert wl.slots % self.G == 0
        self.Bg = wl.slots // self.G
        self.kv = kv
        self.release_enabled = release
        self.keep_outputs = keep_outputs
        self.snapshot_masks = snapshot_masks
        self.shards = [Shard(self.Bg, wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim,
                             wl.max_ctx, fill=fill, kv=kv) for _ in range(self.G)]
        self.queries = {q.qid: q for q in wl.queries}
        self.generated = {q.qid: 0 for q in wl.queries}
        self.inserted_at = {}
        self.arrivals = deque(sorted(wl.queries, key=lambda q: (q.arrival, q.qid)))
        self.queue = deque()     # entries: (qid, length, K, V, home shard or None)
        self.ticket = {}         # qid -> queue order key within a priority class (C25)
        self.prio = {q.qid: q.priority for q in wl.queries}
        self.n_active = wl.initial_active()
        self.outputs: Dict[Tuple[int, int], np.ndarray] = {}
        self.masks: List[List[np.ndarray]] = []
        self.finished_at = {}
        self.pending = [[] for _ in range(self.G)]   # shape policy: reserved (b, qid, l_q)
        if policy == "shape":
            c = wl.control
            assert not (c.preempt or c.preempt_frac or c.resize), "shape policy: no control events"
            assert wl.governor is None and not any(q.priority for q in wl.queries), \
                "shape policy: no priorities / governor (stored K/V re-enter by embedding)"
        self.t = 0

    # ------------------------------------------------------------------ helpers
    def active_per_shard(self):
        return self.n_active // self.G

    def _loc(self, g):
        return g // self.Bg, g % self.Bg

    def _live(self):
        out = []
        for r, sh in enumerate(self.shards):
            for b in sh.occupied():
                out.append((r * self.Bg + b, int(sh.qid[b])))
        return out

    def _victim_order(self, live):
        # C25 lowest priority first; C17 then most recently inserted, ties by higher qid
        return sorted(live, key=lambda x: (self.prio[x[1]], -self.inserted_at[x[1]], -x[1]))

    def _usage(self, r):
        """Live tokens held by shard r (C26)."""
        sh = self.shards[r]
        lens = sh.lens()
        return int(sum(lens[b] for b in sh.occupied()))

    def _budget(self):
        return self.active_per_shard() * self.wl.max_ctx

    def _govern(self, rec):
        """C26: store victims while a shard exceeds hi * T."""
        gov = self.wl.governor
        if gov is None:
            return []
        out = []
        for r, sh in enumerate(self.shards):
            while self._usage(r) > gov[0] * self._budget() and sh.occupied():
                live = [(r * self.Bg + b, int(sh.qid[b])) for b in sh.occupied()]
                g, _ = self._victim_order(live)[0]
                out.append(self._evict(g, rec))
        return out

    def _prefill(self, qid, length):
        wl = self.wl
        sk, sv = wl.scales[1], wl.scales[2]
        K = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_K, wl.layers, qid, 0, length,
                                                wl.kv_heads, wl.head_dim, sk))
        V = bf16_bits_to_f64(query_history_bits(wl.seed, KIND_V, wl.layers, qid, 0, length,
                                                wl.kv_heads, wl.head_dim, sv))
        return K, V

    def _evict(self, g, rec):
        """store the query's K/V, free its row; returns queue entry."""
        r, b = self._loc(g)
        sh = self.shards[r]
        qid = int(sh.qid[b])
        K, V = sh.extract(b)
        length = int(sh.lens()[b])
        sh.remove(b)
        rec.preempted.append((qid, g))
        return (qid, length, K, V, r)

    # ------------------------------------------------------------------ phases
    def _token_qkv(self, qids, pos):
        """q/k/v of one token per slot (keyed by (qid, position)): [L][B][H][D]."""
        wl = self.wl
        return [np.stack([bf16_bits_to_f64(query_token_bits(
            wl.seed, kind, l, qids, pos, H, wl.head_dim, scale)) for l in range(wl.layers)])
            for kind, H, scale in ((KIND_Q, wl.q_heads, wl.scales[0]),
                                   (KIND_K, wl.kv_heads, wl.scales[1]),
                                   (KIND_V, wl.kv_heads, wl.scales[2]))]

    def _shape_decode(self, r, sh, rec):
        """one padded iteration of width W on shard r."""
        wl = self.wl
        new = self.pending[r]
        self.pending[r] = []
        W = max(l for _, _, l in new)
        occ = sh.occupied()
        lens = sh.lens()
        o = None
        if self.kv:
            shp = lambda H: np.zeros((wl.layers, self.Bg, W, H, wl.head_dim))
            q, k, v = shp(wl.q_heads), shp(wl.kv_heads), shp(wl.kv_heads)
            # survivors: their decode token at input position 0
            qids = np.zeros(self.Bg, np.int64)
            pos = np.zeros(self.Bg, np.int64)
            for b in occ:
                qids[b], pos[b] = sh.qid[b], lens[b]
            tq, tk, tv = self._token_qkv(qids, pos)
            for b in occ:
                q[:, b, 0], k[:, b, 0], v[:, b, 0] = tq[:, b], tk[:, b], tv[:, b]
            # new queries: their whole prompt, positions 0..l_q-1
            for b, qd, l in new:
                for t in range(l):
                    tq, tk, tv = self._token_qkv(np.full(self.Bg, qd), np.full(self.Bg, t))
                    q[:, b, t], k[:, b, t], v[:, b, t] = tq[:, b], tk[:, b], tv[:, b]
            o = sh.shape_step(new, q, k, v)
        else:
            sh.shape_step(new)
        rec.width[r] = W
        for b in occ:
            g = r * self.Bg + b
            qid = int(sh.qid[b])
            rec.decoded.append((g, qid, int(lens[b])))
            if self.keep_outputs and o is not None:
                self.outputs[(qid, int(lens[b]))] = o[:, b, 0].copy()
            self.generated[qid] += 1
        for b, qd, l in new:
            rec.prefilled.append((r * self.Bg + b, qd, l))
            if self.keep_outputs and o is not None:
                for t in range(l):
                    self.outputs[(qd, t)] = o[:, b, t].copy()

    def _decode(self, rec):
        wl = self.wl
        rec.width = [1] * self.G
        for r, sh in enumerate(self.shards):
            if self.pending[r]:
                self._shape_decode(r, sh, rec)
                continue
            occ = sh.occupied()
            if not occ:
                sh.step() if not self.kv else sh.step(*self._zeros_qkv())
                continue
            lens = sh.lens()
            pos = np.zeros(self.Bg, np.int64)
            qids = np.zeros(self.Bg, np.int64)
            for b in occ:
                pos[b] = lens[b]          # position of the token decoded now
                qids[b] = sh.qid[b]
            if self.kv:
                q = np.stack([bf16_bits_to_f64(query_token_bits(
                    wl.seed, KIND_Q, l, qids, pos, wl.q_heads, wl.head_dim, wl.scales[0]))
                    for l in range(wl.layers)])
                k = np.stack([bf16_bits_to_f64(query_token_bits(
                    wl.seed, KIND_K, l, qids, pos, wl.kv_heads, wl.head_dim, wl.scales[1]))
                    for l in range(wl.layers)])
                v = np.stack([bf16_bits_to_f64(query_token_bits(
                    wl.seed, KIND_V, l, qids, pos, wl.kv_heads, wl.head_dim, wl.scales[2]))
                    for l in range(wl.layers)])
                o = sh.step(q, k, v)
            else:
                sh.step()
                o = None
            for b in occ:
                g = r * self.Bg + b
                qid = int(qids[b])
                rec.decoded.append((g, qid, int(pos[b])))
                if self.keep_outputs and o is not None:
                    self.outputs[(qid, int(pos[b]))] = o[:, b].copy()
                self.generated[qid] += 1

    def _zeros_qkv(self):
        wl = self.wl
        z = lambda H: np.zeros((wl.layers, self.Bg, H, wl.head_dim))
        return z(wl.q_heads), z(wl.kv_heads), z(wl.kv_heads)

    def _remove_finished(self, rec):
        for r, sh in enumerate(self.shards):
            for b in sh.occupied():
                qid = int(sh.qid[b])
                if self.generated[qid] >= self.queries[qid].A:
                    sh.remove(b)
                    rec.removed.append(r * self.Bg + b)
                    rec.finished.append(qid)
                    self.finished_at[qid] = self.t

    def _release_all(self, rec):
        ps = []
        for sh in self.shards:
            ps.append(sh.release() if self.release_enabled else 0)
        if not rec.released:
            rec.released = ps
        else:
            rec.released = [a + b for a, b in zip(rec.released, ps)]

    def _preempt(self, rec):
        ctl = self.wl.control
        t = self.t
        n = 0
        live = self._live()
        if t in ctl.preempt:
            n = ctl.preempt[t]
        elif t in ctl.preempt_frac:
            n = int(np.floor(ctl.preempt_frac[t] * len(live)))
        n = min(n, len(live))
        if n <= 0:
            return []
        victims = self._victim_order(live)[:n]
        return [self._evict(g, rec) for g, _ in victims]

    def _resize(self, rec):
        ctl = self.wl.control
        if self.t not in ctl.resize:
            return []
        ev = ctl.resize[self.t]
        a = self.active_per_shard()
        if ev == "halve":
            a_new = max(1, a // 2)
        elif ev == "double":
            a_new = min(self.Bg, a * 2)
        else:
            a_new = max(1, min(self.Bg, int(ev) // self.G))
        self.n_active = a_new * self.G
        rec.resized = self.n_active
        out = []
        if a_new < a:
            for r, sh in enumerate(self.shards):
                occ = sh.occupied()
                beyond = [b for b in occ if b >= a_new]
                free_low = [b for b in range(a_new) if sh.qid[b] < 0]
                need = len(beyond) - len(free_low)
                if need > 0:
                    live = [(r * self.Bg + b, int(sh.qid[b])) for b in occ]
                    for g, _ in self._victim_order(live)[:need]:
                        out.append(self._evict(g, rec))
                o2n = sh.compact(a_new)
                for old, new in enumerate(o2n):
                    if old != new:
                        rec.moved.append((r * self.Bg + old, r * self.Bg + new))
        return out

    def _requeue(self, victims):
        """Stored victims re-enter ahead of every earlier entry of their priority,
        in eviction order (C8/C17; C25 orders across priorities)."""
        for i, v in enumerate(victims):
            self.ticket[v[0]] = -(self.t * 100000) + i
            self.queue.append(v)

    def _admissible(self, r, length):
        gov = self.wl.governor
        return gov is None or self._usage(r) + length <= gov[1] * self._budget()

    def _order(self):
        return sorted(range(len(self.queue)),
                      key=lambda i: (-self.prio[self.queue[i][0]], self.ticket[self.queue[i][0]]))

    def _free(self):
        a = self.active_per_shard()
        reserved = {r * self.Bg + b for r in range(self.G) for b, _, _ in self.pending[r]}
        return [r * self.Bg + b for r, sh in enumerate(self.shards) for b in range(a)
                if sh.qid[b] < 0 and r * self.Bg + b not in reserved]

    def _priority_preempt(self, rec):
        """C25, before any insert: the best waiting query, if it has no
        eligible admissible free slot, stores the lowest-priority live query of an
        eligible shard whose priority is lower than its own."""
        if not self.queue:
            return
        qid0, length, _, _, home = self.queue[self._order()[0]]
        if any((home is None or g // self.Bg == home) and self._admissible(g // self.Bg, length)
               for g in self._free()):
            return
        a = self.active_per_shard()
        live = [(g, q) for g, q in self._live()
                if (home is None or g // self.Bg == home) and g % self.Bg < a
                and self.prio[q] < self.prio[qid0]]
        if not live:
            return
        g, _ = self._victim_order(live)[0]
        v = self._evict(g, rec)
        self._release_all(rec)
        self._requeue([v])

    def _insert_phase(self, rec):
        while self.arrivals and self.arrivals[0].arrival <= self.t:
            q = self.arrivals.popleft()
            self.ticket[q.qid] = len(self.ticket) + 1
            self.queue.append((q.qid, q.l_q, None, None, None))
        if self.t > 0 and self.policy == "pd":
            self._priority_preempt(rec)
        while self.queue:
            free = self._free()
            pick = None
            for i in self._order():
                entry = self.queue[i]
                home = entry[4]
                elig = [g for g in free if (home is None or g // self.Bg == home)
                        and self._admissible(g // self.Bg, entry[1])]
                if elig:
                    pick = (i, elig[0])
                    break
            if pick is None:
                break
            i, g = pick
            qid, length, K, V, _ = self.queue[i]
            del self.queue[i]
            if self.policy == "shape":          # raw query: prefilled in the next iteration
                r, b = self._loc(g)
                self.pending[r].append((b, qid, length))
                self.inserted_at[qid] = self.t
                rec.inserted.append((g, qid, length))
                continue
            if self.kv and K is None:
                K, V = self._prefill(qid, length)
            r, b = self._loc(g)
            self.shards[r].insert(b, qid, length, K, V)
            self.inserted_at[qid] = self.t
            rec.inserted.append((g, qid, length))

    # ------------------------------------------------------------------ driver
    def done(self):
        if self.wl.iterations >= 0 and self.t >= self.wl.iterations:
            return True
        return (not self.arrivals and not self.queue and not self._live()
                and not any(self.pending))

    def iteration(self):
        rec = IterationRecord(self.t)
        if self.t > 0:
            self._decode(rec)
            self._remove_finished(rec)
            self._release_all(rec)
            victims = self._preempt(rec)
            victims += self._resize(rec)
            if victims:
                self._release_all(rec)
            gv = self._govern(rec)
            if gv:
                self._release_all(rec)
            victims += gv
            self._requeue(victims)
        self._insert_phase(rec)
        for sh in self.shards:
            rec.S.append(sh.S)
            rec.pad.append(sh.pad.copy())
            rec.qid.append(sh.qid.copy())
            rec.lens.append(sh.lens())
        if self.snapshot_masks:
            self.masks.append([sh.mask.copy() for sh in self.shards])
        self.t += 1
        return rec

    def run(self, max_iters=None):
        recs = []
        while True:
            recs.append(self.iteration())
            if self.done() or (max_iters is not None and self.t >= max_iters):
                break
        return recs
