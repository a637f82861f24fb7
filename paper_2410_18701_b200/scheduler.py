"""Host-side relay-race scheduler of the product path (replicated on every rank).

Baton inserts a new query "as soon as inference of any query is completed, like
a relay race" and, with P&D decoupling, every query in the
batch decodes width-1.  This module only DECIDES (which slots finish, which
queries are stored/re-inserted, where each query goes); the engine
(``engine.py``) executes the decisions through libbaton.  It is deterministic
and replicated: every rank runs the same planner on the same inputs (the
workload, the control events, and the per-iteration completion flags that the
engine all-gathers), so no rank ever broadcasts a decision.

Policy readings: C25 priorities (the queue is served by priority,
then stored victims newest first, then FCFS; at most one preemption of a lower-
priority live query per iteration, before the inserts), C26 the memory governor
((hi, lo) of a rank's token budget: store victims above hi, admit inserts up to
lo); C5 release after removals and before inserts;
C7 inserts of an iteration in ascending slot order; C8 FCFS, lowest free slot,
stored queries re-enter at the queue head; C9 A decode iterations per query;
C17 victims = most recently inserted, ties by higher qid; C18/C19 resize and
stable compaction; C20 global slot g lives on rank g // B_g; C20b a stored
query may only re-enter on the rank holding its stored K/V.
"""
from collections import deque
from dataclasses import dataclass, field
from typing import List, Optional, Tuple


@dataclass
class QueueEntry:
    qid: int
    length: int                 # prefilled / stored K/V length
    home: Optional[int] = None  # rank holding stored K/V (None = fresh query)
    pin: Optional[int] = None   # fresh query prefilled remotely: the rank its K/V went to (C20c)

    def rank(self):
        """The only rank this entry may enter (None: any)."""
        return self.home if self.home is not None else self.pin


@dataclass
class Decisions:
    t: int
    decode: List[Tuple[int, int, int]] = field(default_factory=list)    # (gslot, qid, pos)
    finished: List[Tuple[int, int]] = field(default_factory=list)       # (gslot, qid)
    victims: List[Tuple[int, int, int]] = field(default_factory=list)   # (gslot, qid, length)
    resize: Optional[int] = None                                         # new active per rank
    # victims[:n_pre_compact] were chosen BEFORE this iteration's compaction (their
    # gslots are pre-compaction indices: C17 preemption, resize overflow); the rest
    # (C26 governor, C25 priority preemption) AFTER it, in post-compaction indices
    n_pre_compact: int = 0
    inserts: List[Tuple[int, int, int, Optional[int]]] = field(default_factory=list)  # (gslot, qid, len, home)
    raw: List[Tuple[int, int, int]] = field(default_factory=list)       # shape: reserved (gslot, qid, l_q)
    prefill: List[Tuple[int, int, int]] = field(default_factory=list)   # shape: prefilled now
    completed: List[Tuple[int, int]] = field(default_factory=list)  # (gslot, qid): last token just decoded


class Planner:
    def __init__(self, wl, world=1, policy="baton", pins=None):
        """policy "baton": relay race (remove on completion, insert at once);
        "rtc": the paper's run-to-completion Benchmark -- a finished query
        keeps its slot and keeps decoding (idle EOS tokens) until every query of
        the batch has finished; only an empty batch is refilled (NEXT-4);
        "shape": relay race WITHOUT P&D (vector shaping, NEXT-1) -- a
        new query takes its slot raw and is prefilled inside the batch in the
        next iteration (baton_shape_step), whose input width is the longest such
        prompt; its A decode iterations follow.  No control events.
        The paper's two comparison methods (NEXT-4), on the same kernels:
        "benchmark": the transformers batch-wise strategy -- run-to-completion, and
        the batch's prompts are prefilled together inside the batch, left-padded to
        the longest (a shaped iteration in which every row is new);
        "pd": P&D decoupling without the relay race -- run-to-completion decode
        batches of randomly combined (FCFS) queries whose prompts were prefilled
        separately in batches of similar length (the engine groups them).
        pins: {qid: rank} for fresh queries prefilled on a separate prefill rank and
        handed to that decode rank (NEXT-2, handoff.py): such a query may only take a
        slot of its rank (reading C20c, the fresh-query analogue of C20b)."""
        if policy not in ("baton", "rtc", "shape", "benchmark", "pd"):
            raise ValueError(policy)
        self.rtc = policy in ("rtc", "benchmark", "pd")       # run-to-completion batches
        self.raw_insert = policy in ("shape", "benchmark")     # prefilled inside the batch
        if self.raw_insert or self.rtc:
            c = wl.control
            if policy != "shape" and (c.preempt or c.preempt_frac or c.resize or wl.governor is not None
                                      or any(q.priority for q in wl.queries)):
                raise ValueError(f"{policy} policy: no control events / priorities / governor")
        if policy == "shape":
            c = wl.control
            if c.preempt or c.preempt_frac or c.resize:
                raise ValueError("shape policy: no control events")
            if wl.governor is not None or any(q.priority for q in wl.queries):
                # stored K/V re-enter by embedding, which the shaping path does not
                # have (the oracle Simulator asserts the same)
                raise ValueError("shape policy: no priorities / governor")
        self.pins = dict(pins or {})
        self.raw = {}                                         # shape: gslot -> prompt length
        self.policy = policy
        self.drained = set()                                  # rtc: finished but resident
        self.prio = {q.qid: q.priority for q in wl.queries}
        self.ticket = {}                                      # queue order within a priority
        self.wl = wl
        self.world = world
        if wl.slots % world:
            raise ValueError("slots must divide evenly across ranks")
        self.per_rank = wl.slots // world
        self.active = wl.initial_active() // world          # active slots per rank
        self.occupant = [-1] * wl.slots                      # gslot -> qid
        self.length = [0] * wl.slots                         # gslot -> live length
        self.meta = {q.qid: q for q in wl.queries}
        self.done_tokens = {q.qid: 0 for q in wl.queries}
        self.entered = {}                                    # qid -> iteration of last insert
        self.pending = sorted(wl.queries, key=lambda q: (q.arrival, q.qid))
        self.next_arrival = 0
        self.queue = deque()
        self.t = 0

    # ---------------------------------------------------------------- queries
    def rank_of(self, g):
        return g // self.per_rank

    def local(self, g):
        return g % self.per_rank

    def live(self):
        return [(g, q) for g, q in enumerate(self.occupant) if q >= 0]

    def finished_all(self):
        if self.wl.iterations >= 0 and self.t >= self.wl.iterations:
            return True
        return self.next_arrival >= len(self.pending) and not self.queue and not self.live()

    # ---------------------------------------------------------------- phase 1: decode
    def decode_plan(self):
        """Slots that decode this iteration and the position each one handles."""
        return [(g, q, self.length[g]) for g, q in self.live() if g not in self.raw]

    def prefill_plan(self):
        """shape policy: raw queries prefilled in this iteration's shaped step."""
        return [(g, self.occupant[g], n) for g, n in sorted(self.raw.items())]

    def idle_decodes(self, decode):
        """Decode entries of queries that already produced all their tokens (rtc)."""
        return sum(1 for g, q, pos in decode if pos >= self.meta[q].l_q + self.meta[q].A)

    def local_completion_flags(self, rank):
        """Per local slot: 1 if the query there produced its last token in the
        decode just executed (the engine all-gathers these)."""
        flags = []
        for b in range(self.per_rank):
            g = rank * self.per_rank + b
            q = self.occupant[g]
            flags.append(int(q >= 0 and g not in self.raw and self.done_tokens[q] + 1 >= self.meta[q].A))
        return flags

    def _victims(self, candidates, n):
        # C25 lowest priority first; C17 then most recently inserted, ties by higher qid
        order = sorted(candidates, key=lambda gq: (self.prio[gq[1]], -self.entered[gq[1]], -gq[1]))
        return order[:n]

    def _usage(self, r):
        """Live tokens on rank r (C26)."""
        base = r * self.per_rank
        return sum(self.length[base + b] for b in range(self.per_rank) if self.occupant[base + b] >= 0)

    def _admissible(self, r, length):
        gov = self.wl.governor
        return gov is None or self._usage(r) + length <= gov[1] * self.active * self.wl.max_ctx

    def _requeue(self, entries):
        for i, e in enumerate(entries):
            self.ticket[e.qid] = -(self.t * 100000) + i
            self.queue.append(e)

    def _order(self):
        return sorted(range(len(self.queue)),
                      key=lambda i: (-self.prio[self.queue[i].qid], self.ticket[self.queue[i].qid]))

    def _free(self):
        return [r * self.per_rank + b for r in range(self.world) for b in range(self.active)
                if self.occupant[r * self.per_rank + b] < 0]

    # ---------------------------------------------------------------- one iteration
    def plan(self, all_flags=None):
        """Decide iteration t.  ``all_flags``: concatenated completion flags of
        every rank (from the all-gather) -- used instead of local bookkeeping
        so the decision depends on what the ranks reported."""
        d = Decisions(self.t)
        if self.t > 0:
            d.decode = self.decode_plan()
            for g, q, _ in d.decode:
                self.done_tokens[q] += 1
                self.length[g] += 1
            d.prefill = self.prefill_plan()
            for g, _, n in d.prefill:          # the prompt is now cached (C9: first token)
                self.length[g] = n
            self.raw.clear()
            for g, q in self.live():
                done = (all_flags[g] != 0) if all_flags is not None else (
                    self.done_tokens[q] >= self.meta[q].A)
                if done:
                    d.finished.append((g, q))
            d.completed = [(g, q) for g, q in d.finished if q not in self.drained]
            if self.rtc:
                self.drained.update(q for _, q in d.finished)
                if any(q not in self.drained for _, q in self.live()):
                    d.finished = []                           # the batch runs on
                else:
                    d.finished = list(self.live())
                    self.drained.clear()
            for g, _ in d.finished:
                self.occupant[g] = -1
                self.length[g] = 0
            stored = []
            ctl = self.wl.control
            n_pre = 0
            if self.t in ctl.preempt:
                n_pre = ctl.preempt[self.t]
            elif self.t in ctl.preempt_frac:
                n_pre = int(ctl.preempt_frac[self.t] * len(self.live()))
            n_pre = min(n_pre, len(self.live()))
            if n_pre > 0:
                for g, q in self._victims(self.live(), n_pre):
                    stored.append(self._store(g, q, d))
            if self.t in ctl.resize:
                stored += self._resize(ctl.resize[self.t], d)
            d.n_pre_compact = len(d.victims)
            gov = self.wl.governor
            if gov is not None:                               # C26
                for r in range(self.world):
                    while self._usage(r) > gov[0] * self.active * self.wl.max_ctx:
                        base = r * self.per_rank
                        occ = [(base + b, self.occupant[base + b]) for b in range(self.per_rank)
                               if self.occupant[base + b] >= 0]
                        if not occ:
                            break
                        g, q = self._victims(occ, 1)[0]
                        stored.append(self._store(g, q, d))
            self._requeue(stored)
        self._admit()
        self._fill(d)
        self.t += 1
        return d

    def _store(self, g, q, d):
        d.victims.append((g, q, self.length[g]))
        e = QueueEntry(q, self.length[g], self.rank_of(g))
        self.occupant[g] = -1
        self.length[g] = 0
        return e

    def _resize(self, ev, d):
        if ev == "halve":
            new = max(1, self.active // 2)
        elif ev == "double":
            new = min(self.per_rank, self.active * 2)
        else:
            new = max(1, min(self.per_rank, int(ev) // self.world))
        out = []
        if new < self.active:
            for r in range(self.world):
                base = r * self.per_rank
                occ = [(base + b, self.occupant[base + b]) for b in range(self.per_rank)
                       if self.occupant[base + b] >= 0]
                over = sum(1 for g, _ in occ if g - base >= new)
                room = sum(1 for b in range(new) if self.occupant[base + b] < 0)
                if over > room:
                    for g, q in self._victims(occ, over - room):
                        out.append(self._store(g, q, d))
                # stable compaction into the lowest free slots (mirrors baton_compact)
                for b in range(new, self.per_rank):
                    g = base + b
                    if self.occupant[g] < 0:
                        continue
                    f = next(base + x for x in range(new) if self.occupant[base + x] < 0)
                    self.occupant[f], self.length[f] = self.occupant[g], self.length[g]
                    self.occupant[g], self.length[g] = -1, 0
        self.active = new
        d.resize = new
        return out

    def _admit(self):
        while (self.next_arrival < len(self.pending)
               and self.pending[self.next_arrival].arrival <= self.t):
            q = self.pending[self.next_arrival]
            self.ticket[q.qid] = len(self.ticket) + 1
            self.queue.append(QueueEntry(q.qid, q.l_q, None, self.pins.get(q.qid)))
            self.next_arrival += 1

    def _priority_preempt(self, d):
        """C25, before any insert: the best waiting query, if it has no
        eligible admissible free slot, stores the lowest-priority live query of an
        eligible rank whose priority is lower than its own."""
        if not self.queue:
            return
        e0 = self.queue[self._order()[0]]
        if any((e0.rank() is None or self.rank_of(g) == e0.rank()) and self._admissible(self.rank_of(g), e0.length)
               for g in self._free()):
            return
        live = [(g, q) for g, q in self.live()
                if (e0.rank() is None or self.rank_of(g) == e0.rank()) and self.local(g) < self.active
                and self.prio[q] < self.prio[e0.qid]]
        if not live:
            return
        g, q = self._victims(live, 1)[0]
        self._requeue([self._store(g, q, d)])

    def _fill(self, d):
        if self.rtc and self.live():
            return                                            # batch still running
        if self.t > 0 and self.policy == "baton":
            self._priority_preempt(d)
        while self.queue:
            free = self._free()
            if not free:
                return
            chosen = None
            for idx in self._order():
                e = self.queue[idx]
                for g in free:
                    if (e.rank() is None or self.rank_of(g) == e.rank()) and self._admissible(self.rank_of(g), e.length):
                        chosen = (idx, g)
                        break
                if chosen:
                    break
            if chosen is None:
                return
            idx, g = chosen
            e = self.queue[idx]
            del self.queue[idx]
            self.occupant[g] = e.qid
            self.entered[e.qid] = self.t
            if self.raw_insert:                               # raw: prefilled next iteration
                self.length[g] = 0
                self.raw[g] = e.length
                d.raw.append((g, e.qid, e.length))
                continue
            self.length[g] = e.length
            d.inserts.append((g, e.qid, e.length, e.home))


def local_splice_ops(pl, d, rank):
    """The splice calls rank ``rank`` makes for the decisions ``d`` of planner
    ``pl``, in execution order (local slot indices):

        ("remove", [b...])            finished rows (+ release; C5) -- every t > 0
        ("extract", b, qid)           store a victim's K/V
        ("remove", [b...])            the victims' rows (+ release)
        ("compact", n_active)         batch shrink/grow (C19)
        ("extract", b, qid) ... ("remove", [...])   victims chosen after the resize
        ("insert", [(b, qid, len, home)...])        one batched embed (C7)

    Victims chosen before the compaction (C17 preemption, resize overflow) carry
    pre-compaction slot indices and are stored before ``compact``; the governor's
    (C26) and the priority preemption's (C25) are chosen on the compacted batch
    and are stored after it.  Pure host logic (unit-tested on a host mirror)."""
    ops = []
    if d.t > 0:
        ops.append(("remove", [pl.local(g) for g, _ in d.finished if pl.rank_of(g) == rank]))

    def store(vs):
        loc = [(pl.local(g), q) for g, q, _ in vs if pl.rank_of(g) == rank]
        if loc:
            ops.extend(("extract", b, q) for b, q in loc)
            ops.append(("remove", [b for b, _ in loc]))

    store(d.victims[:d.n_pre_compact])
    if d.resize is not None:
        ops.append(("compact", d.resize))
    store(d.victims[d.n_pre_compact:])
    ins = [(pl.local(g), q, n, home) for g, q, n, home in d.inserts if pl.rank_of(g) == rank]
    if ins:
        ops.append(("insert", ins))
    return ops
