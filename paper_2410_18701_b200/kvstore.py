"""Store for the K/V of stored (preempted / scaled-out) queries: the "prefetchable
GPU&CPU hybrid KV-Cache" of P:L335 (§Overview, Solution 2).

P:L144: a preempted query's "Keys and Values ... are temporarily stored, and it
will be promptly re-inserted"; under memory pressure stored queries are
"moved to the host memory".  The store keeps a stored query's K/V

* in HBM while the stash's HBM budget lasts (``baton_extract`` into device
  buffers: an HBM->HBM copy);
* otherwise in pinned host memory (``baton_extract`` writes it straight over
  PCIe from the copy kernel).

Host-resident entries are PREFETCHED back into HBM on a copy stream ahead of
their re-insert: every iteration the engine passes the planner's service order
of the waiting queue, and host entries among its first ``lookahead`` stored
queries start an async H2D copy into staging buffers while the staging budget
allows.  The re-insert then reads HBM
(``baton_insert`` after waiting on that copy's event only); an entry not (yet)
prefetched is inserted from host memory directly, as before.  Placement never
changes a byte: the re-inserted rows are the extracted rows (tested bit-exact).

Every device byte is moved by libbaton's copy kernel (extract / insert) or by the
copy engine (the prefetch H2D, a plain DMA: the same bytes, no arithmetic).
"""
from dataclasses import dataclass
from typing import Dict, List, Optional

import torch


@dataclass
class Entry:
    qid: int
    rows: int
    nbytes: int
    K: torch.Tensor
    V: torch.Tensor
    where: str                              # "hbm" | "host" | "prefetching"
    ready: Optional[torch.cuda.Event] = None  # prefetch done (where == "prefetching")
    host: Optional[tuple] = None            # the host copy while prefetching


class HybridKVStore:
    def __init__(self, shard, device, hbm_budget=None, host=True, prefetch=True, lookahead=8,
                 staging_budget=4 << 30):
        """hbm_budget: bytes of stored K/V kept in HBM (None = unlimited, i.e. the
        plain HBM stash; 0 with host=True = every store spills to the host).
        staging_budget: HBM for prefetched host entries in flight to their re-insert
        (separate from hbm_budget: a spilled query may be larger than the whole stash
        budget, and the re-insert needs its bytes in HBM anyway)."""
        self.shard = shard
        self.device = device
        self.hbm_budget = hbm_budget
        self.host = host
        self.prefetch_on = prefetch and host
        self.lookahead = lookahead
        self.entries: Dict[int, Entry] = {}
        self.hbm_used = 0
        self.staging_budget = staging_budget
        self.staging_used = 0
        self.stored_bytes = self.peak_stored_bytes = 0       # all placements
        self.copy_stream = torch.cuda.Stream(device=device) if self.prefetch_on else None
        self._inflight: List[tuple] = []     # (event, tensors) kept alive until read
        self._keep: List[tuple] = []         # host K/V taken for the coming insert
        self.timing = None                   # list: (start, end event, bytes) per prefetch
        # counters (bytes / calls) for the measurement
        self.stats = {"stored_hbm": 0, "stored_host": 0, "prefetched": 0,
                      "inserted_from_hbm": 0, "inserted_from_host": 0, "prefetch_bytes": 0,
                      "spill_bytes": 0, "host_insert_bytes": 0}

    def _fits(self, nbytes):
        return self.hbm_budget is None or self.hbm_used + nbytes <= self.hbm_budget

    def __contains__(self, qid):
        return qid in self.entries

    def __len__(self):
        return len(self.entries)

    def store(self, slot, qid):
        """baton_extract of local slot `slot` (query `qid`) into HBM or the host."""
        sh = self.shard
        n = int(sh.baton_query()["lens"][slot])
        shape = (sh.L, sh.Hkv, n, sh.D)
        nbytes = 2 * sh.L * sh.Hkv * n * sh.D * 2
        if not self.host or self._fits(nbytes):
            K, V = sh.baton_extract(slot)
            self.hbm_used += nbytes
            e = Entry(qid, n, nbytes, K, V, "hbm")
            self.stats["stored_hbm"] += 1
        else:
            ko = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
            vo = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
            sh.baton_extract(slot, ko, vo)
            e = Entry(qid, n, nbytes, ko, vo, "host")
            self.stats["stored_host"] += 1
            self.stats["spill_bytes"] += nbytes
        self.entries[qid] = e
        self._account(nbytes)
        return n

    def _account(self, nbytes):
        self.stored_bytes += nbytes
        self.peak_stored_bytes = max(self.peak_stored_bytes, self.stored_bytes)

    def prefetch(self, order):
        """Start H2D copies of host entries among the next `lookahead` stored
        queries in the queue's service order `order` (qids), while they fit."""
        if not self.prefetch_on:
            return
        cur = torch.cuda.current_stream(self.device)
        seen = 0
        for qid in order:
            e = self.entries.get(qid)
            if e is None:
                continue
            seen += 1
            if seen > self.lookahead:
                break
            if e.where != "host" or self.staging_used + e.nbytes > self.staging_budget:
                continue
            # allocated on the decode stream (its caching-allocator pool); the copy
            # stream waits for everything enqueued there so far -- the extract that
            # wrote the host copy and the last use of the reused device blocks
            Kd = torch.empty(e.K.shape, dtype=torch.bfloat16, device=self.device)
            Vd = torch.empty_like(Kd)
            gate = torch.cuda.Event()
            gate.record(cur)
            self.copy_stream.wait_event(gate)
            with torch.cuda.stream(self.copy_stream):
                t0 = None
                if self.timing is not None:
                    t0 = torch.cuda.Event(enable_timing=True)
                    t0.record(self.copy_stream)
                Kd.copy_(e.K, non_blocking=True)
                Vd.copy_(e.V, non_blocking=True)
                ev = torch.cuda.Event(enable_timing=t0 is not None)
                ev.record(self.copy_stream)
                if t0 is not None:
                    self.timing.append((t0, ev, e.nbytes))
            e.host = (e.K, e.V)
            e.K, e.V, e.where, e.ready = Kd, Vd, "prefetching", ev
            self.staging_used += e.nbytes
            self.stats["prefetched"] += 1
            self.stats["prefetch_bytes"] += e.nbytes

    def take(self, qid):
        """The stored K/V of `qid` for its re-insert on the current stream."""
        e = self.entries.pop(qid)
        self.stored_bytes -= e.nbytes
        cur = torch.cuda.current_stream(self.device)
        if e.where == "host":
            self.stats["inserted_from_host"] += 1
            self.stats["host_insert_bytes"] += e.nbytes
            # the insert kernel reads the pinned pages over PCIe: kept alive (and out
            # of the host caching allocator) until it has run (after_insert)
            self._keep.append((e.K, e.V))
            return e.K, e.V
        if e.where == "prefetching":
            cur.wait_event(e.ready)
            self._inflight.append((e.ready, e.host))
            self.staging_used -= e.nbytes
        else:
            self.hbm_used -= e.nbytes
        self.stats["inserted_from_hbm"] += 1
        return e.K, e.V

    def put(self, qid, K, V):
        """A stored query's K/V already in HBM (e.g. a warm start's stash)."""
        nbytes = K.numel() * 2 + V.numel() * 2
        self.entries[qid] = Entry(qid, K.shape[2], nbytes, K, V, "hbm")
        self.hbm_used += nbytes
        self._account(nbytes)

    def after_insert(self):
        """Call after the insert launch that consumed this iteration's take()s."""
        if self._keep:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self._inflight.append((ev, tuple(self._keep)))
            self._keep = []
        self._purge()

    def _purge(self):
        self._inflight = [(ev, t) for ev, t in self._inflight if not ev.query()]
