"""Decode-loop engine: executes the planner's decisions on one GPU's shard.

One process per GPU.  Per iteration (reading of P:L101 / P:L124):

    [t > 0]  tokens for the decoding slots (harness: keyed generator, or a
             pre-generated HBM buffer in the benchmark)
             baton_mask_update                       (a1)
             for every layer: baton_decode_layer     (a2 append + a3 attention)
             completion flags -> all_gather over NCCL (the only collective)
             baton_remove(finished)  (+ release)     (a4)
             baton_extract + baton_remove(victims)   (a6)
             baton_compact                            (a7)
    baton_insert_many(new queries)                   (a5)

Every device byte is produced by libbaton kernels (plus the harness keygen).
"""
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from .baton import (BatonShard, baton_keygen_tokens, baton_keygen_history, baton_prefill_attention,
                    baton_prefill_attention_varlen)
from .comm import gather_completion_flags
from .kvstore import HybridKVStore
from .scheduler import Planner, local_splice_ops

KIND_Q, KIND_K, KIND_V = 0, 1, 2
PREFILL_BATCH_MEAN = 256      # batched (varlen) P&D prefill when prompts average <= this many tokens


@dataclass
class StepStats:
    t: int
    decoded: int = 0
    idle: int = 0               # decodes of already-finished queries (run-to-completion baseline)
    inserted: int = 0
    removed: int = 0
    stored: int = 0
    released: int = 0
    live_rows: int = 0          # sum of lens over decoding slots (keys read per layer per head group)
    insert_rows: int = 0        # prefilled rows embedded
    extract_rows: int = 0
    compact_rows: int = 0
    width: int = 1              # shape policy: input width of the iteration
    prefill_rows: int = 0       # shape policy: prompt tokens prefilled in the batch
    bubble_rows: int = 0        # shape policy: padding input tokens computed
    S: int = 0                  # shared logical length after the iteration (host mirror)
    completed: int = 0          # queries whose last token was decoded in this iteration
    live_slots: int = 0         # occupied slots after the iteration
    kv_live_rows: int = 0       # sum of lens over occupied slots after the iteration


class Engine:
    def __init__(self, wl, rank=0, world=1, device=None, group=None, keep_outputs=False,
                 keep_layers=None, token_source=None, prefill_source=None, use_graph=True,
                 stash_host=False, policy="baton", prefill_attention=False, async_prefill=False,
                 prefill_lookahead=None, prefill_grouping=None, trace=False,
                 stash_hbm_bytes=None, pins=None, device_flags=None):
        """prefill_grouping: "length" -- a8 of several fresh prompts runs in batches of
        similar length, one varlen launch each (the PD method's prefill, P:L220;
        default for policy "pd"); None -- batched only when the prompts are short.
        trace: record a CUDA event after every iteration (per-iteration device time
        for the JSONL log, ``write_log``).
        device_flags (default: on when world > 1): each rank's completion flags are
        computed on the device from the live lengths after the decode (lens >= the
        slot's target length l_q + A, the stand-in for the model's EOS) and all-gathered
        from there; the replicated planner then decides on what the ranks' devices
        reported.  Off: the planner's own bookkeeping (identical decisions, no exchange
        needed on one GPU)."""
        self.wl = wl
        self.rank = rank
        self.world = world
        self.group = group
        self.device = torch.device(device or "cuda")
        self.planner = Planner(wl, world, policy=policy, pins=pins)
        self.B = self.planner.per_rank
        # libbaton requires max_ctx % 16 == 0 (16-B aligned mask rows for the bulk
        # copies); a larger capacity changes no result (C24 caps l_q + A anyway)
        cap = (wl.max_ctx + 15) // 16 * 16
        self.shard = BatonShard(wl.layers, self.B, wl.q_heads, wl.kv_heads, wl.head_dim,
                                cap, device=self.device)
        L, B, D = wl.layers, self.B, wl.head_dim
        self.q = torch.zeros((L, B, wl.q_heads, D), dtype=torch.bfloat16, device=self.device)
        self.k_new = torch.zeros((L, B, wl.kv_heads, D), dtype=torch.bfloat16, device=self.device)
        self.v_new = torch.zeros_like(self.k_new)
        self.out = torch.zeros((L, B, wl.q_heads, D), dtype=torch.bfloat16, device=self.device)
        self.d_qid = torch.full((B,), -1, dtype=torch.int32, device=self.device)
        self.d_pos = torch.zeros((B,), dtype=torch.int32, device=self.device)
        self.keep_outputs = keep_outputs
        self.keep_layers = keep_layers
        self.outputs: Dict[Tuple[int, int], np.ndarray] = {}
        self.token_source = token_source
        self.prefill_source = prefill_source
        self.shape_source = None          # shape policy: (t, dec, pre, W) -> q, k, v
        # P&D accounting: run a8 (baton_prefill_attention, every layer) on each fresh
        # insert, so a policy comparison charges the decoupled prefill its attention
        self.prefill_attention = prefill_attention
        # asynchronous P&D: queued fresh queries are prefilled on a side
        # stream ahead of their insert (keyed K/V + a8 when prefill_attention);
        # the insert waits on that query's event only
        self.async_prefill = async_prefill
        self.prefill_stream = torch.cuda.Stream(device=self.device) if async_prefill else None
        self.prefill_lookahead = prefill_lookahead or 2 * self.B
        self.prefetched: Dict[int, Tuple[torch.Tensor, torch.Tensor, torch.cuda.Event]] = {}
        self.gather_s, self.gathers = 0.0, 0   # completion-flag all-gathers (world > 1)
        self.use_graph = use_graph
        self.staging = {(self.q.data_ptr(), self.k_new.data_ptr(), self.v_new.data_ptr())}
        # P:L147 "moved to the host memory": stored K/V in pinned host memory (the
        # extract/insert copy kernels read/write it over PCIe), else an HBM stash
        # P:L144/P:L147/P:L335: stored K/V in HBM (stash_host=False), in pinned host
        # memory (True: extract/insert copy kernels write/read it over PCIe), or the
        # prefetchable hybrid ("hybrid": HBM up to stash_hbm_bytes, then host; host
        # entries near the queue head prefetched back to HBM ahead of re-insert)
        self.stash_host = stash_host
        hybrid = stash_host == "hybrid"
        self.stash = HybridKVStore(self.shard, self.device,
                                   hbm_budget=stash_hbm_bytes if hybrid else (0 if stash_host else None),
                                   host=bool(stash_host), prefetch=hybrid)
        self.last_decisions = None
        self.prefill_grouping = prefill_grouping or ("length" if policy == "pd" else None)
        self.trace = trace
        self.trace_events = []
        self.device_flags = (world > 1) if device_flags is None else device_flags
        self.d_target = torch.zeros((self.B,), dtype=torch.int32, device=self.device)
        self._target_host = [0] * self.B

    def register_staging(self, q, k, v):
        """Declare a fixed (q, k_new, v_new) buffer set a token source may return
        (e.g. double-buffered H2D staging): decoded in place, no copy."""
        self.staging.add((q.data_ptr(), k.data_ptr(), v.data_ptr()))

    # ---------------------------------------------------------------- inputs (harness)
    def _gen_tokens(self, dec_local):
        wl = self.wl
        qid = np.full(self.B, -1, np.int32)
        pos = np.zeros(self.B, np.int32)
        for b, q, p in dec_local:
            qid[b], pos[b] = q, p
        self.d_qid.copy_(torch.from_numpy(qid))
        self.d_pos.copy_(torch.from_numpy(pos))
        L, B, D = wl.layers, self.B, wl.head_dim
        baton_keygen_tokens(self.q, self.d_qid, self.d_pos, L, B, wl.q_heads, D, KIND_Q, 0,
                            wl.seed, wl.scales[0])
        baton_keygen_tokens(self.k_new, self.d_qid, self.d_pos, L, B, wl.kv_heads, D, KIND_K, 0,
                            wl.seed, wl.scales[1])
        baton_keygen_tokens(self.v_new, self.d_qid, self.d_pos, L, B, wl.kv_heads, D, KIND_V, 0,
                            wl.seed, wl.scales[2])
        return self.q, self.k_new, self.v_new

    def _prefill(self, qid, length):
        if self.prefill_source is not None:
            return self.prefill_source(qid, length)
        wl = self.wl
        shape = (wl.layers, wl.kv_heads, length, wl.head_dim)
        K = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
        V = torch.empty_like(K)
        baton_keygen_history(K, wl.layers, wl.kv_heads, wl.head_dim, qid, 0, length, KIND_K,
                             wl.seed, wl.scales[1])
        baton_keygen_history(V, wl.layers, wl.kv_heads, wl.head_dim, qid, 0, length, KIND_V,
                             wl.seed, wl.scales[2])
        return K, V

    def _prefill_attn(self, qid, n, K, V):
        prefill_attention_one(self.wl, self.device, qid, n, K, V)

    def _batchable(self, items):
        return batchable(items, self.prefill_grouping)

    def _prefill_attn_batch(self, items):
        prefill_attention_batch(self.wl, self.device, items, self.prefill_grouping)

    # ---------------------------------------------------------------- one iteration
    def done(self):
        return self.planner.finished_all()

    def _shape_tokens(self, dec, pre, W):
        """Keyed q/k/v of a shaped iteration, token-major [L][B][W][H][D]: input
        position 0 of a decoding slot is its token, positions t < l of a prefilled
        slot its prompt tokens, everything else a (zero) padding token.  One keygen
        launch per tensor over all B*W input tokens."""
        wl = self.wl
        L, B, D = wl.layers, self.B, wl.head_dim
        qid = np.full((B, W), -1, np.int32)
        pos = np.zeros((B, W), np.int32)
        for b, q, p in dec:
            qid[b, 0], pos[b, 0] = q, p
        for b, q, n in pre:
            qid[b, :n] = q
            pos[b, :n] = np.arange(n)
        d_qid = torch.from_numpy(qid.reshape(-1)).to(self.device)
        d_pos = torch.from_numpy(pos.reshape(-1)).to(self.device)
        out = []
        for kind, H, sc in ((KIND_Q, wl.q_heads, wl.scales[0]), (KIND_K, wl.kv_heads, wl.scales[1]),
                            (KIND_V, wl.kv_heads, wl.scales[2])):
            t = torch.empty((L, B, W, H, D), dtype=torch.bfloat16, device=self.device)
            baton_keygen_tokens(t, d_qid, d_pos, L, B * W, H, D, kind, 0, wl.seed, sc)
            out.append(t)
        return out

    def _shape_decode(self, stats, dec, pre):
        """one shaped iteration (survivors decode, raw queries prefill)."""
        wl = self.wl
        W = max(n for _, _, n in pre)
        if self.shape_source is not None:
            q, k, v = self.shape_source(self.planner.t, dec, pre, W)
        else:
            q, k, v = self._shape_tokens(dec, pre, W)
        out = torch.empty((wl.layers, self.B, W, wl.q_heads, wl.head_dim), dtype=torch.bfloat16,
                          device=self.device)
        self.shard.baton_shape_step(W, [b for b, _, _ in pre], [n for _, _, n in pre], q, k, v, out)
        stats.width = W
        stats.prefill_rows = sum(n for _, _, n in pre)
        stats.bubble_rows = (len(dec) + len(pre)) * W - len(dec) - stats.prefill_rows
        if self.keep_outputs:
            layers = self.keep_layers if self.keep_layers is not None else range(wl.layers)
            o = out[list(layers)].float().cpu().numpy()
            for b, qq, p in dec:
                self.outputs[(qq, p)] = o[:, b, 0].copy()
            for b, qq, n in pre:
                for t in range(n):
                    self.outputs[(qq, t)] = o[:, b, t].copy()
        return dec

    def decode(self, stats):
        with torch.cuda.nvtx.range("baton.decode"):
            return self._decode(stats)

    def _decode(self, stats):
        """a1 + per layer a2/a3 for the slots the planner says are live."""
        pl = self.planner
        dec = [(pl.local(g), q, p) for g, q, p in pl.decode_plan() if pl.rank_of(g) == self.rank]
        stats.decoded = len(dec)
        pre = [(pl.local(g), q, n) for g, q, n in pl.prefill_plan() if pl.rank_of(g) == self.rank]
        if pre:
            stats.live_rows = sum(p + 1 for _, _, p in dec)
            return self._shape_decode(stats, dec, pre)
        stats.idle = sum(1 for b, q, p in dec if p >= pl.meta[q].l_q + pl.meta[q].A)
        stats.live_rows = sum(p + 1 for _, _, p in dec)
        if self.token_source is not None:
            q, k, v = self.token_source(pl.t, dec)
        else:
            q, k, v = self._gen_tokens(dec)
        sh = self.shard
        if self.use_graph:
            # one graph replay: mask update + every layer's fused append/attention.
            # Registered staging sets are used in place (libbaton keeps a graph per
            # pointer set); anything else is copied into the engine's own staging.
            ptrs = (q.data_ptr(), k.data_ptr(), v.data_ptr())
            if ptrs not in self.staging:
                for src, dst in ((q, self.q), (k, self.k_new), (v, self.v_new)):
                    if src.data_ptr() != dst.data_ptr():
                        dst.copy_(src, non_blocking=True)
                q, k, v = self.q, self.k_new, self.v_new
            sh.baton_decode_step(q, k, v, self.out)
        else:
            sh.baton_mask_update()
            for l in range(self.wl.layers):
                sh.baton_decode_layer(l, q[l], self.out[l], k[l], v[l])
        if self.keep_outputs and dec:
            layers = self.keep_layers if self.keep_layers is not None else range(self.wl.layers)
            o = self.out[list(layers)].float().cpu().numpy()
            for b, qq, p in dec:
                self.outputs[(qq, p)] = o[:, b].copy()
        return dec

    def _gather_flags(self, local_flags):
        if self.world == 1:
            return gather_completion_flags(local_flags, self.world, self.group, self.device)
        t0 = time.perf_counter()
        out = gather_completion_flags(local_flags, self.world, self.group, self.device)
        self.gather_s += time.perf_counter() - t0   # host-blocking: the collective + its D2H
        self.gathers += 1
        return out

    def _device_flags(self):
        """This rank's completion flags on the device, after the decode: the slot's live
        length reached its target (l_q + A)."""
        return ((self.shard.d_lens >= self.d_target) & (self.d_target > 0)).to(torch.int32)

    def _sync_targets(self):
        """The device copy of each local slot's target length, after the splice."""
        pl = self.planner
        tgt = [0] * self.B
        for g, q in pl.live():
            if pl.rank_of(g) == self.rank and g not in pl.raw:
                tgt[pl.local(g)] = pl.meta[q].l_q + pl.meta[q].A
        if tgt != self._target_host:
            self._target_host = tgt
            self.d_target.copy_(torch.tensor(tgt, dtype=torch.int32), non_blocking=True)

    def iteration(self):
        pl = self.planner
        stats = StepStats(pl.t)
        flags = None
        if pl.t > 0:
            self.decode(stats)
            # completion flags of every rank
            if self.world > 1:
                local = self._device_flags() if self.device_flags else pl.local_completion_flags(self.rank)
                with torch.cuda.nvtx.range("baton.allgather"):
                    flags = self._gather_flags(local)
        d = pl.plan(flags)
        self.last_decisions = d
        stats.completed = sum(1 for g, _ in d.completed if pl.rank_of(g) == self.rank)
        with torch.cuda.nvtx.range("baton.splice"):
            self._splice(d, stats)
        if self.device_flags:
            self._sync_targets()
        if self.async_prefill:
            self._prefetch()
        stats.S = self.shard.S
        mine = [(g, q) for g, q in pl.live() if pl.rank_of(g) == self.rank]
        stats.live_slots = len(mine)
        stats.kv_live_rows = sum(pl.length[g] for g, _ in mine)
        if self.trace:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.trace_events.append(ev)
        return stats

    def _splice(self, d, stats):
        pl = self.planner
        sh = self.shard
        ops = local_splice_ops(pl, d, self.rank)
        ins = []
        for i, op in enumerate(ops):
            kind = op[0]
            if kind == "remove":
                # removal + release every iteration (C5); a no-op call enqueues nothing.
                # ops[0] (t > 0) removes the finished rows, later removes free victims
                stats.released += sh.baton_remove(op[1])
                if i == 0:
                    stats.removed = len(op[1])
                else:
                    stats.stored += len(op[1])
            elif kind == "extract":
                _, b, q = op
                stats.extract_rows += self.stash.store(b, q)     # the library's live length
            elif kind == "compact":
                before = sh.baton_query()
                o2n = sh.baton_compact(op[1])
                stats.compact_rows = int(sum(before["lens"][b] for b in range(self.B) if o2n[b] != b))
            else:
                ins = op[1]
        if ins:
            slots, ks, vs, lens = [], [], [], []
            fresh = []                          # synchronous P&D: one batched a8 below
            for b, q, n, home in ins:
                if home is not None:
                    K, V = self.stash.take(q)
                elif q in self.prefetched:
                    K, V, ev = self.prefetched.pop(q)
                    torch.cuda.current_stream(self.device).wait_event(ev)
                    # allocated on the prefill stream, read on this one
                    K.record_stream(torch.cuda.current_stream(self.device))
                    V.record_stream(torch.cuda.current_stream(self.device))
                else:
                    K, V = self._prefill(q, n)
                    if self.prefill_attention:
                        fresh.append((q, n, K, V))
                slots.append(b)
                ks.append(K)
                vs.append(V)
                lens.append(n)
            if fresh:
                self._prefill_attn_batch(fresh)
            sh.baton_insert_many(slots, ks, vs, lens)
            self.stash.after_insert()
            stats.inserted = len(ins)
            stats.insert_rows = sum(lens)
        if len(self.stash):
            # hybrid store: start the H2D of host-resident stored queries that come
            # up next in the queue's service order (this rank's only, C20b)
            self.stash.prefetch([pl.queue[i].qid for i in pl._order()
                                 if pl.queue[i].home == self.rank])

    def _prefetch(self):
        """Launch the prefill of the next queued fresh queries on the side stream."""
        pl = self.planner
        todo = []
        for e in list(pl.queue)[:self.prefill_lookahead]:
            if e.home is None and e.qid not in self.prefetched:
                todo.append(e)
        if not todo:
            return
        with torch.cuda.stream(self.prefill_stream):
            kv = [(e.qid, e.length) + self._prefill(e.qid, e.length) for e in todo]
            if self.prefill_attention and self._batchable(kv):
                self._prefill_attn_batch(kv)     # one event: short prompts finish together
                ev = torch.cuda.Event()
                ev.record(self.prefill_stream)
                for qid, _, K, V in kv:
                    self.prefetched[qid] = (K, V, ev)
                return
            for qid, n, K, V in kv:              # an insert waits for its own query only
                if self.prefill_attention:
                    self._prefill_attn(qid, n, K, V)
                ev = torch.cuda.Event()
                ev.record(self.prefill_stream)
                self.prefetched[qid] = (K, V, ev)

    def run(self, max_iters=None):
        all_stats = []
        if self.trace:
            self.trace_start = torch.cuda.Event(enable_timing=True)
            self.trace_start.record()
            self.trace_events = []
        while not self.done():
            all_stats.append(self.iteration())
            if max_iters is not None and len(all_stats) >= max_iters:
                break
        return all_stats

    def log_records(self, stats):
        """Per-iteration records (SURVEY.md §5 metrics log; the Fig. 6-8 traces of
        P:L299-309): live slots, S, sum of live lengths, K/V bytes moved by the
        splice, decoded / idle / completed counts and, when traced, the device time
        at the end of the iteration.  Synchronises when traced."""
        wl = self.wl
        tau_l = 2 * wl.kv_heads * wl.head_dim * 2 * wl.layers      # K+V bytes per token, all layers
        t_ms = None
        if self.trace and self.trace_events:
            torch.cuda.synchronize(self.device)
            t_ms = [self.trace_start.elapsed_time(e) for e in self.trace_events[-len(stats):]]
        recs = []
        for i, s in enumerate(stats):
            r = {"t": s.t, "decoded": s.decoded, "idle": s.idle, "completed": s.completed,
                 "inserted": s.inserted, "removed": s.removed, "stored": s.stored,
                 "live_slots": s.live_slots, "S": s.S, "kv_live_rows": s.kv_live_rows,
                 "kv_live_bytes": s.kv_live_rows * tau_l,
                 "kv_dense_bytes": self.B * s.S * tau_l,   # the paper's dense [B][S] tensors
                 "live_rows_read": s.live_rows,
                 "splice_bytes": 2 * (s.insert_rows + s.extract_rows + s.compact_rows) * tau_l,
                 "width": s.width, "prefill_rows": s.prefill_rows, "bubble_rows": s.bubble_rows}
            if t_ms is not None:
                r["t_ms"] = t_ms[i]
            recs.append(r)
        return recs

    def write_log(self, path, stats):
        """The per-iteration records as JSON lines."""
        import json
        with open(path, "w") as f:
            for r in self.log_records(stats):
                f.write(json.dumps(r) + "\n")


def prefill_groups(items, by_length=False, ratio=1.25, max_prompts=64, max_tiles=1024):
    """Split fresh prompts (qid, n, ...) into varlen prefill launches (at most 64
    prompts and 1024 query tiles each).  by_length: the PD method's grouping
    ("queries with similar sequence lengths will be grouped into a batch";
    P:L335 "the similarity of length principle") -- sorted by length, a new group
    whenever a prompt exceeds the group's shortest by more than `ratio`."""
    order = sorted(items, key=lambda it: it[1]) if by_length else list(items)
    groups, cur, tiles = [], [], 0
    for it in order:
        t = -(-it[1] // 128)
        if cur and (len(cur) == max_prompts or tiles + t > max_tiles
                    or (by_length and it[1] > ratio * cur[0][1])):
            groups.append(cur)
            cur, tiles = [], 0
        cur.append(it)
        tiles += t
    if cur:
        groups.append(cur)
    return groups


def prefill_attention_one(wl, device, qid, n, K, V):
    """a8 over every layer of a fresh query's prompt (output discarded): q from the
    keyed generator (the model's projection stand-in), K/V the query's prefilled K/V."""
    Q = torch.empty((wl.layers, wl.q_heads, n, wl.head_dim), dtype=torch.bfloat16, device=device)
    baton_keygen_history(Q, wl.layers, wl.q_heads, wl.head_dim, qid, 0, n, KIND_Q, wl.seed,
                         wl.scales[0])
    O = torch.empty_like(Q)
    for l in range(wl.layers):
        baton_prefill_attention(Q[l], K[l], V[l], O[l], n, wl.q_heads, wl.kv_heads, wl.head_dim)


def batchable(items, grouping=None):
    if grouping == "length":
        return len(items) > 1
    return len(items) > 1 and sum(it[1] for it in items) <= PREFILL_BATCH_MEAN * len(items)


def prefill_attention_batch(wl, device, items, grouping=None):
    """a8 for several fresh queries (qid, n, K, V) at once (output discarded): per
    layer ONE baton_prefill_attention_varlen launch per group of prompts packed along
    the token axis (NEXT-2; grouping "length": the PD method's similar-length groups).
    The packed q/k/v come from the same keyed generator as the per-query prefill
    (identical values), written straight into the packed layout."""
    # Batching pays where launches dominate (short prompts: 3x for eight 30-200-token
    # prompts, scripts/probes/prefill_batch_probe.py).  Without length grouping, long
    # prompts keep one launch per query and layer: packing them regenerates their K/V
    # (the keyed generator runs at ~250 GB/s), which costs more than the launches saved.
    if not batchable(items, grouping):
        for it in items:
            prefill_attention_one(wl, device, *it)
        return
    L, D = wl.layers, wl.head_dim
    for grp in prefill_groups(items, by_length=grouping == "length"):
        T = sum(n for _, n, _, _ in grp)
        bufs = {}
        for kind, H, sc in ((KIND_Q, wl.q_heads, wl.scales[0]), (KIND_K, wl.kv_heads, wl.scales[1]),
                            (KIND_V, wl.kv_heads, wl.scales[2])):
            t = torch.empty((L, H, T, D), dtype=torch.bfloat16, device=device)
            s0 = 0
            for qid, n, _, _ in grp:
                baton_keygen_history(t[:, :, s0:], L, H, D, qid, 0, n, kind, wl.seed, sc,
                                     head_stride=T * D, layer_stride=H * T * D)
                s0 += n
            bufs[kind] = t
        O = torch.empty_like(bufs[KIND_Q])
        lens = [n for _, n, _, _ in grp]
        for l in range(L):
            baton_prefill_attention_varlen(bufs[KIND_Q][l], bufs[KIND_K][l], bufs[KIND_V][l], O[l], lens,
                                           wl.q_heads, wl.kv_heads, D)
