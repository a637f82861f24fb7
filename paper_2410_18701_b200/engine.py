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


class Engine:
    def __init__(self, wl, rank=0, world=1, device=None, group=None, keep_outputs=False,
                 keep_layers=None, token_source=None, prefill_source=None, use_graph=True,
                 stash_host=False, policy="baton", prefill_attention=False, async_prefill=False,
                 prefill_lookahead=None):
        self.wl = wl
        self.rank = rank
        self.world = world
        self.group = group
        self.device = torch.device(device or "cuda")
        self.planner = Planner(wl, world, policy=policy)
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
        self.stash: Dict[int, Tuple[torch.Tensor, torch.Tensor]] = {}
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
        self.stash_host = stash_host
        self.last_decisions = None

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
        """a8 over every layer of a fresh query's prompt (output discarded)."""
        wl = self.wl
        Q = torch.empty((wl.layers, wl.q_heads, n, wl.head_dim), dtype=torch.bfloat16, device=self.device)
        baton_keygen_history(Q, wl.layers, wl.q_heads, wl.head_dim, qid, 0, n, KIND_Q, wl.seed,
                             wl.scales[0])
        O = torch.empty_like(Q)
        for l in range(wl.layers):
            baton_prefill_attention(Q[l], K[l], V[l], O[l], n, wl.q_heads, wl.kv_heads, wl.head_dim)

    @staticmethod
    def _batchable(items):
        return len(items) > 1 and sum(n for _, n, _, _ in items) <= PREFILL_BATCH_MEAN * len(items)

    def _prefill_attn_batch(self, items):
        """a8 for several fresh queries at once (output discarded): per layer ONE
        baton_prefill_attention_varlen launch over their prompts packed along the token
        axis (NEXT-2).  The packed q/k/v come from the same keyed generator as the
        per-query prefill (identical values), written straight into the packed layout."""
        # Batching pays where launches dominate (short prompts: 3x for eight 30-200-token
        # prompts, scripts/probes/prefill_batch_probe.py).  Long prompts keep one
        # launch per query and layer: packing them would regenerate their K/V (the
        # keyed generator runs at ~250 GB/s), which costs more than the launches saved.
        if not self._batchable(items):
            for it in items:
                self._prefill_attn(*it)
            return
        wl = self.wl
        L, D = wl.layers, wl.head_dim
        groups, cur, tiles = [], [], 0          # launch limits: 64 prompts, 1024 query tiles
        for it in items:
            t = -(-it[1] // 128)
            if cur and (len(cur) == 64 or tiles + t > 1024):
                groups.append(cur)
                cur, tiles = [], 0
            cur.append(it)
            tiles += t
        groups.append(cur)
        for grp in groups:
            T = sum(n for _, n, _, _ in grp)
            bufs = {}
            for kind, H, sc in ((KIND_Q, wl.q_heads, wl.scales[0]), (KIND_K, wl.kv_heads, wl.scales[1]),
                                (KIND_V, wl.kv_heads, wl.scales[2])):
                t = torch.empty((L, H, T, D), dtype=torch.bfloat16, device=self.device)
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

    def iteration(self):
        pl = self.planner
        stats = StepStats(pl.t)
        flags = None
        if pl.t > 0:
            self.decode(stats)
            local = pl.local_completion_flags(self.rank)
            # completion flags + occupancy summary of every rank
            flags = self._gather_flags(local) if self.world > 1 else None
        d = pl.plan(flags)
        self.last_decisions = d
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
                n = int(sh.baton_query()["lens"][b])       # the library's live length
                if self.stash_host:
                    shape = (self.wl.layers, self.wl.kv_heads, n, self.wl.head_dim)
                    ko = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
                    vo = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
                    self.stash[q] = sh.baton_extract(b, ko, vo)
                else:
                    self.stash[q] = sh.baton_extract(b)
                stats.extract_rows += n
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
                    K, V = self.stash.pop(q)
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
            stats.inserted = len(ins)
            stats.insert_rows = sum(lens)
        if self.async_prefill:
            self._prefetch()
        stats.S = sh.S
        return stats

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
        while not self.done():
            all_stats.append(self.iteration())
            if max_iters is not None and len(all_stats) >= max_iters:
                break
        return all_stats
