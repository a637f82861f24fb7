"""NEXT-2: disaggregated P&D -- prefill on its own rank, K/V handed to the decode rank.

P:L132: "all original queries ... are initially prefilled" separately and the
decode batch embeds their Keys/Values; "asynchronous P&D decoupling";
P:L335: prefill batches are composed "using the similarity of length principle",
and decoupling "allows parallel computation with decoupled prefilling and
decoding".  Here the prefill runs on a PREFILL rank (its own GPU) while the
decode ranks run the relay race; each new query's prefilled K/V travel to the
decode rank that will embed it:

* ``assign_pins``: the prefill rank sends the queries to the decode ranks
  round-robin in admission order (arrival, qid).  A remotely prefilled query may
  only take a slot of the rank holding its K/V (reading C20c; Planner ``pins``),
  so every decode rank embeds its queries in the same FCFS order in which they
  were sent -- point-to-point messages then match by order, with no tags.
* ``PrefillServer`` (prefill rank): for each chunk of queries in admission order,
  the K/V (keyed generator: the model's K/V projections stand-in), the prompt's
  attention (a8, ``prefill_attention_batch`` in length groups), then one send of K
  and one of V to the query's decode rank.  At most ``max_inflight`` queries' sends
  are outstanding.
* ``HandoffReceiver`` (decode rank): the Engine's ``prefill_source``.  It posts the
  receives of its next ``lookahead`` queries ahead of their inserts; the insert
  waits on that query's receive only (``work.wait()``: with NCCL the decode stream
  waits on the transfer, the host does not block).

Transport: NCCL point-to-point between the two GPUs (NVLink on the box: a
prefill GPU's K/V arrive in the decode GPU's HBM directly); over gloo (CPU tests,
and two ranks sharing one GPU) tensors travel through host memory as int16 bits.
The completion-flag all-gather stays among the decode ranks (their own group).
"""
import torch
import torch.distributed as dist

from .engine import prefill_attention_batch, KIND_K, KIND_V
from .baton import baton_keygen_history


def admission_order(wl):
    return [q for q in sorted(wl.queries, key=lambda q: (q.arrival, q.qid))]


def assign_pins(wl, n_decode):
    """{qid: decode rank index}: round-robin over the decode ranks in admission order."""
    return {q.qid: i % n_decode for i, q in enumerate(admission_order(wl))}


class Transport:
    """Point-to-point K/V transfer between world ranks."""

    def __init__(self, device=None):
        self.gpu = dist.get_backend() == "nccl"
        self.device = device

    def isend(self, t, dst):
        if self.gpu:
            return dist.isend(t, dst), t
        h = t.contiguous().view(torch.int16).cpu()          # bf16 bits through the host
        return dist.isend(h, dst), h

    def irecv(self, shape, src):
        if self.gpu:
            buf = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
            return dist.irecv(buf, src), buf
        h = torch.empty(shape, dtype=torch.int16)
        return dist.irecv(h, src), h

    def land(self, buf):
        """A received buffer as a bf16 tensor on the decode device."""
        if self.gpu:
            return buf
        t = buf.view(torch.bfloat16)
        return t.to(self.device, non_blocking=False) if self.device is not None else t


def keyed_kv(wl, device):
    """Default K/V source of the prefill rank: the query's keyed history."""
    def make(qid, n):
        shape = (wl.layers, wl.kv_heads, n, wl.head_dim)
        K = torch.empty(shape, dtype=torch.bfloat16, device=device)
        V = torch.empty_like(K)
        baton_keygen_history(K, wl.layers, wl.kv_heads, wl.head_dim, qid, 0, n, KIND_K, wl.seed,
                             wl.scales[1])
        baton_keygen_history(V, wl.layers, wl.kv_heads, wl.head_dim, qid, 0, n, KIND_V, wl.seed,
                             wl.scales[2])
        return K, V
    return make


class PrefillServer:
    def __init__(self, wl, pins, decode_ranks, device=None, kv_source=None, attention=True,
                 chunk=8, max_inflight=16):
        """decode_ranks: world rank of each decode rank index (pins map to indices)."""
        self.wl, self.pins, self.decode_ranks = wl, pins, decode_ranks
        self.device = device
        self.kv_source = kv_source or keyed_kv(wl, device)
        self.attention = attention
        self.chunk, self.max_inflight = chunk, max_inflight
        self.transport = Transport(device)
        self.sent = []                  # (qid, rows) in send order
        self.bytes = 0

    def serve(self):
        order = admission_order(self.wl)
        inflight = []
        for i in range(0, len(order), self.chunk):
            part = order[i:i + self.chunk]
            items = [(q.qid, q.l_q) + tuple(self.kv_source(q.qid, q.l_q)) for q in part]
            if self.attention and self.wl.head_dim == 128:   # a8 is built for head_dim 128
                prefill_attention_batch(self.wl, self.device, items, grouping="length")
            for qid, n, K, V in items:
                dst = self.decode_ranks[self.pins[qid]]
                inflight.append([self.transport.isend(K, dst), self.transport.isend(V, dst)])
                self.sent.append((qid, n))
                self.bytes += 2 * K.numel() * 2
                while len(inflight) > self.max_inflight:
                    for w, _ in inflight.pop(0):
                        w.wait()
        for pair in inflight:
            for w, _ in pair:
                w.wait()


class HandoffReceiver:
    def __init__(self, wl, me, pins, src, device=None, lookahead=4):
        """me: this decode rank's index; src: the prefill rank (world rank)."""
        self.wl = wl
        self.order = [q for q in admission_order(wl) if pins[q.qid] == me]
        self.src, self.lookahead = src, lookahead
        self.transport = Transport(device)
        self.next = 0
        self.posted = {}
        self.received = []

    def _post(self):
        wl = self.wl
        while len(self.posted) < self.lookahead and self.next < len(self.order):
            q = self.order[self.next]
            shape = (wl.layers, wl.kv_heads, q.l_q, wl.head_dim)
            self.posted[q.qid] = (self.transport.irecv(shape, self.src),
                                  self.transport.irecv(shape, self.src))
            self.next += 1

    def __call__(self, qid, n):
        self._post()
        if qid not in self.posted:
            raise RuntimeError(f"handoff: query {qid} not expected next on this rank")
        (wk, bk), (wv, bv) = self.posted.pop(qid)
        wk.wait()
        wv.wait()
        K, V = self.transport.land(bk), self.transport.land(bv)
        assert K.shape[2] == n
        self.received.append(qid)
        self._post()
        return K, V

    def drain(self):
        """Receive (and drop) every query still to come -- a run that ends early (an
        iteration limit) must still match the prefill rank's sends."""
        while self.posted or self.next < len(self.order):
            self._post()
            for (wk, _), (wv, _) in list(self.posted.values()):
                wk.wait()
                wv.wait()
            self.posted.clear()
