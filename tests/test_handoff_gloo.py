"""NEXT-2 handoff on CPU (gloo, world size 3): rank 0 is the prefill rank, ranks 1
and 2 decode.  The prefill rank sends each new query's K/V to its pinned decode
rank (round-robin in admission order, reading C20c); the decode ranks run their
replicated planner with the completion-flag all-gather in their own group and,
at every insert, receive exactly that query's keyed K/V bytes -- in the order
their planner inserts them.  No GPU: K/V are the NumPy keyed generator's bits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from baton_inputs import config_workload, KIND_K, KIND_V, query_history_bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _wl():
    wl = config_workload("13b", gpus=2, n_queries=90)
    wl.layers, wl.q_heads, wl.kv_heads, wl.head_dim = 2, 4, 2, 16   # small tensors, same schedule
    wl.slots = 8
    return wl


def _bits(wl, kind, qid, n):
    return query_history_bits(wl.seed, kind, wl.layers, qid, 0, n, wl.kv_heads, wl.head_dim,
                              wl.scales[1 if kind == KIND_K else 2]).astype(np.int16)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_18701_b200.handoff import (assign_pins, PrefillServer, HandoffReceiver,
                                                   admission_order)
        from paper_2410_18701_b200.scheduler import Planner
        from paper_2410_18701_b200.comm import gather_completion_flags
        wl = _wl()
        n_dec = world - 1
        pins = assign_pins(wl, n_dec)
        decode_group = dist.new_group(list(range(1, world)))
        if rank == 0:
            def kv(qid, n):
                return (torch.from_numpy(_bits(wl, KIND_K, qid, n)).view(torch.bfloat16),
                        torch.from_numpy(_bits(wl, KIND_V, qid, n)).view(torch.bfloat16))
            srv = PrefillServer(wl, pins, list(range(1, world)), kv_source=kv, attention=False,
                                chunk=5, max_inflight=6)
            srv.serve()
            out_q.put((rank, [q for q, _ in srv.sent], srv.bytes))
            dist.barrier()
            return
        me = rank - 1
        recv = HandoffReceiver(wl, me, pins, src=0, lookahead=3)
        pl = Planner(wl, n_dec, pins=pins)
        inserted, ok, trace = [], True, []
        while not pl.finished_all():
            flags = None
            if pl.t > 0:
                flags = gather_completion_flags(pl.local_completion_flags(me), n_dec, group=decode_group)
            d = pl.plan(flags)
            trace.append((d.t, tuple(d.inserts), tuple(d.finished)))
            for g, q, n, home in d.inserts:
                if pl.rank_of(g) != me:
                    continue
                assert home is None and pins[q] == me            # C20c
                K, V = recv(q, n)
                ok &= np.array_equal(K.view(torch.int16).numpy(), _bits(wl, KIND_K, q, n))
                ok &= np.array_equal(V.view(torch.int16).numpy(), _bits(wl, KIND_V, q, n))
                inserted.append(q)
        mine = [q.qid for q in admission_order(wl) if pins[q.qid] == me]
        recv.drain()
        out_q.put((rank, inserted, ok, mine, trace))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_prefill_rank_hands_kv_to_decode_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=300)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sent, nbytes = res[0]
    wl = _wl()
    assert sorted(sent) == sorted(x.qid for x in wl.queries)
    for r in (1, 2):
        inserted, ok, mine, trace = res[r]
        assert ok                               # every byte is the query's keyed K/V
        assert inserted == mine                 # all of its queries, in send order
    assert res[1][3] == res[2][3]               # replicated planners agree
    assert nbytes == sum(2 * x.l_q * wl.layers * wl.kv_heads * wl.head_dim * 2 for x in wl.queries)


def test_pins_round_robin_and_planner_respects_them():
    from paper_2410_18701_b200.handoff import assign_pins
    from paper_2410_18701_b200.scheduler import Planner
    wl = _wl()
    pins = assign_pins(wl, 2)
    assert sorted(set(pins.values())) == [0, 1]
    pl = Planner(wl, 2, pins=pins)
    n = 0
    while not pl.finished_all():
        for g, q, _, _ in pl.plan().inserts:
            assert pl.rank_of(g) == pins[q]
            n += 1
    assert n == len(wl.queries)
