"""World-size-2 CPU test (gloo) of the N>1 host path: each rank contributes the
completion flags of its own slots, one all-gather per iteration gives every
rank the same view, and the replicated planners take identical decisions --
equal to the oracle's G-shard serving loop."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from baton_inputs import config_workload, random_stream


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_18701_b200.scheduler import Planner
        from paper_2410_18701_b200.comm import gather_completion_flags
        if name == "stress":
            wl = config_workload("stress", gpus=world, n_queries=300)
            wl.iterations = 150
        else:
            wl = config_workload("13b", gpus=world, n_queries=200)
        pl = Planner(wl, world)
        trace = []
        while not pl.finished_all():
            flags = None
            if pl.t > 0:
                flags = gather_completion_flags(pl.local_completion_flags(rank), world)
            d = pl.plan(flags)
            trace.append((d.t, tuple(d.decode), tuple(d.finished), tuple(d.victims), d.resize,
                          tuple(d.inserts)))
        out_q.put((rank, trace))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["13b", "stress"])
def test_two_rank_replicated_planner(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    # and equal to the oracle's 2-shard loop
    from oracle import Simulator
    if name == "stress":
        wl = config_workload("stress", gpus=2, n_queries=300)
        wl.iterations = 150
    else:
        wl = config_workload("13b", gpus=2, n_queries=200)
    sim = Simulator(wl, G=2)
    for t, dec, fin, vic, rs, ins in res[0]:
        rec = sim.iteration()
        assert sorted(dec) == sorted(rec.decoded)
        assert sorted(g for g, _ in fin) == sorted(rec.removed)
        assert [(g, q, l) for g, q, l, _ in ins] == rec.inserted
    assert sim.done()
