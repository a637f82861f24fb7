"""Host side of bench.py's configs (no GPU): the workloads each config builds at
N GPUs, the steady-state windows, and -- over 2 gloo ranks -- that the window
plan every rank derives locally (bench.window_plan on its replicated planner) is
exactly what the ranks decide together when they exchange completion flags
through the all-gather each iteration (comm.py), for every config."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench

CONFIGS = ["7b", "13b", "70b", "stress"]


@pytest.mark.parametrize("config", CONFIGS)
@pytest.mark.parametrize("world", [1, 2, 8])
def test_workload_shapes(config, world):
    wl, scaling = bench.bench_workload(config, world)
    assert wl.slots % world == 0
    per = wl.slots // world
    if config == "13b":
        assert scaling == "strong" and wl.slots == 64      # 64 slots split over the GPUs
    else:
        assert scaling == "weak"
        assert per == {"7b": 32, "70b": 16, "stress": 32}[config]
    if config == "70b":
        assert (wl.q_heads, wl.kv_heads, wl.max_ctx) == (64, 8, 4096)
        assert len(wl.queries) == 64 * world
    if config == "stress":
        # configs[4] at 8 GPUs: 16 -> 256 active slots, 25% stored every 16 iterations
        assert wl.active == 2 * world and max(wl.control.resize.values()) == 32 * world
        assert set(wl.control.preempt_frac) == set(range(16, 641, 16))


@pytest.mark.parametrize("config", CONFIGS)
def test_windows_in_steady_state(config):
    from paper_2410_18701_b200.scheduler import Planner
    wl, _ = bench.bench_workload(config, 1)
    span = 40
    starts, (lo, hi) = bench.steady_windows(wl, 1, 5, span)
    assert len(starts) == 5 and starts == sorted(starts) and lo <= starts[0]
    assert starts[-1] + span <= hi + 1
    p = Planner(wl, 1)
    for t0 in starts:
        bench.fast_forward(p, t0)
        assert p.t == t0 and len(p.decode_plan()) == p.active      # every active slot live


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, config, n_iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_18701_b200.scheduler import Planner
        from paper_2410_18701_b200.comm import gather_completion_flags
        wl, _ = bench.bench_workload(config, world)
        starts, _ = bench.steady_windows(wl, world, 3, n_iters)
        t0 = starts[0]
        pl = Planner(wl, world)
        bench.fast_forward(pl, t0)
        local_dec, local_fresh = bench.window_plan(pl, n_iters, rank)
        # the same iterations decided together: local flags -> all-gather -> plan
        dec, fresh = [], []
        for _ in range(n_iters):
            dec.append([(pl.local(g), q, pos) for g, q, pos in pl.decode_plan()
                        if pl.rank_of(g) == rank])
            flags = gather_completion_flags(pl.local_completion_flags(rank), world)
            d = pl.plan(flags)
            fresh += [(q, n, d.t) for g, q, n, home in d.inserts
                      if pl.rank_of(g) == rank and home is None]
        out_q.put((rank, starts, dec == local_dec, fresh == local_fresh,
                   sum(len(x) for x in dec)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("config", CONFIGS)
def test_two_rank_window_plan(config):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_iters = 24
    procs = [ctx.Process(target=_worker, args=(r, 2, port, config, n_iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0]                    # identical windows on every rank
    for r in (0, 1):
        assert res[r][1] and res[r][2]               # local plan == exchanged decisions
    wl, _ = bench.bench_workload(config, 2)
    from paper_2410_18701_b200.scheduler import Planner
    p = Planner(wl, 2)
    bench.fast_forward(p, res[0][0][0])
    total = 0
    for _ in range(n_iters):
        total += len(p.decode_plan())
        bench.fast_forward(p, p.t + 1)
    assert res[0][3] + res[1][3] == total            # the ranks' decodes partition the batch's
