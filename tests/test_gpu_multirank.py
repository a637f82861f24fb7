"""The N>1 engine path on one GPU: two ranks (processes) share cuda:0 and talk
over gloo (NCCL refuses two ranks on one device).  Each rank owns half of the
global slots (C20) and runs the fused decode / splice kernels on its shard; the
only exchange is the per-iteration all-gather of completion flags.  Every
rank's metadata, mask and live K/V bytes must equal the matching shard of the
oracle's 2-shard serving loop after every iteration, and its attention outputs
must be within C13."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    from baton_inputs import Workload, Query, ControlEvents
    rng = np.random.default_rng(5)
    qs = [Query(i, int(i // 3), int(rng.integers(1, 40)), int(rng.integers(1, 15))) for i in range(40)]
    return Workload("mr", qs, layers=2, q_heads=8, kv_heads=1, head_dim=128, slots=8, max_ctx=64,
                    gpus=2, control=ControlEvents(preempt={6: 1, 13: 2}))


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_18701_b200.engine import Engine
        from oracle import Simulator
        wl = _workload()
        eng = Engine(wl, rank=rank, world=world, device="cuda:0", group=dist.group.WORLD,
                     keep_outputs=True)
        sim = Simulator(wl, G=world, kv=True, keep_outputs=True)
        errs = []
        while not sim.done():
            sim.iteration()
            eng.iteration()
            torch.cuda.synchronize()
            sh, osh = eng.shard, sim.shards[rank]
            m = sh.baton_query()
            occ = osh.qid >= 0
            if m["S"] != osh.S or not np.array_equal(m["lens"], osh.lens()):
                errs.append(f"t{sim.t}: S/lens")
            if not np.array_equal(sh.mask[:, :osh.S].cpu().numpy(), osh.mask):
                errs.append(f"t{sim.t}: mask")
            for b in np.nonzero(occ)[0]:
                Ko, _ = osh.live_kv(b)
                Kd, _ = sh.live_kv(b)
                kd = Kd.float().cpu().numpy()
                if not np.array_equal(kd, Ko.astype(np.float32)):
                    errs.append(f"t{sim.t}: K slot {b}")
        assert eng.done()
        worst = 0.0
        mine = {k: v for k, v in eng.outputs.items()}
        for k, o in mine.items():
            ref = sim.outputs[k]
            num = np.abs(o - ref).max(-1)
            den = np.maximum(np.abs(ref).max(-1), 1e-30)
            worst = max(worst, float((num / den).max()))
        out_q.put((rank, errs, worst, len(mine)))
    except Exception as e:   # report instead of hanging the peer
        out_q.put((rank, [repr(e)], 1.0, 0))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    total = 0
    for rank, errs, worst, n in res:
        assert errs == [], (rank, errs[:5])
        assert worst <= 1e-2, (rank, worst)
        total += n
    from baton_inputs import Workload
    assert total == sum(qq.A for qq in _workload().queries)
