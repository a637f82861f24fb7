"""bench.py's N>1 path (slots sharded over ranks, max-over-ranks timing, the
per-iteration completion-flag all-gather) run as 2 ranks on ONE GPU over gloo: the
same code the driver's 2/4/8-GPU runs take, minus NCCL (which needs a GPU per
rank).  Checks the JSON line, not the speed (both ranks share the GPU)."""
import json
import os
import subprocess
import sys

import pytest

from gpu_util import require_cuda

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,port", [("7b", 29731), ("13b", 29732), ("70b", 29733),
                                         ("stress", 29734)])
def test_bench_two_ranks_one_gpu(config, port):
    require_cuda()
    env = dict(os.environ, BATON_BENCH_BACKEND="gloo", BATON_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--config", config, "--gpus", "2", "--steps", "4", "--warmup", "3", "--windows", "2",
           "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 4
    assert d["scaling"] == ("strong" if config == "13b" else "weak")
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["parallelism"] == "slots/2 GPU" and len(d["windows"]) == 2
    assert d["multi_gpu"]["allgather_us_per_iter"] > 0
    assert 1.0 <= d["multi_gpu"]["rank_attn_bytes_max_over_mean"] < 2.0
    # tokens are summed over ranks (each decodes its own slots): more than one rank's
    # worth per step
    per_rank = {"7b": 32, "13b": 32, "70b": 16, "stress": 2}[config]
    tokens_per_step = d["value"] * d["ms_per_step"] / 1e3
    assert tokens_per_step > per_rank, tokens_per_step
