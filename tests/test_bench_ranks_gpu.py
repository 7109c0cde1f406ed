"""bench.py's multi-rank path end to end on a one-GPU box: `--gpus 2`
without torchrun relaunches itself under torch.distributed.run, each rank
builds its own context and session over its own image shard, the parity
mismatches are summed and the elapsed time is the max over ranks, and rank 0
prints one line with n_gpus = 2 covering both shards. LB_RANKS_ON_ONE_GPU
puts both ranks on cuda:0 over gloo (functional only: the ranks share the
GPU, so the timings mean nothing)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_two_rank_bench_on_one_gpu():
    env = dict(os.environ, PYTHONPATH=str(ROOT), LB_RANKS_ON_ONE_GPU="1", LB_POOL_RESERVE="0")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--batch", "2", "--no-extras"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["parity"]["images"] == 4 and d["parity"]["mismatches"] == 0
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 2 * 784 * 8
    assert "2 GPU(s)" in d["config"]["parallelism"]
