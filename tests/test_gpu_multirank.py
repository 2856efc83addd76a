"""The N>1 bench path on one GPU: two ranks launched by torchrun share cuda:0
and exchange archives every generation through the gloo backend (host-staged
allgather; on a multi-GPU box the same code path gathers device blobs over
NCCL). Checks the rank-0 JSON line: whole-job value over both islands, max over
ranks, island merges counted in the kernel launches."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["islands", "shard"])
def test_two_rank_bench_on_one_gpu(mode):
    env = dict(os.environ, TGB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "cfg1", "--no-cpu-baseline", "--mode", mode]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    per_step = d["value"] * d["ms_per_step"] / 1000.0
    if mode == "islands":
        assert "merged every 1" in d["config"]["parallelism"] and d["scaling"] == "weak"
        assert per_step == pytest.approx(2 * d["config"]["batch_per_gpu"], rel=1e-6)
    else:
        assert "batch shard" in d["config"]["parallelism"] and d["scaling"] == "strong"
        assert per_step == pytest.approx(d["config"]["batch_per_gpu"], rel=1e-6)
