"""The bench's N > 1 path on one GPU: two ranks under torchrun with the gloo backend
(BENCH_DIST_BACKEND=gloo; NCCL rejects two ranks on one device).  Covers the episode
sharding, the all-reduce of the shared-parameter gradient, max-over-ranks timing and the
rank-0 JSON line of bench.py end to end; NCCL itself needs the multi-GPU box."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("config,scaling,episodes_total", [("c2", "weak", 2), ("c4", "strong", 64)])
def test_two_ranks_on_one_gpu(config, scaling, episodes_total):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--config", config, "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    if config == "c4":
        env["BENCH_HORIZON"] = "64"
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    assert d["config"]["episodes_total"] == episodes_total
    assert d["value"] > 0 and d["e2e"]["value"] > 0
