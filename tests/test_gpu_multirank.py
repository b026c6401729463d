"""The bench's N > 1 path on one GPU: two ranks under torchrun with the gloo backend
(BENCH_DIST_BACKEND=gloo; NCCL rejects two ranks on one device).  Covers the episode
sharding, the all-reduce of the shared-parameter gradient, max-over-ranks timing and the
rank-0 JSON line of bench.py end to end; NCCL itself needs the multi-GPU box."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
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


def test_nccl_backend_single_rank():
    """The bench under torchrun with the NCCL backend (its default) on the one GPU this pool
    gives: process-group init with device_id, the all-reduce of the shared-parameter gradient,
    the agreed checkpoint interval (all-reduce MIN) and the max-over-ranks timing all go through
    NCCL.  NCCL_DEBUG=INFO must show the communicator came up (nranks 1)."""
    env = dict(os.environ, NCCL_DEBUG="INFO", BENCH_HORIZON="64")
    env.pop("BENCH_DIST_BACKEND", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
           "--config", "c4", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0
    log = out.stdout + out.stderr
    assert "NCCL INFO" in log and "nranks 1" in log, log[-3000:]


def _t6_worker(rank, world, port, T, out):
    """one C4 episode per rank on the same GPU, theta_bar all-reduced over gloo"""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import gpu_run
        from paper_1910_00935_b200 import workloads as W
        from paper_1910_00935_b200.dist import allreduce_shared_grad, episode_shard
        torch.cuda.set_device(0)
        p = W.config("c4", steps=T)
        shard = episode_shard(world, rank, world)
        got = gpu_run(p, [W.make_inputs(p, episode=e) for e in shard], k_ckpt=32)
        g = torch.from_numpy(np.ascontiguousarray(got["dtheta"])).cuda()
        allreduce_shared_grad(g)
        out[rank] = g.cpu().numpy()
    finally:
        dist.destroy_process_group()


def test_allreduced_theta_bar_equals_single_process_sum():
    """SURVEY 4.2 T6 / 8(e) on the CUDA path: two ranks (gloo, both on this GPU), one C4 episode
    each at a post-contact horizon, all-reduce(SUM) of theta_bar == one process holding both
    episodes (rel <= 1e-6; the two differ only in the fp32 summation order of the per-block
    actuator-gradient partials)."""
    import torch.multiprocessing as mp
    from helpers import gpu_run
    from paper_1910_00935_b200 import workloads as W
    T = 128
    p = W.config("c4", steps=T)
    single = gpu_run(p, [W.make_inputs(p, episode=e) for e in range(2)], k_ckpt=32)["dtheta"]
    out = mp.Manager().dict()
    mp.spawn(_t6_worker, args=(2, _port(), T, out), nprocs=2, join=True)
    np.testing.assert_array_equal(out[0], out[1])  # every rank holds the same sum
    r = np.linalg.norm(out[0] - single) / np.linalg.norm(single)
    print(f"[T6] |theta_bar| {np.linalg.norm(single):.3e}, all-reduced vs single process rel {r:.2e}")
    assert np.linalg.norm(single) > 1e-4
    assert r < 1e-6
