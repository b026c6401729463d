"""The N > 1 path on CPU: world_size-2 gloo process group.

Each rank takes its shard of the episodes (paper_1910_00935_b200.dist.episode_shard),
computes the per-episode controller gradients (the CPU oracle stands in for the
GPU library here -- this test covers the sharding and the collective, not the
kernels), and all-reduces the shared-parameter gradient.  The result must equal
the single-process sum over all episodes; the max-over-ranks timing helper and
the weak-scaling throughput formula are checked too.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_00935_b200 import workloads as W
from paper_1910_00935_b200.dist import (allreduce_shared_grad, episode_shard, max_over_ranks,
                                        weak_scaling_value)

TOTAL_EPISODES = 5  # uneven split on purpose: ranks get 3 and 2


def _cfg():
    return W.tiny(3, steps=4, hidden=3, bound=3, floor=True, v_base=(0.2, -1.5, 0.1), seed=21)


def _episode_grad(e):
    from oracle import Oracle
    p = _cfg()
    inp = W.make_inputs(p, episode=e)
    r = Oracle(p).run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"])
    return r["dtheta"], r["loss"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = episode_shard(TOTAL_EPISODES, rank, world)
        g = torch.zeros(len(_episode_grad(0)[0]), dtype=torch.float64)
        for e in shard:
            g += torch.from_numpy(_episode_grad(e)[0])
        allreduce_shared_grad(g)
        ms = max_over_ranks(10.0 * (rank + 1))
        out[rank] = (g.numpy().copy(), ms, list(shard))
    finally:
        dist.destroy_process_group()


def test_episode_shard_partitions():
    for total in (1, 5, 64):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            parts = [list(episode_shard(total, r, world)) for r in range(world)]
            assert sum(parts, []) == list(range(total))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        episode_shard(4, 2, 2)


def test_two_rank_gloo_allreduce_matches_single_process_sum():
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    ref = sum(_episode_grad(e)[0] for e in range(TOTAL_EPISODES))
    assert np.abs(ref).max() > 0
    for rank in range(world):
        g, ms, shard = out[rank]
        np.testing.assert_allclose(g, ref, rtol=1e-12, atol=1e-18)
        assert ms == pytest.approx(20.0)  # max over ranks of 10, 20
    assert out[0][2] + out[1][2] == list(range(TOTAL_EPISODES))


def test_weak_scaling_value():
    # 2 ranks x 1,061,208 particles x 2,048 steps in 1.5 s (max over ranks)
    v = weak_scaling_value(1061208 * 2048, 2, 1500.0)
    assert v == pytest.approx(1061208 * 2048 * 2 / 1.5)


def test_bench_workload_shards():
    """bench.py's work split: C4's 64 episodes over N ranks (strong; --shard-of N sizes rank 0's
    share on one GPU), one episode per rank otherwise (weak)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "bench_mod", os.path.join(os.path.dirname(os.path.dirname(__file__)), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for n in (1, 2, 4, 8):
        parts = [list(bench._workload("c4", n, r)[1]) for r in range(n)]
        assert sum(parts, []) == list(range(64)) and all(len(q) == 64 // n for q in parts)
        assert bench._workload("c4", n, 0)[2] == "strong"
        p, shard, kind = bench._workload("c5", n, n - 1)
        assert list(shard) == [n - 1] and kind == "weak"
