"""the controller optimisation loop (paper_1910_00935_b200.optimize).

CPU tests drive the loop with the CPU oracle standing in for the GPU library (an adapter with
the mpm.Sim call surface): one descent step lowers the loss; the world-size-2 gloo run
(episodes sharded, theta_bar all-reduced) reproduces the single-process run over the same
episodes and keeps theta identical on both ranks.  The GPU test optimises the C2 soft robot
("the robot learns to move forward") through the C-ABI.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_00935_b200 import optimize as O
from paper_1910_00935_b200 import workloads as W


class OracleSim:
    """mpm.Sim call surface over the CPU oracle (test infrastructure only)."""

    def __init__(self, p):
        from oracle import Oracle
        self.o, self.p = Oracle(p), p

    def set_state(self, x, v, C, F, aid):
        self.s = [np.asarray(a.cpu().numpy()) for a in (x, v, C, F, aid)]

    def set_controller(self, theta):
        self.theta = theta.cpu().numpy().astype(np.float64)

    def forward(self, T):
        x, v, C, F, aid = self.s
        self.res = [self.o.run(x[e], v[e], C[e], F[e], aid[e], self.theta, steps=T) for e in range(len(x))]

    def loss(self):
        return np.array([r["loss"] for r in self.res])

    def backward(self, T):
        pass

    def grads(self, out):
        g = sum(r["dtheta"] for r in self.res)
        out["dtheta"].copy_(torch.from_numpy(np.asarray(g)).to(out["dtheta"].dtype))
        return out


def _cfg():
    # tiny 3D robot-like block on the sticky floor: the move-forward loss depends on theta
    # only through the wall contact (internal forces alone keep the centre of mass ballistic)
    return W.tiny(3, steps=6, hidden=3, bound=3, floor=True, v_base=(0.2, -1.5, 0.1), seed=21,
                  loss="move_forward")


def test_descent_step_lowers_the_loss():
    p = _cfg()
    r = O.optimize(p, iters=3, lr=1e-2, method="gd", sim=OracleSim(p), device="cpu")
    assert r["grad_norm"][0] > 0
    assert r["loss"][1] < r["loss"][0], r["loss"]
    assert r["loss"][2] < r["loss"][1], r["loss"]


def test_adam_matches_its_definition():
    th = torch.tensor([1.0, -2.0, 0.5], dtype=torch.float64)
    opt = O.Adam(th, lr=0.1)
    g = torch.tensor([0.3, -0.1, 0.0], dtype=torch.float64)
    opt.step(g)
    # first step: m_hat = g, v_hat = g^2 -> theta -= lr * g / (|g| + eps)
    want = torch.tensor([1.0 - 0.1 * 0.3 / (0.3 + 1e-8), -2.0 + 0.1 * 0.1 / (0.1 + 1e-8), 0.5])
    assert torch.allclose(th, want.double(), atol=1e-12)


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
        p = _cfg()
        r = O.optimize(p, iters=2, lr=1e-2, method="adam", episodes=2, sim=OracleSim(p), device="cpu",
                       rank=rank, world=world)
        out[rank] = (r["theta"].numpy().copy(), r["loss"], r["episodes"])
    finally:
        dist.destroy_process_group()


def test_two_rank_loop_matches_single_process():
    p = _cfg()
    ref = O.optimize(p, iters=2, lr=1e-2, method="adam", episodes=2, sim=OracleSim(p), device="cpu")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0][2] == [0] and out[1][2] == [1]
    np.testing.assert_array_equal(out[0][0], out[1][0])  # same update on every rank
    np.testing.assert_allclose(out[0][0], ref["theta"].numpy(), rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(out[0][1], ref["loss"], rtol=1e-9)


@pytest.mark.gpu
def test_c2_robot_learns_to_move_forward():
    """C2 (2D soft robot, 6,400 particles, 4 muscles, 1,024 steps): Adam on the controller
    through the CUDA path lowers the move-forward loss -x_bar_T . e_0."""
    r = O.optimize("c2", iters=16, lr=0.05, method="adam", clip=1.0, log=print)
    L = r["loss"]
    assert all(np.isfinite(L))
    assert min(L) < L[0] - 0.05, L  # the centre of mass ends >= 0.05 further along +x
    assert L[-1] < L[0], L


@pytest.mark.gpu
def test_c2cl_closed_loop_robot_learns_to_move_forward():
    """The closed-loop controller optimised end to end (f2) on C2."""
    r = O.optimize("c2cl", iters=16, lr=0.05, method="adam", clip=1.0, log=print)
    L = r["loss"]
    assert all(np.isfinite(L))
    assert min(L) < L[0] - 0.05, L
    assert L[-1] < L[0], L


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tiny3d", "c2@256"])
def test_adam_loop_through_the_cuda_path_matches_the_oracle_loop(case):
    """f2 parity: 3 Adam iterations of optimize() driven by the CUDA path (mpm.Sim through the
    C-ABI) and by the fp64 oracle (OracleSim) from the same theta_0 give the same losses and
    the same theta_3 (rel <= 1e-3): the loop, not just a descending loss, is checked."""
    if case == "tiny3d":
        p, kw = _cfg(), dict(lr=1e-2)
    else:
        p, kw = W.config("c2", steps=256), dict(lr=0.05, clip=1.0)
    gpu = O.optimize(p, iters=3, method="adam", **kw)
    ref = O.optimize(p, iters=3, method="adam", sim=OracleSim(p), device="cpu", **kw)
    th, th_ref = gpu["theta"].cpu().double().numpy(), ref["theta"].numpy()
    th0 = W.make_inputs(p)["theta"].astype(np.float64)
    step_rel = np.linalg.norm(th - th_ref) / np.linalg.norm(th_ref - th0)  # vs the distance moved
    print(f"[f2] {case}: losses gpu {gpu['loss']} oracle {ref['loss']}; theta_3 rel {np.linalg.norm(th - th_ref) / np.linalg.norm(th_ref):.2e}, "
          f"rel to the update {step_rel:.2e}")
    np.testing.assert_allclose(gpu["loss"], ref["loss"], rtol=1e-4, atol=1e-7)
    assert np.linalg.norm(th - th_ref) / np.linalg.norm(th_ref) < 1e-3
    assert step_rel < 1e-2
