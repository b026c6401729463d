"""End-to-end controller optimisation through the differentiable MLS-MPM step
(SURVEY.md section 8(f), row f2 -- the experiment the hot path exists for).

PAPER.md P:305 (``diffmpm``): "we use gradient descent to optimize the controller ... the
robot learns to move forward"; P:20 (Fig. 1): the controller is optimised through a
512-2048-step simulation "within tens of iterations"; P:612 (Fig. 6): 3D robots with 16
muscles.  Each iteration is one use of the C-ABI the way ``ti.Tape`` is used in the paper
(P:245-263):

    set_state(S_0) -> set_controller(theta) -> forward(T) -> loss -> backward(T) -> grads(theta_bar)
    [-> all-reduce(SUM) of theta_bar over the episode shards (the one collective, 8(e))]
    -> theta <- update(theta, theta_bar)

The parameter update is a few element-wise torch ops on the controller weights (<= 1K floats):
it is outside the hot path, so it stays plain PyTorch (plain gradient descent, or Adam).
Every rank applies the same update to the same all-reduced gradient, so theta stays identical
across ranks without a broadcast.
"""
from __future__ import annotations

import numpy as np
import torch

from . import workloads as W
from .dist import allreduce_shared_grad, episode_shard


class Adam:
    """Adam (Kingma & Ba) on one flat parameter tensor, in place."""

    def __init__(self, theta: torch.Tensor, lr: float, betas=(0.9, 0.999), eps: float = 1e-8):
        self.theta, self.lr, (self.b1, self.b2), self.eps = theta, float(lr), betas, float(eps)
        self.m = torch.zeros_like(theta)
        self.v = torch.zeros_like(theta)
        self.t = 0

    def step(self, grad: torch.Tensor) -> None:
        self.t += 1
        self.m.mul_(self.b1).add_(grad, alpha=1.0 - self.b1)
        self.v.mul_(self.b2).addcmul_(grad, grad, value=1.0 - self.b2)
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        self.theta.sub_(self.lr * mh / (vh.sqrt() + self.eps))


class GD:
    """Plain gradient descent (the paper's optimiser for diffmpm)."""

    def __init__(self, theta: torch.Tensor, lr: float):
        self.theta, self.lr = theta, float(lr)

    def step(self, grad: torch.Tensor) -> None:
        self.theta.sub_(self.lr * grad)


def episode_inputs(p: dict, episodes, device) -> dict:
    """Stacked [E][N] initial states of the given episode indices (seeded, synthetic)."""
    per = [W.make_inputs(p, episode=e) for e in episodes]
    n = {len(q["x"]) for q in per}
    if len(n) != 1:
        raise ValueError("episodes of one shard must have the same particle count")
    out = {k: torch.from_numpy(np.stack([q[k] for q in per])).to(device) for k in ("x", "v", "C", "F", "aid")}
    out["theta"] = torch.from_numpy(per[0]["theta"]).to(device)
    return out


def optimize(p: dict | str, iters: int, lr: float, method: str = "adam", episodes: int | None = None,
             steps: int | None = None, k_ckpt: int | None = None, sim=None, device="cuda",
             rank: int = 0, world: int = 1, clip: float | None = None, log=None) -> dict:
    """Optimise the shared controller weights of config `p` for `iters` iterations.

    episodes: total episodes over all ranks (default: the config's); rank r simulates the
    contiguous shard dist.episode_shard(episodes, r, world).  sim: an object with the
    mpm.Sim call surface (default: a new mpm.Sim on `device`).  clip: rescale the (all-reduced)
    gradient to this L2 norm when it is larger -- a 1,024-step contact-rich rollout is a very
    deep program and yields occasional exploding gradients ("obtaining
    robust gradients in physical simulation ... is not always easy").  Returns the per-iteration
    total loss (summed over all episodes, all ranks), the final theta and gradient norms.
    """
    if isinstance(p, str):
        p = W.config(p)
    if W.n_theta(p) == 0:
        raise ValueError(f"config {p.get('name')} has no controller to optimise")
    T = int(steps if steps is not None else p["steps"])
    E_tot = int(episodes if episodes is not None else p.get("episodes", 1))
    shard = episode_shard(E_tot, rank, world)
    inp = episode_inputs(p, shard, device)
    E, N = inp["x"].shape[0], inp["x"].shape[1]
    if sim is None:
        from . import mpm
        sim = mpm.sim_from_config(p, N, episodes=E, max_steps=T, k_ckpt=k_ckpt)
    theta = inp["theta"].clone()
    opt = Adam(theta, lr) if method == "adam" else GD(theta, lr)
    grad = torch.zeros_like(theta)
    losses, gnorms = [], []
    for it in range(int(iters)):
        sim.set_state(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"])
        sim.set_controller(theta)
        sim.forward(T)
        L = torch.as_tensor(np.asarray(sim.loss(), np.float64).sum(), dtype=torch.float64)
        sim.backward(T)
        sim.grads({"dtheta": grad})
        allreduce_shared_grad(grad)
        Lt = L.to(grad.device if world > 1 and grad.is_cuda else "cpu")
        allreduce_shared_grad(Lt)
        losses.append(float(Lt))
        gn = float(grad.norm())
        gnorms.append(gn)
        if log:
            log(f"iter {it:3d}  loss {losses[-1]: .6e}  |grad| {gn:.3e}")
        if clip is not None and gn > clip:
            grad.mul_(clip / gn)
        opt.step(grad)
    return {"loss": losses, "grad_norm": gnorms, "theta": theta, "episodes": list(shard), "T": T}
