"""Seeded synthetic workloads.

This module holds NONE of the method's arithmetic: it only lays out particles
on jittered lattices, assigns actuator ids and draws initial velocities and
controller weights.  Both the CUDA path (via the C-ABI) and the CPU oracle
consume its output, which is generated in fp64 and rounded ONCE to fp32 so
that both sides see bit-identical inputs.

Shapes follow the paper's workloads: 2D, 6.4K particles (Table 1 caption,
PAPER.md P:313); a 3D robot with 16 muscles and ~30K particles (Fig. 6
caption); 512-2048 time steps (Fig. 1 caption).
"""
from __future__ import annotations

import copy

import numpy as np

# shared defaults (SURVEY.md 8(d) "Small shared defaults"; R3-R9)
_BASE = dict(E=25.0, nu=0.25, p_mass=1.0, p_vol=1.0, eps_mass=1e-10, bound=3,
             n_sin=4, omega=20.0, dt=1e-3, kappa=4.0, act_axis=1, hidden=32,
             theta_std=0.01, k_ckpt=1, closed_loop=False, obs_sx=10.0, obs_sv=1.0)

CONFIGS: dict[str, dict] = {
    # C1a: 2D elastic block in free flight (no wall contact), COM loss, d/dv0
    "c1a": dict(_BASE, dim=2, n_grid=64, model="fixed_corotated", gravity=3.8, steps=128,
                loss="com_target", target=[0.55, 0.6, 0.0], n_act=0, hidden=0,
                shape="block2d", lower=(0.375, 0.50), counts=(32, 32), h=1.0 / 128,
                v_base=(1.0, 0.5), spin=2.0, v_noise=0.1, seed=1),
    # C1b: same block hitting the sticky floor
    "c1b": dict(_BASE, dim=2, n_grid=64, model="fixed_corotated", gravity=3.8, steps=128,
                loss="com_target", target=[0.55, 0.3, 0.0], n_act=0, hidden=0,
                shape="block2d", lower=(0.375, 0.08), counts=(32, 32), h=1.0 / 128,
                v_base=(0.5, -1.0), spin=2.0, v_noise=0.1, seed=11),
    # C2: 2D soft robot, 4 muscles, 6,400 particles, 1,024 steps (configs[1])
    "c2": dict(_BASE, dim=2, n_grid=128, model="fixed_corotated", gravity=3.8, steps=1024,
               loss="move_forward", target=[0.0, 0.0, 0.0], n_act=4,
               shape="robot2d", origin=(0.1, 0.03), h=1.0 / 256, seed=2),
    # C3: 3D robot, 16 muscles, 29,952 particles, 512 steps, checkpoint every 32
    "c3": dict(_BASE, dim=3, n_grid=64, model="neohookean", gravity=10.0, steps=512, k_ckpt=32,
               loss="move_forward", target=[0.0, 0.0, 0.0], n_act=16,
               shape="robot3d", origin=(0.1, 0.0625, 0.359), h=1.0 / 128, seed=3),
    # C4: 64 independent C3 episodes (shared controller), origin jitter +-0.03 in x, z
    "c4": dict(_BASE, dim=3, n_grid=64, model="neohookean", gravity=10.0, steps=512, k_ckpt=32,
               loss="move_forward", target=[0.0, 0.0, 0.0], n_act=16,
               shape="robot3d", origin=(0.1, 0.0625, 0.359), h=1.0 / 128, seed=4000,
               episodes=64, origin_jitter=0.03),
    # closed-loop variants of C2 / C3 -- the controller also sees, per muscle,
    # its mean position relative to the body's centre of mass and its mean velocity (R22)
    "c2cl": dict(_BASE, dim=2, n_grid=128, model="fixed_corotated", gravity=3.8, steps=1024,
                 loss="move_forward", target=[0.0, 0.0, 0.0], n_act=4, closed_loop=True,
                 shape="robot2d", origin=(0.1, 0.03), h=1.0 / 256, seed=2),
    "c3cl": dict(_BASE, dim=3, n_grid=64, model="neohookean", gravity=10.0, steps=512, k_ckpt=32,
                 loss="move_forward", target=[0.0, 0.0, 0.0], n_act=16, closed_loop=True,
                 shape="robot3d", origin=(0.1, 0.0625, 0.359), h=1.0 / 128, seed=3),
    # the 3D robot coupled with a block of weakly compressible liquid
    # ("a robot (30K) coupled with liquid (13K)"; R23) that falls on its body
    "c3liquid": dict(_BASE, dim=3, n_grid=64, model="neohookean", gravity=10.0, steps=512, k_ckpt=32,
                     loss="move_forward", target=[0.0, 0.0, 0.0], n_act=16,
                     shape="robot3d_liquid", origin=(0.1, 0.0625, 0.359), h=1.0 / 128, seed=6,
                     liquid_lower=(0.15, 0.34, 0.375), liquid_counts=(24, 24, 24)),
    # C5: 3D cube, 102^3 = 1,061,208 particles, 128^3 grid, 2,048 steps, k = 32
    "c5": dict(_BASE, dim=3, n_grid=128, model="neohookean", gravity=10.0, steps=2048, k_ckpt=32,
               loss="com_target", target=[0.6, 0.3, 0.5], n_act=0, hidden=0,
               shape="cube3d", lower=(0.3, 0.1, 0.3), counts=(102, 102, 102), h=1.0 / 256,
               v_base=(0.2, -1.0, 0.1), v_rank_jitter=0.05, seed=5),
}


def config(name: str, **overrides) -> dict:
    p = copy.deepcopy(CONFIGS[name])
    p.update(overrides)
    p["name"] = name
    return p


def n_theta(p: dict) -> int:
    H, S, A = int(p.get("hidden", 0)), int(p.get("n_sin", 4)), int(p.get("n_act", 0))
    if A == 0:
        return 0
    if p.get("closed_loop"):  # R22: + per-muscle observations (2d per actuator group)
        S += 2 * int(p["dim"]) * A
    return H * S + H + A * H + A if H > 0 else A * S + A


# ------------------------------------------------------------------ geometry
def _lattice(rng, lower, counts, h):
    """cell-centred lattice with spacing h and uniform jitter +-h/4 per axis."""
    axes = [lower[k] + (np.arange(counts[k]) + 0.5) * h for k in range(len(counts))]
    grid = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, len(counts))
    return grid + rng.uniform(-0.25 * h, 0.25 * h, size=grid.shape)


def _robot2d(rng, origin, h):
    """body 96h x 40h on four legs 16h x 40h at x offsets {0, 16h, 64h, 80h};
    each leg is one muscle (4 muscles), the body is passive."""
    ox, oy = origin
    parts, aids = [], []
    for j, xo in enumerate((0, 16, 64, 80)):
        parts.append(_lattice(rng, (ox + xo * h, oy), (16, 40), h))
        aids.append(np.full(16 * 40, j, np.int32))
    parts.append(_lattice(rng, (ox, oy + 40 * h), (96, 40), h))
    aids.append(np.full(96 * 40, -1, np.int32))
    return np.concatenate(parts), np.concatenate(aids)


def _robot3d(rng, origin, h):
    """body 48h x 12h x 36h on four legs 12h x 16h x 12h at the x-z corners;
    each leg split 2 x 2 in x-z into 4 muscles of 6h x 16h x 6h (16 muscles)."""
    ox, oy, oz = origin
    parts, aids = [], []
    aid = 0
    for lx in (0, 36):
        for lz in (0, 24):
            for sx in (0, 6):
                for sz in (0, 6):
                    parts.append(_lattice(rng, (ox + (lx + sx) * h, oy, oz + (lz + sz) * h),
                                          (6, 16, 6), h))
                    aids.append(np.full(6 * 16 * 6, aid, np.int32))
                    aid += 1
    parts.append(_lattice(rng, (ox, oy + 16 * h, oz), (48, 12, 36), h))
    aids.append(np.full(48 * 12 * 36, -1, np.int32))
    return np.concatenate(parts), np.concatenate(aids)


def make_inputs(p: dict | str, episode: int = 0, rank: int = 0) -> dict:
    """Initial state for one episode: x, v (N x d), C, F (N x d x d), aid (N),
    theta (n_theta).  All float arrays fp32 (rounded once from fp64)."""
    if isinstance(p, str):
        p = config(p)
    d = int(p["dim"])
    seed = int(p["seed"]) + int(episode) + int(rank)
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = p["shape"]
    if shape in ("block2d", "cube3d", "block"):
        x = _lattice(rng, p["lower"], p["counts"], p["h"])
        aid = np.full(len(x), -1, np.int32)
        if "act_ids" in p and int(p.get("n_act", 0)) > 0:  # tiny test blocks: alternate actuator ids
            aid = (np.arange(len(x)) % int(p["n_act"])).astype(np.int32)
    elif shape == "robot2d":
        x, aid = _robot2d(rng, p["origin"], p["h"])
    elif shape == "robot3d_liquid":  # robot (30K) + liquid (13K)
        x, aid = _robot3d(rng, np.array(p["origin"], np.float64), p["h"])
        xl = _lattice(rng, p["liquid_lower"], p["liquid_counts"], p["h"])
        mat = np.concatenate([np.zeros(len(x), np.int32), np.ones(len(xl), np.int32)])
        x = np.concatenate([x, xl])
        aid = np.concatenate([aid, np.full(len(xl), -1, np.int32)])
    elif shape == "robot3d":
        origin = np.array(p["origin"], np.float64)
        if p.get("origin_jitter"):
            j = p["origin_jitter"]
            origin = origin + np.array([rng.uniform(-j, j), 0.0, rng.uniform(-j, j)])
        x, aid = _robot3d(rng, origin, p["h"])
    else:
        raise ValueError(shape)
    N = len(x)
    if shape != "robot3d_liquid":
        mat = np.zeros(N, np.int32)
        if p.get("fluid_every"):  # tiny mixed blocks: every k-th particle is fluid (and passive)
            mat[:: int(p["fluid_every"])] = 1
            aid = np.where(mat == 1, -1, aid).astype(np.int32)
    v = np.zeros((N, d))
    if "v_base" in p:
        vb = np.array(p["v_base"][:d], np.float64)
        if p.get("v_rank_jitter") and rank:
            vb = vb + rng.uniform(-p["v_rank_jitter"], p["v_rank_jitter"], size=d)
        v += vb
    if p.get("spin"):
        r = x - x.mean(axis=0)
        v[:, 0] += -p["spin"] * r[:, 1]
        v[:, 1] += p["spin"] * r[:, 0]
    if p.get("v_noise"):
        v += rng.normal(0.0, p["v_noise"], size=v.shape)
    C = np.zeros((N, d, d))
    if p.get("C_noise"):
        C += rng.normal(0.0, p["C_noise"], size=C.shape)
    F = np.broadcast_to(np.eye(d), (N, d, d)).copy()
    if p.get("F_noise"):
        F += rng.normal(0.0, p["F_noise"], size=F.shape)
    th_rng = np.random.Generator(np.random.PCG64(int(p["seed"]) + 7919))  # shared across episodes
    theta = th_rng.normal(0.0, p.get("theta_std", 0.01), size=n_theta(p))
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return dict(x=f32(x), v=f32(v), C=f32(C), F=f32(F), aid=np.ascontiguousarray(aid, np.int32),
                mat=np.ascontiguousarray(mat, np.int32),
                theta=f32(theta))


def tiny(dim: int, n_particles: int | None = None, model: str | None = None, n_grid: int = 8,
         bound: int = 1, steps: int = 8, seed: int = 0, n_act: int = 2, hidden: int = 0,
         floor: bool = False, **kw) -> dict:
    """Tiny configurations for finite-difference pins (2-8 particles, 8^d grid)."""
    model = model or ("fixed_corotated" if dim == 2 else "neohookean")
    n_particles = n_particles or (6 if dim == 2 else 8)
    counts = {(2, 6): (3, 2), (2, 4): (2, 2), (3, 8): (2, 2, 2), (3, 4): (2, 2, 1)}.get((dim, n_particles))
    if counts is None:
        raise ValueError("tiny() supports 4 or 6 (2D) and 4 or 8 (3D) particles")
    h = 1.0 / (2 * n_grid)
    lower = tuple([0.44] * dim)
    if floor:
        lower = tuple([0.44] + [0.2] + [0.44] * (dim - 2))
    p = dict(_BASE, dim=dim, n_grid=n_grid, model=model, gravity=3.8 if dim == 2 else 10.0,
             steps=steps, bound=bound, loss="com_target", target=[0.5, 0.5, 0.5][:3],
             n_act=n_act, hidden=hidden, shape="block", lower=lower, counts=counts, h=h,
             v_base=tuple([0.3, -0.2, 0.1][:dim]), spin=1.0, v_noise=0.2, C_noise=0.5,
             F_noise=0.05, theta_std=0.5, seed=seed, act_ids=True, name=f"tiny{dim}d")
    p.update(kw)
    return p
