"""CUDA path (through the C-ABI) vs the fp64 CPU oracle, element by element on
the same seeded inputs.  Gates (BASELINE.json north_star): final particle
states rel <= 1e-4 (per array, ||d||/||ref||), gradients rel-L2 <= 1e-3, plus an
element-wise bound max|d|/max|ref| <= 10x those; every comparison is recorded
(tests/helpers.py: record)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from helpers import (GRAD_TOL, check, compare_arrays, compare_episode, gpu_run, inputs, oracle_pair,
                     oracle_run, oracle_tape, rel)
from paper_1910_00935_b200 import workloads as W

pytestmark = pytest.mark.gpu

TINY = {
    "2d_fcr_act_hidden": lambda: W.tiny(2, steps=12, hidden=4, seed=1),
    "3d_nh_act": lambda: W.tiny(3, steps=5, seed=2),
    "2d_fcr_sticky_floor": lambda: W.tiny(2, steps=10, bound=3, seed=3, floor=True, v_base=(0.3, -1.5)),
    "2d_nh": lambda: W.tiny(2, steps=8, model="neohookean", seed=4),
    "3d_nh_hidden_floor": lambda: W.tiny(3, steps=10, hidden=3, bound=3, seed=6, floor=True,
                                         v_base=(0.2, -1.5, 0.1)),
}


@pytest.mark.parametrize("case", list(TINY))
def test_tiny_every_adjoint_path(case):
    """Seed every component of S_T (L = <lam, S_T>) so every adjoint path
    (x, v, C, F, theta) is exercised; compare with the oracle's tape."""
    p = TINY[case]()
    inp = W.make_inputs(p)
    N, d = inp["x"].shape
    rng = np.random.default_rng(7)
    lam = [rng.standard_normal((N, d)), rng.standard_normal((N, d)),
           rng.standard_normal((N, d, d)), rng.standard_normal((N, d, d))]
    lam = [l.astype(np.float32) for l in lam]
    ref = oracle_tape(p, inp, p["steps"], lam)
    got = gpu_run(p, inp, seed=lam)
    pairs = {k: (got[k][0], ref[k]) for k in "xvCF"}
    pairs.update({k: (got[k].reshape(ref[k].shape), ref[k]) for k in ("dx0", "dv0", "dC0", "dF0", "dtheta")})
    check(compare_arrays(f"tiny/{case}", pairs), case)


@pytest.mark.parametrize("name", ["c1a", "c1b"])
def test_block_full_horizon(name):
    p, inp = inputs(name)
    got = gpu_run(p, inp)
    rows, ref = compare_episode(name, p, inp, got, grads=("dx0", "dv0"))
    check(rows, name)
    if name == "c1a":  # no wall contact: closed form dL/dC0 = dL/dF0 = 0
        scale = np.abs(got["dv0"]).max()
        assert np.abs(got["dC0"]).max() < 1e-3 * scale and np.abs(got["dF0"]).max() < 1e-3 * scale


def test_robot2d_c2_full_horizon():
    p, inp = inputs("c2")
    got = gpu_run(p, inp)
    rows, _ = compare_episode("c2@1024", p, inp, got, grads=("dx0", "dv0", "dtheta"))
    check(rows, "c2")


def test_robot3d_c3_full_horizon_checkpointed():
    """C3 at its full horizon (SURVEY 8(c) "Parity gates"; "512~2048 time steps"): 3D robot,
    16 muscles, H = 32, 512 steps with k = 32 (16 segments)."""
    p, inp = inputs("c3")
    assert p["steps"] == 512
    got = gpu_run(p, inp, k_ckpt=32)
    rows, ref = compare_episode("c3@512", p, inp, got, grads=("dx0", "dv0", "dtheta"))
    check(rows, "c3")
    assert np.linalg.norm(ref["dtheta"]) > 1e-4  # the robot walks: theta_bar is not rounding noise


def test_batched_episodes_c4_post_contact():
    """4 independent C4 episodes in one launch, 128 steps (k = 32): past the landing, so each
    episode's theta_bar is ~1e-3 (not the ~1e-9 rounding noise of a body still in free fall).
    Per-episode states / initial-state gradients and the summed controller gradient equal the
    per-episode oracle runs."""
    T = 128
    p = W.config("c4", steps=T)
    inps = [W.make_inputs(p, episode=e) for e in range(4)]
    got = gpu_run(p, inps, k_ckpt=32)
    with ThreadPoolExecutor(8) as ex:
        futs = [ex.submit(oracle_run, p, inp, T, prec) for inp in inps for prec in ("f64", "f32")]
        res = [f.result() for f in futs]
    dth = dth32 = 0
    for e in range(4):
        ref, ref32 = res[2 * e], res[2 * e + 1]
        assert np.linalg.norm(ref["dtheta"]) > 1e-4, e
        rows, _ = compare_episode("c4@128", p, inps[e], got, e=e, grads=("dx0", "dv0"), refs=(ref, ref32))
        check(rows, f"c4[{e}]")
        dth = dth + ref["dtheta"]
        dth32 = dth32 + ref32["dtheta"]
    rows = compare_arrays("c4@128/sum_dtheta", {"dtheta": (got["dtheta"], dth)},
                          {"dtheta": (rel(dth32, dth), 0.0)})
    check(rows, "c4 sum dtheta")


@pytest.mark.parametrize("k", [1, 7, 64])
def test_checkpoint_interval_invariance(k):
    """Segment size does not change the result: every reduction has a
    fixed order, so the gradients are bitwise equal for any k (SPEC S:333 pattern)."""
    p, inp = inputs("c3", steps=64)
    base = gpu_run(p, inp, k_ckpt=64)
    got = gpu_run(p, inp, k_ckpt=k)
    for key in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta", "loss"):
        assert np.array_equal(got[key], base[key]), (k, key, rel(got[key], base[key]))


def test_bitwise_run_to_run_and_batch_invariance():
    """Same inputs twice -> identical bytes; an episode's results do not depend
    on the other episodes batched with it."""
    p = W.config("c4", steps=24)
    inps = [W.make_inputs(p, episode=e) for e in range(3)]
    a = gpu_run(p, inps, k_ckpt=8)
    b = gpu_run(p, inps, k_ckpt=8)
    for key in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta", "loss"):
        assert np.array_equal(a[key], b[key]), key
    solo = gpu_run(p, inps[1:2], k_ckpt=8)
    for key in ("x", "dx0", "dv0", "dF0"):
        assert np.array_equal(solo[key][0], a[key][1]), key


def test_particle_order_invariance():
    """Permuting the caller's particle order permutes the outputs (R20), up to fp32
    reassociation: the particle id (= caller index) orders the particles inside a cell,
    so a permutation changes only the order of equal-cell terms in the node sums."""
    p, inp = inputs("c1b", steps=32)
    base = gpu_run(p, inp)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(inp["x"]))
    pin = {k: (v[perm] if k != "theta" else v) for k, v in inp.items()}
    got = gpu_run(p, pin)
    for key in ("x", "v", "dx0", "dv0"):
        assert rel(got[key][0], base[key][0][perm]) < 1e-5, key


def test_c5_full_size_one_step():
    """Full C5 size (1,061,208 particles, 128^3 grid), the launch configuration
    bench.py times: one forward step and one reverse step vs the oracle on every
    particle (fp64 oracle on the GPU's fp32 input).  The initial state is
    perturbed (velocity, affine and deformation noise) so that every term of the
    step -- stress, affine momentum, the adjoints -- is non-trivial."""
    p, inp = inputs("c5", steps=1, v_noise=0.3, C_noise=2.0, F_noise=0.02)
    N, d = inp["x"].shape
    rng = np.random.default_rng(3)
    lam = [rng.standard_normal((N, d)).astype(np.float32),
           rng.standard_normal((N, d)).astype(np.float32),
           rng.standard_normal((N, d, d)).astype(np.float32),
           rng.standard_normal((N, d, d)).astype(np.float32)]
    got = gpu_run(p, inp, steps=1, k_ckpt=32, seed=lam)
    ref = oracle_tape(p, inp, 1, lam)
    for k in "xvCF":
        assert rel(got[k][0], ref[k]) < 1e-5, k
    for k in ("dx0", "dv0", "dC0", "dF0"):
        assert rel(got[k][0], ref[k]) < 1e-4, k


def test_c5_full_size_ballistic_and_closed_form():
    """Before the cube reaches the floor (T = 40) the centre of mass is exactly
    ballistic and dL/dv0 has the closed form 2(xbar_T - x*) T dt / N for every
    particle (properties that hold at any size)."""
    T = 40
    p, inp = inputs("c5", steps=T)
    got = gpu_run(p, inp, steps=T, k_ckpt=8)
    x0 = inp["x"].astype(np.float64).mean(0)
    v0 = inp["v"].astype(np.float64).mean(0)
    dt, g = p["dt"], p["gravity"]
    pred = x0 + T * dt * v0 - np.array([0.0, dt * dt * g * T * (T + 1) / 2, 0.0])
    com = got["x"][0].astype(np.float64).mean(0)
    assert np.abs(com - pred).max() < 2e-6
    N = len(inp["x"])
    gexp = 2 * (com - np.array(p["target"])) * T * dt / N
    assert rel(got["dv0"][0], np.tile(gexp, (N, 1))) < GRAD_TOL
    assert got["x"][0][:, 1].min() > 3.0 / 128 + 1.0 / 128  # no floor contact yet


def test_error_paths():
    from paper_1910_00935_b200 import mpm
    p = W.tiny(3, steps=4)
    inp = W.make_inputs(p)
    N = len(inp["x"])
    sim = mpm.sim_from_config(p, N, max_steps=4)
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(1)
    assert e.value.status == 6  # forward before set_state
    x = inp["x"].copy()
    x[0, 0] = 0.01  # stencil leaves the grid
    sim.set_state(x, inp["v"], inp["C"], inp["F"], inp["aid"])
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(2)
    assert e.value.status == 4
    F = inp["F"].copy()
    F[1] = np.diag([1.0, 1.0, -1.0])  # J < 0 under Neo-Hookean
    sim.set_state(inp["x"], inp["v"], inp["C"], F, inp["aid"])
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(2)
    assert e.value.status == 5
    sim.set_state(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"])
    sim.forward(3)
    with pytest.raises(mpm.MpmError) as e:
        sim.backward(3)  # no loss / seed yet
    assert e.value.status == 6
    sim.loss()
    with pytest.raises(mpm.MpmError) as e:
        sim.backward(2)  # != recorded steps
    assert e.value.status == 6
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(5)  # > max_steps
    assert e.value.status == 1
    sim.close()


def test_active_block_capacity_is_an_error():
    from paper_1910_00935_b200 import mpm
    p, inp = inputs("c1a", steps=4)
    sim = mpm.sim_from_config(p, len(inp["x"]), max_steps=4, max_active_blocks=2)
    sim.set_state(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"])
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(4)
    assert e.value.status == 2
    sim.close()


def test_cuda_graph_replay_is_bitwise_identical():
    """forward/backward tapes captured as CUDA graphs on a side stream (and replayed on
    the second iteration) give the same bytes as eager launches on the default stream"""
    import torch
    p = W.config("c4", steps=40)
    inps = [W.make_inputs(p, episode=e) for e in range(2)]
    eager = gpu_run(p, inps, k_ckpt=8)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g1 = gpu_run(p, inps, k_ckpt=8)
    for key in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta", "loss"):
        assert np.array_equal(eager[key], g1[key]), key
    from paper_1910_00935_b200 import mpm
    with torch.cuda.stream(s):  # same handle twice: the second iteration replays the graphs
        N = len(inps[0]["x"])
        sim = mpm.sim_from_config(p, N, episodes=2, max_steps=40, k_ckpt=8)
        cat = lambda k: np.ascontiguousarray(np.stack([i[k] for i in inps]))  # noqa: E731
        outs = []
        for _ in range(2):
            sim.set_state(cat("x"), cat("v"), cat("C"), cat("F"), cat("aid"))
            sim.set_controller(inps[0]["theta"])
            sim.forward(40)
            sim.loss()
            sim.backward(40)
            outs.append(sim.grads())
        sim.close()
    for key in ("dx0", "dv0", "dtheta"):
        assert np.array_equal(outs[0][key], outs[1][key]) and np.array_equal(outs[0][key], eager[key]), key


def test_native_library_is_what_runs():
    """the kernels launched are ours (launch counter of libmpm_b200.so)"""
    p, inp = inputs("c1a", steps=8)
    got = gpu_run(p, inp, steps=8)
    assert got["launches"] >= 8 * 4 + 8 * 2


def test_block_particle_overflow_is_an_error():
    """more than 1728 particles (27 per cell on average) in one 4^3 block: MPM_ERR_UNSUPPORTED,
    never a silent drop (mpm.h)."""
    from paper_1910_00935_b200 import mpm
    p = W.tiny(3, steps=2, n_act=0, hidden=0, bound=1)
    rng = np.random.default_rng(3)
    N = 1800
    x = (0.3125 + 0.25 * rng.random((N, 3))).astype(np.float32)  # base cells 2..3: all in block 0
    v = np.zeros((N, 3), np.float32)
    C = np.zeros((N, 3, 3), np.float32)
    F = np.broadcast_to(np.eye(3, dtype=np.float32), (N, 3, 3)).copy()
    sim = mpm.sim_from_config(p, N, max_steps=2)
    sim.set_state(x, v, C, F, None)
    with pytest.raises(mpm.MpmError) as e:
        sim.forward(2)
    assert e.value.status == 7
    sim.close()


def test_c5_full_size_64_steps_through_landing():
    """SURVEY 8(c) horizons: C5 at full size (1,061,208 particles, 128^3) for 64 steps with the
    checkpoint interval the bench uses (k = 2) -- the cube lands on the sticky floor near step
    50, so contact, the select rule and the re-forward are all exercised -- vs the fp64 oracle
    on every particle (states, L, dL/dx0, dL/dv0).  ~6 min of CPU oracle (fp64 and fp32 builds
    in two threads)."""
    p, inp = inputs("c5", steps=64)
    got = gpu_run(p, inp, steps=64, k_ckpt=2)
    rows, ref = compare_episode("c5@64", p, inp, got, steps=64, grads=("dx0", "dv0"))
    check(rows, "c5@64")
    assert ref["x"][:, 1].min() < 3.5 / 128  # it did reach the floor


def test_dense_2d_block_multi_chunk():
    """2D blocks holding more than one shared-memory chunk of particle rows (> 576 particles in an
    8^2-cell block: ~12 particles per cell at h = dx / 3.5), so p2g's and the U_bar scatter's
    chunk loops run more than once: states and gradients vs the oracle, and checkpoint invariance."""
    p = W.config("c1a", steps=32, counts=(56, 56), h=1.0 / 224)
    inp = W.make_inputs(p)
    x = inp["x"].astype(np.float32)
    b = np.floor(x * np.float32(64) - np.float32(0.5)).astype(np.int64) // 8
    _, per_block = np.unique(b[:, 0] * 8 + b[:, 1], return_counts=True)
    assert per_block.max() > 576 and per_block.max() <= 1728, per_block.max()
    got = gpu_run(p, inp)
    rows, _ = compare_episode("c1a_dense2d@32", p, inp, got, grads=("dx0", "dv0", "dC0", "dF0"))
    check(rows, "dense2d")
    got4 = gpu_run(p, inp, k_ckpt=4)
    for key in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "loss"):
        assert np.array_equal(got[key], got4[key]), key


def test_binning_scan_beside_a_concurrent_kernel():
    """The one-launch binning scan looks back only over chunks whose CTAs started earlier (atomic
    chunk tickets), so it makes progress whatever else occupies the SMs: a C4 batch (16 episodes,
    65,536 grid blocks -> 64 scan chunks per step) runs while another stream keeps the GPU busy
    with large matmuls, finishes, and gives the same bytes as a solo run."""
    import torch
    p = W.config("c4", steps=24)
    inps = [W.make_inputs(p, episode=e) for e in range(16)]
    solo = gpu_run(p, inps, k_ckpt=8)
    other = torch.cuda.Stream()
    a = torch.randn(8192, 8192, device="cuda")
    with torch.cuda.stream(other):
        for _ in range(40):
            a = torch.tanh(a @ a * 1e-4)
    busy = gpu_run(p, inps, k_ckpt=8)
    torch.cuda.synchronize()
    for key in ("x", "v", "C", "F", "dx0", "dv0", "dtheta", "loss"):
        assert np.array_equal(solo[key], busy[key]), key


def test_workspace_bytes_for_steps():
    """mpm_workspace_bytes_for(steps) (SURVEY 8(b)'s form) sizes a tape of `steps` without changing
    the handle: equal to mpm_workspace_bytes at max_steps, growing with steps."""
    import ctypes as ct
    from paper_1910_00935_b200 import mpm
    p = W.config("c3", steps=64)
    sim = mpm.sim_from_config(p, 29952, max_steps=64, k_ckpt=1, probe_only=True)
    L = mpm.load()
    b64, b128, b1 = ct.c_size_t(), ct.c_size_t(), ct.c_size_t()
    assert L.mpm_workspace_bytes_for(sim.h, 64, ct.byref(b64)) == 0
    assert L.mpm_workspace_bytes_for(sim.h, 128, ct.byref(b128)) == 0
    assert L.mpm_workspace_bytes_for(sim.h, 1, ct.byref(b1)) == 0
    assert b64.value == sim.workspace_bytes and b1.value < b64.value < b128.value
    assert L.mpm_workspace_bytes_for(sim.h, 0, ct.byref(b1)) == 1
    now = ct.c_size_t()
    assert L.mpm_workspace_bytes(sim.h, ct.byref(now)) == 0 and now.value == sim.workspace_bytes
    sim.close()
