"""Weakly compressible fluid particles (R23) on the CUDA path vs
the fp64 CPU oracle, through the C-ABI (mpm_set_materials), on the same seeded inputs."""
import numpy as np
import pytest

from helpers import check, compare_arrays, compare_episode, gpu_run, inputs, oracle_tape
from paper_1910_00935_b200 import workloads as W

pytestmark = pytest.mark.gpu

TINY = {
    "2d_fcr_mixed_floor": lambda: W.tiny(2, steps=10, hidden=3, seed=12, fluid_every=2, bound=3, floor=True,
                                         v_base=(0.3, -1.5)),
    "3d_nh_mixed": lambda: W.tiny(3, steps=6, hidden=0, seed=13, fluid_every=3),
    "2d_nh_all_fluid": lambda: W.tiny(2, steps=8, model="neohookean", seed=14, fluid_every=1, n_act=0),
}


@pytest.mark.parametrize("case", list(TINY))
def test_tiny_fluid_every_adjoint_path(case):
    p = TINY[case]()
    inp = W.make_inputs(p)
    assert inp["mat"].any()
    N, d = inp["x"].shape
    rng = np.random.default_rng(17)
    lam = [rng.standard_normal((N, d)), rng.standard_normal((N, d)),
           rng.standard_normal((N, d, d)), rng.standard_normal((N, d, d))]
    lam = [l.astype(np.float32) for l in lam]
    ref = oracle_tape(p, inp, p["steps"], lam)
    got = gpu_run(p, inp, seed=lam)
    pairs = {k: (got[k][0], ref[k]) for k in "xvCF"}
    pairs.update({k: (got[k].reshape(ref[k].shape), ref[k]) for k in ("dx0", "dv0", "dC0", "dF0", "dtheta")
                  if ref[k].size})
    check(compare_arrays(f"tiny_fluid/{case}", pairs), case)
    # the fluid particles' F is isotropic after every step (R23)
    F = got["F"][0][inp["mat"] == 1]
    off = F - np.einsum("nii->n", F)[:, None, None] / d * np.eye(d)
    assert np.abs(off).max() < 1e-6 * np.abs(F).max()


def test_fluid_checkpoint_invariant_and_reproducible():
    """the segment re-forward applies the same F reset bit for bit (k = 1 vs k = 4)."""
    p = W.tiny(3, steps=12, hidden=3, seed=15, fluid_every=2, bound=3, floor=True, v_base=(0.2, -1.5, 0.1))
    inp = W.make_inputs(p)
    a = gpu_run(p, inp, k_ckpt=1)
    b = gpu_run(p, inp, k_ckpt=4)
    c = gpu_run(p, inp, k_ckpt=4)
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
        np.testing.assert_array_equal(b[k], c[k], err_msg=k)


def _shared_nodes(x, mat, n_grid):
    """grid nodes inside the 3^d stencils of both a solid and a fluid particle"""
    b = np.floor(x.astype(np.float64) * n_grid - 0.5).astype(np.int64)
    d = x.shape[1]
    offs = np.stack(np.meshgrid(*[np.arange(3)] * d, indexing="ij"), -1).reshape(-1, d)

    def nodes(bb):
        n = (bb[:, None, :] + offs[None]).reshape(-1, d)
        return set(map(tuple, np.unique(n, axis=0)))
    return len(nodes(b[mat == 0]) & nodes(b[mat != 0]))


def test_robot3d_with_liquid_c3liquid_coupled():
    """P:612's robot (30K) coupled with liquid (13.8K), 176 steps, k = 32: the liquid has landed
    on the robot (solid and fluid particles share hundreds of grid nodes -- two-way coupling
    through the shared grid), states and gradients vs the oracle."""
    T = 176
    p, inp = inputs("c3liquid", steps=T)
    got = gpu_run(p, inp, k_ckpt=32)
    rows, ref = compare_episode("c3liquid@176", p, inp, got, grads=("dx0", "dv0", "dtheta"))
    check(rows, "c3liquid")
    shared = _shared_nodes(ref["x"], inp["mat"], p["n_grid"])
    print(f"[parity] c3liquid@176: solid and fluid share {shared} grid nodes")
    assert shared > 100


def test_clearing_materials_restores_the_solid_run():
    """mpm_set_materials(NULL) after a fluid run gives the all-solid results bit for bit."""
    from paper_1910_00935_b200 import mpm
    p = W.tiny(2, steps=6, hidden=3, seed=21, fluid_every=2)
    inp = W.make_inputs(p)
    N = len(inp["x"])

    def run(mat):
        sim = mpm.sim_from_config(p, N, max_steps=6)
        sim.set_state(inp["x"][None], inp["v"][None], inp["C"][None], inp["F"][None], inp["aid"][None])
        sim.set_controller(inp["theta"])
        if mat is not None:
            sim.set_materials(mat)
            sim.set_materials(None)
        sim.forward(6)
        sim.loss()
        sim.backward(6)
        out = {**sim.get_state(), **sim.grads()}
        sim.close()
        return out

    a, b = run(None), run(inp["mat"][None])
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
