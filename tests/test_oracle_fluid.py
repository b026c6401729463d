"""Pins of the oracle's weakly compressible fluid material (R23).

R23: a fluid particle keeps only the volumetric term of the material model (mu = 0:
NH -> tau = lambda ln J I, FCR -> tau = lambda (J - 1) J I) and, after the deformation update,
forgets its shear: F_{t+1} = J^(1/d) I with J = det((I + dt C) F).  Pinned by
* the P2G stress-scale identity (4/dx^2) sum_i P_i delta_i^T = -dt V (4/dx^2) tau + m C
  (the same identity that pins the solid's stress) against the closed-form fluid stress, for an
  arbitrary (sheared, rotated) F: the fluid's stress depends on J alone;
* the F reset against its closed form;
* whole-trajectory central differences with mixed solid / fluid particles (2D FCR, 3D NH), so
  the reset's and the mu = 0 stress's adjoints are checked.
"""
import numpy as np
import pytest

from oracle import Oracle
from paper_1910_00935_b200 import workloads as W


def _one_particle(dim, model, F, C=None):
    p = W.tiny(dim, model=model, n_act=0, hidden=0)
    o = Oracle(p)
    o.set_materials([1])
    x = np.full((1, dim), 0.5 + 0.3 / p["n_grid"])
    v = np.zeros((1, dim))
    C = np.zeros((1, dim, dim)) if C is None else C
    return p, o, x, v, C, F[None]


@pytest.mark.parametrize("dim,model", [(2, "fixed_corotated"), (2, "neohookean"), (3, "neohookean")])
def test_fluid_stress_is_volumetric_only(dim, model):
    rng = np.random.default_rng(4)
    F = np.eye(dim) + 0.2 * rng.standard_normal((dim, dim))
    if np.linalg.det(F) < 0.2:
        F = F + 0.5 * np.eye(dim)
    p, o, x, v, C, Fb = _one_particle(dim, model, F)
    grid, _ = o.p2g(x, v, C, Fb)
    n, dx = p["n_grid"], 1.0 / p["n_grid"]
    idx = np.indices([n] * dim).reshape(dim, -1).T * dx
    dpos = idx - x[0]
    M2 = (4 / dx ** 2) * (grid[:, :dim].T @ dpos)  # = A = -dt V (4/dx^2) tau (C = 0, v = 0)
    mu, lam = o.lame()
    Ft = F  # C = 0: (I + dt C) F = F
    J = np.linalg.det(Ft)
    vol = lam * np.log(J) if model == "neohookean" else lam * (J - 1) * J
    A = -p["dt"] * p["p_vol"] * 4 / dx ** 2 * vol * np.eye(dim)
    np.testing.assert_allclose(M2, A, rtol=1e-10, atol=1e-12 * np.abs(A).max())


@pytest.mark.parametrize("dim", [2, 3])
def test_fluid_F_reset(dim):
    rng = np.random.default_rng(5)
    F = np.eye(dim) + 0.1 * rng.standard_normal((dim, dim))
    C = 3.0 * rng.standard_normal((1, dim, dim))
    p, o, x, v, C, Fb = _one_particle(dim, "neohookean" if dim == 3 else "fixed_corotated", F, C)
    _, Fn = o.p2g(x, v, C, Fb)
    J = np.linalg.det((np.eye(dim) + p["dt"] * C[0]) @ F)
    np.testing.assert_allclose(Fn[0], J ** (1.0 / dim) * np.eye(dim), rtol=1e-13, atol=1e-15)
    # a solid particle keeps (I + dt C) F
    o.set_materials([0])
    _, Fs = o.p2g(x, v, C, Fb)
    np.testing.assert_allclose(Fs[0], (np.eye(dim) + p["dt"] * C[0]) @ F, rtol=1e-13)


FD_FLUID = {
    "2d_fcr_mixed": lambda: W.tiny(2, steps=10, hidden=3, seed=12, fluid_every=2, bound=3, floor=True,
                                   v_base=(0.3, -1.5)),
    "3d_nh_mixed": lambda: W.tiny(3, steps=6, hidden=0, seed=13, fluid_every=3),
}


@pytest.mark.parametrize("case", list(FD_FLUID))
def test_mixed_material_trajectory_fd(case):
    """Central differences (h = 1e-6, fp64) of a random linear loss <lam, S_T> w.r.t. every
    element of x0, v0, C0, F0 and theta vs the reverse sweep (rel <= 1e-6)."""
    from test_oracle_pins import _fwd_loss, _tape
    p = FD_FLUID[case]()
    inp = {k: (v.astype(np.float64) if v.dtype == np.float32 else v) for k, v in W.make_inputs(p).items()}
    assert inp["mat"].any() and not inp["mat"].all()
    o = Oracle(p).set_materials(inp["mat"])
    rng = np.random.default_rng(31)
    T = p["steps"]
    N, d = inp["x"].shape
    lam = [rng.standard_normal((N, d)), rng.standard_normal((N, d)),
           rng.standard_normal((N, d, d)), rng.standard_normal((N, d, d))]
    L, bars, thb = _tape(o, inp, T, lam)
    grads = dict(zip("xvCF", bars)); grads["theta"] = thb
    h = 1e-6
    for key in ["x", "v", "C", "F", "theta"]:
        arr = inp[key]
        g = grads[key].ravel()
        fd = np.zeros(arr.size)
        for i in range(arr.size):
            ip, im = dict(inp), dict(inp)
            ap = arr.copy().ravel(); ap[i] += h
            am = arr.copy().ravel(); am[i] -= h
            ip[key] = ap.reshape(arr.shape); im[key] = am.reshape(arr.shape)
            fd[i] = (_fwd_loss(o, ip, T, lam) - _fwd_loss(o, im, T, lam)) / (2 * h)
        err = np.linalg.norm(fd - g) / max(np.linalg.norm(fd), 1e-300)
        assert err < 1e-6, (case, key, err)


def test_all_solid_materials_change_nothing():
    p = W.tiny(2, steps=8, hidden=3, seed=2)
    inp = W.make_inputs(p)
    a = Oracle(p).run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"])
    b = Oracle(p).set_materials(np.zeros(len(inp["x"]))).run(inp["x"], inp["v"], inp["C"], inp["F"],
                                                               inp["aid"], inp["theta"])
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta"):
        np.testing.assert_array_equal(a[k], b[k])
