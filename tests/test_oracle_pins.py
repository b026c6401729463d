"""Pins of the CPU oracle against things other than itself (CPU only).

Each test checks the oracle against a closed form, an invariant of the
discrete method, a hand-evaluated fixture (tests/golden/) or central finite
differences of the oracle's own FORWARD map (which pins the separately
hand-written reverse).  A plausible mistake anywhere (a dropped term, a
wrong sign or index, a transposed operand) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

from oracle import Oracle, OracleError
from paper_1910_00935_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line.split())
    return rows


def _cfg2(**kw):
    return W.tiny(2, **kw)


def _cfg3(**kw):
    return W.tiny(3, n_particles=8, **kw)


# ---------------------------------------------------------------- B-spline
def test_bspline_golden_values():
    o = Oracle(_cfg2())
    for row in _golden_rows("bspline_weights.txt"):
        f, *vals = map(float, row)
        w, dw = o.bspline(f)
        np.testing.assert_allclose(w, vals[:3], atol=1e-15)
        np.testing.assert_allclose(dw, vals[3:], atol=1e-15)


def test_bspline_moments_and_derivative():
    """sum w = 1, sum w (o - f) = 0, sum w (o - f)^2 = 1/4 for all f in [1/2, 3/2);
    dw matches central differences of w."""
    o = Oracle(_cfg2())
    o_ = np.arange(3.0)
    for f in np.linspace(0.5, 1.4999, 37):
        w, dw = o.bspline(f)
        assert abs(w.sum() - 1) < 1e-14
        assert abs((w * (o_ - f)).sum()) < 1e-14
        assert abs((w * (o_ - f) ** 2).sum() - 0.25) < 1e-14
        h = 1e-6
        wp, _ = o.bspline(f + h)
        wm, _ = o.bspline(f - h)
        np.testing.assert_allclose((wp - wm) / (2 * h), dw, atol=1e-8)


# --------------------------------------------------------------- material
def test_lame_golden():
    (row,) = [r for r in _golden_rows("closed_forms.txt") if r[0] == "lame"]
    E, nu, mu, lam = map(float, row[1:])
    o = Oracle(_cfg2(E=E, nu=nu))
    assert o.lame() == pytest.approx((mu, lam), rel=1e-14)


def test_stress_closed_forms():
    rows = {r[0]: list(map(float, r[1:])) for r in _golden_rows("closed_forms.txt")}
    # rest state is stress free (both models)
    for cfg in (_cfg2(model="fixed_corotated"), _cfg2(model="neohookean"), _cfg3()):
        o = Oracle(cfg)
        assert np.abs(o.stress(np.eye(o.d))).max() < 1e-14
    o = Oracle(_cfg2(model="fixed_corotated"))
    s0, s1, t0, t1 = rows["fcr_diag"]
    tau = o.stress(np.diag([s0, s1]))
    np.testing.assert_allclose(np.diag(tau), [t0, t1], rtol=1e-12)
    assert abs(tau[0, 1]) < 1e-14 and abs(tau[1, 0]) < 1e-14
    o = Oracle(_cfg3())
    s, t = rows["nh_uniform3"]
    np.testing.assert_allclose(o.stress(s * np.eye(3)), t * np.eye(3), rtol=1e-8, atol=1e-14)


@pytest.mark.parametrize("dim,model", [(2, "fixed_corotated"), (2, "neohookean"), (3, "neohookean")])
def test_stress_is_energy_gradient(dim, model):
    """tau = (d psi / d F) F^T, with d psi/dF by central differences of the
    strain energy (hyperelastic definition of the Kirchhoff stress)."""
    cfg = _cfg2(model=model) if dim == 2 else _cfg3()
    o = Oracle(cfg)
    rng = np.random.default_rng(3)
    for _ in range(5):
        F = np.eye(dim) + 0.2 * rng.standard_normal((dim, dim))
        P = np.zeros((dim, dim))
        h = 1e-6
        for i in range(dim):
            for j in range(dim):
                E = np.zeros((dim, dim)); E[i, j] = h
                P[i, j] = (o.energy(F + E) - o.energy(F - E)) / (2 * h)
        np.testing.assert_allclose(o.stress(F), P @ F.T, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("dim,model", [(2, "fixed_corotated"), (2, "neohookean"), (3, "neohookean")])
def test_stress_rotation_covariance(dim, model):
    cfg = _cfg2(model=model) if dim == 2 else _cfg3()
    o = Oracle(cfg)
    rng = np.random.default_rng(5)
    F = np.eye(dim) + 0.2 * rng.standard_normal((dim, dim))
    Q, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    np.testing.assert_allclose(o.stress(Q @ F), Q @ o.stress(F) @ Q.T, atol=1e-12)


@pytest.mark.parametrize("dim,model", [(2, "fixed_corotated"), (2, "neohookean"), (3, "neohookean")])
def test_stress_adjoint_fd(dim, model):
    cfg = _cfg2(model=model) if dim == 2 else _cfg3()
    o = Oracle(cfg)
    rng = np.random.default_rng(7)
    for _ in range(5):
        F = np.eye(dim) + 0.3 * rng.standard_normal((dim, dim))
        tb = rng.standard_normal((dim, dim))
        Fb = o.stress_adj(F, tb)
        h = 1e-6
        for i in range(dim):
            for j in range(dim):
                E = np.zeros((dim, dim)); E[i, j] = h
                fd = (np.sum(tb * o.stress(F + E)) - np.sum(tb * o.stress(F - E))) / (2 * h)
                assert abs(fd - Fb[i, j]) < 1e-6 * (1 + abs(fd))


def test_degenerate_deformation_errors():
    o = Oracle(_cfg3())
    with pytest.raises(OracleError) as e:
        o.stress(np.diag([1.0, 1.0, -0.5]))
    assert e.value.status == 5
    o = Oracle(_cfg2(model="fixed_corotated"))
    with pytest.raises(OracleError):
        o.stress(np.array([[1.0, 0.0], [0.0, -1.0]]))  # a = b = 0 -> r = 0


# ------------------------------------------------------------- controller
@pytest.mark.parametrize("hidden", [0, 4])
def test_controller_adjoint_fd(hidden):
    cfg = _cfg2(hidden=hidden, n_act=3)
    o = Oracle(cfg)
    rng = np.random.default_rng(11)
    th = rng.standard_normal(o.n_theta()) * 0.7
    ab = rng.standard_normal(3)
    for t in (0, 5, 17):
        g = o.controller_adj(th, t, ab)
        h = 1e-6
        for i in range(len(th)):
            e = np.zeros_like(th); e[i] = h
            fd = (ab @ o.controller(th + e, t) - ab @ o.controller(th - e, t)) / (2 * h)
            assert abs(fd - g[i]) < 1e-7 * (1 + abs(fd))


def test_controller_closed_form_one_layer():
    """H = 0, theta = [W, b]: alpha = tanh(W phi + b) with phi_j = sin(omega t dt + 2 pi j / n_sin)."""
    cfg = _cfg2(hidden=0, n_act=2)
    o = Oracle(cfg)
    W_ = np.array([[0.1, -0.2, 0.3, 0.05], [0.0, 0.4, -0.1, 0.2]])
    b = np.array([0.01, -0.03])
    t = 7
    phi = np.sin(cfg["omega"] * t * cfg["dt"] + 2 * np.pi * np.arange(4) / 4)
    np.testing.assert_allclose(o.controller(np.concatenate([W_.ravel(), b]), t),
                               np.tanh(W_ @ phi + b), rtol=1e-14)


def _golden_map(name):
    return {r[0]: np.array([float(x) for x in r[1:]]) for r in _golden_rows(name)}


def test_controller_two_layer_worked_example():
    """H > 0 (R9): the hand-built worked example of tests/golden/controller_observe.txt --
    theta laid out [W1, b1, W2, b2], hidden tanh, W2 of shape n_act x H, exact intermediates
    h = (0.5, -0.25) and alpha = (0.5, -0.75, 0.125)."""
    g = _golden_map("controller_observe.txt")
    o = Oracle(_cfg2(hidden=2, n_act=3))
    assert o.n_theta() == len(g["open_theta"]) == 19
    np.testing.assert_allclose(o.controller(g["open_theta"], 0), g["open_alpha"], rtol=0, atol=1e-14)


def test_controller_two_layer_saturated_hidden_layer():
    """H > 0 limit: with a hidden pre-activation of magnitude >= 40, tanh(z) = sign(z) exactly in
    fp64, so alpha = tanh(W2 sign(W1 phi + b1) + b2) -- a closed form that no longer contains the
    hidden tanh; checked at several t and for H != n_act (a transposed W2 or a dropped hidden
    nonlinearity fails it)."""
    H, A, S = 5, 3, 4
    cfg = _cfg2(hidden=H, n_act=A)
    o = Oracle(cfg)
    rng = np.random.default_rng(5)
    W1 = rng.choice([-1.0, 1.0], size=(H, S)) * 100.0
    b1 = rng.standard_normal(H) * 10.0
    W2 = rng.standard_normal((A, H)) * 0.3
    b2 = rng.standard_normal(A) * 0.1
    th = np.concatenate([W1.ravel(), b1, W2.ravel(), b2])
    checked, signs = 0, set()
    for t in range(0, 200, 7):
        phi = np.sin(cfg["omega"] * t * cfg["dt"] + 2 * np.pi * np.arange(S) / S)
        z = W1 @ phi + b1
        if np.min(np.abs(z)) < 40:
            continue
        np.testing.assert_allclose(o.controller(th, t), np.tanh(W2 @ np.sign(z) + b2), rtol=0, atol=1e-15)
        checked += 1
        signs.add(tuple(np.sign(z)))
    assert checked >= 5 and len(signs) >= 2  # several t, with different hidden sign patterns


def test_controller_zero_output_layer_gives_tanh_of_bias():
    """H > 0: W2 = 0 makes alpha = tanh(b2) whatever W1, b1 and t (the output layer alone)."""
    H, A = 4, 3
    o = Oracle(_cfg2(hidden=H, n_act=A))
    rng = np.random.default_rng(8)
    b2 = np.array([0.3, -1.2, 0.0])
    th = np.concatenate([rng.standard_normal(H * 4), rng.standard_normal(H), np.zeros(A * H), b2])
    for t in (0, 9):
        np.testing.assert_allclose(o.controller(th, t), np.tanh(b2), rtol=0, atol=1e-16)


# ------------------------------------------------------------ P2G / grid / G2P
def _random_state(o, N, rng, center=0.5, spread=0.08):
    d = o.d
    x = center + spread * (rng.random((N, d)) - 0.5)
    v = rng.standard_normal((N, d))
    C = rng.standard_normal((N, d, d))
    F = np.eye(d) + 0.1 * rng.standard_normal((N, d, d))
    return x, v, C, F


@pytest.mark.parametrize("dim", [2, 3])
def test_p2g_mass_momentum_conservation(dim):
    cfg = W.tiny(dim, n_particles=6 if dim == 2 else 8, n_grid=16)
    o = Oracle(cfg)
    rng = np.random.default_rng(1)
    x, v, C, F = _random_state(o, 40, rng)
    aid = rng.integers(-1, 2, size=40)
    grid, Fn = o.p2g(x, v, C, F, aid, np.array([0.3, -0.6]))
    M = grid[:, dim].sum()
    assert abs(M - 40 * cfg["p_mass"]) < 1e-12 * M
    np.testing.assert_allclose(grid[:, :dim].sum(0), cfg["p_mass"] * v.sum(0), rtol=1e-12, atol=1e-11)
    # F update: F_{t+1} = (I + dt C) F
    np.testing.assert_allclose(Fn, (np.eye(dim) + cfg["dt"] * C) @ F, rtol=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
def test_p2g_affine_second_moment(dim):
    """Single particle: (4/dx^2) sum_i P_i (x_i - x_p)^T = m v (x.)... = A with
    A = -dt V 4/dx^2 tau(F~) + m C  (the APIC/MLS affine moment), because the
    B-spline second moment is dx^2/4 and its first moment vanishes."""
    cfg = W.tiny(dim, n_particles=6 if dim == 2 else 8, n_grid=16)
    o = Oracle(cfg)
    rng = np.random.default_rng(2)
    x, v, C, F = _random_state(o, 1, rng)
    v[:] = 0.0
    grid, Fn = o.p2g(x, v, C, F)
    n = cfg["n_grid"]; dx = 1.0 / n
    idx = np.stack(np.unravel_index(np.arange(n ** dim), (n,) * dim), -1)
    rel = idx * dx - x[0]
    mom = 4 / dx ** 2 * np.einsum("ia,ib->ab", grid[:, :dim], rel)
    tau = o.stress(Fn[0])
    A = -cfg["dt"] * cfg["p_vol"] * 4 / dx ** 2 * tau + cfg["p_mass"] * C[0]
    np.testing.assert_allclose(mom, A, rtol=1e-11, atol=1e-10)


def test_grid_op_truth_table():
    """Sticky walls (R6): z = OR_k (i_k < beta and u_k < 0) or (i_k > n - beta and u_k > 0);
    gravity -dt g on axis 1 applied before the test; U = z ? 0 : u."""
    cfg = W.tiny(2, n_grid=16, bound=3, gravity=10.0, dt=1e-3, eps_mass=0.0)
    o = Oracle(cfg)
    n = 16
    grid = np.zeros((n * n, 3))
    cases = [  # (i0, i1), P, M, expected U
        ((8, 8), (0.2, 0.4), 2.0, (0.1, 0.2 - 0.01)),
        ((2, 8), (-0.2, 0.4), 2.0, (0.0, 0.0)),        # low x wall, moving into it
        ((2, 9), (0.2, 0.4), 2.0, (0.1, 0.19)),        # low x wall, moving away
        ((3, 8), (-0.2, 0.4), 2.0, (-0.1, 0.19)),      # i = beta is not a wall node
        ((14, 8), (0.2, 0.4), 2.0, (0.0, 0.0)),        # i > n - beta
        ((13, 9), (0.2, 0.4), 2.0, (0.1, 0.19)),       # i = n - beta is not
        ((8, 1), (0.2, 0.0), 2.0, (0.0, 0.0)),         # floor: gravity makes u_y < 0
        ((9, 1), (0.2, 0.1), 2.0, (0.1, 0.04)),        # floor, moving up fast enough
        ((8, 15), (0.2, 0.1), 2.0, (0.0, 0.0)),        # ceiling, moving up
        ((9, 9), (0.0, 0.0), 0.0, None),               # empty node (nan without eps)
    ]
    for (i0, i1), P, M, _ in cases:
        grid[i0 * n + i1] = (P[0], P[1], M)
    U = o.grid_op(grid)
    for (i0, i1), P, M, exp in cases[:-1]:
        np.testing.assert_allclose(U[i0 * n + i1], exp, atol=1e-15)
    o2 = Oracle(W.tiny(2, n_grid=16, bound=3, gravity=10.0, eps_mass=1e-10))
    U2 = o2.grid_op(np.zeros((n * n, 3)))
    assert np.all(U2[:, 0] == 0) and np.all(np.isin(U2[:, 1], [0.0, -10.0 * cfg["dt"]]))


@pytest.mark.parametrize("dim", [2, 3])
def test_g2p_affine_reproduction(dim):
    """U_i = B x_i + b  =>  v_p = B x_p + b, C_p = B exactly (B-spline moments)."""
    cfg = W.tiny(dim, n_particles=6 if dim == 2 else 8, n_grid=16)
    o = Oracle(cfg)
    rng = np.random.default_rng(4)
    B = rng.standard_normal((dim, dim)); b = rng.standard_normal(dim)
    n = cfg["n_grid"]
    idx = np.stack(np.unravel_index(np.arange(n ** dim), (n,) * dim), -1) / n
    U = idx @ B.T + b
    x = 0.5 + 0.3 * (rng.random((25, dim)) - 0.5)
    xn, vn, Cn = o.g2p(x, U)
    np.testing.assert_allclose(vn, x @ B.T + b, atol=1e-13)
    np.testing.assert_allclose(Cn, np.broadcast_to(B, Cn.shape), atol=1e-12)
    np.testing.assert_allclose(xn, x + cfg["dt"] * vn, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_rigid_translation_invariant(dim):
    """F = I, C = 0, uniform v, g = 0, eps = 0, away from walls: stress free,
    v, C, F unchanged, x_t = x_0 + t dt v (north_star invariant)."""
    cfg = W.tiny(dim, n_particles=6 if dim == 2 else 8, n_grid=16, gravity=0.0, eps_mass=0.0)
    o = Oracle(cfg)
    rng = np.random.default_rng(6)
    N = 30
    x = 0.45 + 0.1 * rng.random((N, dim))
    v = np.tile(rng.standard_normal(dim) * 0.5, (N, 1))
    C = np.zeros((N, dim, dim)); F = np.tile(np.eye(dim), (N, 1, 1))
    x0 = x.copy()
    for t in range(10):
        x, v2, C, F = o.step(x, v, C, F)
        np.testing.assert_allclose(v2, v, rtol=0, atol=1e-13)
        v = v2
    assert np.abs(C).max() < 1e-11
    np.testing.assert_allclose(F, np.tile(np.eye(dim), (N, 1, 1)), atol=1e-13)
    np.testing.assert_allclose(x, x0 + 10 * cfg["dt"] * v, atol=1e-13)


def test_com_ballistic_c1a():
    """Away from walls the centre of mass is exactly ballistic, independent of
    the material:  x_T = x_0 + T dt v_0 - dt^2 g T (T + 1)/2 e_y."""
    p = W.config("c1a", steps=64)
    inp = W.make_inputs(p)
    o = Oracle(p)
    r = o.run(inp["x"], inp["v"], inp["C"], inp["F"], steps=64)
    x0 = inp["x"].astype(np.float64).mean(0); v0 = inp["v"].astype(np.float64).mean(0)
    T, dt, g = 64, p["dt"], p["gravity"]
    pred = x0 + T * dt * v0 - np.array([0.0, dt * dt * g * T * (T + 1) / 2])
    np.testing.assert_allclose(r["x"].mean(0), pred, atol=1e-9)


def test_c1a_closed_form_gradient():
    """L = |xbar_T - x*|^2 without wall contact => dL/dv0_p = 2(xbar_T - x*) T dt m/M,
    dL/dx0_p = 2(xbar_T - x*) m/M, dL/dC0 = dL/dF0 = 0."""
    p = W.config("c1a")
    inp = W.make_inputs(p)
    o = Oracle(p)
    r = o.run(inp["x"], inp["v"], inp["C"], inp["F"])
    N = len(inp["x"]); T = p["steps"]
    g = 2 * (r["x"].mean(0) - np.array(p["target"][:2])) / N
    np.testing.assert_allclose(r["dv0"], np.tile(g * T * p["dt"], (N, 1)), rtol=1e-6)
    np.testing.assert_allclose(r["dx0"], np.tile(g, (N, 1)), rtol=1e-4)
    assert np.abs(r["dC0"]).max() < 1e-10 * np.abs(g).max()
    assert np.abs(r["dF0"]).max() < 1e-6 * np.abs(g).max()
    # the block stays clear of the walls, so the closed form applies
    assert r["x"].min() > 0.45 and r["x"].max() < 0.85


# ------------------------------------------------- whole-trajectory adjoints
def _tape(o, inp, T, lam):
    """python-level tape over oracle.step / oracle.step_adj with the linear
    loss L = <lam, S_T> (every state component seeded)."""
    x, v, C, F = (inp[k].astype(np.float64) for k in "xvCF")
    aid, th = inp["aid"], inp["theta"].astype(np.float64)
    hist = []
    for t in range(T):
        al = o.controller(th, t) if o.cfg.n_act else None
        hist.append((x, v, C, F, al))
        x, v, C, F = o.step(x, v, C, F, aid, al)
    L = sum(np.sum(l * s) for l, s in zip(lam, (x, v, C, F)))
    bars = [l.copy() for l in lam]
    thb = np.zeros_like(th)
    for t in reversed(range(T)):
        xs, vs, Cs, Fs, al = hist[t]
        *bars, ab = o.step_adj(xs, vs, Cs, Fs, *bars, aid, al)
        if o.cfg.n_act:
            thb += o.controller_adj(th, t, ab[: o.cfg.n_act])
    return L, bars, thb


def _fwd_loss(o, inp, T, lam):
    x, v, C, F = (inp[k].astype(np.float64) for k in "xvCF")
    th = inp["theta"].astype(np.float64)
    for t in range(T):
        al = o.controller(th, t) if o.cfg.n_act else None
        x, v, C, F = o.step(x, v, C, F, inp["aid"], al)
    return sum(np.sum(l * s) for l, s in zip(lam, (x, v, C, F)))


FD_CASES = {
    "2d_fcr_act_hidden": lambda: W.tiny(2, steps=12, hidden=4, seed=1),
    "3d_nh_act": lambda: W.tiny(3, n_particles=8, steps=5, seed=2),
    "2d_fcr_sticky_floor": lambda: W.tiny(2, steps=10, bound=3, n_grid=8, seed=3, floor=True,
                                          v_base=(0.3, -1.5)),
    "2d_nh": lambda: W.tiny(2, steps=8, model="neohookean", seed=4),
}


@pytest.mark.parametrize("case", list(FD_CASES))
def test_trajectory_adjoint_finite_differences(case):
    """Central differences (h = 1e-6, fp64) of L = <lam, S_T> w.r.t. every
    element of x0, v0, C0, F0 and theta vs the reverse sweep (rel <= 1e-6;
    observed 1e-10..1e-7)."""
    p = FD_CASES[case]()
    inp = {k: (v.astype(np.float64) if v.dtype == np.float32 else v)
           for k, v in W.make_inputs(p).items()}
    o = Oracle(p)
    rng = np.random.default_rng(99)
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
    if case == "2d_fcr_sticky_floor":
        # the floor must actually be active for this case to pin the select rule
        x = inp["x"]; v = inp["v"]
        hit = False
        for t in range(T):
            grid, _ = o.p2g(x, v, inp["C"], inp["F"])
            U = o.grid_op(grid)
            n = p["n_grid"]
            iy = np.arange(n * n) % n
            if np.any((grid[:, 2] > 0) & (iy < p["bound"]) & (U[:, 1] == 0)):
                hit = True
                break
            x, v, _, _ = o.step(x, v, inp["C"], inp["F"])
        assert hit


def test_run_matches_python_tape_and_checkpointing():
    """oracle_run (tape with segment checkpointing) equals the plain
    python-level tape, bitwise for every segment size k in {1, 3, T}."""
    p = W.tiny(2, steps=9, hidden=4, seed=8)
    inp = W.make_inputs(p)
    o = Oracle(p)
    res = [o.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"], k_ckpt=k)
           for k in (1, 3, 9, 4)]
    for r in res[1:]:
        for key in ("x", "dx0", "dv0", "dC0", "dF0", "dtheta"):
            assert np.array_equal(r[key], res[0][key]), key
    # python tape with the COM seed
    N, d = inp["x"].shape
    x, v, C, F = (inp[k].astype(np.float64) for k in "xvCF")
    th = inp["theta"].astype(np.float64)
    for t in range(9):
        x, v, C, F = o.step(x, v, C, F, inp["aid"], o.controller(th, t))
    L, xb = o.loss(x)
    assert L == pytest.approx(res[0]["loss"], rel=1e-15)
    inp64 = {k: (a.astype(np.float64) if a.dtype == np.float32 else a) for k, a in inp.items()}
    _, bars, thb = _tape(o, inp64, 9, [xb, np.zeros((N, d)), np.zeros((N, d, d)), np.zeros((N, d, d))])
    np.testing.assert_allclose(bars[1], res[0]["dv0"], rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(thb, res[0]["dtheta"], rtol=1e-12, atol=1e-18)


def test_adjoint_linearity():
    """Running the adjoint with a doubled seed exactly doubles every adjoint."""
    p = W.tiny(3, n_particles=8, steps=1, seed=5)
    inp = W.make_inputs(p)
    o = Oracle(p)
    rng = np.random.default_rng(0)
    N, d = inp["x"].shape
    seeds = [rng.standard_normal((N, d)), rng.standard_normal((N, d)),
             rng.standard_normal((N, d, d)), rng.standard_normal((N, d, d))]
    al = o.controller(inp["theta"], 0)
    a = o.step_adj(inp["x"], inp["v"], inp["C"], inp["F"], *seeds, inp["aid"], al)
    b = o.step_adj(inp["x"], inp["v"], inp["C"], inp["F"], *[2 * s for s in seeds], inp["aid"], al)
    for u, w in zip(a, b):
        assert np.array_equal(2 * u, w)


def test_loss_seed_and_kinds():
    p = W.tiny(2)
    o = Oracle(p)
    x = np.array([[0.2, 0.3], [0.4, 0.7]])
    L, xb = o.loss(x, kind=0, target=[0.1, 0.1])
    assert L == pytest.approx((0.3 - 0.1) ** 2 + (0.5 - 0.1) ** 2)
    np.testing.assert_allclose(xb, np.tile([2 * 0.2 / 2, 2 * 0.4 / 2], (2, 1)))
    L, xb = o.loss(x, kind=1)
    assert L == pytest.approx(-0.3)
    np.testing.assert_allclose(xb, np.tile([-0.5, 0.0], (2, 1)))


def test_out_of_domain_is_an_error():
    o = Oracle(W.tiny(2, n_grid=8))
    x = np.array([[0.05, 0.5]])  # base = floor(0.4 - 0.5) = -1
    with pytest.raises(OracleError) as e:
        o.p2g(x, np.zeros((1, 2)), np.zeros((1, 2, 2)), np.eye(2)[None])
    assert e.value.status == 4
    x = np.array([[0.5, 0.9]])  # base + 2 = 8 > n - 1
    with pytest.raises(OracleError):
        o.g2p(x, np.zeros((64, 2)))


def test_f32_build_tracks_f64():
    """The fp32 build of the same source agrees with fp64 on C1a/C1b within the
    drift budget the parity gate relies on (SURVEY.md 8(c) feasibility)."""
    for name in ("c1a", "c1b"):
        p = W.config(name, steps=64)
        inp = W.make_inputs(p)
        r64 = Oracle(p).run(inp["x"], inp["v"], inp["C"], inp["F"])
        r32 = Oracle(p, "f32").run(inp["x"], inp["v"], inp["C"], inp["F"])
        for k in "xvCF":
            err = np.linalg.norm(r32[k] - r64[k]) / np.linalg.norm(r64[k])
            assert err < 1e-4, (name, k, err)
        err = np.linalg.norm(r32["dv0"] - r64["dv0"]) / np.linalg.norm(r64["dv0"])
        assert err < 1e-3, (name, err)


def test_workload_shapes():
    """The synthetic workloads have the paper's sizes."""
    assert len(W.make_inputs("c2")["x"]) == 6400
    inp = W.make_inputs("c3")
    assert len(inp["x"]) == 29952 and inp["aid"].max() == 15
    assert np.bincount(inp["aid"][inp["aid"] >= 0]).tolist() == [576] * 16
    assert W.n_theta(W.config("c3")) == 688 and W.n_theta(W.config("c2")) == 292
    a, b = W.make_inputs("c2"), W.make_inputs("c2")
    assert all(np.array_equal(a[k], b[k]) for k in a)
    assert math.prod(W.config("c5")["counts"]) == 1061208
