"""Pins of the oracle's closed-loop controller (R22).

R22: the controller input is [phi(t), o_t] with, per actuator group a,
o_t[a] = (s_x (mean_a x_t - mean x_t), s_v mean_a v_t).  Pinned here by
* an identity: with every particle in some group, sum_a n_a o_x[a] = 0 (offsets from the
  centre of mass cancel) and o_x is invariant to a rigid shift of all positions;
* the transpose relation of observe / observe_adj (dot-product test against central
  differences of observe);
* the controller's input adjoint and weight adjoint against central differences;
* reduction to the (separately pinned) open-loop controller when the observation weights are
  zero -- bitwise equal trajectories, losses and gradients;
* whole-trajectory central differences of the closed-loop episode (x0, v0, C0, F0, theta) with
  floor contact, so the loss depends on theta (rel <= 1e-6).
"""
import os

import numpy as np
import pytest

from oracle import Oracle
from paper_1910_00935_b200 import workloads as W


def _cl(dim=2, **kw):
    base = dict(steps=8, hidden=3, bound=3, floor=True, seed=5, closed_loop=True)
    if dim == 2:
        base.update(v_base=(0.3, -1.5))
    else:
        base.update(v_base=(0.2, -1.5, 0.1))
    base.update(kw)
    return W.tiny(dim, **base)


def _state(o, N, rng):
    d = o.d
    x = 0.5 + 0.1 * (rng.random((N, d)) - 0.5)
    v = rng.standard_normal((N, d))
    return x, v


@pytest.mark.parametrize("dim", [2, 3])
def test_observation_identities(dim):
    p = _cl(dim, n_act=3)
    o = Oracle(p)
    rng = np.random.default_rng(1)
    N = 12
    x, v = _state(o, N, rng)
    aid = np.arange(N) % 3  # every particle in a group
    ob = o.observe(x, v, aid).reshape(3, 2, dim)
    n = np.bincount(aid, minlength=3)
    np.testing.assert_allclose((n[:, None] * ob[:, 0, :]).sum(axis=0), 0.0, atol=1e-13)
    ob2 = o.observe(x + np.array([0.01, -0.02, 0.03][:dim]), v, aid).reshape(3, 2, dim)
    np.testing.assert_allclose(ob2[:, 0, :], ob[:, 0, :], atol=1e-13)
    np.testing.assert_array_equal(ob2[:, 1, :], ob[:, 1, :])
    # an empty group observes zero
    ob3 = o.observe(x, v, np.where(aid == 2, -1, aid)).reshape(3, 2, dim)
    assert np.all(ob3[2] == 0)


@pytest.mark.parametrize("dim", [2, 3])
def test_observe_adjoint_is_the_transpose(dim):
    p = _cl(dim, n_act=2)
    o = Oracle(p)
    rng = np.random.default_rng(2)
    N = 10
    x, v = _state(o, N, rng)
    aid = np.array([0, 1, -1, 0, 1, 1, -1, 0, 0, 1])
    ob_bar = rng.standard_normal(o.n_obs())
    xb, vb = o.observe_adj(N, aid, ob_bar)
    dx, dv = rng.standard_normal((N, dim)), rng.standard_normal((N, dim))
    h = 1e-6
    jd = (o.observe(x + h * dx, v + h * dv, aid) - o.observe(x - h * dx, v - h * dv, aid)) / (2 * h)
    lhs = ob_bar @ jd
    rhs = np.sum(xb * dx) + np.sum(vb * dv)
    assert abs(lhs - rhs) < 1e-8 * (1 + abs(lhs))


@pytest.mark.parametrize("hidden", [0, 4])
def test_controller_obs_adjoint_fd(hidden):
    p = _cl(2, n_act=3, hidden=hidden)
    o = Oracle(p)
    rng = np.random.default_rng(3)
    th = rng.standard_normal(o.n_theta()) * 0.5
    obs = rng.standard_normal(o.n_obs())
    ab = rng.standard_normal(3)
    h = 1e-6
    for t in (0, 9):
        thb, obb = o.controller_obs_adj(th, t, obs, ab)
        for i in range(len(th)):
            e = np.zeros_like(th); e[i] = h
            fd = (ab @ o.controller_obs(th + e, t, obs) - ab @ o.controller_obs(th - e, t, obs)) / (2 * h)
            assert abs(fd - thb[i]) < 1e-7 * (1 + abs(fd))
        for j in range(len(obs)):
            e = np.zeros_like(obs); e[j] = h
            fd = (ab @ o.controller_obs(th, t, obs + e) - ab @ o.controller_obs(th, t, obs - e)) / (2 * h)
            assert abs(fd - obb[j]) < 1e-7 * (1 + abs(fd))


@pytest.mark.parametrize("hidden", [0, 3])
def test_zero_observation_weights_reduce_to_open_loop(hidden):
    pc = _cl(2, hidden=hidden)
    po = dict(pc, closed_loop=False)
    oc, oo = Oracle(pc), Oracle(po)
    inp = W.make_inputs(po)
    S, A, n_obs = pc["n_sin"], pc["n_act"], oc.n_obs()
    tho = inp["theta"].astype(np.float64)
    # embed the open-loop weights; the observation columns of the first layer are zero
    if hidden:
        H = hidden
        W1 = tho[: H * S].reshape(H, S)
        thc = np.concatenate([np.hstack([W1, np.zeros((H, n_obs))]).ravel(), tho[H * S:]])
    else:
        Wm = tho[: A * S].reshape(A, S)
        thc = np.concatenate([np.hstack([Wm, np.zeros((A, n_obs))]).ravel(), tho[A * S:]])
    ro = oo.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], tho)
    rc = oc.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], thc)
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0"):
        np.testing.assert_array_equal(rc[k], ro[k], err_msg=k)
    assert rc["loss"] == ro["loss"]
    # theta_bar on the shared weights is the same; the observation columns carry the
    # (nonzero) sensitivity to the observation weights
    if hidden:
        g = rc["dtheta"][: hidden * (S + n_obs)].reshape(hidden, S + n_obs)
        np.testing.assert_allclose(g[:, :S].ravel(), ro["dtheta"][: hidden * S], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(rc["dtheta"][hidden * (S + n_obs):], ro["dtheta"][hidden * S:], rtol=1e-12,
                                   atol=1e-15)
    assert np.linalg.norm(rc["dtheta"]) > 0


FD_CL = {
    "2d_fcr_floor_hidden": lambda: _cl(2, steps=10, hidden=3, seed=7),
    "3d_nh_floor": lambda: _cl(3, steps=6, hidden=0, seed=8, n_grid=8),
}


@pytest.mark.parametrize("case", list(FD_CL))
def test_closed_loop_trajectory_fd(case):
    """Central differences (h = 1e-6, fp64) of the episode loss w.r.t. every element of
    x0, v0, C0, F0 and theta vs the reverse sweep, closed loop, floor contact
    (rel <= 1e-6; C0 <= 1e-5)."""
    p = FD_CL[case]()
    inp = {k: (v.astype(np.float64) if v.dtype == np.float32 else v) for k, v in W.make_inputs(p).items()}
    inp["theta"] = inp["theta"] * 0.5
    o = Oracle(p)
    r = o.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"])
    grads = {"x": r["dx0"], "v": r["dv0"], "C": r["dC0"], "F": r["dF0"], "theta": r["dtheta"]}
    assert np.linalg.norm(r["dtheta"]) > 1e-8  # the loss depends on the controller

    def loss(q):
        return o.run(q["x"], q["v"], q["C"], q["F"], q["aid"], q["theta"])["loss"]

    h = 1e-6
    for key in ["x", "v", "C", "F", "theta"]:
        arr = inp[key]
        g = np.asarray(grads[key]).ravel()
        fd = np.zeros(arr.size)
        for i in range(arr.size):
            ip, im = dict(inp), dict(inp)
            ap = arr.copy().ravel(); ap[i] += h
            am = arr.copy().ravel(); am[i] -= h
            ip[key] = ap.reshape(arr.shape); im[key] = am.reshape(arr.shape)
            fd[i] = (loss(ip) - loss(im)) / (2 * h)
        err = np.linalg.norm(fd - g) / max(np.linalg.norm(fd), 1e-300)
        print(case, key, err, np.linalg.norm(g))
        # C0 enters the COM loss only through the (small) contact response: its central
        # differences carry ~1e-6 relative cancellation noise at h = 1e-6
        assert err < (1e-5 if key == "C" else 1e-6), (case, key, err)


GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "controller_observe.txt")


def _golden():
    out = {}
    with open(GOLDEN) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                k, *v = line.split()
                out[k] = np.array([float(x) for x in v])
    return out


def test_observation_worked_example():
    """R22 on the hand-evaluated five-particle example of tests/golden/controller_observe.txt
    (s_x = 10, s_v = 2; a passive particle shifts the centre of mass but no group velocity):
    pins both o_x and o_v, their layout and the scales."""
    g = _golden()
    o = Oracle(_cl(2, n_act=2, obs_sv=2.0))
    x = g["obs_x"].reshape(5, 2)
    v = g["obs_v"].reshape(5, 2)
    aid = g["obs_aid"].astype(np.int32)
    np.testing.assert_allclose(o.observe(x, v, aid), g["obs_expected"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
def test_observed_velocity_identities(dim):
    """o_v (R22) is pinned by (i) sum_a n_a o_v[a] = s_v * (sum of v over grouped particles),
    (ii) a Galilean shift v -> v + c moves o_v[a] by s_v c for every non-empty group and leaves
    o_x unchanged, (iii) o_v does not depend on x, (iv) an empty group observes zero."""
    A, sv = 3, 2.5
    o = Oracle(_cl(dim, n_act=A, obs_sv=sv))
    rng = np.random.default_rng(4)
    N = 17
    x, v = _state(o, N, rng)
    aid = rng.integers(-1, A - 1, size=N).astype(np.int32)  # group A-1 stays empty
    aid[:2] = [0, 1]
    ob = o.observe(x, v, aid).reshape(A, 2, dim)
    n = np.bincount(aid[aid >= 0], minlength=A)
    np.testing.assert_allclose((n[:, None] * ob[:, 1, :]).sum(0), sv * v[aid >= 0].sum(0), rtol=1e-13, atol=1e-13)
    c_ = rng.standard_normal(dim)
    ob2 = o.observe(x, v + c_, aid).reshape(A, 2, dim)
    for a in range(A):
        if n[a]:
            np.testing.assert_allclose(ob2[a, 1], ob[a, 1] + sv * c_, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(ob2[:, 0], ob[:, 0], rtol=0, atol=1e-15)
    ob3 = o.observe(x + 0.01 * rng.standard_normal(x.shape), v, aid).reshape(A, 2, dim)
    np.testing.assert_array_equal(ob3[:, 1], ob[:, 1])
    assert np.all(ob[A - 1] == 0)


def test_closed_loop_controller_worked_example():
    """Closed-loop MLP input order u = [phi(t), o_t] (R22): the hand-built example of
    tests/golden/controller_observe.txt (h = (0.5, -0.25), alpha = 0.5)."""
    g = _golden()
    o = Oracle(_cl(2, n_act=1, hidden=2))
    assert o.n_theta() == len(g["closed_theta"]) == 21
    np.testing.assert_allclose(o.controller_obs(g["closed_theta"], 0, g["closed_obs"]), g["closed_alpha"],
                               rtol=0, atol=1e-14)
