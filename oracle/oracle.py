"""ctypes front end of the C oracle (oracle_mpm.c).  TEST INFRASTRUCTURE ONLY.

Argument marshalling only: every number is computed in oracle_mpm.c.  The
configuration dict uses the same keys as the workload generator
(``paper_1910_00935_b200/workloads.py``), which holds none of the method's
arithmetic.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_mpm.c")
_HDR = os.path.join(_HERE, "oracle_mpm.h")

STATUS = {0: "ok", 1: "invalid argument", 4: "out of domain", 5: "non-finite"}


class OracleError(RuntimeError):
    def __init__(self, fn, status):
        super().__init__(f"oracle {fn}: status {status} ({STATUS.get(status, '?')})")
        self.status = status


def lib_path(precision: str = "f64") -> str:
    return os.path.join(_HERE, f"liboracle_{precision}.so")


def build(precision: str | None = None, force: bool = False) -> None:
    """Compile the oracle with plain gcc -O2 (single-threaded, untuned)."""
    for prec in ([precision] if precision else ["f64", "f32"]):
        out = lib_path(prec)
        if (not force and os.path.exists(out)
                and os.path.getmtime(out) >= max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))):
            continue
        real = "double" if prec == "f64" else "float"
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-shared", "-fPIC",
                               f"-DORACLE_REAL={real}", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)


class _Cfg(ct.Structure):
    _fields_ = [("dim", ct.c_int32), ("n_grid", ct.c_int32), ("bound", ct.c_int32),
                ("model", ct.c_int32), ("n_act", ct.c_int32), ("act_axis", ct.c_int32),
                ("n_sin", ct.c_int32), ("hidden", ct.c_int32),
                ("dt", ct.c_double), ("E", ct.c_double), ("nu", ct.c_double),
                ("p_mass", ct.c_double), ("p_vol", ct.c_double), ("gravity", ct.c_double),
                ("eps_mass", ct.c_double), ("kappa", ct.c_double), ("omega", ct.c_double),
                ("closed_loop", ct.c_int32), ("obs_sx", ct.c_double), ("obs_sv", ct.c_double),
                ("mat", ct.c_void_p)]


MODELS = {"neohookean": 0, "nh": 0, "fixed_corotated": 1, "fcr": 1}
LOSSES = {"com_target": 0, "move_forward": 1}


def make_cfg(p: dict) -> _Cfg:
    c = _Cfg()
    c.dim = int(p["dim"]); c.n_grid = int(p["n_grid"]); c.bound = int(p.get("bound", 3))
    m = p.get("model", "neohookean")
    c.model = MODELS[m] if isinstance(m, str) else int(m)
    c.n_act = int(p.get("n_act", 0)); c.act_axis = int(p.get("act_axis", 1))
    c.n_sin = int(p.get("n_sin", 4)); c.hidden = int(p.get("hidden", 0))
    c.dt = float(p["dt"]); c.E = float(p["E"]); c.nu = float(p["nu"])
    c.p_mass = float(p.get("p_mass", 1.0)); c.p_vol = float(p.get("p_vol", 1.0))
    c.gravity = float(p.get("gravity", 0.0)); c.eps_mass = float(p.get("eps_mass", 1e-10))
    c.kappa = float(p.get("kappa", 0.0)); c.omega = float(p.get("omega", 20.0))
    c.closed_loop = int(bool(p.get("closed_loop", False)))
    c.obs_sx = float(p.get("obs_sx", 10.0)); c.obs_sv = float(p.get("obs_sv", 1.0))
    return c


class Oracle:
    """One configuration bound to the f64 (default) or f32 oracle build."""

    def __init__(self, params: dict, precision: str = "f64"):
        build(precision)
        self.lib = ct.CDLL(lib_path(precision))
        self.dtype = np.float64 if precision == "f64" else np.float32
        self.p = dict(params)
        self.cfg = make_cfg(params)
        self._mat = None  # per-particle materials (R23), kept alive for cfg.mat
        self.d = self.cfg.dim
        self.n = self.cfg.n_grid
        self.nn = self.n ** self.d
        self._declare()

    # --------------------------------------------------------------- helpers
    def _declare(self):
        P = ct.c_void_p
        L = self.lib
        cfgp = ct.POINTER(_Cfg)
        sig = {
            "oracle_bspline": (None, [self._rt(), P, P]),
            "oracle_lame": (None, [cfgp, P, P]),
            "oracle_stress": (ct.c_int, [cfgp, P, P]),
            "oracle_stress_adj": (ct.c_int, [cfgp, P, P, P]),
            "oracle_energy": (ct.c_int, [cfgp, P, P]),
            "oracle_n_theta": (ct.c_int64, [cfgp]),
            "oracle_controller": (None, [cfgp, P, ct.c_int32, P]),
            "oracle_controller_adj": (None, [cfgp, P, ct.c_int32, P, P]),
            "oracle_n_obs": (ct.c_int, [cfgp]),
            "oracle_controller_obs": (None, [cfgp, P, ct.c_int32, P, P]),
            "oracle_controller_obs_adj": (None, [cfgp, P, ct.c_int32, P, P, P, P]),
            "oracle_observe": (None, [cfgp, ct.c_int64, P, P, P, P]),
            "oracle_observe_adj": (None, [cfgp, ct.c_int64, P, P, P, P]),
            "oracle_p2g": (ct.c_int, [cfgp, ct.c_int64, P, P, P, P, P, P, P, P]),
            "oracle_grid_op": (None, [cfgp, P, P]),
            "oracle_g2p": (ct.c_int, [cfgp, ct.c_int64, P, P, P, P, P]),
            "oracle_step": (ct.c_int, [cfgp, ct.c_int64] + [P] * 10),
            "oracle_g2p_adj": (ct.c_int, [cfgp, ct.c_int64] + [P] * 7),
            "oracle_grid_op_adj": (None, [cfgp, P, P, P]),
            "oracle_p2g_adj": (ct.c_int, [cfgp, ct.c_int64] + [P] * 13),
            "oracle_step_adj": (ct.c_int, [cfgp, ct.c_int64] + [P] * 15),
            "oracle_loss": (ct.c_int, [cfgp, ct.c_int32, P, ct.c_int64, P, P, P]),
            "oracle_run": (ct.c_int, [cfgp, ct.c_int64, ct.c_int32, ct.c_int32] + [P] * 6
                           + [ct.c_int32] + [P] * 11),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def _rt(self):
        return ct.c_double if self.dtype == np.float64 else ct.c_float

    def _a(self, a, shape=None):
        """contiguous array of the oracle's real type (copy if needed)."""
        a = np.ascontiguousarray(np.asarray(a, dtype=self.dtype))
        if shape is not None:
            a = a.reshape(shape)
        return a

    @staticmethod
    def _p(a):
        return None if a is None else a.ctypes.data_as(ct.c_void_p)

    def _check(self, fn, st):
        if st != 0:
            raise OracleError(fn, st)

    def _aid(self, aid, N):
        if aid is None:
            return None
        return np.ascontiguousarray(np.asarray(aid, dtype=np.int32).reshape(N))

    # ------------------------------------------------------------ primitives
    def bspline(self, f):
        w = np.zeros(3, self.dtype); dw = np.zeros(3, self.dtype)
        self.lib.oracle_bspline(float(f), self._p(w), self._p(dw))
        return w, dw

    def lame(self):
        mu = np.zeros(1, self.dtype); lam = np.zeros(1, self.dtype)
        self.lib.oracle_lame(ct.byref(self.cfg), self._p(mu), self._p(lam))
        return float(mu[0]), float(lam[0])

    def stress(self, F):
        F = self._a(F, (self.d, self.d)); tau = np.zeros_like(F)
        self._check("stress", self.lib.oracle_stress(ct.byref(self.cfg), self._p(F), self._p(tau)))
        return tau

    def stress_adj(self, F, tau_bar):
        F = self._a(F, (self.d, self.d)); tb = self._a(tau_bar, (self.d, self.d))
        Fb = np.zeros_like(F)
        self._check("stress_adj", self.lib.oracle_stress_adj(ct.byref(self.cfg), self._p(F),
                                                             self._p(tb), self._p(Fb)))
        return Fb

    def energy(self, F):
        F = self._a(F, (self.d, self.d)); psi = np.zeros(1, self.dtype)
        self._check("energy", self.lib.oracle_energy(ct.byref(self.cfg), self._p(F), self._p(psi)))
        return float(psi[0])

    def n_theta(self):
        return int(self.lib.oracle_n_theta(ct.byref(self.cfg)))

    def controller(self, theta, t):
        th = self._a(theta); a = np.zeros(self.cfg.n_act, self.dtype)
        self.lib.oracle_controller(ct.byref(self.cfg), self._p(th), int(t), self._p(a))
        return a

    def controller_adj(self, theta, t, alpha_bar):
        th = self._a(theta); ab = self._a(alpha_bar); thb = np.zeros_like(th)
        self.lib.oracle_controller_adj(ct.byref(self.cfg), self._p(th), int(t), self._p(ab),
                                       self._p(thb))
        return thb

    def set_materials(self, mat):
        """per-particle material ids (0 solid, 1 fluid; R23), caller order; None = all solid."""
        self._mat = None if mat is None else np.ascontiguousarray(np.asarray(mat, np.int32).ravel())
        self.cfg.mat = None if self._mat is None else self._mat.ctypes.data
        return self

    def n_obs(self):
        return int(self.lib.oracle_n_obs(ct.byref(self.cfg)))

    def controller_obs(self, theta, t, obs):
        th = self._a(theta); o = self._a(obs); a = np.zeros(self.cfg.n_act, self.dtype)
        self.lib.oracle_controller_obs(ct.byref(self.cfg), self._p(th), int(t), self._p(o), self._p(a))
        return a

    def controller_obs_adj(self, theta, t, obs, alpha_bar):
        th = self._a(theta); o = self._a(obs); ab = self._a(alpha_bar)
        thb = np.zeros_like(th); ob = np.zeros(self.n_obs(), self.dtype)
        self.lib.oracle_controller_obs_adj(ct.byref(self.cfg), self._p(th), int(t), self._p(o),
                                           self._p(ab), self._p(thb), self._p(ob))
        return thb, ob

    def observe(self, x, v, aid):
        x = self._a(x); v = self._a(v); N = x.size // self.d
        o = np.zeros(max(self.n_obs(), 1), self.dtype)
        self.lib.oracle_observe(ct.byref(self.cfg), N, self._p(x), self._p(v), self._p(self._aid(aid, N)),
                                self._p(o))
        return o[:self.n_obs()]

    def observe_adj(self, N, aid, obs_bar):
        ob = self._a(obs_bar)
        xb = np.zeros((N, self.d), self.dtype); vb = np.zeros((N, self.d), self.dtype)
        self.lib.oracle_observe_adj(ct.byref(self.cfg), N, self._p(self._aid(aid, N)), self._p(ob),
                                    self._p(xb), self._p(vb))
        return xb, vb

    def _state(self, x, v, C, F):
        d = self.d
        x = self._a(x); N = x.size // d
        return (x.reshape(N, d), self._a(v, (N, d)), self._a(C, (N, d, d)),
                self._a(F, (N, d, d)), N)

    def p2g(self, x, v, C, F, aid=None, alpha=None):
        x, v, C, F, N = self._state(x, v, C, F)
        al = self._a(alpha if alpha is not None else np.zeros(max(self.cfg.n_act, 1)))
        grid = np.zeros((self.nn, self.d + 1), self.dtype); Fn = np.zeros_like(F)
        self._check("p2g", self.lib.oracle_p2g(ct.byref(self.cfg), N, *map(self._p, (x, v, C, F)),
                                               self._p(self._aid(aid, N)), self._p(al),
                                               self._p(grid), self._p(Fn)))
        return grid, Fn

    def grid_op(self, grid):
        g = self._a(grid, (self.nn, self.d + 1)); U = np.zeros((self.nn, self.d), self.dtype)
        self.lib.oracle_grid_op(ct.byref(self.cfg), self._p(g), self._p(U))
        return U

    def g2p(self, x, U):
        x = self._a(x); N = x.size // self.d; x = x.reshape(N, self.d)
        U = self._a(U, (self.nn, self.d))
        xn = np.zeros_like(x); vn = np.zeros_like(x); Cn = np.zeros((N, self.d, self.d), self.dtype)
        self._check("g2p", self.lib.oracle_g2p(ct.byref(self.cfg), N, self._p(x), self._p(U),
                                               self._p(xn), self._p(vn), self._p(Cn)))
        return xn, vn, Cn

    def step(self, x, v, C, F, aid=None, alpha=None):
        x, v, C, F, N = self._state(x, v, C, F)
        al = self._a(alpha if alpha is not None else np.zeros(max(self.cfg.n_act, 1)))
        out = [np.zeros_like(x), np.zeros_like(v), np.zeros_like(C), np.zeros_like(F)]
        self._check("step", self.lib.oracle_step(ct.byref(self.cfg), N,
                                                 *map(self._p, (x, v, C, F)),
                                                 self._p(self._aid(aid, N)), self._p(al),
                                                 *map(self._p, out)))
        return tuple(out)

    def g2p_adj(self, x, U, xb_n, vb_n, Cb_n):
        d = self.d
        x = self._a(x); N = x.size // d; x = x.reshape(N, d)
        U = self._a(U, (self.nn, d))
        xbn, vbn, Cbn = self._a(xb_n, (N, d)), self._a(vb_n, (N, d)), self._a(Cb_n, (N, d, d))
        Ub = np.zeros((self.nn, d), self.dtype); xb = np.zeros_like(x)
        self._check("g2p_adj", self.lib.oracle_g2p_adj(ct.byref(self.cfg), N,
                                                       *map(self._p, (x, U, xbn, vbn, Cbn, Ub, xb))))
        return Ub, xb

    def grid_op_adj(self, grid, U_bar):
        g = self._a(grid, (self.nn, self.d + 1)); Ub = self._a(U_bar, (self.nn, self.d))
        gb = np.zeros_like(g)
        self.lib.oracle_grid_op_adj(ct.byref(self.cfg), self._p(g), self._p(Ub), self._p(gb))
        return gb

    def p2g_adj(self, x, v, C, F, grid_bar, Fb_n, xb_partial, aid=None, alpha=None):
        x, v, C, F, N = self._state(x, v, C, F)
        al = self._a(alpha if alpha is not None else np.zeros(max(self.cfg.n_act, 1)))
        gb = self._a(grid_bar, (self.nn, self.d + 1)); Fbn = self._a(Fb_n, F.shape)
        xb = self._a(xb_partial, x.shape).copy()
        vb, Cb, Fb = np.zeros_like(v), np.zeros_like(C), np.zeros_like(F)
        ab = np.zeros(max(self.cfg.n_act, 1), self.dtype)
        self._check("p2g_adj", self.lib.oracle_p2g_adj(
            ct.byref(self.cfg), N, *map(self._p, (x, v, C, F)), self._p(self._aid(aid, N)),
            self._p(al), self._p(gb), self._p(Fbn), *map(self._p, (xb, vb, Cb, Fb, ab))))
        return xb, vb, Cb, Fb, ab

    def step_adj(self, x, v, C, F, xb_n, vb_n, Cb_n, Fb_n, aid=None, alpha=None):
        x, v, C, F, N = self._state(x, v, C, F)
        al = self._a(alpha if alpha is not None else np.zeros(max(self.cfg.n_act, 1)))
        bars_n = [self._a(xb_n, x.shape), self._a(vb_n, v.shape), self._a(Cb_n, C.shape),
                  self._a(Fb_n, F.shape)]
        out = [np.zeros_like(x), np.zeros_like(v), np.zeros_like(C), np.zeros_like(F)]
        ab = np.zeros(max(self.cfg.n_act, 1), self.dtype)
        self._check("step_adj", self.lib.oracle_step_adj(
            ct.byref(self.cfg), N, *map(self._p, (x, v, C, F)), self._p(self._aid(aid, N)),
            self._p(al), *map(self._p, bars_n), *map(self._p, out), self._p(ab)))
        return tuple(out) + (ab,)

    def loss(self, x, kind=None, target=None):
        kind = LOSSES[self.p.get("loss", "com_target")] if kind is None else kind
        tgt = self._a(target if target is not None else self.p.get("target", [0, 0, 0]))
        x = self._a(x); N = x.size // self.d
        L = np.zeros(1, self.dtype); xb = np.zeros((N, self.d), self.dtype)
        self._check("loss", self.lib.oracle_loss(ct.byref(self.cfg), int(kind), self._p(tgt), N,
                                                 self._p(x), self._p(L), self._p(xb)))
        return float(L[0]), xb

    def run(self, x0, v0, C0, F0, aid=None, theta=None, steps=None, k_ckpt=None,
            loss_kind=None, target=None):
        """Whole episode: S_T, L and dL/d(x0, v0, C0, F0, theta)."""
        x, v, C, F, N = self._state(x0, v0, C0, F0)
        T = int(self.p["steps"] if steps is None else steps)
        k = int(self.p.get("k_ckpt", 1) if k_ckpt is None else k_ckpt)
        kind = LOSSES[self.p.get("loss", "com_target")] if loss_kind is None else loss_kind
        tgt = self._a(target if target is not None else self.p.get("target", [0, 0, 0]))
        nth = self.n_theta()
        th = self._a(theta if theta is not None else np.zeros(nth))
        outS = [np.zeros_like(x), np.zeros_like(v), np.zeros_like(C), np.zeros_like(F)]
        grads = [np.zeros_like(x), np.zeros_like(v), np.zeros_like(C), np.zeros_like(F),
                 np.zeros(max(nth, 1), self.dtype)]
        L = np.zeros(1, self.dtype)
        st = self.lib.oracle_run(ct.byref(self.cfg), N, T, k, *map(self._p, (x, v, C, F)),
                                 self._p(self._aid(aid, N)), self._p(th), int(kind), self._p(tgt),
                                 *map(self._p, outS), self._p(L), *map(self._p, grads))
        self._check("run", st)
        return {"x": outS[0], "v": outS[1], "C": outS[2], "F": outS[3], "loss": float(L[0]),
                "dx0": grads[0], "dv0": grads[1], "dC0": grads[2], "dF0": grads[3],
                "dtheta": grads[4][:nth]}
