"""Thin ctypes binding of libmpm_b200.so (include/mpm.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch supplies the device workspace and the stream.  If the
library is missing this module raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPM_B200_LIB: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("MPM_B200_LIB") or os.path.join(_HERE, "libmpm_b200.so")

MPM_OK = 0
STATUS_NAMES = {0: "MPM_OK", 1: "MPM_ERR_INVALID_ARG", 2: "MPM_ERR_OOM", 3: "MPM_ERR_CUDA",
                4: "MPM_ERR_OUT_OF_DOMAIN", 5: "MPM_ERR_NONFINITE", 6: "MPM_ERR_BAD_SEQUENCE",
                7: "MPM_ERR_UNSUPPORTED"}
MODEL_NEOHOOKEAN, MODEL_FIXED_COROTATED = 0, 1
LOSS_COM_TARGET, LOSS_MOVE_FORWARD = 0, 1

EXPORTS = ["mpm_create", "mpm_destroy", "mpm_last_error", "mpm_default_params", "mpm_get_params",
           "mpm_set_params", "mpm_set_stream", "mpm_workspace_bytes", "mpm_workspace_bytes_for", "mpm_bind_workspace",
           "mpm_set_state", "mpm_n_theta", "mpm_set_controller", "mpm_forward", "mpm_loss",
           "mpm_seed_adjoint", "mpm_backward", "mpm_grads", "mpm_get_state", "mpm_launch_count",
           "mpm_grad_v0_sum", "mpm_set_profiling", "mpm_reset_kernel_stats", "mpm_kernel_stats", "mpm_active_nodes",
           "mpm_active_nodes_at", "mpm_set_materials", "mpm_set_subdomain", "mpm_dd_link",
           "mpm_set_state_ids", "mpm_dd_forward", "mpm_dd_loss", "mpm_dd_backward", "mpm_dd_rows",
           "mpm_get_state_ids"]


class MpmError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str = ""):
        super().__init__(f"{fn}: {STATUS_NAMES.get(status, status)} {msg}".strip())
        self.status = status


class mpm_params(ct.Structure):
    _fields_ = [("gravity", ct.c_float), ("p_mass", ct.c_float), ("p_vol", ct.c_float),
                ("eps_mass", ct.c_float), ("bound", ct.c_int32), ("model", ct.c_int32),
                ("k_ckpt", ct.c_int32), ("max_steps", ct.c_int32), ("n_actuators", ct.c_int32),
                ("act_strength", ct.c_float), ("act_axis", ct.c_int32), ("n_sin", ct.c_int32),
                ("omega", ct.c_float), ("ctrl_hidden", ct.c_int32), ("n_episodes", ct.c_int32),
                ("deterministic", ct.c_int32), ("loss_kind", ct.c_int32),
                ("loss_target", ct.c_float * 3), ("max_active_blocks", ct.c_int32),
                ("grid_store_blocks", ct.c_int64), ("closed_loop", ct.c_int32),
                ("obs_scale_x", ct.c_float), ("obs_scale_v", ct.c_float)]


_lib = None


def load() -> ct.CDLL:
    """Load the CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1910_00935_b200.build` "
                              "(the hot path has no CPU fallback)")
        L = ct.CDLL(LIB_PATH)
        H, P, S = ct.c_void_p, ct.c_void_p, ct.c_int
        sig = {
            "mpm_create": [ct.c_int64, ct.c_int32, ct.c_int32, ct.c_float, ct.c_float, ct.c_float,
                           ct.POINTER(ct.c_void_p)],
            "mpm_destroy": [H], "mpm_default_params": [ct.c_int32, ct.POINTER(mpm_params)],
            "mpm_get_params": [H, ct.POINTER(mpm_params)],
            "mpm_set_params": [H, ct.POINTER(mpm_params)], "mpm_set_stream": [H, P],
            "mpm_workspace_bytes": [H, ct.POINTER(ct.c_size_t)],
            "mpm_workspace_bytes_for": [H, ct.c_int32, ct.POINTER(ct.c_size_t)],
            "mpm_bind_workspace": [H, P, ct.c_size_t], "mpm_set_state": [H, P, P, P, P, P],
            "mpm_n_theta": [H, ct.POINTER(ct.c_int64)], "mpm_set_controller": [H, P, ct.c_int64],
            "mpm_forward": [H, ct.c_int32], "mpm_loss": [H, P], "mpm_seed_adjoint": [H, P, P, P, P],
            "mpm_backward": [H, ct.c_int32], "mpm_grads": [H, P, P, P, P, P],
            "mpm_get_state": [H, P, P, P, P], "mpm_launch_count": [H, ct.POINTER(ct.c_int64)],
            "mpm_grad_v0_sum": [H, P], "mpm_set_profiling": [H, ct.c_int32], "mpm_reset_kernel_stats": [H],
            "mpm_kernel_stats": [H, ct.c_int32, ct.POINTER(ct.c_char_p), ct.POINTER(ct.c_double),
                                 ct.POINTER(ct.c_int64)],
            "mpm_active_nodes": [H, ct.POINTER(ct.c_int64)], "mpm_set_materials": [H, P],
            "mpm_active_nodes_at": [H, ct.c_int32, ct.POINTER(ct.c_int64)],
            "mpm_set_subdomain": [H, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32],
            "mpm_dd_link": [ct.POINTER(ct.c_void_p), ct.c_int32],
            "mpm_set_state_ids": [H, ct.c_int64, P, P, P, P, P],
            "mpm_dd_forward": [ct.POINTER(ct.c_void_p), ct.c_int32, ct.c_int32],
            "mpm_dd_loss": [ct.POINTER(ct.c_void_p), ct.c_int32, P],
            "mpm_dd_backward": [ct.POINTER(ct.c_void_p), ct.c_int32, ct.c_int32],
            "mpm_dd_rows": [H, ct.POINTER(ct.c_int64)],
            "mpm_get_state_ids": [H, P, P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = S
        L.mpm_last_error.argtypes = [H]
        L.mpm_last_error.restype = ct.c_char_p
        _lib = L
    return _lib


def _ptr(a, dtype=np.float32):
    """device or host address of a contiguous torch tensor / numpy array (None -> NULL)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        want = torch.float32 if dtype == np.float32 else torch.int32
        t = a if (a.dtype == want and a.is_contiguous()) else a.to(want).contiguous()
        return ct.c_void_p(t.data_ptr()), t
    arr = np.ascontiguousarray(a, dtype=dtype)
    return ct.c_void_p(arr.ctypes.data), arr


class Sim:
    """One mpm handle with a torch-owned workspace on the current CUDA device."""

    def __init__(self, n_particles: int, n_grid: int, dim: int, dt: float, E: float, nu: float,
                 params: dict | None = None, stream=None, probe_only: bool = False, subdomain=None):
        """subdomain = (x_lo, x_hi, n_body[, migrate_cap]): this handle is one slab of a decomposed
        body (include/mpm.h); n_particles is then its particle capacity."""
        import torch
        self.L = load()
        self.h = ct.c_void_p()
        self._check("mpm_create", self.L.mpm_create(int(n_particles), int(n_grid), int(dim),
                                                    float(dt), float(E), float(nu), ct.byref(self.h)),
                    use_handle=False)
        self.dim, self.N = int(dim), int(n_particles)
        p = mpm_params()
        self._check("mpm_get_params", self.L.mpm_get_params(self.h, ct.byref(p)))
        for k, v in (params or {}).items():
            if k == "loss_target":
                for i, x in enumerate(list(v)[:3]):
                    p.loss_target[i] = float(x)
            else:
                setattr(p, k, v)
        self._check("mpm_set_params", self.L.mpm_set_params(self.h, ct.byref(p)))
        self.params = p
        if subdomain is not None:
            lo, hi, nbody, *cap = subdomain
            self._check("mpm_set_subdomain", self.L.mpm_set_subdomain(self.h, int(lo), int(hi), int(nbody),
                                                                      int(cap[0]) if cap else 0))
        self.E = int(p.n_episodes)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self._check("mpm_set_stream", self.L.mpm_set_stream(self.h, ct.c_void_p(self.stream.cuda_stream)))
        nbytes = ct.c_size_t()
        self._check("mpm_workspace_bytes", self.L.mpm_workspace_bytes(self.h, ct.byref(nbytes)))
        self.workspace_bytes = int(nbytes.value)
        self.n_theta = 0
        if probe_only:  # size query only: no workspace
            return
        self.workspace = torch.empty(self.workspace_bytes + 256, dtype=torch.uint8, device="cuda")
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self._check("mpm_bind_workspace", self.L.mpm_bind_workspace(self.h, ct.c_void_p(aligned),
                                                                    self.workspace_bytes))
        nth = ct.c_int64()
        self._check("mpm_n_theta", self.L.mpm_n_theta(self.h, ct.byref(nth)))
        self.n_theta = int(nth.value)

    # ------------------------------------------------------------------ calls
    def _check(self, fn, st, use_handle=True):
        if st != MPM_OK:
            msg = ""
            if use_handle and self.h:
                msg = (self.L.mpm_last_error(self.h) or b"").decode()
            raise MpmError(fn, st, msg)

    def set_state(self, x, v=None, C=None, F=None, aid=None):
        keep = [_ptr(a) for a in (x, v, C, F)] + [_ptr(aid, np.int32)]
        self._check("mpm_set_state", self.L.mpm_set_state(self.h, *[k[0] for k in keep]))

    def set_materials(self, mat):
        """per-particle material [E][N] (0 solid, 1 fluid; R23), or None = all solid."""
        if mat is None:
            self._check("mpm_set_materials", self.L.mpm_set_materials(self.h, None))
            return
        ptr, keep = _ptr(mat, np.int32)
        self._check("mpm_set_materials", self.L.mpm_set_materials(self.h, ptr))

    def set_controller(self, theta):
        if self.n_theta == 0:
            return
        ptr, keep = _ptr(theta)
        self._check("mpm_set_controller", self.L.mpm_set_controller(self.h, ptr, self.n_theta))

    def forward(self, steps: int):
        self._check("mpm_forward", self.L.mpm_forward(self.h, int(steps)))

    def loss(self, out=None):
        out = np.zeros(self.E, np.float32) if out is None else out
        ptr, keep = _ptr(out)
        self._check("mpm_loss", self.L.mpm_loss(self.h, ptr))
        return out

    def seed_adjoint(self, dx=None, dv=None, dC=None, dF=None):
        keep = [_ptr(a) for a in (dx, dv, dC, dF)]
        self._check("mpm_seed_adjoint", self.L.mpm_seed_adjoint(self.h, *[k[0] for k in keep]))

    def backward(self, steps: int):
        self._check("mpm_backward", self.L.mpm_backward(self.h, int(steps)))

    def _alloc(self, like, shape):
        if like == "numpy":
            return np.zeros(shape, np.float32)
        import torch
        return torch.empty(shape, dtype=torch.float32, device=like)

    def grads(self, out: str | dict = "numpy"):
        """dL/d(x0, v0, C0, F0, theta); out = "numpy" | a torch device | dict of buffers."""
        d, EN = self.dim, self.E * self.N
        shapes = {"dx0": (self.E, self.N, d), "dv0": (self.E, self.N, d),
                  "dC0": (self.E, self.N, d, d), "dF0": (self.E, self.N, d, d),
                  "dtheta": (max(self.n_theta, 0),)}
        bufs = out if isinstance(out, dict) else {k: self._alloc(out, s) for k, s in shapes.items()}
        ptrs = [(_ptr(bufs[k])[0] if bufs.get(k) is not None and (k != "dtheta" or self.n_theta) else None)
                for k in shapes]
        self._check("mpm_grads", self.L.mpm_grads(self.h, *ptrs))
        return bufs

    def grad_v0_sum(self, out=None):
        """sum_p dL/dv0_p per episode: [E][d] (host numpy, or a given buffer)."""
        out = np.zeros((self.E, self.dim), np.float32) if out is None else out
        ptr, keep = _ptr(out)
        self._check("mpm_grad_v0_sum", self.L.mpm_grad_v0_sum(self.h, ptr))
        return out

    def get_state(self, out: str = "numpy"):
        d = self.dim
        shapes = {"x": (self.E, self.N, d), "v": (self.E, self.N, d),
                  "C": (self.E, self.N, d, d), "F": (self.E, self.N, d, d)}
        bufs = {k: self._alloc(out, s) for k, s in shapes.items()}
        self._check("mpm_get_state", self.L.mpm_get_state(self.h, *[_ptr(bufs[k])[0] for k in shapes]))
        return bufs

    # ---- slab subdomain of a decomposed body (f3)
    def set_state_ids(self, x, v, C, F, ids):
        n = int(len(ids))
        keep = [_ptr(a) for a in (x, v, C, F)] + [_ptr(ids, np.int32)]
        self._check("mpm_set_state_ids", self.L.mpm_set_state_ids(self.h, n, *[k[0] for k in keep]))

    def dd_rows(self) -> int:
        c = ct.c_int64()
        self._check("mpm_dd_rows", self.L.mpm_dd_rows(self.h, ct.byref(c)))
        return int(c.value)

    def get_state_ids(self):
        """S_T rows of this subdomain (its particles of step T-1) and their body-wide ids."""
        n, d = self.dd_rows(), self.dim
        out = {"x": np.zeros((n, d), np.float32), "v": np.zeros((n, d), np.float32),
               "C": np.zeros((n, d, d), np.float32), "F": np.zeros((n, d, d), np.float32),
               "ids": np.zeros(n, np.int32)}
        self._check("mpm_get_state_ids", self.L.mpm_get_state_ids(
            self.h, *[_ptr(out[k], np.int32 if k == "ids" else np.float32)[0] for k in ("x", "v", "C", "F", "ids")]))
        return out

    def grads_rows(self, n: int):
        """gradients of the n rows given to set_state_ids (that order)"""
        d = self.dim
        out = {"dx0": np.zeros((n, d), np.float32), "dv0": np.zeros((n, d), np.float32),
               "dC0": np.zeros((n, d, d), np.float32), "dF0": np.zeros((n, d, d), np.float32)}
        self._check("mpm_grads", self.L.mpm_grads(self.h, *[_ptr(out[k])[0] for k in ("dx0", "dv0", "dC0", "dF0")], None))
        return out

    def launch_count(self) -> int:
        c = ct.c_int64()
        self._check("mpm_launch_count", self.L.mpm_launch_count(self.h, ct.byref(c)))
        return int(c.value)

    def set_profiling(self, on: bool):
        self._check("mpm_set_profiling", self.L.mpm_set_profiling(self.h, int(bool(on))))

    def reset_kernel_stats(self):
        self._check("mpm_reset_kernel_stats", self.L.mpm_reset_kernel_stats(self.h))

    def kernel_stats(self) -> dict:
        """{kernel class: (total device ms, launches)} since the last reset."""
        out, i = {}, 0
        while True:
            name, ms, n = ct.c_char_p(), ct.c_double(), ct.c_int64()
            st = self.L.mpm_kernel_stats(self.h, i, ct.byref(name), ct.byref(ms), ct.byref(n))
            if st != MPM_OK:
                break
            out[name.value.decode()] = (float(ms.value), int(n.value))
            i += 1
        return out

    def active_nodes(self, step: int | None = None) -> int:
        """grid nodes with M > 0 at `step` of the recorded forward (default: the last step)"""
        c = ct.c_int64()
        if step is None:
            self._check("mpm_active_nodes", self.L.mpm_active_nodes(self.h, ct.byref(c)))
        else:
            self._check("mpm_active_nodes_at", self.L.mpm_active_nodes_at(self.h, int(step), ct.byref(c)))
        return int(c.value)

    def close(self):
        if self.h:
            self.L.mpm_destroy(self.h)
            self.h = ct.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _handles(sims):
    arr = (ct.c_void_p * len(sims))(*[s.h.value for s in sims])
    return arr, len(sims)


def _dd_call(name, sims, *args):
    arr, n = _handles(sims)
    st = getattr(load(), name)(arr, n, *args)
    if st != MPM_OK:
        msgs = "; ".join((load().mpm_last_error(s.h) or b"").decode() for s in sims)
        raise MpmError(name, st, msgs)


def dd_link(sims):
    """link the slab subdomains of one body (in slab order)"""
    _dd_call("mpm_dd_link", sims)


def dd_forward(sims, steps: int):
    _dd_call("mpm_dd_forward", sims, int(steps))


def dd_loss(sims) -> float:
    out = np.zeros(1, np.float32)
    _dd_call("mpm_dd_loss", sims, ct.c_void_p(out.ctypes.data))
    return float(out[0])


def dd_backward(sims, steps: int):
    _dd_call("mpm_dd_backward", sims, int(steps))


def sim_from_config(p: dict, n_particles: int, episodes: int | None = None,
                    max_steps: int | None = None, k_ckpt: int | None = None, probe_only: bool = False,
                    subdomain=None, **overrides) -> Sim:
    """Build a Sim from a workload config dict (paper_1910_00935_b200.workloads)."""
    dim = int(p["dim"])
    model = p.get("model", "neohookean")
    model = {"neohookean": 0, "nh": 0, "fixed_corotated": 1, "fcr": 1}[model] if isinstance(model, str) else int(model)
    E_ = int(episodes if episodes is not None else p.get("episodes", 1))
    params = dict(gravity=float(p.get("gravity", 0.0)), p_mass=float(p.get("p_mass", 1.0)),
                  p_vol=float(p.get("p_vol", 1.0)), eps_mass=float(p.get("eps_mass", 1e-10)),
                  bound=int(p.get("bound", 3)), model=model,
                  k_ckpt=int(k_ckpt if k_ckpt is not None else p.get("k_ckpt", 1)),
                  max_steps=int(max_steps if max_steps is not None else p["steps"]),
                  n_actuators=int(p.get("n_act", 0)), act_strength=float(p.get("kappa", 0.0)),
                  act_axis=int(p.get("act_axis", 1)), n_sin=int(p.get("n_sin", 4)),
                  omega=float(p.get("omega", 20.0)), ctrl_hidden=int(p.get("hidden", 0)),
                  closed_loop=int(bool(p.get("closed_loop", False))),
                  obs_scale_x=float(p.get("obs_sx", 10.0)), obs_scale_v=float(p.get("obs_sv", 1.0)),
                  n_episodes=E_, deterministic=int(p.get("deterministic", 0)),
                  loss_kind={"com_target": 0, "move_forward": 1}[p.get("loss", "com_target")],
                  loss_target=list(p.get("target", [0, 0, 0])))
    params.update(overrides)
    return Sim(int(n_particles), int(p["n_grid"]), dim, float(p["dt"]), float(p["E"]),
               float(p["nu"]), params, probe_only=probe_only, subdomain=subdomain)
