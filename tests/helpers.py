"""Shared drivers for the parity tests: the same seeded inputs go to the CUDA
path (through the C-ABI) and to the CPU oracle.

Every comparison is recorded (one JSON line per array: L2 and element-wise errors, the gates,
the oracle's own fp32-vs-fp64 deviation and whether the SURVEY 8(c) fallback gate was used) to
$MPM_PARITY_RECORD (default gpurun_out/parity_record.jsonl), from which
profiles/parity_record_r02.jsonl and BASELINE.md section 4 are filled."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_1910_00935_b200 import workloads as W


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def maxerr(a, b):
    """element-wise bound: max_i |a_i - b_i| / max_i |b_i|"""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.abs(b).max() if b.size else 0.0
    d = np.abs(a - b).max() if b.size else 0.0
    return float(d / nb) if nb > 0 else float(d)


STATE_TOL = 1e-4  # north_star: final states rel <= 1e-4 (per array, ||d|| / ||ref||)
GRAD_TOL = 1e-3   # north_star: gradients rel-L2 <= 1e-3
ELEM_FACTOR = 10  # element-wise gate: max |d| / max |ref| <= 10x the L2 gate
STATE_KEYS = ("x", "v", "C", "F", "loss")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def record_path():
    return os.environ.get("MPM_PARITY_RECORD", os.path.join(ROOT, "gpurun_out", "parity_record.jsonl"))


def record(case, rows):
    path = record_path()
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "a") as f:
            for r in rows:
                f.write(json.dumps(dict(case=case, time=time.strftime("%Y-%m-%dT%H:%M:%S"), **r)) + "\n")
    except OSError:
        pass


def compare_arrays(case, pairs, dev32=None, e=0):
    """pairs: {name: (got, ref)}; dev32: {name: (l2, max)} of the oracle's fp32 build vs fp64.
    Gates: the north_star tolerance (or 2x / 4x the oracle-fp32 deviation where that is larger,
    SURVEY 8(c) fallback -- recorded as such).  Returns the rows; check() asserts them."""
    rows = []
    for k, (g, r) in pairs.items():
        base = STATE_TOL if k in STATE_KEYS else GRAD_TOL
        d32 = (dev32 or {}).get(k, (0.0, 0.0))
        l2, mx = rel(g, r), maxerr(g, r)
        l2_gate = max(base, 2.0 * d32[0])
        mx_gate = max(ELEM_FACTOR * base, 4.0 * d32[1])
        rows.append(dict(episode=e, array=k, l2_err=l2, l2_gate=l2_gate, max_err=mx, max_gate=mx_gate,
                         oracle_f32_l2=d32[0] if dev32 else None, oracle_f32_max=d32[1] if dev32 else None,
                         fallback=bool(l2_gate > base or mx_gate > ELEM_FACTOR * base),
                         # passed only thanks to the widened gate
                         fallback_used=bool(l2 >= base or mx >= ELEM_FACTOR * base),
                         passed=bool(l2 < l2_gate and mx < mx_gate)))
    record(case, rows)
    print(f"[parity] {case} e={e}: " + ", ".join(
        f"{r['array']} {r['l2_err']:.1e}/{r['max_err']:.1e} (gates {r['l2_gate']:.0e}/{r['max_gate']:.0e}"
        f"{', fallback gate USED' if r['fallback_used'] else ''})" for r in rows))
    return rows


def check(rows, tag=""):
    bad = [r for r in rows if not r["passed"]]
    assert not bad, (tag, bad)


def oracle_pair(p, inp, steps=None, with_f32=True):
    """fp64 and fp32 oracle runs of the same episode, concurrently (ctypes releases the GIL)"""
    with ThreadPoolExecutor(2) as ex:
        f64 = ex.submit(oracle_run, p, inp, steps)
        f32 = ex.submit(oracle_run, p, inp, steps, "f32") if with_f32 else None
        return f64.result(), (f32.result() if f32 else None)


def episode_pairs(got, ref, e, grads):
    """{name: (gpu, oracle)} for the states, the loss and the listed gradients of episode e"""
    pairs = {k: (got[k][e], ref[k]) for k in "xvCF"}
    for k in grads:
        if k == "dtheta":
            if ref[k].size:
                pairs[k] = (got[k], ref[k])
        elif np.linalg.norm(ref[k]) > 1e-12:
            pairs[k] = (got[k][e], ref[k])
    if got.get("loss") is not None:
        pairs["loss"] = (np.array([got["loss"][e]]), np.array([ref["loss"]]))
    return pairs


def compare_episode(case, p, inp, got, steps=None, e=0, grads=("dx0", "dv0", "dC0", "dF0", "dtheta"),
                    with_f32=True, refs=None):
    """GPU episode e vs the fp64 oracle (+ the fp32 oracle for the fallback gates).
    Returns (rows, fp64 oracle result)."""
    ref, ref32 = refs if refs is not None else oracle_pair(p, inp, steps, with_f32)
    pairs = episode_pairs(got, ref, e, grads)
    dev32 = None
    if ref32 is not None:
        as_got = {k: ref32[k][None] for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0")}
        as_got["dtheta"] = ref32["dtheta"]
        as_got["loss"] = np.array([ref32["loss"]])
        dev32 = {k: (rel(g, r), maxerr(g, r)) for k, (g, r) in episode_pairs(as_got, ref, 0, grads).items()}
    return compare_arrays(case, pairs, dev32, e), ref


def gpu_run(p, inputs, steps=None, k_ckpt=None, episodes=1, seed=None, **over):
    """forward(T) + loss (or a caller seed) + backward(T) + grads through the C-ABI.
    inputs: one dict (episodes = 1) or a list of per-episode dicts."""
    from paper_1910_00935_b200 import mpm
    if isinstance(inputs, dict):
        inputs = [inputs]
    E = len(inputs)
    T = int(steps or p["steps"])
    N = len(inputs[0]["x"])
    sim = mpm.sim_from_config(p, N, episodes=E, max_steps=T, k_ckpt=k_ckpt, **over)
    cat = lambda k: np.ascontiguousarray(np.stack([i[k] for i in inputs]))  # noqa: E731
    sim.set_state(cat("x"), cat("v"), cat("C"), cat("F"), cat("aid"))
    if all("mat" in i for i in inputs) and any(np.any(i["mat"]) for i in inputs):
        sim.set_materials(cat("mat"))
    sim.set_controller(inputs[0]["theta"])
    sim.forward(T)
    st = sim.get_state()
    if seed is None:
        loss = sim.loss()
    else:
        sim.seed_adjoint(*[np.ascontiguousarray(s, np.float32) for s in seed])
        loss = None
    sim.backward(T)
    g = sim.grads()
    out = dict(x=st["x"], v=st["v"], C=st["C"], F=st["F"], loss=loss, dx0=g["dx0"], dv0=g["dv0"],
               dC0=g["dC0"], dF0=g["dF0"], dtheta=g["dtheta"], launches=sim.launch_count())
    sim.close()
    return out


def oracle_run(p, inp, steps=None, precision="f64"):
    from oracle import Oracle
    o = Oracle(p, precision)
    if inp.get("mat") is not None and np.any(inp["mat"]):
        o.set_materials(inp["mat"])
    return o.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"],
                 steps=steps or p["steps"],
                 k_ckpt=1 if (steps or p["steps"]) * len(inp["x"]) <= 5_000_000 else 16)


def oracle_tape(p, inp, T, lam):
    """oracle forward T steps + reverse with the linear loss <lam, S_T>."""
    from oracle import Oracle
    o = Oracle(p)
    if inp.get("mat") is not None and np.any(inp["mat"]):
        o.set_materials(inp["mat"])
    x, v, C, F = (inp[k].astype(np.float64) for k in "xvCF")
    th = inp["theta"].astype(np.float64)
    hist = []
    for t in range(T):
        al = o.controller(th, t) if o.cfg.n_act else None
        hist.append((x, v, C, F, al))
        x, v, C, F = o.step(x, v, C, F, inp["aid"], al)
    bars = [np.asarray(l, np.float64) for l in lam]
    thb = np.zeros_like(th)
    for t in reversed(range(T)):
        xs, vs, Cs, Fs, al = hist[t]
        *bars, ab = o.step_adj(xs, vs, Cs, Fs, *bars, inp["aid"], al)
        if o.cfg.n_act:
            thb += o.controller_adj(th, t, ab[: o.cfg.n_act])
    return dict(x=x, v=v, C=C, F=F, dx0=bars[0], dv0=bars[1], dC0=bars[2], dF0=bars[3], dtheta=thb)


def inputs(name, **over):
    p = W.config(name, **over)
    return p, W.make_inputs(p)
