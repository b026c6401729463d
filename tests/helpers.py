"""Shared drivers for the parity tests: the same seeded inputs go to the CUDA
path (through the C-ABI) and to the CPU oracle."""
import numpy as np

from paper_1910_00935_b200 import workloads as W


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


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
