"""one body decomposed into slab subdomains (include/mpm.h mpm_dd_*,
csrc/engine_dd.cu) -- particles migrate between neighbouring subdomains every step and grid-node
sums at the slab faces read the neighbour's partial tiles, so the decomposed run must equal the
single-domain run BIT FOR BIT: final states, loss and every initial-state gradient (DESIGN.md
section 7).  Here the subdomains are separate handles on one GPU (the peer loads are same-device
loads); across GPUs the same loads go over NVLink."""
import numpy as np
import pytest

from paper_1910_00935_b200 import mpm, workloads as W

pytestmark = pytest.mark.gpu


def _block_x(p, x):
    B = 4 if p["dim"] == 3 else 8
    base = np.floor(x[:, 0].astype(np.float32) * np.float32(p["n_grid"]) - np.float32(0.5)).astype(np.int64)
    return base // B


def _single(p, inp, T, mat=None):
    N = len(inp["x"])
    sim = mpm.sim_from_config(p, N, max_steps=T, k_ckpt=1)
    sim.set_state(inp["x"][None], inp["v"][None], inp["C"][None], inp["F"][None], None)
    if mat is not None:
        sim.set_materials(mat[None])
    sim.forward(T)
    st = sim.get_state()
    L = float(sim.loss()[0])
    sim.backward(T)
    g = sim.grads()
    sim.close()
    out = {k: st[k][0] for k in "xvCF"}
    out.update({k: g[k][0] for k in ("dx0", "dv0", "dC0", "dF0")})
    out["loss"] = L
    return out


def _split(p, inp, T, cuts, cap_frac=0.75, mat=None, cap_per_slab=False):
    """cap_per_slab: each subdomain's capacity from its own particle count (unequal capacities, so
    unequal component strides of the neighbours' state arrays); else cap_frac * N for all."""
    N = len(inp["x"])
    B = 4 if p["dim"] == 3 else 8
    nb = -(-p["n_grid"] // B)
    bounds = [0] + list(cuts) + [nb]
    bx = _block_x(p, inp["x"])
    sims, sel = [], []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        ids = np.nonzero((bx >= lo) & (bx < hi))[0].astype(np.int32)
        sel.append(ids)
        cap = int(1.25 * len(ids)) + 8192 if cap_per_slab else int(cap_frac * N) + 4096
        sims.append(mpm.sim_from_config(p, cap, max_steps=T, k_ckpt=1, subdomain=(lo, hi, N)))
    assert sum(len(s) for s in sel) == N and all(len(s) > 0 for s in sel)
    mpm.dd_link(sims)
    for sim, ids in zip(sims, sel):
        sim.set_state_ids(inp["x"][ids], inp["v"][ids], inp["C"][ids], inp["F"][ids], ids)
        if mat is not None:
            sim.set_materials(mat)
    mpm.dd_forward(sims, T)
    L = mpm.dd_loss(sims)
    parts = [s.get_state_ids() for s in sims]
    mpm.dd_backward(sims, T)
    grads = [s.grads_rows(len(ids)) for s, ids in zip(sims, sel)]
    for s in sims:
        s.close()
    d = p["dim"]
    out = {"x": np.full((N, d), np.nan, np.float32), "v": np.full((N, d), np.nan, np.float32),
           "C": np.full((N, d, d), np.nan, np.float32), "F": np.full((N, d, d), np.nan, np.float32)}
    seen = np.zeros(N, np.int64)
    for q in parts:
        np.add.at(seen, q["ids"], 1)
        for k in "xvCF":
            out[k][q["ids"]] = q[k]
    assert np.all(seen == 1), "every particle is held by exactly one subdomain at T"
    for k in ("dx0", "dv0", "dC0", "dF0"):
        out[k] = np.zeros_like(out["x"] if k in ("dx0", "dv0") else out["C"])
        for ids, g in zip(sel, grads):
            out[k][ids] = g[k]
    out["loss"] = L
    # migration actually happened: some particles end in another slab than they started in
    bounds_a = np.array(bounds)
    start = np.searchsorted(bounds_a, bx, side="right") - 1
    end = np.searchsorted(bounds_a, _block_x(p, out["x"]), side="right") - 1
    out["migrated"] = int(np.sum(start != end))
    return out


def _assert_bitwise(a, b, tag):
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0"):
        assert np.array_equal(a[k], b[k]), (tag, k, float(np.abs(a[k] - b[k]).max()))
    assert a["loss"] == b["loss"], (tag, a["loss"], b["loss"])


def test_c5_two_slabs_bitwise_64_steps():
    """C5 at full size (1,061,208 particles, 128^3), split at x = 0.5 (block column 16), 64 steps
    through the landing on the sticky floor, forward + backward: bitwise equal to one domain."""
    T = 64
    p, inp = W.config("c5", steps=T), None
    inp = W.make_inputs(p)
    ref = _single(p, inp, T)
    got = _split(p, inp, T, cuts=[16], cap_frac=0.6)
    print(f"[f3] c5 2 slabs: {got['migrated']} particles changed slab, loss {got['loss']:.9g}")
    assert got["migrated"] > 0
    _assert_bitwise(got, ref, "c5/2")


def test_c5_four_unequal_slabs_bitwise_32_steps():
    """C5 at full size in 4 slabs of unequal width and capacity (each subdomain sized from its own
    particle count, so the neighbours' state arrays have different component strides), 32 steps:
    bitwise equal to one domain."""
    T = 32
    p = W.config("c5", steps=T)
    inp = W.make_inputs(p)
    ref = _single(p, inp, T)
    got = _split(p, inp, T, cuts=[12, 15, 19], cap_per_slab=True)
    print(f"[f3] c5 4 unequal slabs: {got['migrated']} particles changed slab")
    assert got["migrated"] > 0
    _assert_bitwise(got, ref, "c5/4")


def test_block2d_three_slabs_with_fluid_bitwise():
    """2D block hitting the floor (c1b), 128 steps, three slabs (the middle one has two
    neighbours), every third particle weakly compressible fluid (R23, material by body-wide id)."""
    T = 128
    p = W.config("c1b", steps=T)
    inp = W.make_inputs(p)
    mat = (np.arange(len(inp["x"])) % 3 == 0).astype(np.int32)
    ref = _single(p, inp, T, mat=mat)
    got = _split(p, inp, T, cuts=[3, 4], cap_frac=0.9, mat=mat)
    print(f"[f3] c1b 3 slabs: {got['migrated']} particles changed slab")
    assert got["migrated"] > 0
    _assert_bitwise(got, ref, "c1b/3")


def test_single_slab_equals_single_domain():
    """one subdomain covering the whole grid is the single-domain run (no neighbours)"""
    T = 32
    p = W.config("c1a", steps=T)
    inp = W.make_inputs(p)
    _assert_bitwise(_split(p, inp, T, cuts=[], cap_frac=1.0), _single(p, inp, T), "c1a/1")


def test_decomposition_errors():
    p = W.config("c1b", steps=4)
    inp = W.make_inputs(p)
    N = len(inp["x"])
    # a particle given to the wrong slab is an error, never silently simulated twice
    a = mpm.sim_from_config(p, N, max_steps=4, k_ckpt=1, subdomain=(0, 4, N))
    b = mpm.sim_from_config(p, N, max_steps=4, k_ckpt=1, subdomain=(4, 8, N))
    mpm.dd_link([a, b])
    ids = np.arange(N, dtype=np.int32)
    a.set_state_ids(inp["x"], inp["v"], inp["C"], inp["F"], ids)  # all of them, some belong to b
    b.set_state_ids(inp["x"][:0], inp["v"][:0], inp["C"][:0], inp["F"][:0], ids[:0])
    with pytest.raises(mpm.MpmError) as e:
        mpm.dd_forward([a, b], 4)
    assert e.value.status == 2
    a.close(), b.close()
    # actuated bodies and k_ckpt > 1 are out of the f3 scope: explicit error
    pr = W.config("c2", steps=4)
    c = mpm.sim_from_config(pr, 8000, max_steps=4, k_ckpt=1, subdomain=(0, 16, 6400))
    with pytest.raises(mpm.MpmError) as e:
        mpm.dd_link([c])
    assert e.value.status == 7
    c.close()
    # single-domain entry points refuse a subdomain handle
    s = mpm.sim_from_config(p, N, max_steps=4, k_ckpt=1, subdomain=(0, 8, N))
    with pytest.raises(mpm.MpmError) as e:
        s.set_state(inp["x"][None], inp["v"][None], inp["C"][None], inp["F"][None], None)
    assert e.value.status == 6
    s.close()
