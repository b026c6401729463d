"""Closed-loop controller (R22) on the CUDA path vs the fp64
CPU oracle, through the C-ABI, on the same seeded inputs.  Gates as the open-loop parity tests
(states rel <= 1e-4, gradients rel-L2 <= 1e-3, or 2x the oracle's own fp32-vs-fp64 deviation
on the long robot horizons)."""
import numpy as np
import pytest

from helpers import check, compare_episode, gpu_run, inputs, oracle_run, rel
from paper_1910_00935_b200 import workloads as W

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-4
GRAD_TOL = 1e-3


def _tiny(dim, **kw):
    base = dict(steps=10, hidden=3, bound=3, floor=True, seed=5, closed_loop=True)
    base.update(v_base=(0.3, -1.5) if dim == 2 else (0.2, -1.5, 0.1))
    base.update(kw)
    return W.tiny(dim, **base)


TINY = {
    "2d_fcr_hidden": lambda: _tiny(2, seed=7),
    "2d_fcr_linear": lambda: _tiny(2, hidden=0, seed=9),
    "3d_nh_hidden": lambda: _tiny(3, steps=8, seed=8),
}


@pytest.mark.parametrize("case", list(TINY))
def test_tiny_closed_loop_matches_oracle(case):
    p = TINY[case]()
    inp = W.make_inputs(p)
    inp["theta"] = (inp["theta"] * 0.5).astype(np.float32)
    got = gpu_run(p, inp)
    rows, ref = compare_episode(f"tiny_closed_loop/{case}", p, inp, got, with_f32=False)
    check(rows, case)
    assert np.linalg.norm(ref["dtheta"]) > 0


def test_closed_loop_episodes_are_independent():
    """E = 3 episodes (different inputs) in one launch: each episode's states and initial-state
    gradients equal its own oracle run; theta_bar is their sum."""
    p = _tiny(2, seed=11)
    per = [W.make_inputs(p, episode=e) for e in range(3)]
    for q in per:
        q["theta"] = (q["theta"] * 0.5).astype(np.float32)
    got = gpu_run(p, per)
    thb = 0.0
    for e, q in enumerate(per):
        ref = oracle_run(p, q)
        for k in "xvCF":
            assert rel(got[k][e], ref[k]) < STATE_TOL, (e, k)
        for k in ("dx0", "dv0", "dF0"):
            assert rel(got[k][e], ref[k]) < GRAD_TOL, (e, k, rel(got[k][e], ref[k]))
        thb = thb + ref["dtheta"]
    assert rel(got["dtheta"], thb) < GRAD_TOL


def test_closed_loop_bitwise_reproducible_and_checkpoint_invariant():
    p = _tiny(3, steps=12, seed=3)
    inp = W.make_inputs(p)
    a = gpu_run(p, inp, k_ckpt=1)
    b = gpu_run(p, inp, k_ckpt=1)
    c = gpu_run(p, inp, k_ckpt=5)
    for k in ("x", "v", "C", "F", "dx0", "dv0", "dC0", "dF0", "dtheta"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
        np.testing.assert_array_equal(a[k], c[k], err_msg=k)


def test_robot2d_closed_loop_c2cl():
    """C2 robot with the closed-loop controller (4 muscles x 2d observations), 256 steps."""
    p, inp = inputs("c2cl", steps=256)
    got = gpu_run(p, inp)
    rows, _ = compare_episode("c2cl@256", p, inp, got, grads=("dx0", "dv0", "dtheta"))
    check(rows, "c2cl")


def test_robot3d_closed_loop_c3cl_checkpointed():
    """C3 geometry, 16 muscles x 6 observations (input 100, H = 32), k = 32, 96 steps."""
    p, inp = inputs("c3cl", steps=96)
    got = gpu_run(p, inp, k_ckpt=32)
    rows, _ = compare_episode("c3cl@96", p, inp, got, grads=("dx0", "dv0", "dtheta"))
    check(rows, "c3cl")
