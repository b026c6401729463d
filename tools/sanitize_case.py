"""One small forward + loss + backward through the C-ABI, for compute-sanitizer runs
(tools/sanitize.sh).  Cases exercise every kernel class: the 2D block (c1a), a tiny 3D
closed-loop robot with fluid particles on the sticky floor, and C3 (29,952 particles, many
blocks per CTA: the cp.async.bulk / mbarrier double-buffered tile pipelines, the ticketed scan).
Checkpointing k < T so the segment re-forward runs; CUDA graphs on a side stream."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_00935_b200 import mpm, workloads as W  # noqa: E402


def case(name):
    if name == "c1a":
        return W.config("c1a", steps=8), 4
    if name == "tiny3d_cl_fluid":
        return W.tiny(3, steps=6, hidden=3, closed_loop=True, fluid_every=3, bound=3, floor=True,
                      v_base=(0.2, -1.5, 0.1), seed=3), 4
    if name == "c3":
        return W.config("c3", steps=int(os.environ.get("SAN_STEPS", 6))), 4
    raise SystemExit(f"unknown case {name}")


def main():
    name = sys.argv[1]
    p, k = case(name)
    inp = W.make_inputs(p)
    N = len(inp["x"])
    T = p["steps"]
    with torch.cuda.stream(torch.cuda.Stream()):
        sim = mpm.sim_from_config(p, N, max_steps=T, k_ckpt=k)
        sim.set_state(inp["x"][None], inp["v"][None], inp["C"][None], inp["F"][None], inp["aid"][None])
        if np.any(inp.get("mat", 0)):
            sim.set_materials(inp["mat"][None])
        sim.set_controller(inp["theta"])
        for _ in range(2):  # second iteration replays the captured graphs
            sim.forward(T)
            L = sim.loss()
            sim.backward(T)
            g = sim.grads()
        sim.close()
    del sim
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # leak-check: return torch's cached blocks before exit
    print(f"{name}: N={N} T={T} k={k} loss={L[0]:.6e} |dv0|={np.linalg.norm(g['dv0']):.6e}")


if __name__ == "__main__":
    main()
