"""Short driver for ncu captures: one C5-sized (or other config) forward + backward of a few
steps through the C-ABI.  Not a benchmark -- numbers printed under ncu are never bench values."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_00935_b200 import mpm, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
p = W.config(a.config)
inp = W.make_inputs(p)
N = len(inp["x"])
sim = mpm.sim_from_config(p, N, max_steps=a.steps, k_ckpt=a.k)
dev = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
for _ in range(a.iters):
    sim.set_state(dev["x"], dev["v"], dev["C"], dev["F"], dev["aid"])
    sim.set_controller(dev["theta"])
    sim.forward(a.steps)
    sim.loss()
    sim.backward(a.steps)
torch.cuda.synchronize()
print("done", sim.launch_count())
