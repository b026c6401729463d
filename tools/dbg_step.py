import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_1910_00935_b200 import mpm, workloads as W
from oracle import Oracle
for name, p in [("c1a", W.config("c1a", steps=4)), ("tiny2d", W.tiny(2, steps=4, hidden=3, bound=3, floor=True, seed=7, closed_loop=True, v_base=(0.3, -1.5)))]:
    inp = W.make_inputs(p)
    N = len(inp["x"])
    for T in (1, 2, 3):
        sim = mpm.sim_from_config(p, N, max_steps=T)
        sim.set_state(inp["x"][None], inp["v"][None], inp["C"][None], inp["F"][None], inp["aid"][None])
        sim.set_controller(inp["theta"])
        try:
            sim.forward(T)
            st = sim.get_state()
            ref = Oracle(p).run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"], steps=T)
            print(name, T, "x err", np.abs(st["x"][0] - ref["x"]).max(), "v err", np.abs(st["v"][0] - ref["v"]).max())
        except Exception as e:
            print(name, T, "ERR", e)
        sim.close()
