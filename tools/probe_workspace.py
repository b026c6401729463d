"""Device workspace of C5 at T = 2,048 for k = 1, 2, 4 against the free HBM of the box
(measured round 1: free 190.8 GB; k = 1 274 GB, k = 2 165 GB, k = 4 111 GB)."""
import torch, sys
sys.path.insert(0, ".")
from paper_1910_00935_b200 import mpm, workloads as W
p = W.config("c5"); N = 102**3
free, total = torch.cuda.mem_get_info()
print("free GB", free/1e9, "total", total/1e9)
for k in (1, 2, 4):
    s = mpm.sim_from_config(p, N, max_steps=2048, k_ckpt=k, probe_only=True)
    print(k, s.workspace_bytes/1e9)
    s.close()
