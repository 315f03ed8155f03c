"""A few standalone applies (for ncu captures of the apply-only kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
k5 = int(sys.argv[3]) if len(sys.argv) > 3 else 16   # (config 5: entries per row)
p = configs.config(cfg, k5=k5)
b = int(sys.argv[4]) if len(sys.argv) > 4 else (p.block or 16)
with from_problem(p) as h:
    X = torch.from_numpy(configs.x_block(p.n, b, seed=3)).cuda()
    Y = torch.empty_like(X)
    for _ in range(reps):
        h.apply(X, out=Y)
    torch.cuda.synchronize()
