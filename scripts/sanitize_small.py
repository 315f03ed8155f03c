import sys, numpy as np, torch
sys.path.insert(0, '.')
from gen import configs
from paper_1705_10887_b200 import from_problem
ds = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for p, b in ((configs.config(1), 8), (configs.random_problem(20_011, 1_001, 16, seed=1, name="r"), 16)):
    with from_problem(p) as h:
        h.set_option("dstream", ds)
        X = torch.from_numpy(configs.x_block(p.n, b, seed=1)).cuda()
        Y = h.apply(X)
        if p.m:
            h.eigs(p.m, p.block, max_iters=20, tol=0.0)
torch.cuda.synchronize()
print("ok", ds)
