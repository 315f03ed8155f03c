import sys, time, json, numpy as np, torch
sys.path.insert(0, '.')
from gen import configs
from paper_1705_10887_b200 import from_problem
for cfg in [int(c) for c in sys.argv[1:]]:
    p = configs.config(cfg)
    with from_problem(p) as h:
        h.eigs(p.m, p.block, max_iters=20, tol=0.0)   # warm
        torch.cuda.synchronize()
        for tol in (1e-5, 1e-6):
            t = time.perf_counter()
            lam, V, Z, info = h.eigs(p.m, p.block, max_iters=2000, tol=tol)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            print(json.dumps({"config": cfg, "tol": tol, "iters": info["iters"], "seconds": round(dt, 4),
                              "ms_per_iter": round(1e3 * dt / info["iters"], 4), "converged": info["converged"],
                              "max_residual": info["max_residual"], "lam": [float(x) for x in lam]}), flush=True)
