"""50-iteration eigs time with use_graph = 0 / 1 (warm handle, 3 calls each, median)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import configs
from paper_1705_10887_b200 import from_problem
for cfg in [int(c) for c in sys.argv[1:]] or [1, 2]:
    p = configs.config(cfg)
    res = {}
    with from_problem(p) as h:
        for g in (0, 1):
            h.set_option("use_graph", g)
            ts = []
            for _ in range(4):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); h.eigs(p.m, p.block, max_iters=50, tol=0.0); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[g] = round(float(np.median(ts[1:])), 3)
    print(json.dumps({"config": cfg, "eigs50_ms_by_use_graph": res}), flush=True)
