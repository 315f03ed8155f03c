import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(2)
with from_problem(p) as h:
    for mr in (0, 303104, 0, 303104):
        h.set_option("sp8_min_rows", mr)
        for _ in range(3): h.eigs(8, 32, max_iters=50, tol=0.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10): h.eigs(8, 32, max_iters=50, tol=0.0)
        torch.cuda.synchronize()
        print(json.dumps({"config": 2, "b": 32, "sp8_min_rows": mr, "ms_per_solve": round((time.perf_counter() - t0) * 100, 3)}), flush=True)
