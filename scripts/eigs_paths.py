"""50-iteration eigs time with the sparse-step variants (option fuse: 3 tensor-core step, 2 / 1 fp32 fused, 0 separate)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = configs.config(cfg)
b = int(sys.argv[2]) if len(sys.argv) > 2 else (p.block or 16)
with from_problem(p) as h:
    for fuse in (3, 2, 1, 0, 3):
        h.set_option("fuse", fuse)
        for _ in range(3): h.eigs(p.m, b, max_iters=50, tol=0.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10): h.eigs(p.m, b, max_iters=50, tol=0.0)
        torch.cuda.synchronize()
        print(json.dumps({"config": cfg, "b": b, "fuse": fuse, "ms_per_solve": round((time.perf_counter() - t0) * 100, 3),
                          "sp8_state": h.stat("sp8_state")}), flush=True)
