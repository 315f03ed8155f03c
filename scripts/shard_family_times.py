"""Per-kernel-family device times of the sharded eigensolver at world 1 (config 4 by default): the
per-rank kernel path a multi-GPU solve runs (fp32 sparse kernels, int8 D stream on the rank's tiles)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200.sbmds import shard_from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = configs.config(cfg)
with shard_from_problem(p, 0, 1) as h:
    h.eigs(p.m, p.block, max_iters=5, tol=0.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, _, info = h.eigs(p.m, p.block, max_iters=iters, tol=0.0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
    h.eigs(p.m, p.block, max_iters=iters, tol=0.0); torch.cuda.synchronize()
    fam = {f: round(h.stat(f + "_ns") / 1e6 / iters, 4) for f in FAM}
    h.set_option("profile", 0)
print(json.dumps({"config": cfg, "iters": iters, "gpu_ms_per_iter": info["gpu_ms"] / iters, "wall_ms_per_iter": wall * 1e3 / iters,
                  "family_ms_per_iter": fam}))
