"""Per-family device times of the sharded eigensolver at world 1 vs the plain handle (config arg)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
from paper_1705_10887_b200.sbmds import shard_from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]
p = configs.config(int(sys.argv[1]))
for name, mk in (("shard", lambda: shard_from_problem(p, 0, 1)), ("plain_fuse0", lambda: from_problem(p))):
    with mk() as h:
        if name == "plain_fuse0":
            h.set_option("fuse", 0)
        h.eigs(p.m, p.block, max_iters=10, tol=0.0)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.eigs(p.m, p.block, max_iters=20, tol=0.0); e1.record(); torch.cuda.synchronize()
        print(json.dumps({name: {f: round(h.stat(f + "_ns") / 20e6, 4) for f in FAM}, "ms_per_iter": round(e0.elapsed_time(e1) / 20, 3)}), flush=True)
