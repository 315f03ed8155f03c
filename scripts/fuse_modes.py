"""eigs breakdown (config 4 by default) for the fuse modes given after the config (default 0 1 2 3)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    modes = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 3]
    for f in modes + modes:
        h.set_option("fuse", f)
        h.eigs(p.m, p.block, max_iters=10, tol=0.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.eigs(p.m, p.block, max_iters=50, tol=0.0); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        h.set_option("profile", (1 << len(FAM)) - 1); h.set_option("profile_reset", 1)
        h.eigs(p.m, p.block, max_iters=50, tol=0.0); torch.cuda.synchronize()
        br = {k: round(h.stat(k + "_ns") / 5e7, 4) for k in FAM}
        h.set_option("profile", 0)
        lam = h.eigs(p.m, p.block, max_iters=50, tol=0.0)[0]
        print(json.dumps({"fuse": f, "eigs_ms": round(t, 2), "per_iter_ms": br, "lam": [float(x) for x in lam]}), flush=True)
