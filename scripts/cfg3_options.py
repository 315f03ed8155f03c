"""Config 3 (Morton-ordered icosphere): apply and eigs family times for the sparse-kernel options
(order_columns, blocked, fuse) -- which layout the coherent vertex order wants."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = configs.config(cfg)
b = p.block
X = torch.randn(p.n, b, device="cuda"); Y = torch.empty_like(X)
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]
with from_problem(p) as h:
    for oc in (1, 0):
        for blk in (0, 1, 2, 3):
            h.set_option("order_columns", oc); h.set_option("blocked", blk)
            for _ in range(3): h.apply(X, out=Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
            e0.record()
            for _ in range(10): h.apply(X, out=Y)
            e1.record(); torch.cuda.synchronize()
            fam = {f: round(h.stat(f + "_ns") / 1e7, 4) for f in ("colsum", "csc", "csr")}
            print(json.dumps({"order_columns": oc, "blocked": blk, "apply_ms": round(e0.elapsed_time(e1) / 10, 4), **fam}), flush=True)
            h.set_option("profile", 0)
    h.set_option("order_columns", 1); h.set_option("blocked", 1)
    for fuse in (0, 1, 2):
        h.set_option("fuse", fuse)
        h.eigs(p.m, b, max_iters=5, tol=0.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.eigs(p.m, b, max_iters=50, tol=0.0); e1.record(); torch.cuda.synchronize()
        print(json.dumps({"fuse": fuse, "eigs50_ms": round(e0.elapsed_time(e1), 3)}), flush=True)
