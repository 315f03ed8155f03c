"""Per-kernel-family device times (CUDA events, sbmds 'profile' option) of an eigs solve and of
standalone applies, natural vs reordered rows: which family a change moves."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]
cfg = int(sys.argv[1]); k5 = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = configs.config(cfg, k5=k5)
b = p.block or 16
out = {}
for reorder in (False, True):
    with from_problem(p, reorder_rows=reorder) as h:
        res = {"permuted": h.stat("row_permuted"), "umax": h.stat("blocked_umax")}
        if p.m:
            h.eigs(p.m, b, max_iters=10, tol=0.0)
            h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
            h.eigs(p.m, b, max_iters=20, tol=0.0); torch.cuda.synchronize()
            res["eigs_ms_per_iter"] = {f: round(h.stat(f + "_ns") / 20e6, 4) for f in FAM}
            h.set_option("profile", 0)
        X = torch.randn(p.n, b, device="cuda")
        Y = torch.empty_like(X)
        for _ in range(3): h.apply(X, out=Y)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        for _ in range(10): h.apply(X, out=Y)
        torch.cuda.synchronize()
        res["apply_ms"] = {f: round(h.stat(f + "_ns") / 10e6, 4) for f in FAM}
        out[str(reorder)] = res
print(json.dumps(out))
