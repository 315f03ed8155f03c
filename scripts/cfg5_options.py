"""Config 5: standalone apply time for row order (natural / reordered) x blocked mask, b in {16, 64}."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
k = int(sys.argv[1])
p = configs.config(5, k5=k)
for reorder in (False, True):
    with from_problem(p, reorder_rows=reorder) as h:
        for b in (16, 64):
            X = torch.randn(p.n, b, device="cuda"); Y = torch.empty_like(X)
            for blk in (0, 1, 2, 3):
                h.set_option("blocked", blk)
                for _ in range(2): h.apply(X, out=Y)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
                e0.record()
                for _ in range(5): h.apply(X, out=Y)
                e1.record(); torch.cuda.synchronize()
                fam = {f: round(h.stat(f + "_ns") / 5e6, 3) for f in ("colsum", "csc", "dstream", "csr")}
                print(json.dumps({"k": k, "reorder": reorder, "b": b, "blocked": blk, "umax": h.stat("blocked_umax"),
                                  "apply_ms": round(e0.elapsed_time(e1) / 5, 3), **fam}), flush=True)
                h.set_option("profile", 0)
            del X, Y
