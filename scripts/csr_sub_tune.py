"""CSR SpMM time (b = 1, 4) vs lanes per row on the config-5 structures."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
for k in (8, 16, 64):
    p = configs.config(5, k5=k)
    with from_problem(p) as h:
        for b in (1, 4):
            X = torch.randn((p.n, b), device="cuda"); Y = torch.empty_like(X)
            res = {}
            for L in (1, 2, 4, 8, 16, 32):
                h.set_option("csr_sub_L", L)
                h.apply(X, Y)
                h.set_option("profile", 1 << 4); h.set_option("profile_reset", 1)
                for _ in range(5): h.apply(X, Y)
                torch.cuda.synchronize()
                res[L] = round(h.stat("csr_ns") / 5e6, 4)
                h.set_option("profile", 0)
            h.set_option("csr_sub_L", 0)
            print(json.dumps({"k": k, "b": b, "csr_ms_by_L": res}), flush=True)
