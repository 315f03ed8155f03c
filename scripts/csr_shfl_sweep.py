"""k_spmm_csr_vec4 with and without the shuffled pair loads (option csr_shfl) on config 5:
device time of the CSR family per standalone apply, per width b and entries per row k."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
out = {}
for k5 in (8, 16, 64):
    p = configs.config(5, k5=k5)
    with from_problem(p) as h:
        for b in (4, 8, 16, 32, 64):
            X = torch.randn(p.n, b, device="cuda")
            Y = torch.empty_like(X)
            for shf in (0, 1):
                h.set_option("csr_shfl", shf)
                for _ in range(3): h.apply(X, out=Y)
                h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
                for _ in range(10): h.apply(X, out=Y)
                torch.cuda.synchronize()
                out[f"k={k5} b={b} shfl={shf}"] = round(h.stat("csr_ns") / 10e6, 4)
                h.set_option("profile", 0)
            print(f"k={k5} b={b}: plain {out[f'k={k5} b={b} shfl=0']} ms, shuffled {out[f'k={k5} b={b} shfl=1']} ms", flush=True)
print(json.dumps(out))
