"""Timing diagnostics of the tensor-core sparse step (k_sp8_step) at config 4: per-iteration
'csr' family time with the T product on / off (sp8_dbg = 1 gives invalid results)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    for dbg in (0, 1, 0, 1):
        h.set_option("sp8_dbg", dbg)
        h.eigs(p.m, p.block, max_iters=5, tol=0.0)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        h.eigs(p.m, p.block, max_iters=20, tol=0.0); torch.cuda.synchronize()
        print(json.dumps({"sp8_dbg": dbg, "csr_ms": round(h.stat("csr_ns") / 2e7, 4), "csc_ms": round(h.stat("csc_ns") / 2e7, 4)}), flush=True)
        h.set_option("profile", 0)
