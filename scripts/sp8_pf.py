"""Sparse-step time at config 4 against the images' L2 prefetch distance (option sp8_pf)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(4)
with from_problem(p) as h:
    h.eigs(p.m, p.block, max_iters=5, tol=0.0)
    for pf in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['0', '1', '2', '3', '4', '6', '0'])]:
        h.set_option("sp8_pf", pf)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        h.eigs(p.m, p.block, max_iters=12, tol=0.0)
        torch.cuda.synchronize()
        n = max(1, h.stat("csr_launches"))
        print(json.dumps({"sp8_pf": pf, "csr_ms": round(h.stat("csr_ns") / n / 1e6, 4), "launches": n,
                          "dstream_ms": round(h.stat("dstream_ns") / max(1, h.stat("dstream_launches")) / 1e6, 4)}), flush=True)
        h.set_option("profile", 0)
