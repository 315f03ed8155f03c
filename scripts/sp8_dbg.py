"""Timing diagnostics of the tensor-core sparse step (k_sp8_step) at config 4: per-iteration
'csr' family time with the T product on / off (sp8_dbg = 1 gives invalid results)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    for dbg in (0,):
        h.set_option("sp8_dbg", dbg)
        h.eigs(p.m, p.block, max_iters=5, tol=0.0)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        h.eigs(p.m, p.block, max_iters=20, tol=0.0); torch.cuda.synchronize()
        print(json.dumps({"sp8_dbg": dbg, "csr_ms": round(h.stat("csr_ns") / 2e7, 4), "csc_ms": round(h.stat("csc_ns") / 2e7, 4)}), flush=True)
        h.set_option("profile", 0)

# timeline of CTA 0 (sp8_dbg & 2): events per block, microseconds from the first load
EV = ["load_issued", "mma_N_start", "mma_T_start", "A_got_N", "A_bt_done", "B_gram_done", "B_T_drained", "B_staged",
      "prod_empty_ok", "prod_yp_ok", "mma_T_issued"]
with from_problem(p) as h:
    for dbg in (10, 26):
        h.set_option("sp8_dbg", dbg)
        h.eigs(p.m, p.block, max_iters=4, tol=0.0)   # iterations 2..4 use the step (no RR at 4? RR at 4 = last)
        torch.cuda.synchronize()
        tr = [[h.stat(f"sp8_trace_{e * 64 + i}") for i in range(64)] for e in range(len(EV))]
        t0 = tr[0][0]
        print("sp8_dbg", dbg)
        for i in range(0, 16):
            print(i, " ".join(f"{EV[e]}={(tr[e][i] - t0) / 1000:.2f}" for e in range(len(EV)) if tr[e][i]))
