"""Sparse-step diagnostics at config 4: per-iteration 'csr' family time (the k_sp8_step launches)
with sp8_dbg = 0 (normal), 1 (T product off), 4 (images streamed only, no MMA); timings only."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    h.eigs(p.m, p.block, max_iters=5, tol=0.0)
    for dbg in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['0', '1', '4', '0'])]:
        h.set_option("sp8_dbg", dbg)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        try:
            h.eigs(p.m, p.block, max_iters=12, tol=0.0)
        except Exception as e:
            print("(results invalid in this mode:", str(e)[:60], ")")
        torch.cuda.synchronize()
        n = max(1, h.stat("csr_launches"))
        print(json.dumps({"sp8_dbg": dbg, "csr_ms": round(h.stat("csr_ns") / n / 1e6, 4), "launches": n,
                          "dstream_ms": round(h.stat("dstream_ns") / max(1, h.stat("dstream_launches")) / 1e6, 4),
                          "img_bytes": h.stat("sp8_bytes")}), flush=True)
        h.set_option("profile", 0)
    h.set_option("sp8_dbg", 0)
