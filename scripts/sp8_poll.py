"""k_sp8_step per-launch time at config 4 vs the MMA warp's poll back-off (option sp8_poll, ns)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    h.eigs(p.m, p.block, max_iters=5, tol=0.0)
    for ns in (0, 20, 50, 100, 200, 500, 0):
        h.set_option("sp8_poll", ns)
        h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
        h.eigs(p.m, p.block, max_iters=20, tol=0.0); torch.cuda.synchronize()
        n = max(1, h.stat("csr_launches"))
        print(json.dumps({"sp8_poll": ns, "csr_ms": round(h.stat("csr_ns") / n / 1e6, 4),
                          "fold_ms": round(h.stat("csc_ns") / max(1, h.stat("csc_launches")) / 1e6, 4),
                          "dstream_ms": round(h.stat("dstream_ns") / max(1, h.stat("dstream_launches")) / 1e6, 4)}), flush=True)
        h.set_option("profile", 0)
