"""Per-block timeline of CTA 0 of the tensor-core sparse step (sp8_dbg = 2: results valid) at
config 4: microseconds of each event from the first image load, blocks 0..47."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
EV = ["load_issued", "N_start", "T_start", "A_got_N", "A_digits", "C_gram", "B_T_drained", "B_staged",
      "prod_empty_ok", "N_issued", "T_issued", "A_tmem", "A_waitN", "N_done_seen", "A_btempty", "A_ystored",
      "A_yrempty", "B_atfull", "A8_btfull", "A6_btfull"]
p = configs.config(4)
with from_problem(p) as h:
    h.eigs(p.m, p.block, max_iters=4, tol=0.0)
    h.set_option("sp8_dbg", int(sys.argv[1]) if len(sys.argv) > 1 else 10)
    h.set_option("sp8_poll", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    h.eigs(p.m, p.block, max_iters=3, tol=0.0)
    torch.cuda.synchronize()
    tr = [[h.stat(f"sp8_trace_{(e * 64 if e < 12 else 2048 + (e - 12) * 64) + i}") for i in range(64)] for e in range(len(EV))]
    t0 = tr[0][0]
    print("event " + " ".join(f"{e[:8]:>8}" for e in EV))
    for i in range(48):
        print(f"{i:3d}   " + " ".join(f"{(tr[e][i] - t0) / 1000:8.2f}" if tr[e][i] else "       -" for e in range(len(EV))))
    starts = [h.stat(f"sp8_trace_{768 + c}") for c in range(148)]
    ends = [h.stat(f"sp8_trace_{1024 + c}") for c in range(148)]
    s0 = min(starts)
    print("CTA start spread us", (max(starts) - s0) / 1000, "end spread us", (max(ends) - min(ends)) / 1000,
          "first end", (min(ends) - s0) / 1000, "last end", (max(ends) - s0) / 1000)
