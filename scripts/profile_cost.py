"""Cost of the bench's in-region D-stream events: 50-iteration config-4 solves timed from outside
with and without profile = 1 << 2 (events around k_dstream_sym8, which split its PDL overlap)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(4)
with from_problem(p) as h:
    for _ in range(3):
        h.eigs(p.m, p.block, max_iters=50, tol=0.0)
    for prof in (0, 4, 0, 4, 0, 4):
        h.set_option("profile", prof); h.set_option("profile_reset", 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            h.eigs(p.m, p.block, max_iters=50, tol=0.0)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"profile": prof, "ms_per_solve": round(e0.elapsed_time(e1) / 5, 3)}), flush=True)
    h.set_option("profile", 0)
