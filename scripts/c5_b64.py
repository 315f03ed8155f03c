import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "split", "rotate"]
p = configs.config(5, k5=8)
with from_problem(p) as h:
    for b in (64, 16, 1):
        X = torch.randn(p.n, b, device="cuda"); Y = torch.empty_like(X)
        for ds, dy in ((0, 3), (0, 64), (2 if b > 4 else 1, 3)):
            h.set_option("dstream", ds); h.set_option("dy_max_range", dy)
            for _ in range(3): h.apply(X, out=Y)
            torch.cuda.synchronize()
            h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): h.apply(X, out=Y)
            e1.record(); torch.cuda.synchronize()
            fam = {f: round(h.stat(f + "_ns") / 1e7, 3) for f in FAM}
            print(json.dumps({"b": b, "dstream": ds, "dy": dy, "path": h.stat("dstream_path"), "ms": round(e0.elapsed_time(e1) / 10, 3), **fam}), flush=True)
            h.set_option("profile", 0)
