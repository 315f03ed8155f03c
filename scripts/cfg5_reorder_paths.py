"""Config 5 standalone apply with reordered rows (SBMDS_REORDER_ROWS): per-family device times for
every choice of the row-blocked kernels (option blocked = 0..3: bit 0 = S Y2, bit 1 = S^T X)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "split"]
k5 = int(sys.argv[1]) if len(sys.argv) > 1 else 16
bs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16]
p = configs.config(5, k5=k5)
out = {}
for reorder in (False, True):
    with from_problem(p, reorder_rows=reorder) as h:
        for b in bs:
            X = torch.randn(p.n, b, device="cuda")
            Y = torch.empty_like(X)
            for mask in (0, 1, 2, 3):
                h.set_option("blocked", mask)
                for _ in range(3): h.apply(X, out=Y)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10): h.apply(X, out=Y)
                e1.record(); torch.cuda.synchronize()
                total = e0.elapsed_time(e1) / 10
                h.set_option("profile", (1 << 10) - 1); h.set_option("profile_reset", 1)
                for _ in range(10): h.apply(X, out=Y)
                torch.cuda.synchronize()
                fam = {f: round(h.stat(f + "_ns") / 10e6, 4) for f in FAM}
                h.set_option("profile", 0)
                out[f"reorder={int(reorder)} b={b} blocked={mask}"] = {"ms": round(total, 4), "umax": h.stat("blocked_umax"), **fam}
                print(f"reorder={int(reorder)} b={b} blocked={mask}", out[f"reorder={int(reorder)} b={b} blocked={mask}"], flush=True)
print(json.dumps(out))
