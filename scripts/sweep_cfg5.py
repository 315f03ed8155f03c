"""Config 5 operator-apply bandwidth sweep (BASELINE.json configs[4]):
n = 4M, l = 20k, k in {8, 16, 64}, b in {1, 4, 16, 64}. Per point: applies/s (CUDA events over
20 device-resident applies), whole-apply algorithmic GB/s (4l^2 + 16 nnz + 4(n+1) + 4(l+1) + 8nb),
the D-stream path and its kernel GB/s, the per-family breakdown, and the gathered L2->SM bytes of
the two SpMMs (2 nnz 4b). Prints one JSON object per point; --out writes them all."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem

FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "split"]
ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, nargs="*", default=[8, 16, 64])
ap.add_argument("--b", type=int, nargs="*", default=[1, 4, 16, 64])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=None)
a = ap.parse_args()
rows = []
for k in a.k:
    p = configs.config(5, k5=k)
    with from_problem(p) as h:
        for b in a.b:
            X = torch.randn((p.n, b), device="cuda", generator=torch.Generator("cuda").manual_seed(b))
            Y = torch.empty_like(X)
            for _ in range(3):
                h.apply(X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                h.apply(X, Y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            h.set_option("profile", (1 << 10) - 1)
            h.set_option("profile_reset", 1)
            for _ in range(5):
                h.apply(X, Y)
            torch.cuda.synchronize()
            br = {f: round(h.stat(f + "_ns") / 5e6, 4) for f in FAM}
            h.set_option("profile", 0)
            byt = 4 * p.l * p.l + 16 * p.nnz + 4 * (p.n + 1) + 4 * (p.l + 1) + 8 * p.n * b
            dpath, dbytes = h.stat("dstream_path"), h.stat("dstream_bytes")
            r = {"k": k, "b": b, "n": p.n, "l": p.l, "nnz": p.nnz, "apply_ms": round(ms, 4),
                 "applies_per_s": round(1e3 / ms, 1), "apply_algorithmic_GBps": round(byt / ms / 1e6, 1),
                 "dstream_path": dpath, "dstream_GBps": round(dbytes / (br["dstream"] * 1e6), 1) if br["dstream"] else None,
                 "spmm_gathered_GB": round(2 * p.nnz * 4 * b / 1e9, 2), "per_apply_ms": br}
            print(json.dumps(r), flush=True)
            rows.append(r)
if a.out:
    json.dump(rows, open(a.out, "w"), indent=1)
