"""Per-kernel device-time breakdown of sbmds_apply / sbmds_eigs (CUDA events in libsbmds).

python scripts/profile_breakdown.py [--config 4] [--b 16] [--applies 20] [--eigs] [--quick]
Prints one JSON object; --quick runs a handful of applies (for ncu captures).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import configs  # noqa: E402
from paper_1705_10887_b200 import from_problem  # noqa: E402

FAM = ["colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--k5", type=int, default=16)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--applies", type=int, default=20)
ap.add_argument("--eigs", action="store_true")
ap.add_argument("--quick", action="store_true")
ap.add_argument("--order", type=int, default=1)
ap.add_argument("--dstream", type=int, default=0)
a = ap.parse_args()

p = configs.config(a.config, k5=a.k5)
b = a.b or p.block or 16
h = from_problem(p)
h.set_option("order_columns", a.order)
h.set_option("dstream", a.dstream)
X = torch.randn((p.n, b), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
Y = torch.empty_like(X)
for _ in range(2 if a.quick else 3):
    h.apply(X, Y)
torch.cuda.synchronize()
if a.quick:
    for _ in range(3):
        h.apply(X, Y)
    torch.cuda.synchronize()
    sys.exit(0)
h.set_option("profile", (1 << len(FAM)) - 1)
h.set_option("profile_reset", 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.applies):
    h.apply(X, Y)
e1.record()
torch.cuda.synchronize()
tot = e0.elapsed_time(e1) / a.applies
out = {"config": a.config, "b": b, "n": p.n, "l": p.l, "nnz": p.nnz, "apply_ms": tot,
       "per_apply_ms": {f: h.stat(f + "_ns") / 1e6 / max(1, a.applies) for f in FAM[:5] + ["split"]}, "dstream_path": h.stat("dstream_path"), "dstream_bytes": h.stat("dstream_bytes")}
byt = 4 * p.l * p.l + 16 * p.nnz + 4 * (p.n + 1) + 4 * (p.l + 1) + 8 * p.n * b
out["apply_algorithmic_GBps"] = byt / (tot / 1e3) / 1e9
if a.eigs and p.m:
    h.set_option("profile_reset", 1)
    e0.record()
    lam, V, Z, info = h.eigs(p.m, p.block, max_iters=50, tol=0.0)
    e1.record()
    torch.cuda.synchronize()
    out["eigs_ms"] = e0.elapsed_time(e1)
    out["eigs_breakdown_ms"] = {f: h.stat(f + "_ns") / 1e6 for f in FAM}
    out["eigs_launches"] = {f: h.stat(f + "_launches") for f in FAM}
print(json.dumps(out))
