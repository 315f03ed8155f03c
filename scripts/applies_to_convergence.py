"""Applies to convergence (SURVEY.md §8(f) NEXT-3 comparison): the library's block subspace
iteration (GPU, sbmds_eigs, block b) and its restarted block Lanczos (GPU, option solver = 1)
against the paper's Lanczos (ARPACK eigsh which='LA' through the fp64 oracle on
the host) on the same operator and tolerance. The cost
unit that matters on the GPU is a pass over D: one block apply streams D once for b columns,
one Lanczos matvec streams it for one column.

python scripts/applies_to_convergence.py [configs ...] [--tol 1e-6] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import configs  # noqa: E402
from oracle import sbmds_oracle as O  # noqa: E402
from paper_1705_10887_b200 import from_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", type=int, nargs="*", default=[1, 2, 3])
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--out", default=None)
a = ap.parse_args()
rows = []
for cfg in a.configs:
    p = configs.config(cfg)
    with from_problem(p) as h:
        h.eigs(p.m, p.block, max_iters=5, tol=0.0)    # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lam, V, Z, info = h.eigs(p.m, p.block, max_iters=2000, tol=a.tol)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
        h.set_option("solver", 1)
        h.eigs(p.m, p.block, max_iters=8, tol=0.0)    # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lamL, VL, _, infoL = h.eigs(p.m, p.block, max_iters=2000, tol=a.tol)
        torch.cuda.synchronize()
        t_lz = time.perf_counter() - t0
        h.set_option("solver", 0)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    t0 = time.perf_counter()
    lam_o, V_o, _, nmv = O.eigs_matfree(S, p.D, p.m, tol=a.tol, seed=0)
    t_cpu = time.perf_counter() - t0
    r = {"config": cfg, "n": p.n, "l": p.l, "m": p.m, "block": p.block, "tol": a.tol,
         "subspace_iteration_gpu": {"iters": info["iters"], "block_applies": info["n_applies"],
                                    "D_passes": info["n_applies"], "operator_columns": info["n_applies"] * p.block,
                                    "seconds": round(t_gpu, 4), "max_residual": info["max_residual"]},
         "block_lanczos_gpu": {"block_applies": infoL["n_applies"], "D_passes": infoL["n_applies"],
                               "operator_columns": infoL["n_applies"] * p.block, "seconds": round(t_lz, 4),
                               "max_residual": infoL["max_residual"], "converged": infoL["converged"],
                               "max_rel_eig_diff": float(np.max(np.abs(np.asarray(lamL) - lam_o) / np.abs(lam_o))),
                               "angle": float(O.principal_angle(VL.cpu().numpy().astype(np.float64), V_o))},
         "lanczos_arpack_cpu": {"matvecs": nmv, "D_passes": nmv, "operator_columns": nmv,
                                "seconds": round(t_cpu, 3)},
         "max_rel_eig_diff": float(np.max(np.abs(np.asarray(lam) - lam_o) / np.abs(lam_o))),
         "angle": float(O.principal_angle(V.cpu().numpy().astype(np.float64), V_o))}
    print(json.dumps(r), flush=True)
    rows.append(r)
if a.out:
    json.dump(rows, open(a.out, "w"), indent=1)
