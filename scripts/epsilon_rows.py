"""The paper's approximation-error workload on a synthetic torus:
epsilon(E^) = ||E^_R - E_R||_F^2 / ||E_R||_F^2 over a seeded random subset R of rows, where E
holds exact squared mesh-graph geodesics (Dijkstra, gen/) and the rows of E^ = S D S^T come from
the library's uncentred apply (center = 0) on indicator blocks e_R (E^ is symmetric, so its
columns R are its rows R). One block is also checked against the fp64 oracle (apply_raw).

python scripts/epsilon_rows.py [--config 2] [--rows 256] [--out profiles/r01_epsilon_cfg2.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import _native, configs  # noqa: E402
from gen.mesh import torus_grid  # noqa: E402
from oracle import sbmds_oracle as O  # noqa: E402
from paper_1705_10887_b200 import from_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--rows", type=int, default=256)
ap.add_argument("--block", type=int, default=64)
ap.add_argument("--out", default=None)
a = ap.parse_args()

p = configs.config(a.config)
nu, nv = p.meta["nu"], p.meta["nv"]
verts, _, edges = torus_grid(nu, nv, seed=p.meta["seed"])
w = np.linalg.norm(verts[edges[:, 0]] - verts[edges[:, 1]], axis=1)
g = _native.Graph(p.n, edges, w)
R = np.sort(np.random.default_rng(1705).choice(p.n, a.rows, replace=False))
t0 = time.perf_counter()
E_R = g.dijkstra_rows(R) ** 2                     # exact squared geodesics, |R| x n
t_dij = time.perf_counter() - t0

approx = np.empty((len(R), p.n))
ms = []
with from_problem(p) as h:
    h.set_option("center", 0)
    for c0 in range(0, len(R), a.block):
        rows = R[c0:c0 + a.block]
        X = torch.zeros((p.n, len(rows)), device="cuda")
        X[torch.from_numpy(rows).long().cuda(), torch.arange(len(rows), device="cuda")] = 1.0
        Y = torch.empty_like(X)
        h.apply(X, Y)                               # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.apply(X, Y); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        approx[c0:c0 + len(rows)] = Y.cpu().numpy().T.astype(np.float64)
        if c0 == 0:   # parity of one block against the fp64 oracle
            S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
            ref = O.apply_raw(S, p.D, X.cpu().numpy().astype(np.float64))
            parity = float(np.linalg.norm(Y.cpu().numpy() - ref) / np.linalg.norm(ref))
out = {"config": a.config, "mesh": p.meta.get("mesh"), "n": p.n, "l": p.l, "rows": len(R),
       "epsilon": O.rel_sq_error(approx, E_R),
       "epsilon_landmark_rows_excluded": O.rel_sq_error(approx[~np.isin(R, p.landmarks)],
                                                        E_R[~np.isin(R, p.landmarks)]),
       "parity_first_block_vs_oracle": parity, "block": a.block,
       "apply_ms_per_block": round(float(np.median(ms)), 4),
       "rows_per_s": round(a.block / (float(np.median(ms)) / 1e3), 1),
       "dijkstra_rows_s_host": round(t_dij, 2)}
print(json.dumps(out))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
