#!/usr/bin/env python
"""Error of config 4's landmark-graph stand-in D against exact squared mesh-graph
Dijkstra distances, measured at FULL size (n = 1.8M, l = 50,000) on a seeded sample of landmark
rows (exact SSSP from each sampled landmark to all 50,000 landmarks). Input generation only."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import _native, configs  # noqa: E402
from gen.mesh import torus_grid  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = configs.config(4)
V, F, E = torus_grid(1200, 1500, seed=0)
w = np.linalg.norm(V[E[:, 0]] - V[E[:, 1]], axis=1)
g = _native.Graph(p.n, E, w)
rng = np.random.default_rng(2024)
sample = np.sort(rng.choice(p.l, size=rows, replace=False))
t0 = time.time()
exact = g.dijkstra_rows(p.landmarks[sample], targets=p.landmarks) ** 2
t = time.time() - t0
approx = p.D[sample].astype(np.float64)
off = exact > 0
rel = np.abs(approx - exact)[off] / exact[off]
out = {"config": "config 4 (torus 1200x1500, n=1,800,000, l=50,000)", "sampled_rows": rows,
       "entries": int(off.sum()), "frobenius_rel_error": float(np.linalg.norm(approx - exact) / np.linalg.norm(exact)),
       "mean_rel_error": float(rel.mean()), "median_rel_error": float(np.median(rel)),
       "p99_rel_error": float(np.quantile(rel, 0.99)), "max_rel_error": float(rel.max()),
       "stand_in_never_below_exact": bool((approx >= exact * (1 - 1e-6)).all()),
       "dijkstra_seconds": t, "threads": _native.num_threads()}
print(json.dumps(out, indent=1))
