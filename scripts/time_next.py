#!/usr/bin/env python
"""Times of the round-2 additions at config sizes (device, host clocks around synchronised calls):
the sBHA build (sbmds_sbha_build) on config 1-2 meshes with their FPS landmarks, BMDS
(sbmds_bmds) at configs 1-2 and the subspace-iteration eigs beside it. Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import configs  # noqa: E402
from gen.mesh import torus_grid  # noqa: E402
from paper_1705_10887_b200 import from_problem  # noqa: E402
from paper_1705_10887_b200.sbmds import sbha_build  # noqa: E402

out = {}
for cfg, (nu, nv), prow in ((1, (40, 50), 8), (2, (250, 400), 16)):
    p = configs.config(cfg)
    V, F, _ = torus_grid(nu, nv, seed=0)
    sbha_build(V, F.astype(np.int32), p.landmarks, prow)          # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    rp, ci, vv, info = sbha_build(V, F.astype(np.int32), p.landmarks, prow)
    torch.cuda.synchronize()
    out[f"sbha_cfg{cfg}"] = {"n": p.n, "l": p.l, "p_row": prow, "seconds": time.perf_counter() - t, **info}
    with from_problem(p) as h:
        h.bmds(p.m, p.block, tol=1e-9)
        torch.cuda.synchronize()
        t = time.perf_counter()
        lam_b, _, _, ib = h.bmds(p.m, p.block, tol=1e-9)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t
        t = time.perf_counter()
        lam_s, _, _, is_ = h.eigs(p.m, p.block, max_iters=1000, tol=1e-6)
        torch.cuda.synchronize()
        ts = time.perf_counter() - t
    out[f"bmds_cfg{cfg}"] = {"seconds": tb, "gpu_ms": ib["gpu_ms"], "iters": ib["iters"],
                             "eigenvalues": list(lam_b), "sbmds_seconds": ts, "sbmds_iters": is_["iters"],
                             "sbmds_eigenvalues": list(lam_s)}
print(json.dumps(out))
