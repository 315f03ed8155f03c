export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 600 python -m pytest tests/test_gpu_eigs.py -x -q 2>&1 | tail -3
python - <<'PY'
import sys; sys.path.insert(0,'.')
from gen import configs
from paper_1705_10887_b200 import from_problem
for cfg in (2, 4):
    p = configs.config(cfg)
    with from_problem(p) as h:
        for f in (1, 3):
            h.set_option("fuse", f)
            lam, V, Z, info = h.eigs(p.m, p.block, max_iters=50, tol=0.0)
            lam2, V2, Z2, info2 = h.eigs(p.m, p.block, max_iters=500, tol=1e-6)
            print(cfg, f, "50-iter res", info["max_residual"], "conv iters", info2["iters"], info2["converged"], info2["max_residual"], flush=True)
PY
