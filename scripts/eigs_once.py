"""One short eigs solve (for ncu captures of the eigs-only kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
p = configs.config(cfg)
with from_problem(p) as h:
    h.eigs(p.m, p.block, max_iters=iters, tol=0.0)
