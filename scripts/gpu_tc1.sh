export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 120 python -c "
import numpy as np, torch
from gen import configs
from oracle import sbmds_oracle as O
from paper_1705_10887_b200 import from_problem
p = configs.config(1)
S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val.astype(np.float32))
for b in (8, 16, 32, 64):
    X = configs.x_block(p.n, b, seed=1)
    with from_problem(p) as h:
        for ds in (1, 2):
            h.set_option('dstream', ds)
            Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
            Yo = O.apply(S, p.D, X.astype(np.float64))
            print(b, ds, np.linalg.norm(Y - Yo) / np.linalg.norm(Yo), flush=True)
"
echo rc=$?
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -8
timeout 300 python scripts/profile_breakdown.py --config 4 --eigs 2>&1 | tail -2
