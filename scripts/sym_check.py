import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from gen import configs
from oracle import sbmds_oracle as O
from paper_1705_10887_b200 import from_problem
cases = [(configs.config(1), 16), (configs.config(1), 8), (configs.random_problem(30_011, 2_003, 16, seed=3, name="r"), 16),
         (configs.random_problem(30_011, 2_003, 16, seed=4, name="r"), 5), (configs.config(2), 16), (configs.config(2), 12)]
for p, b in cases:
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    X = configs.x_block(p.n, b, seed=b)
    Yo = O.apply(S, p.D, X.astype(np.float64))
    with from_problem(p) as h:
        for ds in (2, 3):
            h.set_option('dstream', ds)
            Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
            print(p.name, p.l, b, ds, h.stat('dstream_path'), np.linalg.norm(Y - Yo) / np.linalg.norm(Yo), flush=True)
