import sys, numpy as np, torch
sys.path.insert(0, '.')
import scipy.sparse as sp
from gen import configs
from oracle import sbmds_oracle as O
from paper_1705_10887_b200 import Sbmds
n = l = 256
rng = np.random.default_rng(0)
rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int32); vv = np.ones(n, dtype=np.float32)
def run(D, b=16, tag=""):
    X = rng.standard_normal((n, b)).astype(np.float32)
    Yo = O.apply(sp.identity(n, format="csr"), D.astype(np.float64), X.astype(np.float64))
    h = Sbmds(n, l, rp, ci, vv, np.ascontiguousarray(D))
    h.set_option("blocked", 0)
    out = {}
    for ds in (2, 3, 31, 33, 35):
        h.set_option("dstream", min(ds, 3)); h.set_option("sym_dbg", ds - 30 if ds > 30 else 0)
        Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
        out[ds] = Y
        print(tag, ds, np.linalg.norm(Y - Yo) / np.linalg.norm(Yo), flush=True)
    for k in out:
        d = out[k] - Yo
        print("   ", k, "err by row-tile:", [float(np.linalg.norm(d[i*128:(i+1)*128]) / np.linalg.norm(Yo)) for i in range(2)])
    h.close()
A = rng.uniform(0, 10, (n, n)).astype(np.float32); A = (A + A.T) / 2
Dd = A.copy(); Dd[:128, 128:] = 0; Dd[128:, :128] = 0
Do = A.copy(); Do[:128, :128] = 0; Do[128:, 128:] = 0
run(Do, tag="offdiag")
