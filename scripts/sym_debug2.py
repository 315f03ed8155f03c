import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1705_10887_b200 import Sbmds
n = l = 256
rng = np.random.default_rng(0)
rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int32); vv = np.ones(n, dtype=np.float32)
A = rng.uniform(0, 10, (n, n)).astype(np.float32); A = (A + A.T) / 2
D = A.copy(); D[:128, :128] = 0; D[128:, 128:] = 0
h = Sbmds(n, l, rp, ci, vv, np.ascontiguousarray(D)); h.set_option("blocked", 0)
for half in (0, 1):
    X = np.zeros((n, 16), np.float32)
    blk = rng.standard_normal((128, 16)).astype(np.float32); blk -= blk.mean(0)
    X[half*128:(half+1)*128] = blk
    Y2 = D.astype(np.float64) @ X.astype(np.float64)
    ref = Y2 - Y2.mean(0)
    for ds in (2, 3):
        h.set_option("dstream", ds)
        Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
        got = -2 * Y
        for t in range(2):
            sl = slice(t*128, (t+1)*128)
            e = np.linalg.norm(got[sl] - ref[sl]) / max(1e-30, np.linalg.norm(ref))
            print(f"X in tile {half} ds {ds} out tile {t}: rel err {e:.3e}  |ref| {np.linalg.norm(ref[sl]):.3e} |got| {np.linalg.norm(got[sl]):.3e}")
        if ds == 3:
            g, r = got[:128], ref[:128]
            if half == 1:
                # is the result the transpose product instead? D_10 X_1 would be D[128:, :128]^T... compare with D[:128,128:].T @ X1
                alt = D[:128, 128:].T.astype(np.float64) @ X[128:].astype(np.float64)
                alt = alt - 0
                print("   corr with D01 X1:", np.corrcoef(g.ravel(), r.ravel())[0,1])
