#!/usr/bin/env python
"""Write tests/golden/cfg<i>_oracle_eigs.txt: the fp64 ORACLE's top eigenvalues of
-1/2 J S D S^T J for a BASELINE config, by ARPACK Lanczos on the oracle's
matrix-free apply (oracle.eigs_matfree). Calls only gen/ (inputs) and oracle/.

The file also records fingerprints of the generated inputs (n, l, nnz, fp64 sums of D and of
S's values) so a test can confirm it regenerated the same problem before comparing.

  python scripts/oracle_golden_eigs.py 4 [k_extra]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen import configs  # noqa: E402
from oracle import sbmds_oracle as O  # noqa: E402


def main():
    cfg = int(sys.argv[1])
    extra = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    t0 = time.time()
    p = configs.config(cfg)
    tgen = time.time() - t0
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val.astype(np.float32))
    k = p.m + extra
    t0 = time.time()
    lam, V, _, nmv = O.eigs_matfree(S, p.D, k, tol=1e-10, seed=0)
    teig = time.time() - t0
    res = O.residuals(S, p.D, lam, V)
    out = os.path.join(ROOT, "tests", "golden", f"cfg{cfg}_oracle_eigs.txt")
    with open(out, "w") as f:
        f.write(f"# fp64 oracle (oracle.eigs_matfree: ARPACK which='LA', tol=1e-10, v0 seed 0) top-{k}\n")
        f.write(f"# eigenvalues of -1/2 J S D S^T J (PAPER.md:113, :215) for BASELINE config {cfg}\n")
        f.write(f"# ({p.name}); written by scripts/oracle_golden_eigs.py {cfg} {extra} — calls only gen/ + oracle/.\n")
        f.write(f"# {nmv} matvecs, {teig:.0f} s on {os.cpu_count()} cores; generation {tgen:.0f} s.\n")
        f.write(f"n: {p.n}\nl: {p.l}\nnnz: {p.nnz}\n")
        f.write(f"D_sum: {float(np.sum(p.D, dtype=np.float64))!r}\n")
        f.write(f"S_sum: {float(np.sum(p.val.astype(np.float32), dtype=np.float64))!r}\n")
        f.write("lambda: " + " ".join(repr(float(x)) for x in lam) + "\n")
        f.write("residual: " + " ".join(repr(float(x)) for x in res) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
