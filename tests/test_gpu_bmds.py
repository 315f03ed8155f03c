"""GPU: BMDS, the paper's QR route (sbmds_bmds), against the fp64 oracle and
against sbmds_eigs on the same handle (SPEC.md:455 path equivalence: the same eigenvalues, and
embeddings equal up to an orthogonal transform, compared through Z Z^T)."""
import numpy as np
import pytest

from gen import configs
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu
EIG_TOL, ANGLE_TOL = 1e-4, 1e-3


def handle(p, **kw):
    from paper_1705_10887_b200 import from_problem
    return from_problem(p, **kw)


def host(t):
    return t.cpu().numpy().astype(np.float64)


def test_bmds_config1_vs_dense_oracle_and_oracle_bmds():
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o = O.eigs_dense(S, p.D, p.m)
    lam_b, V_b, _ = O.bmds(S, p.D, p.m)
    with handle(p) as h:
        lam, V, Z, info = h.bmds(p.m, p.block, tol=1e-9)
        assert h.stat("bmds_dropped") == 1              # J P 1 = 0 for rows summing to 1
    V, Z = host(V), host(Z)
    assert info["converged"] == 1 and info["n_applies"] == 0
    for ref in (lam_o, lam_b):
        assert np.all(np.abs(lam - ref) <= 1e-6 * np.abs(ref)), (lam, ref)
    assert O.principal_angle(V, V_o) <= ANGLE_TOL and O.principal_angle(V, V_b) <= ANGLE_TOL
    assert np.abs(V.T @ V - np.eye(p.m)).max() < 1e-5
    assert np.allclose(Z, V * np.sqrt(np.maximum(lam, 0))[None, :], rtol=1e-5, atol=1e-7)
    for j in range(p.m):
        assert V[np.argmax(np.abs(V[:, j])), j] > 0


@pytest.mark.parametrize("cfg", [1, 2])
def test_bmds_sbmds_path_equivalence(cfg):
    """BMDS and sBMDS on the same inputs give the same eigenvalues and the same
    embedding up to an orthogonal transform (Z Z^T); config 2 also against ARPACK on the oracle."""
    p = configs.config(cfg)
    with handle(p) as h:
        lam_b, _, Zb, ib = h.bmds(p.m, p.block, tol=1e-9)
        lam_s, _, Zs, is_ = h.eigs(p.m, p.block, max_iters=1000, tol=1e-6)
    Zb, Zs = host(Zb), host(Zs)
    assert ib["converged"] == 1 and is_["converged"] == 1
    assert np.all(np.abs(lam_b - lam_s) <= 1e-6 * np.abs(lam_s)), (lam_b, lam_s)
    # Z Z^T on a row sample (n x n would be 80 GB at config 2)
    rows = np.random.default_rng(cfg).choice(p.n, size=min(p.n, 2000), replace=False)
    Gb, Gs = Zb[rows] @ Zb[rows].T, Zs[rows] @ Zs[rows].T
    assert np.linalg.norm(Gb - Gs) <= 1e-4 * np.linalg.norm(Gs)
    if cfg == 2:
        S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
        lam_o, _, _, _ = O.eigs_matfree(S, p.D, p.m)
        assert np.all(np.abs(lam_b - lam_o) <= EIG_TOL * np.abs(lam_o))


def test_bmds_cf2_exact():
    """CF2 at config 2's S: rank-3 B~ = (JSY)(JSY)^T, eigenpairs = SVD of JSY (closed form)."""
    p = configs.config(2)
    rng = np.random.default_rng(7)
    Yl = rng.standard_normal((p.l, 3)) * [3.0, 2.0, 1.0]
    D = ((Yl[:, None, :] - Yl[None, :, :]) ** 2).sum(-1).astype(np.float32)
    q = configs.Problem("cf2", p.n, p.l, p.row_ptr, p.col_idx, p.val, D)
    S = O.csr(q.n, q.l, q.row_ptr, q.col_idx, q.val32())
    JSY = S @ Yl
    JSY -= JSY.mean(0)
    U, s, _ = np.linalg.svd(JSY, full_matrices=False)
    with handle(q) as h:
        lam, V, Z, info = h.bmds(3, 8, tol=1e-10)
    assert np.all(np.abs(lam - s ** 2) <= 1e-6 * s ** 2)
    assert O.principal_angle(host(V), U) <= 1e-4


def test_bmds_rank_deficient_jp():
    """J P is rank-deficient by construction for a partition of unity (J P 1 = J 1 = 0): the
    semi-definite Cholesky drops exactly that null pivot (stat bmds_dropped = 1). A landmark
    column with no entries adds a second null direction (a zero column of J P); both solves
    still match the dense oracle."""
    p = configs.config(1)
    col = np.asarray(p.col_idx).copy()
    col[col == 7] = 8                                   # landmark 7 loses every entry
    q = configs.Problem("hole", p.n, p.l, p.row_ptr, col, p.val, p.D)
    for prob, drops in ((p, 1), (q, 2)):
        S = O.csr(prob.n, prob.l, prob.row_ptr, prob.col_idx, prob.val32())
        lam_o, V_o, _ = O.eigs_dense(S, prob.D, 3)
        with handle(prob) as h:
            lam, V, Z, info = h.bmds(3, 8, tol=1e-9)
            assert h.stat("bmds_dropped") == drops
        assert np.all(np.abs(lam - lam_o) <= 1e-6 * np.abs(lam_o)), (lam, lam_o)
        assert O.principal_angle(host(V), V_o) <= ANGLE_TOL
