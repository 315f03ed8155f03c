"""GPU: the fixed-point paths keep the fp32 contract on adversarial value ranges, or fall back
(DESIGN.md §4 "precision contract"), and the eigensolver's error statuses.

The int8 D stream stores D on one global quantum (max|D| 2^-22 < q <= max|D| 2^-21); the
tensor-core sparse step stores each 128-row block of S on one quantum. Both check, once per
handle, that the bulk of the values keeps enough significant bits:
  * D: binades between max|D| and the median |D| (stat dq_range) <= dq_max_range (6);
  * S: binades between a block's max|S| and its smallest nonzero row maximum (stat sp8_range)
    <= sp8_max_range (7).
Otherwise auto takes the fp32-grade kernels. Each test states which path it expects and checks
the result against the fp64 oracle at the north_star tolerances.
"""
import numpy as np
import pytest

from gen import configs
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu
TOL, EIG_TOL, ANGLE_TOL = 1e-5, 1e-4, 1e-3


def handle(p, **kw):
    from paper_1705_10887_b200 import from_problem
    return from_problem(p, **kw)


def run_apply(h, X):
    import torch
    Y = h.apply(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_S(p):
    return O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())


def sqdist32(P):
    P = np.asarray(P, dtype=np.float64)
    g = (P ** 2).sum(1)
    D = g[:, None] + g[None, :] - 2 * P @ P.T
    np.maximum(D, 0, out=D)
    np.fill_diagonal(D, 0)
    D = (D + D.T) / 2
    return np.ascontiguousarray(D.astype(np.float32))


def two_cluster_problem(n=40_000, l=5_000, seed=3):
    """Landmarks in two clusters 300 apart (90% spread ~1, 10% spread ~1): squared distances
    within the big cluster are O(1), across O(1e5) -> max|D| / median|D| ~ 1e5 (>= 1e4)."""
    base = configs.random_problem(n, l, 16, seed=seed, name="two_cluster")
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((l, 3))
    far = rng.random(l) < 0.1
    P[far, 0] += 300.0
    D = sqdist32(P)
    return configs.Problem("two_cluster", n, l, base.row_ptr, base.col_idx, base.val, D)


def test_wide_range_d_falls_back_and_meets_the_bar():
    p = two_cluster_problem()
    med = np.median(np.abs(p.D[np.triu_indices(p.l, 1)]))
    assert p.D.max() / med >= 1e4
    S = oracle_S(p)
    X = configs.x_block(p.n, 16, seed=4)
    ref = O.apply(S, p.D, X.astype(np.float64))
    with handle(p) as h:
        Y = run_apply(h, X)
        assert h.stat("dq_state") == -1 and h.stat("dq_range") > 6
        assert h.stat("dstream_path") == 2          # full D on the 3xTF32 tensor-core stream
        # m = 1: the spectrum spans ~4 decades (rank 3, separation >> cluster shape), so only
        # the leading pair is conditioned for fp32-grade arithmetic at the 1e-4 bar
        lam, V, Z, info = h.eigs(1, 16, max_iters=500, tol=1e-6)
        assert h.stat("dstream_path") == 2
    assert relerr(Y, ref) <= TOL
    lam_o, V_o, _, _ = O.eigs_matfree(S, p.D, 1)
    assert np.all(np.abs(lam - lam_o) <= EIG_TOL * np.abs(lam_o)), (lam, lam_o)
    assert O.principal_angle(V.cpu().numpy().astype(np.float64), V_o) <= ANGLE_TOL


def test_wide_range_d_host_upload_skips_the_pack():
    """Host D: create's histogram (taken behind the upload) decides before packing: no int8
    copy is built, and the first full-D apply mirrors the uploaded upper triangle."""
    p = two_cluster_problem(n=30_000, l=4_500, seed=5)
    X = configs.x_block(p.n, 16, seed=2)
    with handle(p, device="numpy") as h:
        assert h.stat("dq_state") == -1 and h.stat("d_packed_in_create") == 0
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 2
    assert relerr(Y, O.apply(oracle_S(p), p.D, X.astype(np.float64))) <= TOL


def test_normal_d_keeps_int8_and_forced_threshold_falls_back():
    """Config-5 recipe D (uniform [0, 100]): 1 binade; the int8 stream is kept. Lowering
    dq_max_range below it re-decides at the next apply and switches the stream; both meet the bar."""
    p = configs.random_problem(40_000, 5_000, 16, seed=9, name="normal_d")
    X = configs.x_block(p.n, 16, seed=4)
    ref = O.apply(oracle_S(p), p.D, X.astype(np.float64))
    with handle(p) as h:
        Y8 = run_apply(h, X)
        assert h.stat("dq_state") == 1 and h.stat("dq_range") <= 2 and h.stat("dstream_path") == 3
        h.set_option("dq_max_range", 0)
        Yt = run_apply(h, X)
        assert h.stat("dq_state") == -1 and h.stat("dstream_path") == 2
        h.set_option("dq_max_range", 6)
        Y8b = run_apply(h, X)
        assert h.stat("dq_state") == 1 and h.stat("dstream_path") == 3
    assert relerr(Y8, ref) <= TOL and relerr(Yt, ref) <= TOL
    assert np.array_equal(Y8, Y8b)


def test_x_with_a_dominant_row_falls_back():
    """X whose row 123 is 1e4 x the others: Y1's columns are dominated by the ~16 landmarks of that
    row (max / rms ~ 17), so the bulk of each column keeps few bits of the per-column fixed point
    (measured on the int8 stream: 2.5e-5 relative error, above the bar). The standalone apply's
    column check sends this apply to the fp32-grade stream; the next, Gaussian X goes back to int8."""
    p = configs.random_problem(40_000, 5_000, 16, seed=10, name="dominant_x")
    X = configs.x_block(p.n, 16, seed=6)
    X[123] *= 1e4
    Xn = configs.x_block(p.n, 16, seed=7)
    with handle(p) as h:
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 2 and h.stat("y_fallbacks") == 1
        Yn = run_apply(h, Xn)
        assert h.stat("dstream_path") == 3 and h.stat("y_fallbacks") == 1
        h.set_option("dstream", 3)                      # forced int8: the error the check avoids
        Y8 = run_apply(h, X)
    ref = O.apply(oracle_S(p), p.D, X.astype(np.float64))
    assert relerr(Y, ref) <= TOL
    assert relerr(Yn, O.apply(oracle_S(p), p.D, Xn.astype(np.float64))) <= TOL
    print("forced int8 on the dominant-row X:", relerr(Y8, ref))


def _eigs_vs_oracle(q, expect_sp8):
    S = oracle_S(q)
    with handle(q) as h:
        lam, V, Z, info = h.eigs(3, 16, max_iters=500, tol=1e-6)
        state, rng = h.stat("sp8_state"), h.stat("sp8_range")
    assert state == (1 if expect_sp8 else -2), (state, rng)
    assert info["converged"] == 1
    lam_o, V_o, _, _ = O.eigs_matfree(S, q.D, 3)
    assert np.all(np.abs(lam - lam_o) <= EIG_TOL * np.abs(lam_o)), (lam, lam_o)
    assert O.principal_angle(V.cpu().numpy().astype(np.float64), V_o) <= ANGLE_TOL
    return rng


def test_s_weights_spanning_decades_within_rows_keep_sp8():
    """Config 2 with every row's non-maximal weights scaled by 10^U(-6, 0): weights span 1e-6..1
    inside each 128-row image but every row keeps its largest weight, so the row maxima stay
    within a few binades of the block's; the tensor-core step is kept and matches the oracle."""
    p = configs.config(2)
    rng = np.random.default_rng(21)
    val = np.asarray(p.val, dtype=np.float64).copy()
    rp = np.asarray(p.row_ptr)
    f = 10.0 ** rng.uniform(-6, 0, size=val.shape)
    for i in range(0, p.n):
        a, b = rp[i], rp[i + 1]
        if b - a > 1:
            j = a + np.argmax(val[a:b])
            f[j] = 1.0
        else:
            f[a:b] = 1.0
    val *= f
    assert val.min() < 1e-6 * val.max()
    q = configs.Problem("cfg2_decades", p.n, p.l, p.row_ptr, p.col_idx, val, p.D)
    assert _eigs_vs_oracle(q, expect_sp8=True) <= 7


def test_s_rows_far_below_their_block_fall_back():
    """Config 2 with every 37th row scaled by 1e-6: those rows sit ~20 binades below their
    block's max, so the images would keep them with ~3 significant bits; the eigs step falls
    back to the fp32 sparse kernels (sp8_state = -2) and matches the oracle."""
    p = configs.config(2)
    val = np.asarray(p.val, dtype=np.float64).copy()
    rp = np.asarray(p.row_ptr)
    for i in range(0, p.n, 37):
        val[rp[i]:rp[i + 1]] *= 1e-6
    q = configs.Problem("cfg2_tiny_rows", p.n, p.l, p.row_ptr, p.col_idx, val, p.D)
    assert _eigs_vs_oracle(q, expect_sp8=False) > 7


# ------------------------------------------------------------------------------ error statuses
def test_rank_deficient_warm_start_takes_the_shifted_cholesky():
    """X0 with a zero column: G = X0^T X0 is singular (an exactly zero pivot), the Cholesky-QR's
    shifted retry (k_small.cuh chol_block) factors it, and the solve still converges to the
    oracle's pairs on the remaining columns."""
    import torch
    p = configs.config(1)
    S = oracle_S(p)
    lam_o, V_o, _ = O.eigs_dense(S, p.D, p.m)
    X0 = torch.from_numpy(configs.x_block(p.n, p.block, seed=3)).cuda()
    X0[:, 5] = 0.0
    with handle(p) as h:
        lam, V, Z, info = h.eigs(p.m, p.block, max_iters=500, tol=1e-6, X0=X0)
        assert h.stat("chol_retries") >= 1
    assert info["status"] == 0 and info["converged"] == 1
    assert np.all(np.abs(lam - lam_o) <= EIG_TOL * np.abs(lam_o))
    assert O.principal_angle(V.cpu().numpy().astype(np.float64), V_o) <= ANGLE_TOL


def test_zero_warm_start_is_a_breakdown():
    """X0 = 0: G = 0 has no Cholesky factor even shifted -> SBMDS_EBREAKDOWN (SPEC.md:53-style
    error, not a silent result)."""
    import torch
    from paper_1705_10887_b200 import SbmdsError
    p = configs.config(1)
    with handle(p) as h:
        X0 = torch.zeros((p.n, p.block), device="cuda")
        with pytest.raises(SbmdsError, match="EBREAKDOWN"):
            h.eigs(p.m, p.block, max_iters=50, tol=1e-6, X0=X0)
        lam, V, Z, info = h.eigs(p.m, p.block, max_iters=500, tol=1e-6)   # the handle stays usable
    assert info["converged"] == 1


def test_no_convergence_status_fills_outputs():
    """max_iters too small for tol: SBMDS_ENOCONV (SPEC.md:53 NonConvergence), with the outputs
    and info still filled (orthonormal V, Z = V Λ^{1/2}, iters = max_iters)."""
    from paper_1705_10887_b200 import SbmdsError
    from paper_1705_10887_b200._lib import SBMDS_ENOCONV
    p = configs.config(1)
    with handle(p) as h:
        lam, V, Z, info = h.eigs(p.m, p.block, max_iters=3, tol=1e-12)
        with pytest.raises(SbmdsError, match="ENOCONV"):
            h.eigs(p.m, p.block, max_iters=3, tol=1e-12, raise_noconv=True)
    assert info["status"] == SBMDS_ENOCONV and info["converged"] == 0 and info["iters"] == 3
    V = V.cpu().numpy().astype(np.float64)
    Z = Z.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(lam)) and np.abs(V.T @ V - np.eye(p.m)).max() < 1e-5
    assert np.allclose(Z, V * np.sqrt(np.maximum(lam, 0))[None, :], rtol=1e-5, atol=1e-7)


@pytest.mark.gpu
def test_nan_in_x_propagates_through_the_standalone_apply():
    """A NaN in X must come out as NaN (as the fp32 kernels give), not as garbage digits of the
    fixed-point paths: the column check sees it in the sum of squares and keeps the fp32-grade
    kernels (stats x_fallbacks / y_fallbacks)."""
    import torch
    from gen import configs
    from paper_1705_10887_b200 import from_problem
    p = configs.config(2)
    X = configs.x_block(p.n, 16, seed=2)
    X[4321, 5] = np.nan
    with from_problem(p) as h:
        h.set_option("sp8_min_rows", 0)
        f0 = h.stat("x_fallbacks")
        Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
        assert h.stat("x_fallbacks") == f0 + 1
    assert np.isnan(Y[:, 5]).all()          # B~ is dense in effect: every row of that column
    assert np.isfinite(Y[:, [0, 1, 15]]).all()
