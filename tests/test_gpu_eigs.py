"""GPU parity: sbmds_eigs (block subspace iteration, CUDA) vs the fp64 oracle.

Tolerances (BASELINE.json north_star): eigenvalues relative error <= 1e-4; embedding
principal subspace angle <= 1e-3 rad. Subspaces are compared only across a spectral
gap (reading R4); Z is compared through Z Z^T (rigid-motion invariant).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from gen import configs
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu
EIG_TOL, ANGLE_TOL = 1e-4, 1e-3


def handle(p, **kw):
    from paper_1705_10887_b200 import from_problem
    return from_problem(p, **kw)


def gpu_eigs(h, m, block, **kw):
    lam, V, Z, info = h.eigs(m, block, **kw)
    return lam, V.cpu().numpy().astype(np.float64), Z.cpu().numpy().astype(np.float64), info


def check_against(lam, V, Z, lam_o, V_o, Z_o):
    assert np.all(np.abs(lam - lam_o) <= EIG_TOL * np.abs(lam_o)), (lam, lam_o)
    assert O.principal_angle(V, V_o) <= ANGLE_TOL
    # orthonormal columns, canonical signs (largest |v_i| positive)
    assert np.abs(V.T @ V - np.eye(V.shape[1])).max() < 1e-5
    for j in range(V.shape[1]):
        i = np.argmax(np.abs(V[:, j]))
        assert V[i, j] > 0
    assert np.allclose(Z, V * np.sqrt(np.maximum(lam, 0))[None, :], rtol=1e-5, atol=1e-7)


def test_eigs_config1_vs_dense():
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o = O.eigs_dense(S, p.D, p.m)
    with handle(p) as h:
        lam, V, Z, info = gpu_eigs(h, p.m, p.block, max_iters=500, tol=1e-6)
    assert info["status"] == 0 and info["converged"] == 1
    check_against(lam, V, Z, lam_o, V_o, Z_o)
    assert np.allclose(Z @ Z.T, Z_o @ Z_o.T, atol=1e-4 * lam_o[0])


def test_eigs_config2_vs_lanczos():
    p = configs.config(2)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, p.m)
    with handle(p) as h:
        lam, V, Z, info = gpu_eigs(h, p.m, p.block, max_iters=500, tol=1e-6)
    check_against(lam, V, Z, lam_o, V_o, Z_o)


def test_eigs_cf2_exact_rank3_at_config2_shape():
    """CF2 at n = 100,000: S of config 2 (rows sum to 1), D = squared distances of landmark
    points y ~ N(0, diag(9,4,1)) => eigenpairs are the SVD of J S Y (no eigensolver needed)."""
    p = configs.config(2)
    rng = np.random.default_rng(5)
    Yl = rng.standard_normal((p.l, 3)) * [3.0, 2.0, 1.0]
    D = ((Yl[:, None, :] - Yl[None, :, :]) ** 2).sum(-1).astype(np.float32)
    q = configs.Problem("cf2", p.n, p.l, p.row_ptr, p.col_idx, p.val, D)
    S = O.csr(q.n, q.l, q.row_ptr, q.col_idx, q.val32())
    JSY = S @ Yl
    JSY -= JSY.mean(0)
    U, s, _ = np.linalg.svd(JSY, full_matrices=False)
    with handle(q) as h:
        lam, V, Z, info = gpu_eigs(h, 3, 8, max_iters=200, tol=1e-6)
    assert np.all(np.abs(lam - s ** 2) <= EIG_TOL * s ** 2)
    assert O.principal_angle(V, U) <= ANGLE_TOL


def test_eigs_negative_top_m_zeroed():
    """CF3 circle (S = I): the top-m algebraic set reaches negative eigenvalues; their Z
    columns are zero and info counts them."""
    N, rho = 40, 1.0
    th = 2 * np.pi * np.arange(N) / N
    diff = np.angle(np.exp(1j * (th[:, None] - th[None, :])))
    D = ((rho * diff) ** 2).astype(np.float32)
    rp = np.arange(N + 1, dtype=np.int64)
    ci = np.arange(N, dtype=np.int32)
    p = configs.Problem("circle", N, N, rp, ci, np.ones(N), D)
    lam_all = np.sort(np.linalg.eigvalsh(O.dense_operator(sp.identity(N, format="csr"), D.astype(np.float64))))[::-1]
    m = 24
    assert lam_all[m - 1] < 0
    with handle(p) as h:
        lam, V, Z, info = gpu_eigs(h, m, 39, max_iters=3000, tol=1e-7)
    assert np.allclose(lam, lam_all[:m], rtol=1e-4, atol=1e-6 * abs(lam_all[0]))
    neg = lam < 0
    assert info["n_negative"] == int(neg.sum())
    assert np.all(Z[:, neg] == 0)


def test_eigs_fixed_iterations_and_warm_start():
    p = configs.config(1)
    with handle(p) as h:
        lam, V, Z, info = gpu_eigs(h, p.m, p.block, max_iters=7, tol=0.0)
        assert info["status"] == 0 and info["iters"] == 7
        import torch
        X0 = torch.zeros((p.n, p.block), device="cuda")
        X0[:, :3] = torch.from_numpy(V.astype(np.float32)).cuda()
        X0[:, 3:] = torch.randn((p.n, p.block - 3), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
        lam2, V2, _, info2 = gpu_eigs(h, p.m, p.block, max_iters=500, tol=1e-5, X0=X0)
        lam3, V3, _, _ = gpu_eigs(h, p.m, p.block, max_iters=500, tol=1e-5, X0=X0)
    assert info2["converged"] == 1
    assert np.array_equal(lam2, lam3) and np.array_equal(V2, V3)   # deterministic


def test_eigs_host_outputs():
    p = configs.config(1)
    with handle(p) as h:
        lam, V, Z, info = h.eigs(p.m, p.block, tol=1e-6, device="numpy")
        lam_d, V_d, Z_d, _ = gpu_eigs(h, p.m, p.block, tol=1e-6)
    assert np.array_equal(lam, lam_d)
    assert np.array_equal(V, V_d.astype(np.float32))


@pytest.mark.parametrize("gram_tc", [0, 1])
def test_eigs_gram_paths_agree(gram_tc):
    """Gram on FP64 tensor cores (DMMA) and on FP64 CUDA cores both solve config 1 to the bar."""
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o = O.eigs_dense(S, p.D, p.m)
    with handle(p) as h:
        h.set_option("gram_tc", gram_tc)
        lam, V, Z, info = gpu_eigs(h, p.m, p.block, max_iters=500, tol=1e-6)
    check_against(lam, V, Z, lam_o, V_o, Z_o)


def test_eigs_block64_and_m_equals_block():
    """block = 64 (the widest tcgen05 path, two swizzle atoms per stage) and m = block."""
    p = configs.config(2)
    rng = np.random.default_rng(8)
    Yl = rng.standard_normal((p.l, 3)) * [3.0, 2.0, 1.0]
    D = ((Yl[:, None, :] - Yl[None, :, :]) ** 2).sum(-1).astype(np.float32)
    q = configs.Problem("cf2", p.n, p.l, p.row_ptr, p.col_idx, p.val, D)
    S = O.csr(q.n, q.l, q.row_ptr, q.col_idx, q.val32())
    JSY = S @ Yl
    JSY -= JSY.mean(0)
    U, s, _ = np.linalg.svd(JSY, full_matrices=False)
    with handle(q) as h:
        lam, V, Z, info = gpu_eigs(h, 3, 64, max_iters=100, tol=1e-6)
        lam8, V8, _, _ = gpu_eigs(h, 8, 8, max_iters=100, tol=0.0)
    assert np.all(np.abs(lam - s ** 2) <= EIG_TOL * s ** 2)
    assert O.principal_angle(V, U) <= ANGLE_TOL
    assert np.allclose(lam8[:3], s ** 2, rtol=1e-4)        # m = block: the rank-3 part, then ~0
    assert np.all(np.abs(lam8[3:]) < 1e-3 * s[0] ** 2)


@pytest.mark.parametrize("cfg,block", [(1, 8), (2, 16), (2, 4), (3, 32)])
def test_fused_sparse_step_matches_unfused(cfg, block):
    """The fused eigs step (A5 + next A2 + Gram in k_blk_spmm_fused) computes the same
    iteration as the separate kernels: eigenvalues, residuals and the Ritz subspace agree
    after a fixed number of iterations (only fp32 summation order differs), and the fused
    path is bitwise deterministic."""
    p = configs.config(cfg)
    m = min(p.m, block)
    with handle(p) as h:
        assert h.stat("blocked_umax") > 0
        out = {}
        for fuse in (1, 0):
            h.set_option("fuse", fuse)
            out[fuse] = gpu_eigs(h, m, block, max_iters=25, tol=0.0, seed=3)
        h.set_option("fuse", 1)
        rep = gpu_eigs(h, m, block, max_iters=25, tol=0.0, seed=3)
    (la, Va, _, ia), (lb, Vb, _, ib) = out[1], out[0]
    assert np.allclose(la, lb, rtol=1e-6), (la, lb)
    assert O.principal_angle(Va, Vb) <= 1e-4
    assert abs(ia["max_residual"] - ib["max_residual"]) <= 1e-4 * max(1.0, abs(ib["max_residual"])) + 1e-9
    assert np.array_equal(la, rep[0]) and np.array_equal(Va, rep[1])


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_graph_replay_matches_eager(cfg):
    """The eigs loop replayed from CUDA graphs (option use_graph) and launched eagerly compute
    the same iteration bitwise: graph capture changes how kernels are launched, not what runs."""
    p = configs.config(cfg)
    m, block = p.m, p.block
    iters = 23 if cfg != 4 else 12
    with handle(p) as h:
        out = {}
        for g in (1, 0):
            h.set_option("use_graph", g)
            out[g] = gpu_eigs(h, m, block, max_iters=iters, tol=0.0, seed=5)
        h.set_option("use_graph", 1)
        conv = gpu_eigs(h, m, block, max_iters=500, tol=1e-6, seed=5)
        h.set_option("use_graph", 0)
    assert np.array_equal(out[1][0], out[0][0]) and np.array_equal(out[1][1], out[0][1])
    assert out[1][3]["iters"] == out[0][3]["iters"] == iters
    assert conv[3]["converged"] == 1


@pytest.mark.parametrize("cfg", [2, 4])
def test_tensor_core_sparse_step(cfg):
    """The eigs sparse step on the int8 tensor cores (k_sp8.cuh: A5 + Grams + next A2 from
    dense 128-row digit images of S) computes the same iteration as the separate fp32 kernels:
    eigenvalues, residuals and the Ritz subspace agree after a fixed number of iterations (the
    24-bit fixed point of S and of the B operands perturbs products by <= ~2^-23 of the scaled
    maxima), and the step is bitwise deterministic."""
    p = configs.config(cfg)
    it = 25 if cfg == 2 else 12
    with handle(p) as h:
        h.set_option("fuse", 0)
        ref = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
        h.set_option("fuse", 3)
        a = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
        assert h.stat("sp8_state") == 1 and h.stat("sp8_umax") <= 128
        rep = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
    (la, Va, _, ia), (lb, Vb, _, ib) = a, ref
    assert np.allclose(la, lb, rtol=1e-5), (la, lb)
    # the degenerate leading torus pair is compared as a pair: the subspace of all m
    assert O.principal_angle(Va, Vb) <= 1e-3
    assert abs(ia["max_residual"] - ib["max_residual"]) <= 1e-3 * max(1.0, abs(ib["max_residual"])) + 1e-7
    assert np.array_equal(la, rep[0]) and np.array_equal(Va, rep[1])


def test_tensor_core_sparse_step_general_s():
    """The tensor-core sparse step with a general S (signed weights, rows not summing to 1, as the
    paper's thresholded P_sparse): the (S 1 - 1) t^T correction and signed digits give
    the same iteration as the fp32 kernels, and the solve converges to the oracle's eigenpairs."""
    p = configs.config(2)
    rng = np.random.default_rng(11)
    val = p.val * (1.0 + 0.3 * rng.standard_normal(p.val.shape))   # some weights change sign
    q = configs.Problem("cfg2_signed", p.n, p.l, p.row_ptr, p.col_idx, val, p.D)
    S = O.csr(q.n, q.l, q.row_ptr, q.col_idx, q.val32())
    assert (q.val32() < 0).any()
    rs = np.asarray(S.sum(axis=1)).ravel()
    assert np.abs(rs - 1).max() > 0.1
    with handle(q) as h:
        h.set_option("fuse", 0)
        ref = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=4)
        h.set_option("fuse", 3)
        a = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=4)
        assert h.stat("sp8_state") == 1
        lam, V, Z, info = gpu_eigs(h, 3, 16, max_iters=500, tol=1e-6)
    assert np.allclose(a[0], ref[0], rtol=1e-5), (a[0], ref[0])
    assert O.principal_angle(a[1], ref[1]) <= 1e-3
    assert info["converged"] == 1
    lam_o, V_o, Z_o, _ = O.eigs_matfree(S, q.D, 3)
    assert np.all(np.abs(lam - lam_o) <= EIG_TOL * np.abs(lam_o)), (lam, lam_o)
    assert O.principal_angle(V, V_o) <= ANGLE_TOL


def test_eigs_config4_bench_configuration():
    """The bench's solve at full size (config 4: 50 fixed iterations, m = 3, b = 16, the
    tensor-core sparse step): the returned pairs satisfy B~ v = θ v to <= 1e-5 of |θ_1| when the
    residual is formed by the fp64 ORACLE's apply (so each θ is within that distance of an
    eigenvalue of B~), V is orthonormal, Z = V Λ^{1/2}, and the solve is deterministic."""
    p = configs.config(4)
    with handle(p) as h:
        lam, V, Z, info = gpu_eigs(h, 3, 16, max_iters=50, tol=0.0, seed=0)
        assert h.stat("sp8_state") == 1
        lam2, V2, _, _ = gpu_eigs(h, 3, 16, max_iters=50, tol=0.0, seed=0)
    assert np.array_equal(lam, lam2) and np.array_equal(V, V2)
    assert np.abs(V.T @ V - np.eye(3)).max() < 1e-5
    assert np.allclose(Z, V * np.sqrt(np.maximum(lam, 0))[None, :], rtol=1e-5, atol=1e-7)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    r = O.residuals(S, p.D, lam, V)
    assert np.all(r <= 1e-5 * abs(lam[0])), (r, lam)


def test_tensor_core_sparse_step_empty_rows():
    """Rows without entries (two whole empty 128-row blocks and ragged ones around them): the
    step's zero images, zero rows of Y and empty dictionaries agree with the fp32 kernels."""
    p = configs.config(2)
    rp = np.asarray(p.row_ptr, dtype=np.int64)
    keep = np.ones(rp[-1], dtype=bool)
    lo, hi = 1000, 1300          # rows [1000, 1300): blocks 8..9 entirely, block 7 and 10 partly
    keep[rp[lo]:rp[hi]] = False
    lens = np.diff(rp)
    lens[lo:hi] = 0
    rp2 = np.zeros_like(rp)
    rp2[1:] = np.cumsum(lens)
    q = configs.Problem("cfg2_holes", p.n, p.l, rp2, np.asarray(p.col_idx)[keep], np.asarray(p.val)[keep], p.D)
    with handle(q) as h:
        h.set_option("fuse", 0)
        ref = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=2)
        h.set_option("fuse", 3)
        a = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=2)
        assert h.stat("sp8_state") == 1
    assert np.allclose(a[0], ref[0], rtol=1e-5), (a[0], ref[0])
    assert O.principal_angle(a[1], ref[1]) <= 1e-3
    assert np.all(a[1][lo:hi] == a[1][lo:hi])   # finite


@pytest.mark.parametrize("cfg", [1, 2])
def test_block_lanczos_matches_oracle(cfg):
    """NEXT-3: the restarted block Lanczos with full reorthogonalisation (option solver = 1, the
    paper's sBMDS eigensolver family) reaches the oracle's top-m eigenpairs to the
    BASELINE tolerances, like the subspace iteration, and is deterministic."""
    p = configs.config(cfg)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    if cfg == 1:
        lam_o, V_o, Z_o = O.eigs_dense(S, p.D, p.m)
    else:
        lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, p.m)
    with handle(p) as h:
        h.set_option("solver", 1)
        lam, V, Z, info = gpu_eigs(h, p.m, p.block, max_iters=400, tol=1e-6)
        lam2, V2, _, _ = gpu_eigs(h, p.m, p.block, max_iters=400, tol=1e-6)
        h.set_option("solver", 0)
    assert info["status"] == 0 and info["converged"] == 1
    check_against(lam, V, Z, lam_o, V_o, Z_o)
    assert np.array_equal(lam, lam2) and np.array_equal(V, V2)


def test_tensor_core_sparse_step_duplicate_entries():
    """Repeated (row, column) entries in S (allowed by the CSR input, summed by every SpMM): the
    tensor-core step's images sum them too, so its iteration matches the fp32 kernels."""
    p = configs.config(2)
    rp = np.asarray(p.row_ptr, dtype=np.int64)
    ci = np.asarray(p.col_idx).copy()
    val = np.asarray(p.val, dtype=np.float64).copy()
    rows = np.arange(0, p.n, 7)                      # every 7th row: its 2nd entry repeats its 1st column
    has2 = (rp[rows + 1] - rp[rows]) >= 2
    e1 = rp[rows[has2]]
    ci[e1 + 1] = ci[e1]
    val[e1 + 1] *= 0.5
    q = configs.Problem("cfg2_dups", p.n, p.l, rp, ci, val, p.D)
    with handle(q) as h:
        h.set_option("fuse", 0)
        ref = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=6)
        h.set_option("fuse", 3)
        a = gpu_eigs(h, 3, 16, max_iters=20, tol=0.0, seed=6)
        assert h.stat("sp8_state") == 1
    assert np.allclose(a[0], ref[0], rtol=1e-5), (a[0], ref[0])
    assert O.principal_angle(a[1], ref[1]) <= 1e-3


def test_deferred_gram_and_fused_y2_digits():
    """Config 2 on the symmetric-half int8 D stream (dstream = 3), so every eigs iteration after
    the first runs the cooperative reduces: the non-Rayleigh-Ritz sparse steps leave their Gram
    sums and Cholesky to the next fold (FoldGram), and the D-partial reduce forms Y2's digit
    planes (k_dreduce_y2d). Switching either off (sp8_dbg 128: Gram in the step's last CTA; 64:
    k_dreduce_pair + k_y2_digits) changes only summation orders: the same iteration within the
    fp32 noise, each path bitwise deterministic, and the solve converges to the oracle."""
    p = configs.config(2)
    it = 25
    with handle(p) as h:
        h.set_option("dstream", 3)
        h.set_option("fuse", 3)
        runs = {}
        for dbg in (0, 128, 64, 128 | 64):
            h.set_option("sp8_dbg", dbg)
            runs[dbg] = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=5)
            assert h.stat("sp8_state") == 1
        h.set_option("sp8_dbg", 0)
        again = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=5)
        lam, V, Z, info = gpu_eigs(h, p.m, 16, max_iters=500, tol=1e-6, seed=5)
    base = runs[0]
    assert np.array_equal(base[0], again[0]) and np.array_equal(base[1], again[1])
    for dbg, r in runs.items():
        assert np.allclose(r[0], base[0], rtol=1e-6), (dbg, r[0], base[0])
        assert O.principal_angle(r[1], base[1]) <= 1e-3, dbg
    assert info["converged"] == 1
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, p.m)
    check_against(lam, V, Z, lam_o, V_o, Z_o)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [2, 4])
def test_int8_gram_steps(cfg):
    """Eigs steps whose Gram only feeds the next Cholesky-QR take G = Y^T Y and 1^T Y from Y's
    24-bit digits on the int8 tensor cores (k_sp8_step GRAM8; exact integer sums of the digitised
    block); the step before a Rayleigh-Ritz step and that step keep the FP64 Gram of the fp32
    rows. Both ways run the same iteration within the fixed point's rounding (the Gram only
    chooses the basis of the next iterate), the int8 path is taken where expected, it is bitwise
    deterministic, and the tolerance-mode solve converges to the oracle."""
    p = configs.config(cfg)
    it = 25 if cfg == 2 else 12
    with handle(p) as h:
        h.set_option("fuse", 3)
        h.set_option("sp8_gram8", 0)
        ref = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
        assert h.stat("sp8_state") == 1 and h.stat("gram8_launches") == 0
        h.set_option("sp8_gram8", 1)
        a = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
        # fixed-iteration solve: Rayleigh-Ritz at the end only; every step but the last two
        assert h.stat("gram8_launches") == it - 2
        rep = gpu_eigs(h, p.m, 16, max_iters=it, tol=0.0, seed=3)
        n8 = h.stat("gram8_launches")
        lam, V, Z, info = gpu_eigs(h, p.m, 16, max_iters=500, tol=1e-6, seed=5)
        # tolerance mode, rr_period 5: steps 1-3 of every 5
        assert h.stat("gram8_launches") - n8 == 3 * (info["iters"] // 5) + min(3, info["iters"] % 5)
    (la, Va, _, ia), (lb, Vb, _, ib) = a, ref
    assert np.allclose(la, lb, rtol=1e-5), (la, lb)
    assert O.principal_angle(Va, Vb) <= 1e-3
    assert ia["orth_error"] <= 1e-9, ia["orth_error"]
    assert np.array_equal(la, rep[0]) and np.array_equal(Va, rep[1])
    assert info["converged"] == 1
    if cfg == 2:
        S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
        lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, p.m)
        check_against(lam, V, Z, lam_o, V_o, Z_o)


@pytest.mark.gpu
def test_eigs_b32_two_half_passes():
    """block = 32 where S is local: the tensor-core sparse step runs as two 16-column passes over
    the images per iteration (Gram -- on the int8 tensor cores from Y's digits on steps that feed no
    Rayleigh-Ritz step -- and Cholesky by their own kernels). Same iteration as the fp32
    fused kernels (sp8_apply = 0 keeps them), bitwise deterministic, converges to the oracle."""
    p = configs.config(2)
    with handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        h.set_option("sp8_apply", 0)
        ref = gpu_eigs(h, 8, 32, max_iters=12, tol=0.0, seed=2)
        h.set_option("sp8_apply", 1)
        h.set_option("sp8_gram8", 0)
        a64 = gpu_eigs(h, 8, 32, max_iters=12, tol=0.0, seed=2)   # FP64 Gram kernel on every step
        assert h.stat("sp8_state") == 1 and h.stat("gram8_launches") == 0
        h.set_option("sp8_gram8", 1)
        a = gpu_eigs(h, 8, 32, max_iters=12, tol=0.0, seed=2)
        # the int8 Gram of the 32-wide block (k_gram8_32) on every step but the last two
        assert h.stat("gram8_launches") == 10
        assert np.allclose(a[0], a64[0], rtol=1e-6), (a[0], a64[0])
        assert O.principal_angle(a[1], a64[1]) <= 1e-4
        rep = gpu_eigs(h, 8, 32, max_iters=12, tol=0.0, seed=2)
        lam, V, Z, info = gpu_eigs(h, 3, 32, max_iters=500, tol=1e-6, seed=5)
    assert np.allclose(a[0], ref[0], rtol=1e-5), (a[0], ref[0])
    assert np.array_equal(a[0], rep[0]) and np.array_equal(a[1], rep[1])
    assert info["converged"] == 1
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, 3)
    check_against(lam, V, Z, lam_o, V_o, Z_o)
