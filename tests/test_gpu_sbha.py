"""GPU: the sBHA build (sbmds_sbha_build) against the fp64 sBHA oracle
(oracle/sbha_oracle.py: dense cotangent Laplacian, M, dense solve of P_u, per-column thresholding).

Parity: the same support per column (the p largest |P_uc|), except where the p-th and (p+1)-th
magnitudes tie to ~1e-9 relative (two fp64 solves in different orders may order them
differently; both choices are then checked valid), and the kept values to 1e-6 of the column's
largest magnitude (fp32 output of an fp64 solve; M_uu's condition number is ~1e6-1e8 here).
"""
import numpy as np
import pytest

from gen import configs
from gen.mesh import icosphere, torus_grid
from oracle import sbha_oracle as B
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu


def planar_grid(N, jitter=0.2, seed=0):
    rng = np.random.default_rng(seed)
    x, y = np.meshgrid(np.linspace(0, 1, N), np.linspace(0, 1, N), indexing="ij")
    h = 1.0 / (N - 1)
    inner = (x > 0) & (x < 1) & (y > 0) & (y < 1)
    x = x + inner * rng.uniform(-jitter, jitter, x.shape) * h
    y = y + inner * rng.uniform(-jitter, jitter, y.shape) * h
    V = np.stack([x.ravel(), y.ravel(), 0.1 * np.sin(3 * x.ravel()) * np.cos(2 * y.ravel())], 1)
    idx = np.arange(N * N).reshape(N, N)
    a, b, c, d = idx[:-1, :-1].ravel(), idx[1:, :-1].ravel(), idx[1:, 1:].ravel(), idx[:-1, 1:].ravel()
    F = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)])
    return V, F


def gpu_sbha(V, F, lm, p_row):
    from paper_1705_10887_b200.sbmds import sbha_build
    rp, ci, vv, info = sbha_build(V, F.astype(np.int32), lm, p_row, device="numpy")
    n, l = len(V), len(lm)
    S = np.zeros((n, l))
    for i in range(n):
        cols = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)                 # columns ascending, no duplicates
        S[i, cols] = vv[rp[i]:rp[i + 1]]
    return S, info, (rp, ci, vv)


def check_against_oracle(V, F, lm, p_row):
    n, l = len(V), len(lm)
    S, info, _ = gpu_sbha(V, F, lm, p_row)
    Pd = B.interpolation(B.mesh_biharmonic(V, F), lm)
    p = B.p_from_prow(n, l, p_row)
    Po = B.threshold(Pd, lm, p)
    assert info["p"] == p and info["nnz"] == l + l * p
    assert np.array_equal(S[lm], np.eye(l))
    u = np.setdiff1d(np.arange(n), lm)
    for c in range(l):
        a = np.abs(Pd[u, c])
        kth = np.sort(a)[::-1][p - 1]
        got, want = set(np.flatnonzero(S[u, c])), set(np.flatnonzero(Po[u, c]))
        for q in got ^ want:                              # only near-ties may differ
            assert abs(a[q] - kth) <= 1e-9 * a.max(), (c, q, a[q], kth)
        assert len(got) == p
        scale = a.max()
        both = np.array(sorted(got & want), dtype=np.int64)
        assert np.abs(S[u[both], c] - Pd[u[both], c]).max() <= 1e-6 * scale
    return S, Po, info


def test_sbha_config1_torus():
    """Config 1's mesh and landmarks (torus 40 x 50, l = 100 FPS), p_row = 8; 30 panels of the band
    Cholesky with a ragged last one."""
    p = configs.config(1)
    V, F, _ = torus_grid(40, 50, seed=0)
    S, Po, info = check_against_oracle(V, F, p.landmarks, 8)
    assert info["window"] < len(V) - p.l                 # a real band, not the dense matrix


def test_sbha_icosphere_irregular_valence():
    V, F = icosphere(3)                                   # 642 vertices, valence 5 and 6
    lm = np.random.default_rng(1).choice(len(V), 40, replace=False).astype(np.int32)
    check_against_oracle(V, F, lm, 6)


def test_sbha_open_planar_mesh():
    """Boundary edges take their single cotangent; p_row = n - l keeps all."""
    V, F = planar_grid(20, seed=2)
    lm = np.random.default_rng(3).choice(len(V), 25, replace=False).astype(np.int32)
    check_against_oracle(V, F, lm, 5)
    S, _, _ = gpu_sbha(V, F, lm, 1e9)                    # p = n - l: the dense P exactly (fp32)
    Pd = B.interpolation(B.mesh_biharmonic(V, F), lm)
    assert np.abs(S - Pd).max() <= 1e-6 * np.abs(Pd).max()
    assert np.abs(S.sum(1) - 1).max() < 1e-5             # rows sum to 1 (constant reproduction)


def test_sbha_multi_panel_band():
    """Torus 90 x 120 (n = 10,800, l = 150): ~166 panels and a W-row sliding window."""
    V, F, _ = torus_grid(90, 120, seed=4)
    lm = np.random.default_rng(5).choice(len(V), 150, replace=False).astype(np.int32)
    check_against_oracle(V, F, lm, 10)


def test_sbha_feeds_sbmds():
    """The built S drives the whole path: sbmds_eigs on (S_gpu, D) matches the dense oracle on the
    oracle's S (config 1's D: squared graph distances between its landmarks)."""
    import torch
    from paper_1705_10887_b200 import Sbmds
    p = configs.config(1)
    V, F, _ = torus_grid(40, 50, seed=0)
    S, Po, _ = check_against_oracle(V, F, p.landmarks, 8)
    _, _, (rp, ci, vv) = gpu_sbha(V, F, p.landmarks, 8)
    with Sbmds(p.n, p.l, rp, ci, vv, p.D) as h:
        lam, Vg, Z, info = h.eigs(3, 8, max_iters=500, tol=1e-6)
    So = O.csr(p.n, p.l, *(lambda M: (np.r_[0, np.cumsum((M != 0).sum(1))], np.nonzero(M)[1], M[M != 0]))(Po))
    lam_o, V_o, _ = O.eigs_dense(So, p.D, 3)
    assert np.all(np.abs(lam - lam_o) <= 1e-4 * np.abs(lam_o)), (lam, lam_o)
    assert O.principal_angle(Vg.cpu().numpy().astype(np.float64), V_o) <= 1e-3
    del torch


def test_sbha_rejects_degenerate_faces():
    from paper_1705_10887_b200 import SbmdsError
    V, F, _ = torus_grid(10, 12, seed=1)
    V = V.copy()
    V[F[0, 1]] = V[F[0, 0]]                               # collapse one edge: zero-area faces
    with pytest.raises(SbmdsError, match="degenerate"):
        gpu_sbha(V, F, np.arange(0, 120, 9, dtype=np.int32), 4)


def test_sbha_config2_full_size_sampled_columns():
    """At config 2's full size (torus 250 x 400, n = 100,000, its 1,000 FPS landmarks, p_row 16):
    sampled columns of the GPU's S against the oracle's sparse-LU solve of the same columns
    (oracle.interpolation_columns) thresholded to the same p -- the sampled-output check at a size
    the dense oracle cannot reach."""
    from oracle import sbha_oracle as Bo
    p = configs.config(2)
    V, F, _ = torus_grid(250, 400, seed=0)
    from paper_1705_10887_b200.sbmds import sbha_build
    rp, ci, vv, info = sbha_build(V, F.astype(np.int32), p.landmarks, 16, device="numpy")
    n, l = p.n, p.l
    assert info["nnz"] == l + l * info["p"] and info["p"] == Bo.p_from_prow(n, l, 16)
    rows = np.repeat(np.arange(n), np.diff(rp))
    is_lm = np.zeros(n, bool)
    is_lm[p.landmarks] = True
    u = np.flatnonzero(~is_lm)
    cols = [0, 1, 137, 500, 999]
    M = Bo.biharmonic_sparse(Bo.cotan_adjacency(V, F), Bo.lumped_mass(V, F))
    Pu = Bo.interpolation_columns(M, p.landmarks, cols)
    for j, c in enumerate(cols):
        sel = (ci == c) & ~is_lm[rows]
        g_rows, g_vals = rows[sel], vv[sel]
        o_rows, o_vals = Bo.threshold_column(Pu[:, j], u, info["p"])
        a = np.abs(Pu[:, j])
        kth = np.sort(a)[::-1][info["p"] - 1]
        pos = {r: q for q, r in enumerate(u)}
        for r in set(g_rows.tolist()) ^ set(o_rows.tolist()):   # only near-ties may differ
            assert abs(a[pos[r]] - kth) <= 1e-9 * a.max(), (c, r)
        common = np.intersect1d(g_rows, o_rows)
        gv = dict(zip(g_rows.tolist(), g_vals.tolist()))
        ov = dict(zip(o_rows.tolist(), o_vals.tolist()))
        err = max(abs(gv[r] - ov[r]) for r in common.tolist())
        assert err <= 1e-6 * a.max(), (c, err)
