"""Pins for the sBHA oracle (oracle/sbha_oracle.py) against SPEC.md's
worked examples (tests/golden/sbha_spec_examples.txt), closed forms and invariants: each pin is
a property the paper or geometry fixes, not the oracle's formula re-typed."""
import os

import numpy as np
import scipy.sparse as sp

from oracle import sbha_oracle as B

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sbha_spec_examples.txt")


def golden():
    out = {}
    for line in open(GOLDEN):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split(":", 1)
            out[k.strip()] = np.array([float(x) for x in v.split()])
    return out


def planar_grid(N, jitter=0.0, seed=0):
    """Unit-square N x N vertex grid, each cell split along one diagonal; optional jitter."""
    rng = np.random.default_rng(seed)
    x, y = np.meshgrid(np.linspace(0, 1, N), np.linspace(0, 1, N), indexing="ij")
    h = 1.0 / (N - 1)
    inner = (x > 0) & (x < 1) & (y > 0) & (y < 1)
    x = x + inner * rng.uniform(-jitter, jitter, x.shape) * h
    y = y + inner * rng.uniform(-jitter, jitter, y.shape) * h
    V = np.stack([x.ravel(), y.ravel(), np.zeros(N * N)], 1)
    idx = np.arange(N * N).reshape(N, N)
    a, b, c, d = idx[:-1, :-1].ravel(), idx[1:, :-1].ravel(), idx[1:, 1:].ravel(), idx[:-1, 1:].ravel()
    F = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)])
    return V, F, inner.ravel()


def test_spec_equilateral_triangle():
    g = golden()
    V = np.array([[0, 0, 0], [1, 0, 0], [0.5, np.sqrt(3) / 2, 0]])
    F = np.array([[0, 1, 2]])
    A = B.cotan_adjacency(V, F).toarray()
    off = A[~np.eye(3, dtype=bool)]
    assert np.allclose(off, g["equilateral_edge_weight"][0], rtol=1e-14)
    assert np.allclose(np.diag(A), 0)
    assert np.allclose(B.lumped_mass(V, F), g["equilateral_mass"][0], rtol=1e-14)


def test_spec_split_square():
    g = golden()
    V = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], dtype=float)
    F = np.array([[0, 1, 2], [0, 2, 3]])
    A = B.cotan_adjacency(V, F).toarray()
    assert abs(A[0, 2] - g["square_diag_weight"][0]) < 1e-15
    for i, j in ((0, 1), (1, 2), (2, 3), (3, 0)):         # boundary edges: one 45-degree cotangent
        assert abs(A[i, j] - g["square_axis_weight"][0]) < 1e-14 and A[i, j] == A[j, i]
    m = B.lumped_mass(V, F)
    assert np.allclose(m[[1, 3]], g["square_mass_corner"][0]) and np.allclose(m[[0, 2]], g["square_mass_diag"][0])


def test_spec_path_graph_biharmonic():
    adj = sp.csr_matrix(np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], dtype=float))
    assert np.array_equal(B.graph_biharmonic(adj), golden()["path_M"].reshape(3, 3))
    assert np.array_equal(B.graph_biharmonic(sp.csr_matrix((2, 2))), np.zeros((2, 2)))


def test_total_area_and_linear_precision_on_planar_mesh():
    """Sum of lumped masses = area (1 for the unit square); the cotangent Laplacian (V - A) of any
    planar triangulation annihilates linear functions at interior vertices (linear precision)."""
    V, F, inner = planar_grid(9, jitter=0.3, seed=1)
    m = B.lumped_mass(V, F)
    assert abs(m.sum() - 1.0) < 1e-13
    A = B.cotan_adjacency(V, F)
    L = sp.diags(np.asarray(A.sum(1)).ravel()) - A
    for f in (V[:, 0], V[:, 1], 2 * V[:, 0] - 3 * V[:, 1] + 0.7):
        r = L @ f
        assert np.abs(r[inner]).max() < 1e-12
        assert np.abs(r[~inner]).max() > 1e-6                # (not at the boundary: a real test)


def test_biharmonic_invariants_on_torus():
    from gen.mesh import torus_grid
    V, F, _ = torus_grid(8, 10, seed=2)
    M = B.mesh_biharmonic(V, F)
    s = np.abs(M).max()
    assert np.abs(M - M.T).max() <= 1e-12 * s
    assert np.abs(M @ np.ones(len(V))).max() <= 1e-10 * s
    ev = np.linalg.eigvalsh(M)
    assert ev.min() >= -1e-9 * ev.max() and abs(ev[1]) > 1e-8 * ev.max()   # PSD, null space = constants


def test_interpolation_properties():
    """P: landmark rows are e_t exactly; rows sum to 1 (constant reproduction, M 1 = 0); l = n gives
    I; and P g minimises the biharmonic energy f^T M f over f with f_b = g (any perturbation on
    the free rows raises it) -- the variational form of Eq. 6, not its solve."""
    from gen.mesh import torus_grid
    V, F, _ = torus_grid(8, 10, seed=3)
    n = len(V)
    M = B.mesh_biharmonic(V, F)
    lm = np.array([0, 17, 33, 46, 60, 71])
    P = B.interpolation(M, lm)
    assert np.array_equal(P[lm], np.eye(len(lm)))
    assert np.abs(P.sum(1) - 1).max() < 1e-10
    assert np.array_equal(B.interpolation(M, np.arange(n)), np.eye(n))
    rng = np.random.default_rng(4)
    g = rng.standard_normal(len(lm))
    f = P @ g
    E0 = f @ M @ f
    u = np.setdiff1d(np.arange(n), lm)
    for _ in range(20):
        d = np.zeros(n)
        d[u] = rng.standard_normal(len(u))
        for eps in (1e-3, 1e-1):
            fe = f + eps * d
            assert fe @ M @ fe > E0


def test_thresholding():
    g = golden()
    n, l, prow, p = g["p_example"].astype(int)
    assert B.p_from_prow(n, l, prow) == p
    col = g["threshold_column"]
    P = np.concatenate([[[1.0]], col[:, None]])         # row 0 is the landmark
    kept = B.threshold(P, [0], 2)
    assert np.array_equal(kept[1:, 0], g["threshold_kept"]) and kept[0, 0] == 1.0
    # ties -> lowest row index
    T = B.threshold(np.array([[1.0], [0.3], [-0.3], [0.3]]), [0], 2)
    assert np.array_equal(T[:, 0], [1.0, 0.3, -0.3, 0.0])
    # brute force against all subsets on a random column; p = n - l keeps everything
    rng = np.random.default_rng(5)
    Pr = rng.standard_normal((9, 2))
    Tr = B.threshold(Pr, [4, 7], 3)
    for c in range(2):
        u = [r for r in range(9) if r not in (4, 7)]
        best = sorted(u, key=lambda r: -abs(Pr[r, c]))[:3]
        assert set(np.flatnonzero(Tr[u, c]) ) == {u.index(r) for r in best}
    assert np.array_equal(B.threshold(Pr, [4, 7], 7), Pr)


def test_sbha_interpolation_budget():
    from gen.mesh import torus_grid
    V, F, _ = torus_grid(10, 12, seed=6)
    lm = np.arange(0, 120, 7)
    Ps, p = B.sbha_interpolation(V, F, lm, p_row=4)
    assert p == B.p_from_prow(120, len(lm), 4)
    u = np.setdiff1d(np.arange(120), lm)
    assert (np.count_nonzero(Ps[u], axis=0) <= p).all()
    assert np.array_equal(Ps[lm], np.eye(len(lm)))


def test_sparse_path_pins():
    """The large-mesh oracle path (biharmonic_sparse, interpolation_columns, threshold_column) on its
    own pins: the SPEC.md:204 path-graph M, M 1 = 0 and symmetry on a torus, the solved columns
    reproduce constants (their sum over the landmark columns is 1 on every free row) and minimise
    the biharmonic energy (perturbations raise it), and thresholding keeps the p largest."""
    import scipy.sparse as sp
    from gen.mesh import torus_grid
    g = golden()
    adj = sp.csr_matrix(np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], dtype=float))
    assert np.array_equal(B.biharmonic_sparse(adj, np.ones(3)).toarray(), g["path_M"].reshape(3, 3))
    V, F, _ = torus_grid(20, 24, seed=9)
    n = len(V)
    M = B.biharmonic_sparse(B.cotan_adjacency(V, F), B.lumped_mass(V, F))
    s = abs(M).max()
    assert abs(M - M.T).max() <= 1e-12 * s and np.abs(M @ np.ones(n)).max() <= 1e-10 * s
    lm = np.arange(0, n, 11)
    Pu = B.interpolation_columns(M, lm, np.arange(len(lm)))
    assert np.abs(Pu.sum(1) - 1).max() < 1e-9                         # constants reproduced
    u = np.setdiff1d(np.arange(n), lm)
    Md = M.toarray()
    rng = np.random.default_rng(2)
    gvec = rng.standard_normal(len(lm))
    f = np.zeros(n)
    f[lm] = gvec
    f[u] = Pu @ gvec
    E0 = f @ Md @ f
    for _ in range(10):
        d = np.zeros(n)
        d[u] = rng.standard_normal(len(u))
        assert (f + 1e-2 * d) @ Md @ (f + 1e-2 * d) > E0
    rows, vals = B.threshold_column(np.array([0.1, -0.9, 0.5, 0.9]), np.array([3, 5, 8, 9]), 2)
    assert rows.tolist() == [5, 9] and vals.tolist() == [-0.9, 0.9]   # tie -> both (p = 2), row order
