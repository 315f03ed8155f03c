"""Pins for the fp64 oracle against what the paper and the mathematics fix (not against itself).

Each test names the closed form / worked example it checks.
A plausible slip in the oracle — a dropped -1/2, a missing centring, S vs S^T,
a transposed D, ascending instead of descending order, a missing sqrt in Z —
fails at least one of them (see test_mutations_are_caught).
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sbmds_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sqdist(P):
    P = np.asarray(P, dtype=np.float64)
    return ((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)


def eye_csr(n):
    return sp.identity(n, format="csr", dtype=np.float64)


def load_golden(name):
    """Golden fixtures: '# cite' lines, then 'key: v1 v2 ...' lines."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(":", 1)
            out[k.strip()] = np.array([float(x) for x in v.split()])
    return out


# --------------------------------------------------------------------------- SPEC worked examples
def test_three_collinear_points():
    """points 0,1,2, m=1 -> Z = (-1,0,1) up to sign, λ = 2."""
    g = load_golden("mds_collinear3.txt")
    E = sqdist(g["points"][:, None])
    lam, V, Z = O.eigs_dense(eye_csr(3), E, 1)
    assert np.allclose(lam, g["lambda"], atol=1e-12)
    z = Z[:, 0] * np.sign(Z[2, 0])
    assert np.allclose(z, g["Z"], atol=1e-12)


def test_four_collinear_points_lambda5():
    """-1/2 J E J of 4 collinear unit-spaced points: λ1 = 5 (= Σ centred x²)."""
    g = load_golden("mds_collinear4.txt")
    E = sqdist(g["points"][:, None])
    lam, _, _ = O.eigs_dense(eye_csr(4), E, 2)
    assert np.allclose(lam, g["lambda"], atol=1e-12)


def test_unit_square():
    """unit-square corners, m=2: λ = (1,1) and distances reproduced."""
    g = load_golden("mds_unit_square.txt")
    P = g["points"].reshape(4, 2)
    E = sqdist(P)
    lam, _, Z = O.eigs_dense(eye_csr(4), E, 2)
    assert np.allclose(lam, g["lambda"], atol=1e-12)
    assert np.allclose(sqdist(Z), E, atol=1e-10)


def test_zero_distances():
    """E = 0 -> Z = 0."""
    lam, _, Z = O.eigs_dense(eye_csr(5), np.zeros((5, 5)), 2)
    assert np.allclose(lam, 0) and np.allclose(Z, 0)


def test_diag_spectrum_selection():
    """operator diag(5,4,3,2,1), k=2 -> (5,4): top-m algebraic selection."""
    lam, V, _ = O.mds_dense(np.diag([5.0, 4, 3, 2, 1]), 2)
    assert np.allclose(lam, [5, 4])
    lam, V, _ = O.mds_dense(np.diag([1.0, -9, 3, 2, 0.5]), 2)   # algebraic, not |λ|
    assert np.allclose(lam, [3, 2])


# --------------------------------------------------------------------------- closed forms
def test_cf1_planar_points_recovered():
    """CF1 (north_star): S = I, D = squared Euclidean distances of planar points Y.
    B~ = (JY)(JY)^T: λ = eig((JY)^T JY), Z = JY up to a rigid motion."""
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((60, 2)) * [3.0, 1.0]
    lam, V, Z = O.eigs_dense(eye_csr(60), sqdist(Y), 2)
    JY = Y - Y.mean(0)
    ref = np.sort(np.linalg.eigvalsh(JY.T @ JY))[::-1]
    assert np.allclose(lam, ref, rtol=1e-12)
    # orthogonal Procrustes: min_Q ||Z Q - JY|| = 0
    U, _, Wt = np.linalg.svd(Z.T @ JY)
    assert np.linalg.norm(Z @ (U @ Wt) - JY) < 1e-9 * np.linalg.norm(JY)


def random_pou(n, l, k, rng, landmark_rows=True):
    """Random S with k nnz per row, rows summing to 1 (partition of unity)."""
    rows, cols, vals = [], [], []
    for i in range(n):
        if landmark_rows and i < l:
            rows.append(i); cols.append(i); vals.append(1.0)
            continue
        c = rng.choice(l, size=k, replace=False)
        w = rng.uniform(0.1, 1.0, size=k)
        rows += [i] * k; cols += list(c); vals += list(w / w.sum())
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, l))


def cf2_problem(n=300, l=40, k=5, seed=2):
    rng = np.random.default_rng(seed)
    S = random_pou(n, l, k, rng)
    Yl = rng.standard_normal((l, 3)) * [3.0, 2.0, 1.0]
    D = sqdist(Yl)
    JSY = S @ Yl
    JSY = JSY - JSY.mean(0)
    return S, D, JSY


def test_cf2_apply_is_rank3_gram():
    """CF2: rows of S sum to 1 and D_ab = |y_a - y_b|^2 => B~ = (JSY)(JSY)^T exactly."""
    S, D, JSY = cf2_problem()
    X = np.random.default_rng(3).standard_normal((S.shape[0], 4))
    Y = O.apply(S, D, X)
    ref = JSY @ (JSY.T @ X)
    assert np.linalg.norm(Y - ref) < 1e-11 * np.linalg.norm(ref)
    B = O.dense_operator(S, D)
    assert np.linalg.norm(B - JSY @ JSY.T) < 1e-11 * np.linalg.norm(B)


def test_cf2_eigs_dense_matfree_bmds():
    """CF2 eigenpairs = SVD of JSY (λ_i = σ_i², V = left singular vectors), for all three oracle paths."""
    S, D, JSY = cf2_problem()
    U, s, _ = np.linalg.svd(JSY, full_matrices=False)
    for lam, V, Z in (O.eigs_dense(S, D, 3), O.eigs_matfree(S, D, 3)[:3], O.bmds(S, D, 3)):
        assert np.allclose(lam, s ** 2, rtol=1e-9)
        assert O.principal_angle(V, U) < 1e-7
        assert np.allclose(Z @ Z.T, JSY @ JSY.T, atol=1e-8 * s[0] ** 2)


def test_cf3_circle_negative_and_degenerate_spectrum():
    """CF3: N points on a circle of radius ρ, S = I, D = squared arc length (circulant).
    For k != 0 the Fourier modes are eigenvectors and J leaves them alone:
    λ_k = -1/2 Σ_j D_0j cos(2πkj/N); the k=0 mode is annihilated (λ = 0)."""
    N, rho = 24, 1.7
    th = 2 * np.pi * np.arange(N) / N
    diff = np.angle(np.exp(1j * (th[:, None] - th[None, :])))
    D = (rho * diff) ** 2
    B = O.dense_operator(eye_csr(N), D)
    got = np.sort(np.linalg.eigvalsh(B))
    j = np.arange(N)
    lam = [-0.5 * np.sum(D[0] * np.cos(2 * np.pi * k * j / N)) for k in range(1, N)]
    want = np.sort(np.concatenate([[0.0], lam]))
    assert np.allclose(got, want, atol=1e-10 * np.abs(want).max())
    assert (want < -1e-6).sum() > 0                   # genuinely indefinite
    top, _, _ = O.eigs_dense(eye_csr(N), D, 2)         # cos/sin pair: exactly degenerate
    assert abs(top[0] - top[1]) < 1e-10 * abs(top[0])


def test_cf4_selector_s():
    """CF4: every row of S is a unit vector and each landmark repeats c times (n = c l):
    J_n S = S J_l, so the nonzero eigenvalues of B~ are c · eig(-1/2 J_l D J_l)."""
    rng = np.random.default_rng(4)
    l, c = 12, 5
    n = l * c
    cols = rng.permutation(np.repeat(np.arange(l), c))
    S = sp.csr_matrix((np.ones(n), (np.arange(n), cols)), shape=(n, l))
    A = rng.uniform(0, 10, size=(l, l))
    D = A + A.T
    np.fill_diagonal(D, 0)
    Jl = np.eye(l) - 1.0 / l
    small = np.linalg.eigvalsh(-0.5 * Jl @ D @ Jl)
    big = np.linalg.eigvalsh(O.dense_operator(S, D))
    want = np.sort(c * small)
    got = np.sort(big)
    # the n - l extra eigenvalues are exactly zero; compare after dropping n-l zeros
    got_nz = np.delete(got, np.argsort(np.abs(got))[: n - l])
    assert np.allclose(np.sort(got_nz), want, atol=1e-9 * np.abs(want).max())


# --------------------------------------------------------------------------- brute force / invariants
def test_brute_force_quadruple_sum():
    """Tiny input: B~_ij = -1/2 Σ_pq J_ip (Σ_ab S_pa D_ab S_qb) J_qj written as loops."""
    rng = np.random.default_rng(5)
    n, l = 6, 3
    S = rng.uniform(-0.5, 1.0, size=(n, l))            # general S: negative values, no row-sum constraint
    A = rng.uniform(0, 4, size=(l, l))
    D = A + A.T
    E = [[sum(S[p, a] * D[a, b] * S[q, b] for a in range(l) for b in range(l))
          for q in range(n)] for p in range(n)]
    J = [[(1.0 if i == j else 0.0) - 1.0 / n for j in range(n)] for i in range(n)]
    B = [[-0.5 * sum(J[i][p] * E[p][q] * J[q][j] for p in range(n) for q in range(n))
          for j in range(n)] for i in range(n)]
    B = np.array(B)
    Ssp = sp.csr_matrix(S)
    assert np.allclose(O.dense_operator(Ssp, D), B, atol=1e-12)
    X = rng.standard_normal((n, 2))
    assert np.allclose(O.apply(Ssp, D, X), B @ X, atol=1e-12)


def test_invariants_on_config1():
    """B~ symmetric, B~ 1 = 0, J 1 = 0, columns of B~X sum to 0; rows of S sum to 1, landmark rows e_j."""
    from gen import configs
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val)
    B = O.dense_operator(S, p.D)
    assert np.abs(B - B.T).max() < 1e-12 * np.abs(B).max()
    assert np.abs(B @ np.ones(p.n)).max() < 1e-10 * np.abs(B).max()
    assert np.abs(O.centering(7) @ np.ones(7)).max() < 1e-15
    X = np.random.default_rng(0).standard_normal((p.n, 3))
    Y = O.apply(S, p.D, X)
    assert np.abs(Y.sum(0)).max() < 1e-10 * np.abs(Y).max() * p.n
    assert np.allclose(np.asarray(S.sum(1)).ravel(), 1.0, atol=1e-14)
    lm_rows = S[p.landmarks].toarray()
    assert np.array_equal(lm_rows, np.eye(p.l))


def test_dense_matfree_bmds_agree_on_config1():
    """Config 1: full eigh, Lanczos on matvecs, and the QR route all give the same top-3 pairs."""
    from gen import configs
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val)
    lam_d, V_d, _ = O.eigs_dense(S, p.D, p.m)
    lam_m, V_m, _, _ = O.eigs_matfree(S, p.D, p.m)
    lam_b, V_b, _ = O.bmds(S, p.D, p.m)
    assert np.allclose(lam_m, lam_d, rtol=1e-10)
    assert np.allclose(lam_b, lam_d, rtol=1e-10)
    assert O.principal_angle(V_m, V_d) < 1e-7 and O.principal_angle(V_b, V_d) < 1e-7
    # the dense spectrum has the structure SURVEY.md [Pr1] reports: clean cut at m=3
    lam_all = np.sort(np.linalg.eigvalsh(O.dense_operator(S, p.D)))[::-1]
    assert O.relgap(lam_all, 3) > 1e-2


def test_embedding_and_angle_helpers():
    V = np.eye(4)[:, :3]
    Z = O.embedding(V, np.array([4.0, -1.0, 9.0]))
    assert np.allclose(Z[:, 0], 2 * V[:, 0]) and np.allclose(Z[:, 1], 0) and np.allclose(Z[:, 2], 3 * V[:, 2])
    t = 0.3
    a = np.array([[1.0], [0.0], [0.0]])
    b = np.array([[np.cos(t)], [np.sin(t)], [0.0]])
    assert abs(O.principal_angle(a, b) - t) < 1e-12


def test_mutations_are_caught():
    """Each plausible oracle slip breaks CF2 (so the pins above would fail)."""
    S, D, JSY = cf2_problem(n=80, l=12, k=3)
    X = np.random.default_rng(9).standard_normal((80, 2))
    ref = JSY @ (JSY.T @ X)
    good = O.apply(S, D, X)
    S64 = sp.csr_matrix(S)
    muts = {
        "no_half": -1.0 * (lambda T: T - T.mean(0))(S64 @ (D @ (S64.T @ (X - X.mean(0))))),
        "no_left_J": -0.5 * (S64 @ (D @ (S64.T @ (X - X.mean(0))))),
        "no_right_J": (lambda T: -0.5 * (T - T.mean(0)))(S64 @ (D @ (S64.T @ X))),
        "sign": 0.5 * (lambda T: T - T.mean(0))(S64 @ (D @ (S64.T @ (X - X.mean(0))))),
    }
    assert np.linalg.norm(good - ref) < 1e-10 * np.linalg.norm(ref)
    for name, Ym in muts.items():
        assert np.linalg.norm(Ym - ref) > 1e-3 * np.linalg.norm(ref), name


def test_apply_raw_pins():
    """apply_raw (E^ X = S D S^T X) is pinned three ways: S = I gives D X
    (closed form); columns of E^ e_j equal the dense product S D S^T built entry by entry on a
    tiny case (brute force); and -1/2 J (apply_raw) J equals the centred apply (pinned above)."""
    rng = np.random.default_rng(3)
    l = 7
    A = rng.uniform(0, 10, (l, l))
    D = (A + A.T) / 2
    X = rng.standard_normal((l, 3))
    assert np.allclose(O.apply_raw(sp.identity(l, format="csr"), D, X), D @ X)
    n = 11
    Sd = np.zeros((n, l))
    for i in range(n):
        cols = rng.choice(l, 3, replace=False)
        Sd[i, cols] = rng.uniform(-1, 1, 3)
    S = sp.csr_matrix(Sd)
    E = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            E[i, j] = sum(Sd[i, a] * D[a, c] * Sd[j, c] for a in range(l) for c in range(l))
    Xn = rng.standard_normal((n, 2))
    assert np.allclose(O.apply_raw(S, D, Xn), E @ Xn)
    J = np.eye(n) - np.ones((n, n)) / n
    assert np.allclose(-0.5 * J @ O.apply_raw(S, D, J @ Xn), O.apply(S, D, Xn))
    assert O.rel_sq_error(E, E) == 0.0 and abs(O.rel_sq_error(2 * E, E) - 1.0) < 1e-12


# --------------------------------------------------------------------------- helper pins
def test_residuals_closed_form():
    """residuals() (the SPEC.md:52 residual ||B~v - θv||) on CF2, where B~ = A A^T, A = JSY.
    Exact eigenpairs (λ_i = σ_i², v_i = u_i) give 0. A rotated v = cos t u_1 + sin t z with
    z ⊥ range(A) (so B~z = 0) has B~v = cos t σ_1² u_1, hence, for any θ,
    ||B~v - θv||² = cos²t (σ_1² - θ)² + θ² sin²t — closed form, not the oracle's formula."""
    S, D, JSY = cf2_problem()
    U, s, _ = np.linalg.svd(JSY, full_matrices=False)
    r0 = O.residuals(S, D, s ** 2, U)
    assert r0.shape == (3,) and np.all(r0 < 1e-10 * s[0] ** 2)
    rng = np.random.default_rng(11)
    z = rng.standard_normal(JSY.shape[0])
    z -= U @ (U.T @ z)                                  # z ⊥ span(U) = range(A)
    z /= np.linalg.norm(z)
    for t, theta in ((0.1, s[0] ** 2), (0.4, 0.7 * s[0] ** 2), (1.2, 2.0)):
        v = np.cos(t) * U[:, 0] + np.sin(t) * z
        want = np.sqrt((np.cos(t) * (s[0] ** 2 - theta)) ** 2 + (theta * np.sin(t)) ** 2)
        got = O.residuals(S, D, np.array([theta]), v[:, None])[0]
        assert abs(got - want) < 1e-9 * s[0] ** 2, (t, got, want)


def test_principal_angle_two_dimensional():
    """Largest principal angle between 2-D subspaces with known distinct angles a < b:
    span(e1, e2) vs span(cos a e1 + sin a e3, cos b e2 + sin b e4) -> b (not a), independent
    of the bases chosen (the second is given as a non-orthonormal mix of its vectors)."""
    a, b = 0.2, 0.7
    E = np.eye(6)
    A = E[:, :2]
    B = np.stack([np.cos(a) * E[:, 0] + np.sin(a) * E[:, 2],
                  np.cos(b) * E[:, 1] + np.sin(b) * E[:, 3]], axis=1)
    mix = np.array([[2.0, 1.0], [-0.5, 3.0]])
    for Bb in (B, B @ mix):
        assert abs(O.principal_angle(A, Bb) - b) < 1e-12
        assert abs(O.principal_angle(Bb, A) - b) < 1e-12
    assert O.principal_angle(A, A @ mix) < 1e-7          # same subspace, different basis
    # orthogonal complement: π/2
    assert abs(O.principal_angle(A, E[:, 4:6]) - np.pi / 2) < 1e-12


def test_dense_times_multiblock_closed_form():
    """_dense_times (the D product of the oracle apply) at l = 5000 > 2048 rows per block, with
    a ragged last block: D = squared distances of integer points (exact in fp32), whose product
    has the closed form D T = a (1^T T) - 2 Y (Y^T T) + 1 (a^T T), a_i = |y_i|^2. Checked for
    fp32 and fp64 D, and through the full apply against CF2's rank-3 Gram at the same l."""
    rng = np.random.default_rng(12)
    l = 5000
    Y = rng.integers(-40, 41, size=(l, 3)).astype(np.float64)
    D64 = sqdist(Y)
    assert D64.max() < 2 ** 24
    T = rng.standard_normal((l, 5))
    a = (Y ** 2).sum(1)
    want = np.outer(a, T.sum(0)) - 2 * Y @ (Y.T @ T) + np.outer(np.ones(l), a @ T)
    for D in (D64, D64.astype(np.float32)):
        got = O._dense_times(D, T)
        assert np.linalg.norm(got - want) < 1e-12 * np.linalg.norm(want)
    # full apply: PoU S over these landmarks -> B~ = (JSY)(JSY)^T
    n = 7000
    S = random_pou(n, l, 4, rng)
    X = rng.standard_normal((n, 3))
    A = S @ Y
    A = A - A.mean(0)
    ref = A @ (A.T @ X)
    got = O.apply(S, D64.astype(np.float32), X)
    assert np.linalg.norm(got - ref) < 1e-11 * np.linalg.norm(ref)


def test_relgap_explicit_spectrum():
    """relgap = (λ_m - λ_{m+1}) / |λ_1| (R4) on explicit descending spectra,
    including a negative λ_1 (absolute value in the denominator)."""
    lam = np.array([10.0, 4.0, 3.5, -20.0])
    assert abs(O.relgap(lam, 1) - 0.6) < 1e-15
    assert abs(O.relgap(lam, 2) - 0.05) < 1e-15
    assert abs(O.relgap(lam, 3) - 2.35) < 1e-15
    assert abs(O.relgap(np.array([-1.0, -3.0]), 1) - 2.0) < 1e-15
