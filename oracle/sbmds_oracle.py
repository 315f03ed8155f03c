"""fp64 CPU oracle for the sBMDS hot path — TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module. It shares no code with the CUDA
path (``paper_1705_10887_b200``) and never imports it.

What it computes is the paper's plain definition, in fp64, from the same
fp32-stored inputs upcast exactly:

  * the operator   B~ = -1/2 J Ê J,  Ê = P W P^T  ("extracting the
    eigenvalues of -1/2 J Ê J = -1/2 J P W P^T J"), J = I - (1/n) 1 1^T
    (PAPER.md:111), with P = S (the n x l sparse interpolation operator, CSR) and
    W = D_ll already squared (reading R2);
  * classical MDS on it: "the eigenvalue decomposition ... truncating its
    decomposition to the biggest m eigenvalues ... Z = V_m Λ_m^{1/2}"
    (PAPER.md:113), negative λ among the top m get a zero column;
  * for sizes where the dense n x n matrix does not fit, the same eigenpairs by
    Lanczos on matrix-vector products, as sBMDS does;
  * BMDS, the paper's QR route, as a second independent path.

Pins (tests/test_oracle.py, ``-m "not gpu"``), per function — each against a
closed form, a worked example or brute force, never against a re-typed formula:

  dense_operator / approx_sqdist  brute-force quadruple sum; CF1-CF4; SPEC examples
  apply                           brute force; CF2 (rank-3 Gram); mutation test
  _dense_times (multi-block)      rank-structure closed form of squared distances at
                                  l = 5000 (> 2048-row blocks, ragged tail), fp32 and fp64
  apply_raw / rel_sq_error        S = I closed form; brute-force S D S^T; J-sandwich
  eigs_dense / mds_dense / top_m  SPEC.md:55-57, :414-416 goldens; CF1; CF3 spectrum
  eigs_matfree / bmds             CF2 (eigenpairs = SVD of JSY); dense agreement, cfg 1
  embedding                       explicit λ (negative -> zero column)
  residuals                       CF2: 0 at exact pairs, closed form for a rotated v
  principal_angle                 1-D and 2-D subspaces with known distinct angles (max)
  relgap                          explicit spectra

Every function is pinned; none is "parity unpinned" (DESIGN.md §2 lists the pins).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla


# ----------------------------------------------------------------------------- inputs
def csr(n: int, l: int, row_ptr, col_idx, val) -> sp.csr_matrix:
    """S as an fp64 scipy CSR matrix (exact upcast of the stored values)."""
    return sp.csr_matrix((np.asarray(val, dtype=np.float64),
                          np.asarray(col_idx, dtype=np.int64),
                          np.asarray(row_ptr, dtype=np.int64)), shape=(n, l))


def centering(n: int) -> np.ndarray:
    """J = I - (1/n) 1 1^T, explicitly. Small n only."""
    return np.eye(n) - np.full((n, n), 1.0 / n)


# ----------------------------------------------------------------------------- operator
def approx_sqdist(S, D) -> np.ndarray:
    """Ê = P W P^T with P = S, W = D_ll (Eq. 7). n x n, small n."""
    S = sp.csr_matrix(S, dtype=np.float64)
    SD = np.asarray(S @ np.asarray(D, dtype=np.float64))     # P W   (n x l)
    return SD @ S.T.toarray()                                # (P W) P^T


def dense_operator(S, D) -> np.ndarray:
    """B~ = -1/2 J Ê J with the double centring written out.

    J E J subtracts the row means and the column means and adds back the grand
    mean; small n only (n x n dense).
    """
    E = approx_sqdist(S, D)
    row = E.mean(axis=1, keepdims=True)
    col = E.mean(axis=0, keepdims=True)
    JEJ = E - row - col + E.mean()
    return -0.5 * JEJ


def _dense_times(D, T: np.ndarray, block_rows: int = 2048) -> np.ndarray:
    """D @ T in fp64 with D upcast exactly in row blocks (D may be fp32 and large)."""
    D = np.asarray(D)
    out = np.empty((D.shape[0], T.shape[1]), dtype=np.float64)
    for i in range(0, D.shape[0], block_rows):
        out[i:i + block_rows] = D[i:i + block_rows].astype(np.float64) @ T
    return out


def apply(S, D, X) -> np.ndarray:
    """Y = -1/2 J S D S^T J X, right to left, fp64, explicit centred copies.

    PAPER.md:221-222: the matvec uses sparse P, "J is a sum of identity and a
    rank-one matrix", and "W is small"; SPEC.md:428 stages center -> P^T -> W -> P
    -> center -> scale. X is n x b (or n); returned with X's shape, fp64.
    """
    S = sp.csr_matrix(S, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    if vec:
        X = X[:, None]
    Xc = X - X.mean(axis=0, keepdims=True)          # J X
    T1 = np.asarray(S.T @ Xc)                        # P^T (J X)
    T2 = _dense_times(D, T1)                         # W (...)
    T3 = np.asarray(S @ T2)                          # P (...)
    Y = -0.5 * (T3 - T3.mean(axis=0, keepdims=True))  # -1/2 J (...)
    return Y[:, 0] if vec else Y


def apply_raw(S, D, X) -> np.ndarray:
    """E^ X = S D S^T X (no centring, no -1/2), right to left, fp64.

    PAPER.md:152-156: K_BHA = P W P^T, "two interpolation operations"; with W = D_ll of squared
    distances (reading R2) this is the approximation E^ of the squared-distance matrix whose
    rows the paper's error estimate compares with exact rows.
    """
    S = sp.csr_matrix(S, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    if vec:
        X = X[:, None]
    Y = np.asarray(S @ _dense_times(D, np.asarray(S.T @ X)))
    return Y[:, 0] if vec else Y


def rel_sq_error(A, B) -> float:
    """epsilon(A) = ||A - B||_F^2 / ||B||_F^2, fp64."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    return float(np.sum((A - B) ** 2) / np.sum(B ** 2))


# ----------------------------------------------------------------------------- MDS
def embedding(V: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """Z = V_m Λ_m^{1/2}; a negative λ gets a zero column."""
    return V * np.sqrt(np.maximum(lam, 0.0))[None, :]


def top_m(lam: np.ndarray, V: np.ndarray, m: int):
    """The m biggest (algebraic, "biggest m eigenvalues") eigenpairs, descending."""
    order = np.argsort(-lam, kind="stable")[:m]
    return lam[order], V[:, order]


def mds_dense(B: np.ndarray, m: int):
    """Classical MDS of an explicit operator B = -1/2 J E J: full eigh, top m."""
    lam, V = np.linalg.eigh(B)
    lam, V = top_m(lam, V, m)
    return lam, V, embedding(V, lam)


def eigs_dense(S, D, m: int):
    """Top-m eigenpairs and Z of -1/2 J S D S^T J by a full dense eigendecomposition."""
    return mds_dense(dense_operator(S, D), m)


def eigs_matfree(S, D, m: int, tol: float = 1e-12, seed: int = 0, ncv: int | None = None):
    """Same eigenpairs by Lanczos on matvecs only ("uses the Lanczos method").

    scipy's ARPACK (implicitly restarted Lanczos), which='LA' = largest algebraic.
    Returns (lam, V, Z, n_matvec).
    """
    S = sp.csr_matrix(S, dtype=np.float64)
    n = S.shape[0]
    Dd = np.asarray(D)
    if Dd.dtype != np.float64 and Dd.nbytes <= 24e9:
        Dd = Dd.astype(np.float64)
    count = [0]

    def mv(x):
        count[0] += 1
        return apply(S, Dd, np.asarray(x).reshape(n))

    op = spla.LinearOperator((n, n), matvec=mv, dtype=np.float64)
    v0 = np.random.default_rng(seed).standard_normal(n)
    lam, V = spla.eigsh(op, k=m, which="LA", tol=tol, v0=v0, ncv=ncv)
    lam, V = top_m(lam, V, m)
    return lam, V, embedding(V, lam), count[0]


def bmds(S, D, m: int):
    """BMDS, the paper's QR route: QR = J P; eig of -1/2 R W R^T;
    Z = Q Ṽ_m Λ_m^{1/2}. Needs the dense n x l matrix J P (moderate n*l only)."""
    S = sp.csr_matrix(S, dtype=np.float64)
    JP = S.toarray()
    JP -= JP.mean(axis=0, keepdims=True)
    Q, R = np.linalg.qr(JP, mode="reduced")
    small = -0.5 * (R @ np.asarray(D, dtype=np.float64) @ R.T)
    small = 0.5 * (small + small.T)
    lam, U = np.linalg.eigh(small)
    lam, U = top_m(lam, U, m)
    V = Q @ U
    return lam, V, embedding(V, lam)


def residuals(S, D, lam: np.ndarray, V: np.ndarray) -> np.ndarray:
    """||B~ v_i - λ_i v_i||_2 per column (the SPEC.md:52 residual)."""
    R = apply(S, D, V) - V * lam[None, :]
    return np.linalg.norm(R, axis=0)


# ----------------------------------------------------------------------------- comparisons
def principal_angle(Va: np.ndarray, Vb: np.ndarray) -> float:
    """Largest principal angle between span(Va) and span(Vb) (host fp64):
    asin || (I - Qa Qa^T) Qb ||_2 with Q* orthonormal bases."""
    Qa = scipy.linalg.orth(np.asarray(Va, dtype=np.float64))
    Qb = scipy.linalg.orth(np.asarray(Vb, dtype=np.float64))
    P = Qb - Qa @ (Qa.T @ Qb)
    s = np.linalg.norm(P, 2) if P.size else 0.0
    return float(np.arcsin(min(1.0, s)))


def relgap(lam_sorted_desc: np.ndarray, m: int) -> float:
    """(λ_m - λ_{m+1}) / |λ_1| for a descending spectrum (reading R4)."""
    return float((lam_sorted_desc[m - 1] - lam_sorted_desc[m]) / abs(lam_sorted_desc[0]))
