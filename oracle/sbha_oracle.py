"""fp64 CPU oracle for the sBHA build — TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s baseline legs may import it. It
shares no code with the CUDA path and never imports it. The plain definitions, in fp64, dense
where the paper's formula is a matrix expression (small meshes only):

  * cotangent adjacency A_ij = (cot α_ij + cot β_ij) / 2, the angles opposite edge ij
    (PAPER.md:97-100); a boundary edge gets its single cotangent / 2;
  * lumped mass D_ii = 1/3 of the total area of the triangles incident on i;
  * V = diag(sum_j A_ij), the biharmonic operator M = (V - A)^T D^{-1} (V - A);
    the graph variant D = I, A = 0/1 adjacency;
  * the interpolation operator P = [I_l ; -M_uu^{-1} M_ub] (Eq. 6), with the
    rows of the landmarks b the identity and u the remaining rows in increasing order;
  * the same columns for large meshes by a sparse LU of M_uu (interpolation_columns; M from
    scipy sparse products, biharmonic_sparse);
  * thresholding: each column of P_u keeps its p largest-magnitude entries (PAPER.md:175-191
    "chooses the p biggest elements in magnitude ... for each column"), ties to the lowest row
    (SPEC.md:325), kept values unchanged; p = ceil((n - l) p_row / l).

Pins (tests/test_sbha_oracle.py, ``-m "not gpu"``): SPEC.md:178-188 worked examples (equilateral
triangle, split square), the path-graph M of SPEC.md:204 written out by hand, total area,
linear precision of the cotangent Laplacian on a flat grid, M 1 = 0 and symmetry, P's
constant reproduction and identity rows, the variational characterisation of P (every
perturbation of P_u g raises g^T M g-energy), brute-force thresholding, p = n - l keeping all;
biharmonic_sparse / interpolation_columns / threshold_column by the path-graph M of SPEC.md:204,
M 1 = 0, constant reproduction of the solved columns and the energy minimality above.
Every function here is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def cotan_adjacency(verts, faces, n: int | None = None) -> sp.csr_matrix:
    """A_ij = sum over the triangles containing edge ij of cot(angle opposite ij) / 2."""
    V = np.asarray(verts, dtype=np.float64)
    F = np.asarray(faces, dtype=np.int64)
    n = len(V) if n is None else n
    rows, cols, vals = [], [], []
    for a, b, c in F:
        for (i, j, k) in ((a, b, c), (b, c, a), (c, a, b)):     # edge ij, opposite vertex k
            u, w = V[i] - V[k], V[j] - V[k]
            cot = float(np.dot(u, w) / np.linalg.norm(np.cross(u, w)))
            rows += [i, j]
            cols += [j, i]
            vals += [cot / 2, cot / 2]
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def lumped_mass(verts, faces, n: int | None = None) -> np.ndarray:
    """D_ii = (1/3) sum of the areas of the faces containing i."""
    V = np.asarray(verts, dtype=np.float64)
    n = len(V) if n is None else n
    m = np.zeros(n)
    for a, b, c in np.asarray(faces, dtype=np.int64):
        area = 0.5 * np.linalg.norm(np.cross(V[b] - V[a], V[c] - V[a]))
        m[[a, b, c]] += area / 3
    return m


def biharmonic(A: sp.spmatrix, mass: np.ndarray) -> np.ndarray:
    """M = (V - A)^T D^{-1} (V - A), dense fp64 (small n)."""
    Ad = np.asarray(sp.csr_matrix(A).toarray(), dtype=np.float64)
    L = np.diag(Ad.sum(axis=1)) - Ad
    return L.T @ np.diag(1.0 / np.asarray(mass, dtype=np.float64)) @ L


def mesh_biharmonic(verts, faces) -> np.ndarray:
    return biharmonic(cotan_adjacency(verts, faces), lumped_mass(verts, faces))


def graph_biharmonic(adj) -> np.ndarray:
    """Generic graph: D = I, A = 0/1 adjacency."""
    A = sp.csr_matrix(adj, dtype=np.float64)
    return biharmonic(A, np.ones(A.shape[0]))


def interpolation(M: np.ndarray, landmarks) -> np.ndarray:
    """P (n x l): row landmarks[t] = e_t; rows u = -M_uu^{-1} M_ub (dense solve)."""
    M = np.asarray(M, dtype=np.float64)
    n = M.shape[0]
    b = np.asarray(landmarks, dtype=np.int64)
    l = len(b)
    u = np.setdiff1d(np.arange(n), b)                   # increasing order
    P = np.zeros((n, l))
    P[b, np.arange(l)] = 1.0
    if len(u):
        P[u] = -np.linalg.solve(M[np.ix_(u, u)], M[np.ix_(u, b)])
    return P


def p_from_prow(n: int, l: int, p_row: float) -> int:
    """p = ceil((n - l) p_row / l), clamped to [1, n - l]."""
    return max(1, min(n - l, math.ceil((n - l) * p_row / l)))


def threshold(P: np.ndarray, landmarks, p: int) -> np.ndarray:
    """Each column's p largest |P_uc| over the non-landmark rows u kept (ties: lowest row)."""
    P = np.asarray(P, dtype=np.float64)
    n, l = P.shape
    is_lm = np.zeros(n, dtype=bool)
    is_lm[np.asarray(landmarks, dtype=np.int64)] = True
    u = np.flatnonzero(~is_lm)
    out = np.zeros_like(P)
    out[is_lm] = P[is_lm]
    for c in range(l):
        col = P[u, c]
        order = sorted(range(len(u)), key=lambda r: (-abs(col[r]), u[r]))[:p]
        out[u[order], c] = col[order]
    return out


def biharmonic_sparse(A: sp.spmatrix, mass: np.ndarray) -> sp.csr_matrix:
    """M = (V - A)^T D^{-1} (V - A) with scipy sparse products (large meshes; the same formula as
    biharmonic, kept sparse)."""
    A = sp.csr_matrix(A, dtype=np.float64)
    L = sp.diags(np.asarray(A.sum(axis=1)).ravel()) - A
    return sp.csr_matrix(L.T @ sp.diags(1.0 / np.asarray(mass, dtype=np.float64)) @ L)


def interpolation_columns(M: sp.spmatrix, landmarks, cols) -> np.ndarray:
    """Columns `cols` of P_u = -M_uu^{-1} M_ub by a sparse LU of M_uu (scipy
    SuperLU, a library factorisation), for meshes whose dense M does not fit. Returns
    (n - l) x len(cols), rows = the free vertices in increasing order."""
    import scipy.sparse.linalg as spla
    M = sp.csc_matrix(M, dtype=np.float64)
    n = M.shape[0]
    b = np.asarray(landmarks, dtype=np.int64)
    u = np.setdiff1d(np.arange(n), b)
    Muu = M[u][:, u].tocsc()
    rhs = -M[u][:, b[np.asarray(cols)]].toarray()
    return spla.splu(Muu).solve(rhs)


def threshold_column(col: np.ndarray, u: np.ndarray, p: int):
    """One column's kept (row, value) pairs: the p largest |col| over the free rows u (ties: lowest
    row), in increasing row order."""
    order = sorted(range(len(u)), key=lambda r: (-abs(col[r]), u[r]))[:p]
    order = sorted(order, key=lambda r: u[r])
    return u[order], col[order]


def sbha_interpolation(verts, faces, landmarks, p_row: float):
    """The sparse interpolation operator P_sparse of a triangle mesh: (P_sparse, p)."""
    n = len(verts)
    l = len(landmarks)
    P = interpolation(mesh_biharmonic(verts, faces), landmarks)
    p = p_from_prow(n, l, p_row)
    return threshold(P, landmarks, p), p
