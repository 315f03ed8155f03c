"""Synthetic meshes that stand in for the paper's datasets (input generation only).

PAPER.md:286 uses Brain, Bunny, Dragon and TOSCA meshes, none of which exist in
this container; BASELINE.json configs 1-4 replace them by a jittered torus grid
and a bumpy icosphere of the paper's sizes. Recipe details BASELINE.json leaves
open follow SURVEY.md §8(c) reading 10 and are restated in DESIGN.md §3.
"""
from __future__ import annotations

import numpy as np


def torus_grid(nu: int, nv: int, R: float = 3.0, r: float = 1.0, jitter: float = 0.1,
               seed: int = 0):
    """Torus (R, r) as an nu x nv triangulated parameter grid.

    Vertex (i, j) -> index i*nv + j at u = 2pi(i + du)/nu, v = 2pi(j + dv)/nv with
    du, dv ~ U[-jitter, jitter] (cells). Each quad (i,j),(i+1,j),(i+1,j+1),(i,j+1)
    is split along the (i,j)-(i+1,j+1) diagonal. Returns (verts (n,3) f64,
    faces (2n,3) i64, edges (3n,2) i64).
    """
    rng = np.random.default_rng(seed)
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    du = rng.uniform(-jitter, jitter, size=(nu, nv))
    dv = rng.uniform(-jitter, jitter, size=(nu, nv))
    u = 2 * np.pi * (i + du) / nu
    v = 2 * np.pi * (j + dv) / nv
    verts = np.stack([(R + r * np.cos(v)) * np.cos(u),
                      (R + r * np.cos(v)) * np.sin(u),
                      r * np.sin(v)], axis=-1).reshape(-1, 3)
    idx = (i * nv + j)
    ip = ((i + 1) % nu) * nv + j
    jp = i * nv + (j + 1) % nv
    ipjp = ((i + 1) % nu) * nv + (j + 1) % nv
    faces = np.concatenate([np.stack([idx, ip, ipjp], -1).reshape(-1, 3),
                            np.stack([idx, ipjp, jp], -1).reshape(-1, 3)]).astype(np.int64)
    edges = np.concatenate([np.stack([idx, ip], -1).reshape(-1, 2),
                            np.stack([idx, jp], -1).reshape(-1, 2),
                            np.stack([idx, ipjp], -1).reshape(-1, 2)]).astype(np.int64)
    return verts, faces, edges


def icosphere(s: int):
    """Unit icosphere after s midpoint subdivisions: n = 10*4^s + 2."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(s):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e.sort(axis=1)
        uniq, inv = np.unique(e, axis=0, return_inverse=True)
        inv = inv.reshape(3, -1)
        mid = v[uniq[:, 0]] + v[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        base = len(v)
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        ab, bc, ca = inv[0] + base, inv[1] + base, inv[2] + base
        v = np.concatenate([v, mid])
        f = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)])
    return v, f


def mesh_edges(faces: np.ndarray) -> np.ndarray:
    e = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
    e.sort(axis=1)
    return np.unique(e, axis=0)


def real_sph_harm(ell: int, m: int, xyz: np.ndarray) -> np.ndarray:
    """Real spherical harmonic Y_ell^m evaluated at unit vectors xyz."""
    from scipy.special import sph_harm_y
    theta = np.arccos(np.clip(xyz[:, 2], -1.0, 1.0))       # polar
    phi = np.arctan2(xyz[:, 1], xyz[:, 0])                  # azimuth
    if m == 0:
        return np.real(sph_harm_y(ell, 0, theta, phi))
    y = sph_harm_y(ell, abs(m), theta, phi)
    return np.sqrt(2.0) * (np.imag(y) if m < 0 else np.real(y))


def morton_order(v: np.ndarray) -> np.ndarray:
    """Vertex order along the Z-order (Morton) curve of the coordinates, 20 bits per axis
    (ties by index): the spatially coherent numbering scanned and remeshed meshes carry."""
    v = np.asarray(v, dtype=np.float64)
    span = float((v.max(0) - v.min(0)).max()) or 1.0
    q = ((v - v.min(0)) / span * (2 ** 20 - 1)).astype(np.uint64)

    def spread(x):
        x = x & np.uint64(0x1FFFFF)
        x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
        x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
        x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
        x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
        x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
        return x

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


def bumpy_sphere(s: int, n_harm: int = 8, amp: float = 0.05, seed: int = 0, order: str = "morton"):
    """Icosphere radius r = 1 + amp * sum_i Y_i / max|Y_i|, seeded ell in [2,8], m in [-ell, ell].

    order "morton" (default) numbers the vertices along the Z-order curve of their positions
    (faces remapped), like the coherent orders of real mesh files; "subdivision" keeps the
    icosphere's construction order (midpoints appended per level), in which 128 consecutive
    vertices of s = 8 touch up to 4,611 of 5,000 landmarks."""
    v, f = icosphere(s)
    rng = np.random.default_rng(seed)
    radius = np.ones(len(v))
    for _ in range(n_harm):
        ell = int(rng.integers(2, 9))
        m = int(rng.integers(-ell, ell + 1))
        y = real_sph_harm(ell, m, v)
        radius += amp * y / np.max(np.abs(y))
    v = v * radius[:, None]
    if order == "morton":
        perm = morton_order(v)                   # new index i holds old vertex perm[i]
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))
        v, f = v[perm], inv[f]
    elif order != "subdivision":
        raise ValueError(order)
    return v, f
