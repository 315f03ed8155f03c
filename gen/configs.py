"""Seeded synthetic workloads shaped like BASELINE.json ``configs`` (input generation only).

Nothing here computes any part of the sBMDS method; it only builds the inputs
S (n x l CSR) and D_ll (l x l squared landmark distances) that both the CUDA
path and the oracle consume, plus the X blocks the parity tests feed in.

Recipe (BASELINE.json configs 1-4 + SURVEY.md §8(c) reading 10):
  mesh      torus grid with +-0.1 cell jitter, or icosphere + 8 seeded harmonics
  graph     mesh edges weighted by Euclidean length
  landmarks farthest-point sampling, first = seeded random vertex
  D_ll      squared Dijkstra distances between landmarks, exactly symmetric
  sigma     mean over landmarks of the distance to the nearest other landmark
  S         landmark rows e_j (1 nnz); other rows: k nearest landmarks by graph
            distance, weights exp(-d^2/sigma^2) normalised to sum 1, columns sorted
Config 5: random clustered rows (window 256) and D = (U + U^T)/2, U ~ U[0,100].
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
from typing import Optional

import numpy as np

from . import _native
from .mesh import bumpy_sphere, mesh_edges, torus_grid


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    l: int
    row_ptr: np.ndarray      # int64 (n+1)
    col_idx: np.ndarray      # int32 (nnz)
    val: np.ndarray          # float64 for mesh configs (rounded to f32 at the ABI), float32 for cfg 5
    D: np.ndarray            # float32 (l, l) row-major, symmetric
    m: int = 3
    block: int = 8
    iters: Optional[int] = None
    landmarks: Optional[np.ndarray] = None
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def val32(self) -> np.ndarray:
        return np.ascontiguousarray(self.val.astype(np.float32))


def _cache_dir() -> Optional[str]:
    d = os.environ.get("SBMDS_GEN_CACHE", os.path.expanduser("~/.cache/sbmds_gen"))
    if d in ("", "0", "off"):
        return None
    try:
        os.makedirs(d, exist_ok=True)
        return d
    except OSError:
        return None


def _cached(key: str, builder):
    d = _cache_dir()
    tag = hashlib.sha1(key.encode()).hexdigest()[:16]
    path = os.path.join(d, tag) if d else None
    names = ("row_ptr", "col_idx", "val", "D", "landmarks")
    if path and os.path.exists(os.path.join(path, "done")):
        arrs = {k: np.load(os.path.join(path, k + ".npy")) for k in names}
        meta = dict(np.load(os.path.join(path, "meta.npy"), allow_pickle=True).item())
        return arrs, meta
    arrs, meta = builder()
    if path:
        try:
            os.makedirs(path, exist_ok=True)
            for k in names:
                np.save(os.path.join(path, k + ".npy"), arrs[k])
            np.save(os.path.join(path, "meta.npy"), np.array(meta, dtype=object))
            open(os.path.join(path, "done"), "w").close()
        except OSError:
            pass
    return arrs, meta


def mesh_problem(verts: np.ndarray, edges: np.ndarray, l: int, k: int, seed: int,
                 d_mode: str = "exact"):
    """Landmarks, D_ll and S for a mesh (graph of its edges, Euclidean lengths).

    d_mode "exact": D_ll = squared mesh-graph Dijkstra distances (configs 1-3).
    d_mode "landmark_graph": config-4 stand-in, squared shortest paths on the graph
    joining landmarks within 3x the FPS covering radius.
    """
    n = len(verts)
    w = np.linalg.norm(verts[edges[:, 0]] - verts[edges[:, 1]], axis=1)
    g = _native.Graph(n, edges, w)
    first = int(np.random.default_rng(seed + 7919).integers(n))
    landmarks, min_dist = g.fps(l, first)
    cover = float(min_dist.max()) if l < n else float(w.min())
    if d_mode == "exact":
        D = g.landmark_sqdist(landmarks)
    elif d_mode == "landmark_graph":
        D = g.landmark_graph_sqdist(landmarks, 3.0 * cover)
    else:
        raise ValueError(d_mode)
    W = np.sqrt(D.astype(np.float64))
    np.fill_diagonal(W, np.inf)
    sigma = float(np.mean(W.min(axis=1))) if l > 1 else 1.0
    del W
    kk = min(k, l)
    radius = float("inf") if l <= 200 else (1.5 * np.sqrt(0.276 * kk) + 1.0) * sigma
    lab, dist = g.knearest(landmarks, kk, radius)
    wts = np.exp(-(dist ** 2 - dist[:, :1] ** 2) / sigma ** 2)
    wts /= wts.sum(axis=1, keepdims=True)
    order = np.argsort(lab, axis=1, kind="stable")
    lab = np.take_along_axis(lab, order, 1)
    wts = np.take_along_axis(wts, order, 1)
    is_lm = np.zeros(n, dtype=bool)
    is_lm[landmarks] = True
    cnt = np.where(is_lm, 1, kk).astype(np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(cnt)
    col_idx = np.empty(row_ptr[-1], dtype=np.int32)
    val = np.empty(row_ptr[-1], dtype=np.float64)
    nl = ~is_lm
    pos = row_ptr[:-1][nl][:, None] + np.arange(kk)[None, :]
    col_idx[pos] = lab[nl]
    val[pos] = wts[nl]
    lm_pos = row_ptr[:-1][landmarks]
    col_idx[lm_pos] = np.arange(l, dtype=np.int32)
    val[lm_pos] = 1.0
    meta = {"sigma": sigma, "first": first, "d_mode": d_mode, "cover": cover}
    return {"row_ptr": row_ptr, "col_idx": col_idx, "val": val, "D": D,
            "landmarks": landmarks.astype(np.int32)}, meta


def torus_problem(nu: int, nv: int, l: int, k: int, seed: int = 0, name: str = "torus",
                  d_mode: str = "exact"):
    def build():
        verts, _, edges = torus_grid(nu, nv, seed=seed)
        return mesh_problem(verts, edges, l, k, seed, d_mode)
    arrs, meta = _cached(f"torus/{nu}/{nv}/{l}/{k}/{seed}/{d_mode}/v1", build)
    meta.update(mesh=f"torus {nu}x{nv}", nu=nu, nv=nv, seed=seed)
    return Problem(name, nu * nv, l, arrs["row_ptr"], arrs["col_idx"], arrs["val"], arrs["D"],
                   landmarks=arrs["landmarks"], meta=meta)


def sphere_problem(s: int, l: int, k: int, seed: int = 0, name: str = "bumpy_sphere"):
    def build():
        verts, faces = bumpy_sphere(s, seed=seed)
        return mesh_problem(verts, mesh_edges(faces), l, k, seed)
    arrs, meta = _cached(f"sphere/{s}/{l}/{k}/{seed}/v2-morton", build)
    meta.update(mesh=f"bumpy icosphere s={s} (vertices in Morton order)", s=s, seed=seed)
    return Problem(name, 10 * 4 ** s + 2, l, arrs["row_ptr"], arrs["col_idx"], arrs["val"],
                   arrs["D"], landmarks=arrs["landmarks"], meta=meta)


def random_problem(n: int, l: int, k: int, seed: int = 0, window: int = 256,
                   name: str = "random"):
    def build():
        col, val = _native.random_rows(n, l, k, min(window, l), seed)
        row_ptr = np.arange(n + 1, dtype=np.int64) * k
        D = _native.random_sym(l, seed)
        return {"row_ptr": row_ptr, "col_idx": col, "val": val, "D": D,
                "landmarks": np.zeros(0, dtype=np.int32)}, {}
    arrs, meta = _cached(f"random/{n}/{l}/{k}/{seed}/{window}/v1", build)
    meta.update(window=window, seed=seed)
    return Problem(name, n, l, arrs["row_ptr"], arrs["col_idx"], arrs["val"], arrs["D"],
                   meta=meta)


def config(i: int, seed: int = 0, k5: int = 16) -> Problem:
    """BASELINE.json configs[i-1] (1-based, as SURVEY.md numbers them)."""
    if i == 1:
        p = torus_problem(40, 50, 100, 8, seed, name="cfg1_torus40x50")
        p.m, p.block = 3, 8
    elif i == 2:
        p = torus_problem(250, 400, 1000, 16, seed, name="cfg2_torus250x400")
        p.m, p.block = 3, 16
    elif i == 3:
        p = sphere_problem(8, 5000, 32, seed, name="cfg3_bumpy_sphere_s8")
        p.m, p.block = 8, 32
    elif i == 4:
        p = torus_problem(1200, 1500, 50000, 32, seed, name="cfg4_torus1200x1500",
                          d_mode="landmark_graph")
        p.m, p.block, p.iters = 3, 16, 50
    elif i == 5:
        p = random_problem(4_000_000, 20_000, k5, seed, name=f"cfg5_random_k{k5}")
        p.m, p.block = 0, 0
    else:
        raise ValueError(f"no config {i}")
    return p


def x_block(n: int, b: int, seed: int = 0, dtype=np.float32) -> np.ndarray:
    """X ~ N(0,1), n x b row-major (BASELINE.json config 5)."""
    rng = np.random.default_rng(seed + 104729)
    return rng.standard_normal((n, b), dtype=np.float32 if dtype == np.float32 else np.float64)
