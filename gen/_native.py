"""ctypes loader for the input-generator helper ``gen/native/geodesic.cpp``.

Input generation only. Builds in-tree with g++/OpenMP on
first use; ``__graft_entry__.build()`` builds it ahead of time.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "native", "geodesic.cpp")
LIB = os.path.join(_HERE, "lib", "libsbmdsgen.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-O3", "-march=x86-64-v2", "-std=c++17", "-fopenmp", "-shared", "-fPIC",
               SRC, "-o", tmp]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB)
            i64, i32, u64, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
            L.gen_dijkstra_rows.argtypes = [i64, p, p, p, i64, p, i64, p, p]
            L.gen_fps.argtypes = [i64, p, p, p, i64, i32, p, p]
            L.gen_knearest.argtypes = [i64, p, p, p, i64, p, i32, ctypes.c_double, p, p]
            L.gen_knearest.restype = i64
            L.gen_landmark_graph_sqdist.argtypes = [i64, p, p, p, i64, p, ctypes.c_double, p]
            L.gen_random_rows.argtypes = [i64, i64, i32, i32, u64, p, p]
            L.gen_landmark_sqdist.argtypes = [i64, p, p, p, i64, p, p]
            L.gen_random_sym.argtypes = [i64, u64, p]
            L.gen_num_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


class Graph:
    """Undirected weighted graph in symmetric CSR (both directions stored)."""

    def __init__(self, n: int, edges: np.ndarray, weights: np.ndarray):
        e = np.asarray(edges, dtype=np.int64)
        wts = np.asarray(weights, dtype=np.float64)
        src = np.concatenate([e[:, 0], e[:, 1]])
        dst = np.concatenate([e[:, 1], e[:, 0]])
        ww = np.concatenate([wts, wts])
        order = np.lexsort((dst, src))
        src, dst, ww = src[order], dst[order], ww[order]
        self.n = int(n)
        self.ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(self.ptr, src + 1, 1)
        self.ptr = np.cumsum(self.ptr).astype(np.int64)
        self.idx = np.ascontiguousarray(dst.astype(np.int32))
        self.w = np.ascontiguousarray(ww)

    def dijkstra_rows(self, sources, targets=None) -> np.ndarray:
        s = np.ascontiguousarray(np.asarray(sources, dtype=np.int32))
        t = np.arange(self.n, dtype=np.int32) if targets is None else \
            np.ascontiguousarray(np.asarray(targets, dtype=np.int32))
        out = np.empty((len(s), len(t)), dtype=np.float64)
        lib().gen_dijkstra_rows(self.n, _p(self.ptr), _p(self.idx), _p(self.w),
                                len(s), _p(s), len(t), _p(t), _p(out))
        return out

    def fps(self, l: int, first: int):
        lm = np.empty(l, dtype=np.int32)
        md = np.empty(self.n, dtype=np.float64)
        rc = lib().gen_fps(self.n, _p(self.ptr), _p(self.idx), _p(self.w), l, int(first),
                           _p(lm), _p(md))
        if rc != 0:
            raise ValueError("graph is disconnected: farthest point unreachable")
        return lm, md

    def knearest(self, landmarks, k: int, radius: float = float("inf")):
        """Exact k nearest landmarks (label, dist) per vertex, sorted by (dist, label).

        Searches are truncated at ``radius`` and retried with 1.5x the radius until
        every vertex's k-th candidate is strictly inside it (then the answer is exact).
        """
        lm = np.ascontiguousarray(np.asarray(landmarks, dtype=np.int32))
        lab = np.empty((self.n, k), dtype=np.int32)
        dist = np.empty((self.n, k), dtype=np.float64)
        while True:
            bad = lib().gen_knearest(self.n, _p(self.ptr), _p(self.idx), _p(self.w), len(lm),
                                     _p(lm), int(k), float(radius), _p(lab), _p(dist))
            if bad == 0:
                return lab, dist
            if radius == float("inf"):
                raise ValueError("fewer than k landmarks reachable from some vertex")
            radius *= 1.5

    def landmark_graph_sqdist(self, landmarks, radius: float) -> np.ndarray:
        lm = np.ascontiguousarray(np.asarray(landmarks, dtype=np.int32))
        D = np.empty((len(lm), len(lm)), dtype=np.float32)
        rc = lib().gen_landmark_graph_sqdist(self.n, _p(self.ptr), _p(self.idx), _p(self.w),
                                             len(lm), _p(lm), float(radius), _p(D))
        if rc != 0:
            raise ValueError("landmark graph is disconnected; increase radius")
        return D


    def landmark_sqdist(self, landmarks) -> np.ndarray:
        lm = np.ascontiguousarray(np.asarray(landmarks, dtype=np.int32))
        D = np.empty((len(lm), len(lm)), dtype=np.float32)
        rc = lib().gen_landmark_sqdist(self.n, _p(self.ptr), _p(self.idx), _p(self.w), len(lm),
                                       _p(lm), _p(D))
        if rc != 0:
            raise ValueError("graph is disconnected: landmark pair unreachable")
        return D


def random_sym(l: int, seed: int) -> np.ndarray:
    D = np.empty((l, l), dtype=np.float32)
    lib().gen_random_sym(l, seed & (2**64 - 1), _p(D))
    return D


def random_rows(n: int, l: int, k: int, window: int, seed: int):
    col = np.empty(n * k, dtype=np.int32)
    val = np.empty(n * k, dtype=np.float32)
    rc = lib().gen_random_rows(n, l, k, window, seed & (2**64 - 1), _p(col), _p(val))
    if rc != 0:
        raise ValueError("bad random_rows arguments")
    return col, val


def num_threads() -> int:
    return int(lib().gen_num_threads())
