"""Python binding of libsbmds (include/sbmds.h): argument marshalling only.

Every step of the operator and of the eigensolver runs in the CUDA library; this
module turns torch tensors / numpy arrays into pointers and a stream handle.
torch CUDA tensors are passed as device pointers (asynchronous on the current
stream); numpy arrays and CPU tensors are passed as host pointers (the library
stages them and synchronises).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from ._lib import (NCCL_UNIQUE_ID_BYTES, SBMDS_BORROW_D, SBMDS_ENOCONV, SBMDS_REORDER_ROWS, SBMDS_VALIDATE,
                   SbmdsError, SbmdsInfo, check, lib)

try:
    import torch
except Exception:  # pragma: no cover - torch is in the image
    torch = None


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _ptr(x, dtype) -> int:
    """Pointer to a contiguous buffer of `dtype` (torch tensor or numpy array)."""
    if _is_torch(x):
        want = {np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        if x.dtype != want or not x.is_contiguous():
            raise TypeError(f"expected a contiguous {want} tensor, got {x.dtype}")
        return x.data_ptr()
    if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags.c_contiguous:
        raise TypeError(f"expected a C-contiguous numpy {np.dtype(dtype)} array")
    return x.ctypes.data


def _stream(stream) -> int:
    if stream is not None:
        return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)
    if torch is not None and torch.cuda.is_available():
        return int(torch.cuda.current_stream().cuda_stream)
    return 0


def launch_count() -> int:
    """Kernels libsbmds has launched in this process (bench.py's gpu_launches)."""
    return int(lib().sbmds_launch_count())


class Sbmds:
    """Handle over S (n x l CSR) and D_ll (l x l, symmetric squared landmark distances).

    Mirrors sbmds_create / sbmds_apply / sbmds_eigs / sbmds_destroy.
    """

    def __init__(self, n: int, l: int, row_ptr, col_idx, val, D, *, validate: bool = False,
                 borrow_d: bool = False, reorder_rows: bool = False, stream=None):
        self.n, self.l = int(n), int(l)
        nnz = int(row_ptr[-1])
        flags = ((SBMDS_VALIDATE if validate else 0) | (SBMDS_BORROW_D if borrow_d else 0) |
                 (SBMDS_REORDER_ROWS if reorder_rows else 0))
        self._keep = (row_ptr, col_idx, val, D) if borrow_d else ()
        h = ctypes.c_void_p()
        check(lib().sbmds_create(self.n, self.l, nnz, _ptr(row_ptr, np.int64),
                                 _ptr(col_idx, np.int32), _ptr(val, np.float32), _ptr(D, np.float32),
                                 flags, _stream(stream), ctypes.byref(h)))
        self._h = h

    # -- lifecycle ---------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().sbmds_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls -------------------------------------------------------------------------
    def apply(self, X, out=None, stream=None):
        """Y = -1/2 J S D S^T J X for an n x b block (b <= 64)."""
        if X.ndim != 2 or X.shape[0] != self.n:
            raise ValueError(f"X must be n x b with n={self.n}")
        b = int(X.shape[1])
        if out is None:
            out = torch.empty_like(X) if _is_torch(X) else np.empty_like(X)
        check(lib().sbmds_apply(self._h, b, _ptr(X, np.float32), _ptr(out, np.float32),
                                _stream(stream)))
        return out

    def eigs(self, m: int, block: int, max_iters: int = 500, tol: float = 1e-5, seed: int = 0,
             X0=None, V=None, Z=None, device: str = "cuda", stream=None, raise_noconv=False):
        """Top-m eigenpairs of B~ and Z = V_m Λ_m^{1/2}. Returns (eigvals, V, Z, info)."""
        if V is None:
            V = (torch.empty((self.n, m), dtype=torch.float32, device=device)
                 if device != "numpy" else np.empty((self.n, m), dtype=np.float32))
        if Z is None:
            Z = (torch.empty((self.n, m), dtype=torch.float32, device=device)
                 if device != "numpy" else np.empty((self.n, m), dtype=np.float32))
        ev = np.zeros(m, dtype=np.float64)
        info = SbmdsInfo()
        x0 = _ptr(X0, np.float32) if X0 is not None else None
        st = lib().sbmds_eigs(self._h, int(m), int(block), int(max_iters), float(tol), int(seed),
                              x0, ev.ctypes.data, _ptr(V, np.float32), _ptr(Z, np.float32),
                              ctypes.byref(info), _stream(stream))
        if st == SBMDS_ENOCONV and not raise_noconv:
            pass
        else:
            check(st)
        d = {k: getattr(info, k) for k, _ in SbmdsInfo._fields_}
        d["status"] = int(st)
        return ev, V, Z, d

    def bmds(self, m: int, block: int, max_iters: int = 2000, tol: float = 1e-8, seed: int = 0, stream=None,
             raise_noconv=False):
        """BMDS (sbmds_bmds): (eigvals, V, Z, info) on the device."""
        V = torch.empty((self.n, m), dtype=torch.float32, device="cuda")
        Z = torch.empty((self.n, m), dtype=torch.float32, device="cuda")
        ev = np.zeros(m, dtype=np.float64)
        info = SbmdsInfo()
        st = lib().sbmds_bmds(self._h, int(m), int(block), int(max_iters), float(tol), int(seed), ev.ctypes.data,
                              V.data_ptr(), Z.data_ptr(), ctypes.byref(info), _stream(stream))
        if not (st == SBMDS_ENOCONV and not raise_noconv):
            check(st)
        d = {k: getattr(info, k) for k, _ in SbmdsInfo._fields_}
        d["status"] = int(st)
        return ev, V, Z, d

    def set_option(self, key: str, value: int):
        check(lib().sbmds_set_option(self._h, key.encode(), int(value)))

    def stat(self, key: str) -> int:
        v = ctypes.c_int64()
        check(lib().sbmds_get_stat(self._h, key.encode(), ctypes.byref(v)))
        return int(v.value)


class SbmdsShard(Sbmds):
    """Shard handle: rows [row0, row0 + n_local) of an n_global-row S, tile range
    `rank` of `world` of D's upper triangle (sbmds_create_shard). apply() needs a communicator
    (attach_nccl) when world > 1; stage() drives one stage with caller-owned exchange buffers."""

    def __init__(self, n_global: int, row0: int, n_local: int, l: int, row_ptr, col_idx, val, D, rank: int,
                 world: int, *, validate: bool = False, stream=None):
        self.n, self.l = int(n_local), int(l)
        self.n_global, self.row0, self.rank, self.world = int(n_global), int(row0), int(rank), int(world)
        nnz = int(row_ptr[-1])
        flags = SBMDS_VALIDATE if validate else 0
        self._keep = ()
        h = ctypes.c_void_p()
        check(lib().sbmds_create_shard(self.n_global, self.row0, self.n, self.l, nnz, _ptr(row_ptr, np.int64),
                                       _ptr(col_idx, np.int32), _ptr(val, np.float32), _ptr(D, np.float32),
                                       self.rank, self.world, flags, _stream(stream), ctypes.byref(h)))
        self._h = h

    def attach_nccl(self, unique_id: bytes):
        buf = ctypes.create_string_buffer(bytes(unique_id), NCCL_UNIQUE_ID_BYTES)
        check(lib().sbmds_shard_attach_nccl(self._h, buf))

    def exchange_bytes(self, b: int, stage: int) -> int:
        return int(lib().sbmds_shard_exchange_bytes(self.l, int(b), int(stage)))

    def stage(self, stage: int, b: int, X=None, exch_in=None, exch_out=None, Y=None, stream=None):
        """One stage of the sharded apply on device tensors (exchange buffers: uint8 tensors of
        exchange_bytes(b, stage) bytes; the caller sums stage k's out over ranks into stage k+1's in)."""
        ptr = lambda t: None if t is None else t.data_ptr()   # noqa: E731
        check(lib().sbmds_shard_stage(self._h, int(stage), int(b), ptr(X), ptr(exch_in), ptr(exch_out), ptr(Y),
                                      _stream(stream)))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 creates it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    check(lib().sbmds_nccl_unique_id(buf))
    return buf.raw


def sbha_build(verts, faces, landmarks, p_row: float, device: str = "cuda", stream=None):
    """S = P_sparse of a triangle mesh (sbmds_sbha_build): (row_ptr int64, col_idx int32, val f32, info).
    verts (n x 3 float64) and faces (nf x 3 int32) as numpy arrays or device tensors."""
    from ._lib import SbhaInfo
    V = np.ascontiguousarray(verts, dtype=np.float64) if not _is_torch(verts) else verts
    F = np.ascontiguousarray(faces, dtype=np.int32) if not _is_torch(faces) else faces
    lm = np.ascontiguousarray(landmarks, dtype=np.int32)
    n, nf, l = int(V.shape[0]), int(F.shape[0]), int(lm.shape[0])
    p = int(lib().sbmds_sbha_p(n, l, float(p_row)))
    if p < 1:
        raise ValueError("need 1 <= l < n and p_row > 0")
    nnz = l + l * p
    if device == "numpy":
        rp, ci, vv = np.empty(n + 1, np.int64), np.empty(nnz, np.int32), np.empty(nnz, np.float32)
        ptrs = (rp.ctypes.data, ci.ctypes.data, vv.ctypes.data)
    else:
        rp = torch.empty(n + 1, dtype=torch.int64, device=device)
        ci = torch.empty(nnz, dtype=torch.int32, device=device)
        vv = torch.empty(nnz, dtype=torch.float32, device=device)
        ptrs = (rp.data_ptr(), ci.data_ptr(), vv.data_ptr())
    vp = V.data_ptr() if _is_torch(V) else V.ctypes.data
    fp = F.data_ptr() if _is_torch(F) else F.ctypes.data
    info = SbhaInfo()
    check(lib().sbmds_sbha_build(n, vp, nf, fp, l, lm.ctypes.data, float(p_row), *ptrs, ctypes.byref(info),
                                 _stream(stream)))
    return rp, ci, vv, {k: getattr(info, k) for k, _ in SbhaInfo._fields_}


def split_rows(row_ptr, world: int):
    """Contiguous row ranges [r0, r1) per rank with balanced stored entries (host logic)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n, nnz = len(rp) - 1, int(rp[-1])
    cuts = [0]
    for g in range(1, world):
        r = int(np.searchsorted(rp, nnz * g / world, side="left"))
        cuts.append(min(max(r, cuts[-1] + 1), n - (world - g)))
    cuts.append(n)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def shard_tiles(l: int, S: int, rank: int, world: int) -> np.ndarray:
    """The upper 128 x 128 tiles (I << 16 | J) rank `rank` streams (sbmds_shard_tiles)."""
    cnt = int(lib().sbmds_shard_tiles(int(l), int(S), int(rank), int(world), None, 0))
    if cnt < 0:
        raise ValueError("bad shard plan arguments")
    out = np.empty(cnt, dtype=np.uint32)
    lib().sbmds_shard_tiles(int(l), int(S), int(rank), int(world), out.ctypes.data, cnt)
    return out


def shard_from_problem(p, rank: int, world: int, device: Optional[str] = "cuda", **kw) -> SbmdsShard:
    """Build rank `rank`'s shard of a gen.configs.Problem (rows split by split_rows)."""
    r0, r1 = split_rows(p.row_ptr, world)[rank]
    rp = np.asarray(p.row_ptr, dtype=np.int64)
    lo, hi = int(rp[r0]), int(rp[r1])
    rpl = np.ascontiguousarray(rp[r0:r1 + 1] - lo)
    ci = np.ascontiguousarray(np.asarray(p.col_idx)[lo:hi], dtype=np.int32)
    vv = np.ascontiguousarray(np.asarray(p.val)[lo:hi], dtype=np.float32)
    D = np.ascontiguousarray(p.D, dtype=np.float32)
    if device and device != "numpy":
        rpl, ci, vv, D = (torch.from_numpy(a).to(device) for a in (rpl, ci, vv, D))
    return SbmdsShard(p.n, r0, r1 - r0, p.l, rpl, ci, vv, D, rank, world, **kw)


def from_problem(p, device: Optional[str] = "cuda", **kw) -> Sbmds:
    """Convenience: build a handle from a gen.configs.Problem (host or device upload)."""
    rp = np.ascontiguousarray(p.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(p.col_idx, dtype=np.int32)
    vv = np.ascontiguousarray(p.val, dtype=np.float32)
    D = np.ascontiguousarray(p.D, dtype=np.float32)
    if device and device != "numpy":
        rp, ci, vv, D = (torch.from_numpy(a).to(device) for a in (rp, ci, vv, D))
    return Sbmds(p.n, p.l, rp, ci, vv, D, **kw)


__all__ = ["Sbmds", "SbmdsShard", "SbmdsError", "from_problem", "shard_from_problem", "launch_count",
           "nccl_unique_id", "split_rows", "shard_tiles", "sbha_build"]
