"""GPU: the sharded apply (include/sbmds.h "Sharded apply") against the oracle.

One GPU only (gpurun), so the ranks of a world > 1 are emulated the only safe way: shard handles
of every rank live in one process and the test drives them stage by stage, one after another,
summing the exchange buffers itself between stages (no kernel ever waits on another rank).
The in-library NCCL path (sbmds_apply after sbmds_shard_attach_nccl) runs at world 1.
"""
import numpy as np
import pytest

from gen import configs
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_apply(p, X):
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    return O.apply(S, p.D, X.astype(np.float64))


def staged_apply(p, world, X, **opts):
    """All ranks' four stages on one GPU, sums by the test (what NCCL allreduce does)."""
    import torch
    from paper_1705_10887_b200.sbmds import shard_from_problem, split_rows
    hs = [shard_from_problem(p, r, world) for r in range(world)]
    for h in hs:
        for k, v in opts.items():
            h.set_option(k, v)
    rows = split_rows(p.row_ptr, world)
    b, l = X.shape[1], p.l
    Xs = [torch.from_numpy(np.ascontiguousarray(X[a:c])).cuda() for a, c in rows]
    buf = lambda st: torch.empty(hs[0].exchange_bytes(b, st), dtype=torch.uint8, device="cuda")  # noqa: E731
    toff = hs[0].exchange_bytes(b, 2) - 8 * b
    # stage 0: s = sum_g 1^T X_g
    outs = [buf(0) for _ in hs]
    for h, Xg, o in zip(hs, Xs, outs):
        h.stage(0, b, X=Xg, exch_out=o)
    s = sum(o.view(torch.float64) for o in outs).contiguous().view(torch.uint8)
    # stage 1: Y1 = sum_g (S_g^T X_g - w_g s^T)
    outs = [buf(1) for _ in hs]
    for h, Xg, o in zip(hs, Xs, outs):
        h.stage(1, b, X=Xg, exch_in=s, exch_out=o)
    Y1 = sum(o.view(torch.float32) for o in outs).contiguous().view(torch.uint8)
    # stage 2: Y2 | t = sum_g (tiles of rank g)
    outs = [buf(2) for _ in hs]
    for h, o in zip(hs, outs):
        h.stage(2, b, exch_in=Y1, exch_out=o)
    y2t = torch.zeros_like(outs[0])
    y2t[:4 * l * b].view(torch.float32)[:] = sum(o[:4 * l * b].view(torch.float32) for o in outs)
    y2t[toff:].view(torch.float64)[:] = sum(o[toff:].view(torch.float64) for o in outs)
    # stage 3: local rows
    Ys = []
    for h, Xg in zip(hs, Xs):
        Y = torch.empty_like(Xg)
        h.stage(3, b, exch_in=y2t, Y=Y)
        Ys.append(Y)
    torch.cuda.synchronize()
    paths = [h.stat("dstream_path") for h in hs]
    for h in hs:
        h.close()
    return np.vstack([Y.cpu().numpy() for Y in Ys]), paths


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("b", [16, 8, 32, 4])
def test_staged_shards_match_oracle(world, b):
    """l = 5000 (40 row tiles, 820 upper tiles): every width streams each rank's tile range on the
    int8 symmetric-half kernel (b = 4 at width 8, Y1 widened and Y2 narrowed around it); with
    dstream = 1 (FFMA, not tiled by rank) rank 0 streams all of D and the others add zeros."""
    p = configs.random_problem(40_000, 5_000, 16, seed=b + world, name="shard")
    X = configs.x_block(p.n, b, seed=b)
    Y, paths = staged_apply(p, world, X)
    assert paths == [3] * world
    assert relerr(Y, oracle_apply(p, X)) <= TOL
    if b == 4:
        Yf, pf = staged_apply(p, world, X, dstream=1)
        assert pf[0] == 1 and relerr(Yf, oracle_apply(p, X)) <= TOL
    assert relerr(Y, oracle_apply(p, X)) <= TOL


def test_staged_shards_ragged_config2():
    """Config 2 (mesh S, l = 1000: the full-D 3xTF32 stream on rank 0) split over 2 ranks."""
    p = configs.config(2)
    X = configs.x_block(p.n, 16, seed=3)
    Y, _ = staged_apply(p, 2, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


def test_nccl_world1_apply():
    """The in-library NCCL path: a world-1 communicator attached, sbmds_apply runs the four stages
    with ncclAllReduce in between; the result meets the oracle bar and equals the staged path."""
    import torch
    from paper_1705_10887_b200 import SbmdsError
    from paper_1705_10887_b200.sbmds import nccl_unique_id, shard_from_problem
    p = configs.random_problem(40_000, 5_000, 16, seed=31, name="shard_nccl")
    X = configs.x_block(p.n, 16, seed=2)
    with shard_from_problem(p, 0, 1) as h:
        h.attach_nccl(nccl_unique_id())
        Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
        assert h.stat("dstream_path") == 3
    Ys, _ = staged_apply(p, 1, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL
    assert np.array_equal(Y, Ys)


def test_shard_apply_needs_a_communicator():
    import torch
    from paper_1705_10887_b200 import SbmdsError
    from paper_1705_10887_b200.sbmds import shard_from_problem
    p = configs.random_problem(20_000, 1_000, 8, seed=4, name="shard_err")
    with shard_from_problem(p, 1, 2) as h:
        with pytest.raises(SbmdsError, match="EINVAL"):
            h.apply(torch.zeros((h.n, 4), device="cuda"))
        with pytest.raises(SbmdsError, match="EINVAL"):
            h.eigs(3, 8)


def _manual_shards(p, cuts, device="cuda"):
    """Shard handles over arbitrary contiguous row ranges (not split_rows' balance)."""
    import torch
    from paper_1705_10887_b200.sbmds import SbmdsShard
    rp = np.asarray(p.row_ptr, dtype=np.int64)
    hs = []
    W = len(cuts) - 1
    for g in range(W):
        r0, r1 = cuts[g], cuts[g + 1]
        lo, hi = int(rp[r0]), int(rp[r1])
        arrs = [np.ascontiguousarray(rp[r0:r1 + 1] - lo), np.ascontiguousarray(np.asarray(p.col_idx)[lo:hi], np.int32),
                np.ascontiguousarray(np.asarray(p.val)[lo:hi], np.float32), np.ascontiguousarray(p.D, np.float32)]
        if device != "numpy":
            arrs = [torch.from_numpy(a).cuda() for a in arrs]
        hs.append(SbmdsShard(p.n, r0, r1 - r0, p.l, *arrs, g, W))
    return hs


@pytest.mark.parametrize("cuts_frac,b,device", [((0, 0.07, 0.5, 0.93, 1.0), 5, "cuda"),
                                                ((0, 0.3, 1.0), 16, "numpy")])
def test_uneven_partitions_and_host_inputs(cuts_frac, b, device):
    """Arbitrary row ranges (7% / 43% / 43% / 7%) with b = 5 (bp = 8 padding), and host inputs (a
    host D crosses as its upper strips and each rank packs only its own tiles) over 2 ranks."""
    import torch
    p = configs.random_problem(40_000, 5_000, 16, seed=17, name="shard_uneven")
    cuts = [int(round(f * p.n)) for f in cuts_frac]
    hs = _manual_shards(p, cuts, device)
    X = configs.x_block(p.n, b, seed=4)
    W, l = len(hs), p.l
    Xs = [torch.from_numpy(np.ascontiguousarray(X[cuts[g]:cuts[g + 1]])).cuda() for g in range(W)]
    buf = lambda st: torch.empty(hs[0].exchange_bytes(b, st), dtype=torch.uint8, device="cuda")  # noqa: E731
    toff = hs[0].exchange_bytes(b, 2) - 8 * b
    outs = [buf(0) for _ in hs]
    for h, Xg, o in zip(hs, Xs, outs):
        h.stage(0, b, X=Xg, exch_out=o)
    s = sum(o.view(torch.float64) for o in outs).contiguous().view(torch.uint8)
    outs = [buf(1) for _ in hs]
    for h, Xg, o in zip(hs, Xs, outs):
        h.stage(1, b, X=Xg, exch_in=s, exch_out=o)
    Y1 = sum(o.view(torch.float32) for o in outs).contiguous().view(torch.uint8)
    outs = [buf(2) for _ in hs]
    for h, o in zip(hs, outs):
        h.stage(2, b, exch_in=Y1, exch_out=o)
    y2t = torch.zeros_like(outs[0])
    y2t[:4 * l * b].view(torch.float32)[:] = sum(o[:4 * l * b].view(torch.float32) for o in outs)
    y2t[toff:].view(torch.float64)[:] = sum(o[toff:].view(torch.float64) for o in outs)
    Ys = []
    for h, Xg in zip(hs, Xs):
        Y = torch.empty_like(Xg)
        h.stage(3, b, exch_in=y2t, Y=Y)
        Ys.append(Y)
    torch.cuda.synchronize()
    paths = [h.stat("dstream_path") for h in hs]
    for h in hs:
        h.close()
    got = np.vstack([Y.cpu().numpy() for Y in Ys])
    assert paths == [3] * W
    assert relerr(got, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("cfg,nccl", [(1, False), (2, True), (2, False)])
def test_sharded_eigensolver_world1(cfg, nccl):
    """The sharded subspace iteration (local rows, allreduced Grams, the global sign rule) on a
    world-1 shard -- with the NCCL communicator attached (every allreduce issued) or without --
    against the oracle's eigenpairs; a warm start and the Philox start both."""
    import torch
    from paper_1705_10887_b200.sbmds import nccl_unique_id, shard_from_problem
    p = configs.config(cfg)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o, V_o = (O.eigs_dense(S, p.D, p.m)[:2] if cfg == 1 else O.eigs_matfree(S, p.D, p.m)[:2])
    with shard_from_problem(p, 0, 1) as h:
        if nccl:
            h.attach_nccl(nccl_unique_id())
        lam, V, Z, info = h.eigs(p.m, p.block, max_iters=500, tol=1e-6)
        X0 = torch.from_numpy(configs.x_block(p.n, p.block, seed=2)).cuda()
        lam2, _, _, info2 = h.eigs(p.m, p.block, max_iters=500, tol=1e-6, X0=X0)
    V = V.cpu().numpy().astype(np.float64)
    Z = Z.cpu().numpy().astype(np.float64)
    assert info["converged"] == 1 and info2["converged"] == 1
    for l_ in (lam, lam2):
        assert np.all(np.abs(l_ - lam_o) <= 1e-4 * np.abs(lam_o)), (l_, lam_o)
    assert O.principal_angle(V, V_o) <= 1e-3
    assert np.abs(V.T @ V - np.eye(p.m)).max() < 1e-5
    for j in range(p.m):
        assert V[np.argmax(np.abs(V[:, j])), j] > 0
    assert np.allclose(Z, V * np.sqrt(np.maximum(lam, 0))[None, :], rtol=1e-5, atol=1e-7)
