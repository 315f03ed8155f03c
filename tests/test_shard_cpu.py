"""World-size-2 gloo tests (CPU, no GPU) of the sharded apply's partition and reduction plan
(include/sbmds.h "Sharded apply").

Each rank asks the library (host code only) for its tile range of D's upper triangle and
checks its schedule; the ranks then all-gather their tiles (every upper tile exactly once over
the ranks) and run the four stages of the plan on the CPU in fp64 -- rows split by
split_rows, w_g = S_g^T 1 / n_global, tile contributions D_IJ Y1_J and D_IJ^T Y1_I, t_g =
(D w_g)^T Y1 -- with gloo all_reduce(sum) between stages. The gathered result must equal the oracle's
apply: a wrong w split, a missed or doubled tile, or a wrong rank-one term fails it.
"""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L_CASES = (1029, 2003, 300)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(l):
    sys.path.insert(0, ROOT)
    from gen import configs
    return configs.random_problem(4 * l + 17, l, 8, seed=l, window=min(256, l), name="shard_cpu")


def _stages(p, rank, world, tiles, dist, X):
    """The library's four shard stages, written out on the CPU in fp64 (the plan, not the kernels)."""
    import torch
    from paper_1705_10887_b200.sbmds import split_rows
    r0, r1 = split_rows(p.row_ptr, world)[rank]
    rp = np.asarray(p.row_ptr)
    n, l = p.n, p.l
    Sg = np.zeros((r1 - r0, l))
    for i in range(r0, r1):
        for e in range(rp[i], rp[i + 1]):
            Sg[i - r0, p.col_idx[e]] += np.float32(p.val[e])
    Xg = X[r0:r1]
    D = p.D.astype(np.float64)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    s = allreduce(Xg.sum(0))                                   # stage 0
    wg = Sg.sum(0) / n
    Y1 = allreduce(Sg.T @ Xg - np.outer(wg, s))                # stage 1
    Y2g = np.zeros_like(Y1)                                    # stage 2: my tiles only
    for v in tiles:
        I, J = int(v) >> 16, int(v) & 0xFFFF
        ri, rj = slice(128 * I, min(l, 128 * I + 128)), slice(128 * J, min(l, 128 * J + 128))
        Y2g[ri] += D[ri, rj] @ Y1[rj]
        if I < J:
            Y2g[rj] += D[ri, rj].T @ Y1[ri]
    tg = (D @ wg) @ Y1                                         # t_g = (D w_g)^T Y1 (local w_g)
    Y2 = allreduce(Y2g)
    t = allreduce(tg)
    return r0, r1, -0.5 * (Sg @ Y2 - t[None, :])               # stage 3


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1705_10887_b200._lib import lib
    from paper_1705_10887_b200.sbmds import shard_tiles
    dist.init_process_group("gloo")
    out = {}
    try:
        for l in L_CASES:
            # the rank's schedule as the int8 stream (S = 5, gN = 51, contiguous) and the pair stream use it
            errs = [int(lib().sbmds_shard_plan_selfcheck(l, S, gN, ctas, c, rank, 2))
                    for (S, gN, c) in ((5, 51, 1), (8, 32, 1), (8, 1, 0)) for ctas in (1, 74, 148)]
            tiles = shard_tiles(l, 5, rank, 2)
            allt = [torch.zeros(0, dtype=torch.int64) for _ in range(2)]
            cnt = [torch.zeros(1, dtype=torch.int64) for _ in range(2)]
            dist.all_gather(cnt, torch.tensor([len(tiles)], dtype=torch.int64))
            mx = int(max(c.item() for c in cnt))
            pad = torch.full((mx,), -1, dtype=torch.int64)
            pad[:len(tiles)] = torch.from_numpy(tiles.astype(np.int64))
            allt = [torch.zeros(mx, dtype=torch.int64) for _ in range(2)]
            dist.all_gather(allt, pad)
            union = np.concatenate([a.numpy()[a.numpy() >= 0] for a in allt])
            p = _problem(l)
            X = np.random.default_rng(l + 1).standard_normal((p.n, 5))
            r0, r1, Yg = _stages(p, rank, 2, tiles, dist, X)
            out[l] = (errs, union.tolist(), r0, r1, Yg, X)
        q.put((rank, out))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_shard_plan_and_reduction_world2():
    sys.path.insert(0, ROOT)
    from oracle import sbmds_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for l in L_CASES:
        (e0, u0, a0, b0, Y0, X), (e1, u1, a1, b1, Y1, _) = res[0][l], res[1][l]
        assert all(e == 0 for e in e0 + e1), (l, e0, e1)
        NT = (l + 127) // 128
        want = sorted((I << 16) | J for I in range(NT) for J in range(I, NT))
        assert u0 == u1 and sorted(u0) == want                  # every upper tile exactly once
        assert a0 == 0 and b0 == a1 and b1 == 4 * l + 17          # the rows are covered once
        p = _problem(l)
        S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
        ref = O.apply(S, p.D, X)
        got = np.vstack([Y0, Y1])
        assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref), l


def test_shard_tiles_are_contiguous_balanced_ranges():
    """Host plan: the ranks' tile lists concatenate to the world-1 walk order, sizes differ by <= 1."""
    sys.path.insert(0, ROOT)
    from paper_1705_10887_b200.sbmds import shard_tiles
    for l, world in ((50_000, 8), (2003, 3), (129, 4)):
        full = shard_tiles(l, 5, 0, 1)
        parts = [shard_tiles(l, 5, r, world) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)
        sizes = [len(x) for x in parts]
        assert max(sizes) - min(sizes) <= 1


def test_split_rows_balances_entries():
    sys.path.insert(0, ROOT)
    from paper_1705_10887_b200.sbmds import split_rows
    rp = np.concatenate([[0], np.cumsum(np.r_[np.full(500, 1), np.full(500, 9)])])
    parts = split_rows(rp, 4)
    assert parts[0][0] == 0 and parts[-1][1] == 1000
    assert all(parts[i][1] == parts[i + 1][0] for i in range(3))
    loads = [rp[b] - rp[a] for a, b in parts]
    assert max(abs(x - rp[-1] / 4) for x in loads) <= 2 * 9      # within two rows of the ideal
    from paper_1705_10887_b200._lib import lib
    assert lib().sbmds_shard_tiles(100, 5, 2, 2, None, 0) < 0        # rank outside the world
    assert lib().sbmds_shard_plan_selfcheck(100, 5, 51, 4, 1, 0, 0) < 0


def _eigs_worker(rank, port, q):
    """The sharded subspace iteration's reduction plan (sbmds.cu eigs_shard) in fp64 with gloo:
    local rows of the iterate, s / Y1 / Y2 | t / G / H' summed over the ranks, t_g = (D w_g)^T Y1
    R^-1 for the folded iterate X = Y R^-1, Cholesky and Rayleigh-Ritz identical on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from gen import configs
    from paper_1705_10887_b200.sbmds import split_rows
    dist.init_process_group("gloo")
    try:
        p = configs.config(1)
        n, l, b, m = p.n, p.l, p.block, p.m
        r0, r1 = split_rows(p.row_ptr, 2)[rank]
        rp = np.asarray(p.row_ptr)
        Sg = np.zeros((r1 - r0, l))
        for i in range(r0, r1):
            for e in range(rp[i], rp[i + 1]):
                Sg[i - r0, p.col_idx[e]] += np.float32(p.val[e])
        D = p.D.astype(np.float64)
        wg = Sg.sum(0) / n
        vg = D @ wg

        def ar(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        Y = np.random.default_rng(7).standard_normal((n, b))[r0:r1]    # the global start's rows
        G = ar(Y.T @ Y)
        s = ar(Y.sum(0))
        for it in range(60):
            R = np.linalg.cholesky(G).T                                   # G = R^T R
            Ri = np.linalg.inv(R)
            Y1 = ar(Sg.T @ Y - np.outer(wg, s))
            Y2 = D @ (Y1 @ Ri)                                            # (each rank's tiles, summed)
            t = ar((vg @ Y1) @ Ri)
            Yn = -0.5 * (Sg @ Y2 - t[None, :])
            G = ar(Yn.T @ Yn)
            Hp = ar(Y.T @ Yn)
            s = ar(Yn.sum(0))
            Y = Yn
            Yprev_Ri = Ri
        H = Yprev_Ri.T @ Hp                                                # X^T B~ X with X = Y_k R^-1
        theta = np.sort(np.linalg.eigvalsh(0.5 * (H + H.T)))[::-1][:m]
        q.put((rank, theta))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_sharded_eigensolver_plan_world2():
    sys.path.insert(0, ROOT)
    from gen import configs
    from oracle import sbmds_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_eigs_worker, args=(r, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p_ in ps:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    lam_o = O.eigs_dense(S, p.D, p.m)[0]
    assert np.array_equal(res[0], res[1])                                 # both ranks, the same problem
    assert np.all(np.abs(res[0] - lam_o) <= 1e-8 * np.abs(lam_o)), (res[0], lam_o)
