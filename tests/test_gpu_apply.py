"""GPU parity: sbmds_apply (CUDA, through the C ABI) vs the fp64 oracle, element by element.

Tolerance (BASELINE.json north_star): relative Frobenius error <= 1e-5 in fp32.
Inputs are the seeded generators of gen/ (configs 1, 2, shrunken 3/5 shapes) plus
edge cases: ragged l, empty columns, negative / non-normalised S, duplicates, b in 1..64.
"""
import numpy as np
import pytest

from gen import configs
from oracle import sbmds_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _torch():
    import torch
    return torch


def make_handle(p, **kw):
    from paper_1705_10887_b200 import from_problem
    return from_problem(p, **kw)


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_apply(h, X):
    torch = _torch()
    Xt = torch.from_numpy(X).cuda()
    Y = h.apply(Xt)
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def oracle_apply(p, X):
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())  # the fp32 values the ABI receives
    return O.apply(S, p.D, X.astype(np.float64))


def synth_problem(n, l, k, seed, negative=False, rowsum_one=True, empty_cols=0, dup=False):
    """Random CSR S (variable row lengths 1..k), symmetric D; not a paper workload — edge cases."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, k + 1, size=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(lens)
    usable = l - empty_cols
    cols = np.concatenate([np.sort(rng.choice(usable, size=c, replace=dup)) for c in lens]).astype(np.int32)
    vals = rng.uniform(0.05, 1.0, size=row_ptr[-1])
    if negative:
        vals *= np.where(rng.random(row_ptr[-1]) < 0.3, -1.0, 1.0)
    if rowsum_one:
        sums = np.add.reduceat(vals, row_ptr[:-1])
        vals = vals / np.repeat(sums, lens)
    A = rng.uniform(0, 100, size=(l, l)).astype(np.float32)
    D = np.ascontiguousarray((A + A.T) / 2)
    p = configs.Problem("synth", n, l, row_ptr, cols, vals, D)
    return p


@pytest.mark.parametrize("b", [8, 1, 3, 16, 64])
def test_apply_config1(b):
    p = configs.config(1)
    X = configs.x_block(p.n, b, seed=b)
    with make_handle(p) as h:
        Y = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("b", [16, 4, 1, 5])
def test_apply_config2(b):
    p = configs.config(2)
    X = configs.x_block(p.n, b, seed=b)
    with make_handle(p) as h:
        Y = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("k,b", [(8, 1), (16, 4), (16, 16), (64, 64), (8, 32), (16, 2)])
def test_apply_random_structure(k, b):
    """Config-5 recipe at a size the oracle finishes in seconds (several tiles + ragged tail)."""
    p = configs.random_problem(60_001, 2_003, k, seed=k + b, name="cfg5_small")
    X = configs.x_block(p.n, b, seed=7)
    with make_handle(p) as h:
        Y = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("case", ["negative", "not_normalised", "empty_cols", "duplicates", "l_ragged"])
def test_apply_edge_cases(case):
    kw = dict(n=5000, l=333, k=12, seed=11)
    if case == "negative":
        p = synth_problem(**kw, negative=True)
    elif case == "not_normalised":
        p = synth_problem(**kw, rowsum_one=False)
    elif case == "empty_cols":
        p = synth_problem(**kw, empty_cols=40)
    elif case == "duplicates":
        p = synth_problem(**kw, dup=True)
    else:
        p = synth_problem(n=3001, l=1029, k=9, seed=3)
    for b in (1, 4, 7, 16):
        X = configs.x_block(p.n, b, seed=b)
        with make_handle(p) as h:
            Y = run_apply(h, X)
        assert relerr(Y, oracle_apply(p, X)) <= TOL, (case, b)


def test_apply_invariants_and_determinism():
    """Columns of B~X sum to 0; X1^T(B~X2) = (B~X1)^T X2 (CSR vs CSC); B~1 = 0; bitwise repeatable."""
    p = configs.config(2)
    X1 = configs.x_block(p.n, 16, seed=1)
    X2 = configs.x_block(p.n, 16, seed=2)
    with make_handle(p) as h:
        Y1 = run_apply(h, X1)
        Y2 = run_apply(h, X2)
        Y1b = run_apply(h, X1)
        ones = np.ones((p.n, 4), dtype=np.float32)
        Y0 = run_apply(h, ones)
    scale = np.abs(Y1).max()
    assert np.abs(Y1.astype(np.float64).sum(0)).max() <= 1e-5 * scale * np.sqrt(p.n)
    a = X1.astype(np.float64).T @ Y2.astype(np.float64)
    bm = Y1.astype(np.float64).T @ X2.astype(np.float64)
    assert np.abs(a - bm).max() <= 1e-5 * np.abs(a).max()
    assert np.abs(Y0).max() <= 1e-5 * scale
    assert np.array_equal(Y1, Y1b)


def test_apply_host_buffers_match_device():
    """The C ABI accepts host pointers (numpy) and stages them itself."""
    p = configs.config(1)
    X = configs.x_block(p.n, 8, seed=3)
    from paper_1705_10887_b200 import from_problem
    with from_problem(p, device="numpy") as hh, make_handle(p) as hd:
        Yh = hh.apply(X)
        Yd = run_apply(hd, X)
    assert np.array_equal(Yh, Yd)


def test_apply_column_of_operator():
    """B~ e_j equals column j of the dense oracle operator (SPEC.md:432 style)."""
    p = configs.config(1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    B = O.dense_operator(S, p.D)
    E = np.zeros((p.n, 4), dtype=np.float32)
    idx = [0, 17, 999, 1999]
    E[idx, range(4)] = 1.0
    with make_handle(p) as h:
        Y = run_apply(h, E)
    assert relerr(Y, B[:, idx]) <= TOL


def test_errors_are_reported():
    from paper_1705_10887_b200 import Sbmds, SbmdsError
    p = configs.config(1)
    with make_handle(p) as h:
        torch = _torch()
        X = torch.zeros((p.n, 65), device="cuda")
        with pytest.raises(SbmdsError):
            h.apply(X)
    bad = p.col_idx.copy()
    bad[5] = p.l
    with pytest.raises(SbmdsError, match="EINVAL"):
        Sbmds(p.n, p.l, p.row_ptr, bad, p.val32(), p.D)
    Dn = p.D.copy()
    Dn[0, 1] += 1.0
    with pytest.raises(SbmdsError, match="symmetric"):
        Sbmds(p.n, p.l, p.row_ptr, p.col_idx, p.val32(), Dn, validate=True)


@pytest.mark.parametrize("dstream", [1, 2])
@pytest.mark.parametrize("b", [8, 16, 32, 64, 12])
def test_apply_both_dstream_paths(dstream, b):
    """FFMA stream (1) and tcgen05 3xTF32 stream (2) both meet the bar, ragged l (l = 2003)."""
    p = configs.random_problem(30_011, 2_003, 16, seed=b, name="cfg5_small")
    X = configs.x_block(p.n, b, seed=b)
    with make_handle(p) as h:
        h.set_option("dstream", dstream)
        Y = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("blocked", [0, 1, 2, 3])
@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
def test_apply_blocked_and_plain_sparse_paths(blocked, b):
    """Row-blocked (smem dictionary) SpMMs and the plain CSR/CSC SpMMs both meet the bar."""
    p = configs.config(2)
    X = configs.x_block(p.n, b, seed=b)
    with make_handle(p) as h:
        h.set_option("blocked", blocked)
        assert 0 < h.stat("blocked_umax") < 200     # torus: ~100 landmarks per 256-row block
        Y = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL


@pytest.mark.parametrize("dstream", [3, 4])
@pytest.mark.parametrize("b", [16, 12, 8, 5, 32, 20])
def test_apply_symmetric_half_stream(b, dstream):
    """NEXT-1: streaming only the upper triangle of D (3: k_dstream_sym8, 4: k_dstream_pair) meets the
    bar; l = 2003 gives 16 row tiles with a ragged last one, so diagonal, off-diagonal and
    transposed tiles, blocks split between pairs and (b = 8) a single block all occur."""
    p = configs.random_problem(30_011, 2_003, 16, seed=b + 100, name="cfg5_small")
    X = configs.x_block(p.n, b, seed=b)
    with make_handle(p) as h:
        h.set_option("dstream", dstream)
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == dstream
    assert relerr(Y, oracle_apply(p, X)) <= TOL


def test_apply_symmetric_half_many_blocks():
    """l = 9001: 71 row tiles, 5 block rows of 16 at b = 8, 9 of 8 at b = 16, 18 of 4 at
    b = 32; every pair's range crosses blocks. Bitwise deterministic, and one handle can
    switch widths (one packed D, one schedule per width)."""
    p = configs.random_problem(40_000, 9_001, 8, seed=7, name="cfg5_mid")
    with make_handle(p) as h:
        h.set_option("dstream", 3)
        for b in (16, 8, 32):
            X = configs.x_block(p.n, b, seed=b)
            Y = run_apply(h, X)
            assert h.stat("dstream_path") == 3
            assert relerr(Y, oracle_apply(p, X)) <= TOL
            assert np.array_equal(Y, run_apply(h, X))


def test_symmetric_half_eigs_config2():
    """The symmetric-half stream inside the eigensolver (config 2) agrees with the full stream."""
    p = configs.config(2)
    with make_handle(p) as h:
        lam_a, _, _, _ = h.eigs(p.m, p.block, max_iters=200, tol=1e-6)
        h.set_option("dstream", 3)
        lam_b, _, _, _ = h.eigs(p.m, p.block, max_iters=200, tol=1e-6)
    assert np.allclose(lam_a, lam_b, rtol=1e-5)


def test_degenerate_inputs():
    """l = 1 (D = [[0]]), nnz = 0 (S = 0) and empty rows: B~X = 0 where the algebra says so,
    and the oracle agrees everywhere."""
    from paper_1705_10887_b200 import Sbmds
    torch = _torch()
    n = 1000
    X = configs.x_block(n, 8, seed=1)
    # l = 1: every row of S is e_1 -> J S = 0 -> B~ = 0
    rp = np.arange(n + 1, dtype=np.int64)
    h = Sbmds(n, 1, rp, np.zeros(n, np.int32), np.ones(n, np.float32), np.zeros((1, 1), np.float32))
    Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
    h.close()
    assert np.abs(Y).max() < 1e-6 * np.abs(X).max()
    # nnz = 0
    h = Sbmds(n, 7, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32),
              np.ones((7, 7), np.float32))
    Y = h.apply(torch.from_numpy(X).cuda()).cpu().numpy()
    h.close()
    assert np.abs(Y).max() == 0.0
    # empty rows interleaved with full ones
    p = synth_problem(n=3000, l=300, k=6, seed=9)
    lens = np.diff(p.row_ptr)
    keep = np.arange(p.n) % 3 != 0                        # every third row empty
    new_lens = np.where(keep, lens, 0)
    rp2 = np.zeros(p.n + 1, np.int64)
    rp2[1:] = np.cumsum(new_lens)
    mask = np.repeat(keep, lens)
    q = configs.Problem("emptyrows", p.n, p.l, rp2, p.col_idx[mask], p.val[mask], p.D)
    for b in (4, 16):
        Xq = configs.x_block(q.n, b, seed=b)
        with make_handle(q) as hq:
            Yq = run_apply(hq, Xq)
        assert relerr(Yq, oracle_apply(q, Xq)) <= TOL


def test_borrowed_device_d():
    """SBMDS_BORROW_D keeps the caller's device D (l % 4 == 0) and gives identical results."""
    p = configs.config(2)
    X = configs.x_block(p.n, 16, seed=2)
    with make_handle(p) as h1, make_handle(p, borrow_d=True) as h2:
        assert h1.stat("d_borrowed") == 0 and h2.stat("d_borrowed") == 1
        assert np.array_equal(run_apply(h1, X), run_apply(h2, X))


def test_invalid_eigs_arguments():
    from paper_1705_10887_b200 import SbmdsError
    p = configs.config(1)
    with make_handle(p) as h:
        for m, block, iters in ((3, 65, 10), (9, 8, 10), (0, 8, 10), (3, 8, 0)):
            with pytest.raises(SbmdsError, match="EINVAL"):
                h.eigs(m, block, max_iters=iters)
        Dbad = p.D.copy()
        Dbad[3, 3] = np.nan
    from paper_1705_10887_b200 import Sbmds
    with pytest.raises(SbmdsError, match="non-finite"):
        Sbmds(p.n, p.l, p.row_ptr, p.col_idx, p.val32(), Dbad, validate=True)


def test_host_d_upper_upload_and_mirror():
    """A host D crosses the host link as its block upper triangle only (D is symmetric); the
    symmetric-half path needs nothing else, and the first full-D apply mirrors the lower
    triangle on the device. Both paths meet the bar; VALIDATE uploads (and checks) all of D."""
    p = configs.random_problem(30_011, 2_003, 16, seed=5, name="cfg5_small")
    X = configs.x_block(p.n, 16, seed=2)
    ref = oracle_apply(p, X)
    l = p.l
    upper = sum(min(128, l - r0) * (l - r0) for r0 in range(0, l, 128)) * 4
    with make_handle(p, device="numpy") as h:
        assert h.stat("h2d_bytes") == upper and h.stat("d_lower_missing") == 1
        h.set_option("dstream", 3)
        assert relerr(run_apply(h, X), ref) <= TOL
        assert h.stat("d_lower_missing") == 1
        h.set_option("dstream", 2)
        assert relerr(run_apply(h, X), ref) <= TOL
        assert h.stat("d_lower_missing") == 0
        h.set_option("dstream", 1)
        assert relerr(run_apply(h, X[:, :4].copy()), oracle_apply(p, X[:, :4].copy())) <= TOL
    with make_handle(p, device="numpy", validate=True) as h:
        assert h.stat("h2d_bytes") == 4 * l * l and h.stat("d_lower_missing") == 0


@pytest.mark.parametrize("l", [1, 5, 127, 128, 129, 300, 1025])
@pytest.mark.parametrize("b", [8, 16, 32])
def test_symmetric_half_small_l(l, b):
    """Forced symmetric-half stream at tile-boundary sizes: one tile (the T CTA sees only a
    diagonal tile and emits an empty flush), l = 127 / 128 / 129, more pairs than blocks."""
    n = max(4 * l, 64)
    p = configs.random_problem(n, l, min(8, l), seed=l + b, window=min(256, l), name="small_l")
    X = configs.x_block(p.n, b, seed=l)
    with make_handle(p) as h:
        h.set_option("dstream", 3)
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 3
    ref = oracle_apply(p, X)
    if l == 1:
        assert np.abs(Y).max() <= 1e-6 * max(1.0, np.abs(X).max())
    else:
        assert relerr(Y, ref) <= TOL


@pytest.mark.parametrize("dstream", [0, 1, 2, 3])
@pytest.mark.parametrize("b", [1, 4, 12, 16, 64])
def test_uncentred_apply(dstream, b):
    """center = 0: sbmds_apply returns E^ X = S D S^T X (the paper's error
    workload, :317) on every D-stream path, to the same bar as the centred apply."""
    p = configs.random_problem(30_011, 2_003, 16, seed=b + 7, name="cfg5_small")
    X = configs.x_block(p.n, b, seed=b + 1)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    ref = O.apply_raw(S, p.D, X.astype(np.float64))
    with make_handle(p) as h:
        h.set_option("center", 0)
        h.set_option("dstream", dstream)
        Y = run_apply(h, X)
        h.set_option("center", 1)
        Yc = run_apply(h, X)
    assert relerr(Y, ref) <= TOL
    assert relerr(Yc, oracle_apply(p, X)) <= TOL   # the centred apply is untouched afterwards


def test_apply_config4_full_size():
    """Parity at BASELINE's full size (config 4: n = 1.8M, l = 50,000, k = 32, b = 16) in the
    launch configuration the library picks by default (CSC SpMM, int8 symmetric-half D stream,
    row-blocked CSR SpMM): every output element against the fp64 oracle's apply (~5 s on the
    host), relative Frobenius error <= 1e-5."""
    p = configs.config(4)
    X = configs.x_block(p.n, 16, seed=21)
    with make_handle(p) as h:
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 3
    Yo = oracle_apply(p, X)
    assert relerr(Y, Yo) <= TOL, relerr(Y, Yo)


def test_host_d_pack_issued_in_create():
    """A host D large enough for the int8 symmetric-half stream (auto path): create takes max |D|
    over the landed strips, builds the stream's schedule while D crosses the link and packs D on
    a handle stream past its return; the first D-stream launch waits for that pack. The host-D
    handle's apply equals the device-D handle's bit for bit (same packing, same max) and meets
    the oracle bar; so does an eigs solve started right after create."""
    p = configs.random_problem(40_000, 5_000, 16, seed=9, name="host_d_pack")
    X = configs.x_block(p.n, 16, seed=4)
    ref = oracle_apply(p, X)
    with make_handle(p, device="numpy") as hh, make_handle(p) as hd:
        assert hh.stat("d_lower_missing") == 1
        assert hh.stat("d_packed_in_create") == 1 and hd.stat("d_packed_in_create") == 0
        lam_h = hh.eigs(3, 16, max_iters=8, tol=0.0)[0]   # the first D-stream launch is inside eigs
        lam_d = hd.eigs(3, 16, max_iters=8, tol=0.0)[0]
        Yh, Yd = run_apply(hh, X), run_apply(hd, X)
        assert hh.stat("dstream_path") == 3 and hd.stat("dstream_path") == 3
    assert np.array_equal(Yh, Yd)
    assert np.array_equal(np.asarray(lam_h), np.asarray(lam_d))
    assert relerr(Yh, ref) <= TOL


@pytest.mark.parametrize("cfgname", ["random", "narrow_window"])
def test_reordered_rows_keep_the_callers_order(cfgname):
    """SBMDS_REORDER_ROWS: the handle keeps S's rows in its own order (here a real permutation:
    random-window rows reorder), X / Y / X0 / V / Z stay in the caller's order. Apply, eigs (with a
    warm start) and BMDS agree with the oracle and with a natural-order handle."""
    import torch
    if cfgname == "random":
        p = configs.random_problem(60_001, 2_003, 16, seed=77, name="cfg5_small")
    else:
        p = configs.random_problem(30_011, 1_029, 8, seed=78, window=100, name="narrow")
    X = configs.x_block(p.n, 16, seed=5)
    ref = oracle_apply(p, X)
    with make_handle(p, reorder_rows=True) as hr, make_handle(p) as hn:
        assert hr.stat("row_permuted") == 1 and hn.stat("row_permuted") == 0
        Yr = run_apply(hr, X)
        lam_r, V_r, Z_r, _ = hr.eigs(3, 16, max_iters=300, tol=1e-6)
        lam_n, V_n, Z_n, _ = hn.eigs(3, 16, max_iters=300, tol=1e-6)
        X0 = torch.from_numpy(configs.x_block(p.n, 16, seed=9)).cuda()
        lam_w, V_w, _, _ = hr.eigs(3, 16, max_iters=300, tol=1e-6, X0=X0)
    assert relerr(Yr, ref) <= TOL
    assert np.allclose(lam_r, lam_n, rtol=1e-5) and np.allclose(lam_w, lam_n, rtol=1e-5)
    Vr, Vn = V_r.cpu().numpy().astype(np.float64), V_n.cpu().numpy().astype(np.float64)
    assert O.principal_angle(Vr, Vn) <= 1e-3
    for j in range(3):                              # the sign rule in the caller's row order
        assert Vr[np.argmax(np.abs(Vr[:, j])), j] > 0


@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_narrow_blocks_on_the_int8_stream(b):
    """b <= 4 at a D large enough for the symmetric half (l = 5000): the int8 stream at width 8 with
    Y1 widened and Y2 narrowed around it (3 l^2 / 2 bytes instead of the FFMA stream's 4 l^2),
    centred and uncentred, against the oracle."""
    p = configs.random_problem(40_000, 5_000, 16, seed=90 + b, name="narrow_b")
    X = configs.x_block(p.n, b, seed=b)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    with make_handle(p) as h:
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 3
        h.set_option("center", 0)
        Yr = run_apply(h, X)
    assert relerr(Y, oracle_apply(p, X)) <= TOL
    assert relerr(Yr, O.apply_raw(S, p.D, X.astype(np.float64))) <= TOL


@pytest.mark.parametrize("b", [33, 48, 64])
def test_wide_blocks_in_two_int8_passes(b):
    """33 <= b <= 64 in a standalone apply at a D large enough for the symmetric half: two passes
    of the width-32 int8 stream over the column halves (Y2 and t merged), vs the oracle; the
    uncentred apply (an R^-1 fold of -2 I) keeps the 3xTF32 stream."""
    p = configs.random_problem(40_000, 5_000, 16, seed=70 + b, name="wide_b")
    X = configs.x_block(p.n, b, seed=b)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    with make_handle(p) as h:
        Y = run_apply(h, X)
        assert h.stat("dstream_path") == 3
        h.set_option("center", 0)
        Yr = run_apply(h, X)
        assert h.stat("dstream_path") == 2
    assert relerr(Y, oracle_apply(p, X)) <= TOL
    assert relerr(Yr, O.apply_raw(S, p.D, X.astype(np.float64))) <= TOL


@pytest.mark.parametrize("kind", ["config2", "signed", "uncentred", "dominant_row"])
def test_apply_on_tensor_core_sparse_kernels(kind):
    """Standalone sbmds_apply at b = 16 where S is local (every 128-row block touches <= 128
    landmarks): A2 = S^T X runs as the T products and A5 = S (Y2 - 1 t^T) as the N products of the
    tensor-core sparse step (k_sp8_step TONLY / without T products; S_B as dense digit images, X
    and Y2 - 1 t^T as 24-bit digits with one scale per column) -- against the oracle, against the
    fp32 kernels (sp8_apply = 0), for a signed, non-normalised S (the (S 1 - 1) t^T term), for the
    uncentred operator (center = 0: A2 stays on the CSC kernel) and for an X with a dominant row
    (the column check sends A2 to the fp32 CSC kernel: x_fallbacks)."""
    p = configs.config(2)
    if kind == "signed":
        rng = np.random.default_rng(5)
        val = p.val * (1.0 + 0.3 * rng.standard_normal(p.val.shape))
        p = configs.Problem("cfg2_signed", p.n, p.l, p.row_ptr, p.col_idx, val, p.D)
    X = configs.x_block(p.n, 16, seed=9)
    if kind == "dominant_row":
        X[777] *= 1.0e4
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    with make_handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        if kind == "uncentred":
            h.set_option("center", 0)
            ref = O.apply_raw(S, p.D, X.astype(np.float64))
        else:
            ref = O.apply(S, p.D, X.astype(np.float64))
        n0, t0, f0 = h.stat("sp8_apply_launches"), h.stat("sp8_apply_t_launches"), h.stat("x_fallbacks")
        Y = run_apply(h, X)
        assert h.stat("sp8_apply_launches") == n0 + 1 and h.stat("sp8_state") == 1
        assert h.stat("sp8_apply_t_launches") == t0 + (1 if kind in ("config2", "signed") else 0)
        assert h.stat("x_fallbacks") == f0 + (1 if kind == "dominant_row" else 0)
        Y_again = run_apply(h, X)
        h.set_option("sp8_apply", 0)
        Y32 = run_apply(h, X)
        assert h.stat("sp8_apply_launches") == n0 + 2
    assert relerr(Y, ref) <= TOL, relerr(Y, ref)
    assert relerr(Y32, ref) <= TOL
    assert relerr(Y, Y32) <= 5e-6
    assert np.array_equal(Y, Y_again)


def test_apply_b32_on_tensor_core_sparse_kernels():
    """b = 32 (config 3's width) on the tensor-core sparse kernels: two passes over the images,
    one per 16-column half of X (strided rows, cp.async staging) and of Y2 / Y."""
    p = configs.config(2)
    X = configs.x_block(p.n, 32, seed=13)
    ref = oracle_apply(p, X)
    with make_handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        n0, t0 = h.stat("sp8_apply_launches"), h.stat("sp8_apply_t_launches")
        Y = run_apply(h, X)
        assert h.stat("sp8_apply_launches") == n0 + 1 and h.stat("sp8_apply_t_launches") == t0 + 1
        Y_again = run_apply(h, X)
        h.set_option("sp8_apply", 0)
        Y32 = run_apply(h, X)
    assert relerr(Y, ref) <= TOL, relerr(Y, ref)
    assert relerr(Y32, ref) <= TOL
    assert relerr(Y, Y32) <= 5e-6
    assert np.array_equal(Y, Y_again)


def test_tensor_core_sparse_kernels_split_blocks():
    """A 128-row block whose rows sit in two distant regions of the mesh touches more landmarks
    than one 128-column image holds (a Morton-numbered mesh has such blocks at the curve's
    jumps): the build halves it (stat sp8_splits) instead of giving up the tensor-core kernels.
    Config 2 with seven 16-row ranges of block 0 swapped with rows far across the mesh: apply (b = 16, 32) and the eigs step
    against the oracle."""
    p0 = configs.config(2)
    n = p0.n
    perm = np.arange(n)
    for q in range(7):   # block 0 then holds 16 rows of each of eight regions: 163 distinct landmarks
        a, b_ = 16 * (q + 1), 12_000 * (q + 1) + 16 * (q + 1)
        perm[a:a + 16], perm[b_:b_ + 16] = np.arange(b_, b_ + 16), np.arange(a, a + 16)
    lens = np.diff(p0.row_ptr)[perm]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(p0.row_ptr[r], p0.row_ptr[r + 1]) for r in perm])
    p = configs.Problem("cfg2_swapped", n, p0.l, row_ptr, p0.col_idx[idx], p0.val[idx], p0.D)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    with make_handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        for b in (16, 32):
            X = configs.x_block(p.n, b, seed=b)
            n0 = h.stat("sp8_apply_launches")
            Y = run_apply(h, X)
            assert h.stat("sp8_state") == 1 and h.stat("sp8_splits") >= 1 and h.stat("sp8_apply_launches") == n0 + 1
            assert h.stat("sp8_blocks") > (n + 127) // 128
            assert relerr(Y, O.apply(S, p.D, X.astype(np.float64))) <= TOL
        torch = _torch()
        lam, V, Z, info = h.eigs(3, 16, max_iters=500, tol=1e-6)
        torch.cuda.synchronize()
        assert info["converged"] == 1 and h.stat("gram8_launches") > 0
    lam_o, V_o, Z_o, _ = O.eigs_matfree(S, p.D, 3)
    assert np.all(np.abs(np.asarray(lam) - lam_o) <= 1e-4 * np.abs(lam_o))
    assert O.principal_angle(V.cpu().numpy().astype(np.float64), V_o) <= 1e-3


def test_apply_graph_capture_without_checks():
    """With dy_max_range >= 64 the standalone apply reads nothing back (include/sbmds.h): after a
    warm-up call it can be captured into a CUDA graph and replayed -- A2 then stays on the CSC
    kernel, A5 on the tensor-core N products -- with the eager call's result bit for bit."""
    torch = _torch()
    p = configs.config(2)
    X = torch.from_numpy(configs.x_block(p.n, 16, seed=4)).cuda()
    Y = torch.empty_like(X)
    Yg = torch.empty_like(X)
    with make_handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        h.set_option("dy_max_range", 64)
        h.apply(X, out=Y)
        torch.cuda.synchronize()
        n5 = h.stat("sp8_apply_launches")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            h.apply(X, out=Yg)
        Yg.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert h.stat("sp8_apply_launches") == n5 + 1 and h.stat("sp8_apply_t_launches") == 0
    assert torch.equal(Y, Yg)
    assert relerr(Y.cpu().numpy(), oracle_apply(p, X.cpu().numpy())) <= TOL


@pytest.mark.parametrize("n_rows", [99_991, 1_030, 1_001])
def test_tensor_core_sparse_kernels_ragged_n(n_rows):
    """n not a multiple of 128 (nor of 4): the last block of the tensor-core sparse kernels is a
    few rows (23 at n = 99,991, 6 at n = 1,030, 105 at n = 1,001 -- an odd count; the library needs
    n >= l = 1,000); apply at b = 16 and 32 on that path against the oracle."""
    p0 = configs.config(2)
    nnz = int(p0.row_ptr[n_rows])
    p = configs.Problem("cfg2_head", n_rows, p0.l, p0.row_ptr[:n_rows + 1].copy(), p0.col_idx[:nnz].copy(),
                        p0.val[:nnz].copy(), p0.D)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    with make_handle(p) as h:
        h.set_option("sp8_min_rows", 0)   # (config 2 is below the default size threshold of these kernels)
        for b in (16, 32):
            X = configs.x_block(p.n, b, seed=b + 3)
            n0 = h.stat("sp8_apply_launches")
            Y = run_apply(h, X)
            ref = O.apply(S, p.D, X.astype(np.float64))
            assert relerr(Y, ref) <= TOL, (n_rows, b, relerr(Y, ref))
            assert h.stat("sp8_apply_launches") == n0 + 1 and h.stat("sp8_state") == 1


@pytest.mark.parametrize("b", [8, 16, 32, 64])
def test_csr_spmm_shuffled_pairs_bitwise(b):
    """k_spmm_csr_vec4 with a group's (column, value) pairs loaded once and broadcast by shuffles
    (option csr_shfl = 1) sums in the same entry order as the plain loop (0): Y is bit-equal, and
    equals the oracle's to the tolerance. Rows of 1..70 entries: shorter than one chunk, longer
    than the four chunks in flight at every width; n is not a multiple of the rows per warp."""
    torch = _torch()
    p = synth_problem(n=4099, l=301, k=70, seed=11, negative=True, rowsum_one=False)
    X = configs.x_block(p.n, b, seed=5)
    Yo = oracle_apply(p, X)
    with make_handle(p) as h:
        h.set_option("blocked", 0)
        h.set_option("sp8_apply", 0)
        ys = []
        for shf in (0, 1):
            h.set_option("csr_shfl", shf)
            ys.append(run_apply(h, X))
    assert np.array_equal(ys[0], ys[1])
    assert relerr(ys[1], Yo) <= TOL
