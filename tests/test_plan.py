"""Host logic of the symmetric-half D stream (no GPU): the walk, the per-CTA ranges and the
partial-slot schedule that k_dstream_sym8 / k_dstream_pair follow. sbmds_plan_selfcheck replays
the kernels' accumulate/flush rules against the host plan and counts violated invariants: each
upper tile once, each tile's row (N) and column (T) contribution in exactly one slot of the
right row tile, consistent reduction lists and slot map."""
import pytest

from paper_1705_10887_b200._lib import lib


@pytest.mark.parametrize("l", [1, 5, 127, 128, 129, 300, 2003, 9001, 50000])
@pytest.mark.parametrize("S,gN,contiguous", [(5, 51, 1), (8, 32, 1), (2, 128, 1), (16, 1, 0), (8, 1, 0)])
@pytest.mark.parametrize("ctas", [1, 7, 74, 148])
def test_plan_selfcheck(l, S, gN, contiguous, ctas):
    if l == 50000 and (ctas != 148 or (S, gN) not in ((5, 51), (8, 1))):
        pytest.skip("large l: the production layouts only (int8 b = 16, fp16 pairs)")
    assert lib().sbmds_plan_selfcheck(l, S, gN, ctas, contiguous) == 0


def test_plan_selfcheck_rejects_bad_arguments():
    assert lib().sbmds_plan_selfcheck(0, 5, 1, 1, 0) < 0
    assert lib().sbmds_plan_selfcheck(100, 17, 1, 1, 0) < 0


@pytest.mark.parametrize("l", [1, 5, 127, 128, 129, 300, 1153, 2003, 9001, 50000])
@pytest.mark.parametrize("SR,SC,gN", [(9, 1, 256), (15, 1, 256), (4, 1, 256), (3, 2, 128), (9, 1, 7)])
@pytest.mark.parametrize("ctas,rank,world", [(1, 0, 1), (7, 0, 1), (148, 0, 1), (148, 1, 2), (74, 2, 3)])
def test_plan_selfcheck_rectangular_blocks(l, SR, SC, gN, ctas, rank, world):
    """Blocks of SR x SC tiles (the int8 stream's 9 x 1 at b = 16, 15 x 1 at b = 8, 4 x 1 at
    b = 32), also as the tile range of a rank of a sharded apply: every upper tile once, every
    contribution in exactly one slot of the right row tile, contiguous slot map consistent."""
    if l == 50000 and (ctas != 148 or (SR, SC, gN) != (9, 1, 256)):
        pytest.skip("large l: the production layout only")
    assert lib().sbmds_plan_selfcheck_rect(l, SR, SC, gN, ctas, 1, rank, world) == 0


def test_rectangular_blocks_write_fewer_partials():
    """The point of 9 x 1 blocks: a column accumulator is flushed once per block, i.e. once per
    SR tiles (counted here by replaying the walk): 5 x 5 blocks flush 1 per 5 tiles."""
    def col_flushes(NT, SR, SC):
        n = 0
        for bi in range((NT + SR - 1) // SR):
            for bj in range((bi * SR) // SC, (NT + SC - 1) // SC):
                cols = {J for r in range(SR) for c in range(SC)
                        for I, J in [(bi * SR + r, bj * SC + c)] if I < NT and J < NT and J > I}
                n += len(cols)
        return n
    NT = 391   # config 4: l = 50,000
    tiles = NT * (NT + 1) // 2
    assert col_flushes(NT, 9, 1) / tiles < 0.12 < 0.19 < col_flushes(NT, 5, 5) / tiles


def test_plan_selfcheck_rect_rejects_bad_arguments():
    assert lib().sbmds_plan_selfcheck_rect(100, 9, 0, 1, 1, 1, 0, 1) < 0
    assert lib().sbmds_plan_selfcheck_rect(100, 17, 1, 1, 1, 1, 0, 1) < 0
    assert lib().sbmds_plan_selfcheck_rect(100, 9, 1, 1, 1, 1, 2, 2) < 0


def _split(n, r0, dsize, limit=128):
    import numpy as np
    r0 = np.ascontiguousarray(r0, dtype=np.int32)
    ds = np.ascontiguousarray(dsize, dtype=np.int32)
    out = np.zeros(2 * len(r0) + 2, dtype=np.int32)
    nb = lib().sbmds_sparse_split_rows(n, len(ds), r0.ctypes.data, ds.ctypes.data, limit, out.ctypes.data, len(out))
    return nb, out[:nb + 1] if nb > 0 else None


def test_sp8_split_rows_rule():
    """The block-splitting rule of the tensor-core sparse kernels (host part of ensure_sp8): only
    blocks over the limit are halved, at a multiple of 4 rows from their start; the boundaries stay
    a partition of [0, n); a block over the limit with fewer than 8 rows cannot be split."""
    import numpy as np
    n = 128 * 5 + 37
    r0 = np.minimum(np.arange(7) * 128, n)           # 6 blocks, the last of 37 rows
    nb, out = _split(n, r0, [100, 129, 128, 300, 20, 200])
    assert nb == 9
    assert list(out) == [0, 128, 192, 256, 384, 448, 512, 640, 660, n]
    assert all(int(b) % 4 == 0 for b in out[:-1]) and out[0] == 0 and out[-1] == n and np.all(np.diff(out) > 0)
    nb2, out2 = _split(n, out, [100, 60, 70, 128, 160, 150, 20, 110, 100])   # second round: two pieces still over
    assert nb2 == 11 and list(out2[4:9]) == [384, 416, 448, 480, 512]
    assert _split(8, [0, 8], [129])[0] == 2 and list(_split(8, [0, 8], [129])[1]) == [0, 4, 8]
    assert _split(7, [0, 7], [129])[0] == -1          # fewer than 8 rows over the limit
    assert _split(6, [0, 4, 6], [10, 500])[0] == -1
    assert _split(640, np.arange(6) * 128, [128] * 5)[0] == 5   # nothing over the limit: unchanged count
    assert lib().sbmds_sparse_split_rows(0, 1, None, None, 128, None, 0) == -2
