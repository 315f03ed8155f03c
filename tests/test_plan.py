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
