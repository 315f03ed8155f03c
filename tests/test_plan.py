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
