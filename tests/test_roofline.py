"""The algorithmic-bytes model behind bench.py's roofline, checked
against brute-force sector counts on small grids."""

import numpy as np
import pytest

from paper_1706_04552_b200 import roofline as R


def _brute(r, c, kind):
    n = 1 << r
    ys, xs = np.mgrid[0:n, 0:n]
    member = (xs & (n - 1 - ys)) == 0
    per = 32 // c  # cells per sector
    sec = lambda m: {(int(y), int(x) // per) for y, x in zip(*np.nonzero(m))}  # noqa: E731
    write = sec(member)
    if kind == 0:
        return len(write), 0
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)] + ([(1, 1), (1, -1), (-1, 1), (-1, -1)] if kind == 2 else [])
    need = np.zeros_like(member)
    for dx, dy in offs:
        sh = np.zeros_like(member)
        sh[max(dy, 0):n + min(dy, 0), max(dx, 0):n + min(dx, 0)] = member[max(-dy, 0):n + min(-dy, 0),
                                                                          max(-dx, 0):n + min(-dx, 0)]
        need |= sh
    return len(write), len(sec(need))


@pytest.mark.parametrize("c", [1, 2, 4])
def test_sector_counts_match_brute_force(c):
    for r in range(0, 10):
        w, _ = _brute(r, c, 0)
        assert R.write_sectors(r, c) == w, (r, c)
        for kind in (1, 2):
            _, rd = _brute(r, c, kind)
            assert R.stencil_read_sectors(r, c, kind == 2) == rd, (r, c, kind)


def test_table_entries_match_counter():
    for key, v in list(R._TABLE.items())[::7]:
        r, c, e = (int(t) for t in key.split(","))
        if r <= 12:
            assert R.stencil_read_sectors(r, c, bool(e)) == v


def test_survey_figures():
    """SURVEY §8d exact byte counts."""
    assert R.write_bytes(16, 1) == 181_398_528
    assert R.write_bytes(16, 4) == 408_146_688
    assert R.pass_bytes(17, 1, 2) == 828_974_656 + 544_195_584
    assert R.pass_bytes(17, 1, 1) == 823_305_952 + 544_195_584
    assert R.stencil_read_bytes(16, 4, False) == 643_873_120
