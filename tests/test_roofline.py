"""The algorithmic-bytes model behind bench.py's roofline, checked
against brute-force sector counts on small grids."""

import numpy as np
import pytest

from paper_1706_04552_b200 import roofline as R


def _brute(r, c, kind, unit=32):
    n = 1 << r
    ys, xs = np.mgrid[0:n, 0:n]
    member = (xs & (n - 1 - ys)) == 0
    per = unit // c  # cells per sector (or fetch unit)
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


@pytest.mark.parametrize("c", [1, 2, 4])
def test_fetch_unit_counts_match_brute_force(c):
    """The 64-byte-fetch read set (hw_bytes) against a brute-force neighbour scan."""
    for r in range(0, 10):
        for kind in (1, 2):
            _, rd = _brute(r, c, kind, unit=64)
            assert R.stencil_read_sectors(r, c, kind == 2, unit=64) == rd, (r, c, kind)


def test_table_entries_match_counter():
    for key, v in list(R._TABLE.items())[::7]:
        parts = [int(t) for t in key.split(",")]
        r, c, e = parts[:3]
        unit = parts[3] if len(parts) > 3 else 32
        if r <= 12:
            assert R.stencil_read_sectors(r, c, bool(e), unit=unit) == v


def test_hw_model_figures():
    """bench.py's hw_model: write = sector RMW (2x), stencil = 64-byte reads + sector writes."""
    assert R.hw_bytes(16, 1, 0) == 2 * 181_398_528
    assert R.hw_bytes(17, 1, 2) == R.stencil_read_bytes_fetch(17, 1, True) + 544_195_584
    assert R.stencil_read_bytes_fetch(17, 1, True) == 1_091_211_008  # ncu: 1101 MB read per launch


def test_survey_figures():
    """SURVEY §8d exact byte counts."""
    assert R.write_bytes(16, 1) == 181_398_528
    assert R.write_bytes(16, 4) == 408_146_688
    assert R.pass_bytes(17, 1, 2) == 828_974_656 + 544_195_584
    assert R.pass_bytes(17, 1, 1) == 823_305_952 + 544_195_584
    assert R.stencil_read_bytes(16, 4, False) == 643_873_120
