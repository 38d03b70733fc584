"""The tuned kernels' tile visiting order (gm_tile_order, host-side, no GPU):
a permutation of the gasket's member tiles, grouped by level-L sub-gasket in
lambda digit order (the ranges partitioned launches address, partition.py) and
row-major inside each group (stencil2.cu rowmajor_table)."""

import numpy as np
import pytest


def _digit_xy(s: int, L: int) -> tuple[int, int]:
    # lambda in digit order (gasket.cuh lambda_digit_order): digit 1 -> (0,1), 2 -> (1,1)
    x = y = 0
    for i in range(L):
        d = s % 3
        s //= 3
        x |= (d == 2) << i
        y |= (d != 0) << i
    return x, y


@pytest.mark.parametrize("q,L", [(0, 0), (1, 0), (4, 0), (4, 2), (6, 3), (7, 5), (8, 8)])
def test_tile_order_is_grouped_rowmajor_permutation(q, L):
    from paper_1706_04552_b200 import _build, native

    _build.build()
    bx, by = native.tile_order(q, L)
    assert bx.size == 3**q
    assert np.all((bx & ~by) == 0)  # member tiles only
    assert len(set(zip(bx.tolist(), by.tolist()))) == 3**q  # each exactly once
    m = q - L
    per = 3**m
    for s in range(3**L):
        sx, sy = _digit_xy(s, L)
        gx, gy = bx[s * per:(s + 1) * per], by[s * per:(s + 1) * per]
        assert np.all(gx >> m == sx) and np.all(gy >> m == sy), s
        key = (gy << 20) | gx
        assert np.all(np.diff(key) > 0), s  # row-major: Y ascending, then l ascending


def test_tile_order_rejects_bad_arguments():
    from paper_1706_04552_b200 import native

    out = np.zeros(3, dtype=np.uint32)
    with pytest.raises(ValueError):
        native.check(native.lib().gm_tile_order(2, 0, out.ctypes.data, out.size))  # capacity < 9
    with pytest.raises(ValueError):
        native.tile_order(3, 4)
