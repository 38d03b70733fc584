"""Algorithmic DRAM bytes of the gasket passes on the dense row-major layout.

A DRAM sector is 32 bytes = 32/c cells of width c.  Sector s of row y holds a
gasket cell iff s (as a bit pattern) is a subset of y >> k, k = log2(32/c)
(membership x & (n-1-y) == 0 splits bitwise), so

    write pass:   sectors = 2^k * 3^(r-k)            (exact, any r >= k)
    stencil read: sectors of the neighbour set of all gasket cells
                  (4- or 8-neighbourhood, the cell itself is not read),
                  counted exactly per row with numpy bitsets.

These are the "algorithmic bytes" of the roofline; the
element-byte figure (c bytes per cell read + written) is reported beside them.
"""

from __future__ import annotations

import functools
import json
from pathlib import Path

import numpy as np

SECTOR = 32
# stencil_read_sectors(r, c, eight) precomputed with this module's counter
# (keys "r,c,eight"); tests/test_roofline.py re-derives entries and checks
# small levels against a brute-force neighbour scan.
_TABLE_PATH = Path(__file__).with_name("stencil_sectors.json")
try:
    _TABLE = json.loads(_TABLE_PATH.read_text())
except (OSError, ValueError):  # pragma: no cover
    _TABLE = {}


def _k(c: int, unit: int = SECTOR) -> int:
    return (unit // c).bit_length() - 1


def write_sectors(r: int, c: int) -> int:
    k = _k(c)
    if r <= k:  # whole rows fit in one sector
        return 1 << r
    return (1 << k) * 3 ** (r - k)


def write_bytes(r: int, c: int) -> int:
    return SECTOR * write_sectors(r, c)


def _subset_rows(Y: np.ndarray, nsec: int) -> np.ndarray:
    s = np.arange(nsec, dtype=np.int64)
    return (s[None, :] & ~Y[:, None]) == 0


@functools.lru_cache(maxsize=None)
def stencil_read_sectors(r: int, c: int, eight: bool, chunk: int = 2048, unit: int = SECTOR) -> int:
    """Exact number of `unit`-byte blocks (default: 32-byte sectors) holding a
    neighbour of some gasket cell."""
    n = 1 << r
    k = _k(c, unit)
    if r <= k:
        # a row is a single (partial) sector: count rows holding any needed cell
        mask = (np.arange(n)[None, :] & (n - 1 - np.arange(n))[:, None]) == 0
        need = np.zeros_like(mask)
        offs = [(1, 0), (-1, 0), (0, 1), (0, -1)] + ([(1, 1), (1, -1), (-1, 1), (-1, -1)] if eight else [])
        for dx, dy in offs:
            sh = np.zeros_like(mask)
            ys = slice(max(dy, 0), n + min(dy, 0))
            yd = slice(max(-dy, 0), n + min(-dy, 0))
            xs = slice(max(dx, 0), n + min(dx, 0))
            xd = slice(max(-dx, 0), n + min(-dx, 0))
            sh[yd, xd] = mask[ys, xs]
            need |= sh
        return int(need.any(axis=1).sum())
    nsec = n >> k
    low = (1 << k) - 1
    total = 0
    for y0 in range(0, n, chunk):
        ys = np.arange(y0, min(n, y0 + chunk), dtype=np.int64)
        need = np.zeros((ys.size, nsec), dtype=bool)
        for dy in (-1, 0, 1):
            yy = ys + dy
            valid = (yy >= 0) & (yy < n)
            yyc = np.clip(yy, 0, n - 1)
            m = yyc  # row y holds the cells x that are bit-subsets of y
            base = _subset_rows(m >> k, nsec) & valid[:, None]
            full_low = ((m & low) == low)[:, None]
            if dy == 0:
                # (x-1, y), (x+1, y): x-1 stays in s unless x's low bits are 0 (always
                # possible) -> s-1; x+1 stays in s (x low bits 0 exists when k >= 1)
                # and crosses into s+1 only when the low bits can all be 1.
                need |= base
                need[:, :-1] |= base[:, 1:]
                need[:, 1:] |= base[:, :-1] & full_low
            else:
                need |= base
                if eight:
                    need[:, :-1] |= base[:, 1:]
                    need[:, 1:] |= base[:, :-1] & full_low
        total += int(need.sum())
    return total


def stencil_read_bytes(r: int, c: int, eight: bool) -> int:
    hit = _TABLE.get(f"{r},{c},{int(eight)}")
    return SECTOR * (int(hit) if hit is not None else stencil_read_sectors(r, c, eight))


# The smallest unit an L2 read miss fetches on B200 is a 64-byte half line (the
# .L2::64B fetch-size hint; scripts/probe_fetch.cu), so the stencil's read set at
# that granularity is what DRAM must deliver at best.  Precomputed like _TABLE
# (keys "r,c,eight,64"); tests/test_roofline.py re-derives small entries.
FETCH = 64


def stencil_read_bytes_fetch(r: int, c: int, eight: bool) -> int:
    hit = _TABLE.get(f"{r},{c},{int(eight)},{FETCH}")
    return FETCH * (int(hit) if hit is not None else stencil_read_sectors(r, c, eight, unit=FETCH))


def hw_bytes(r: int, c: int, kind: int) -> int:
    """DRAM bytes the B200 memory system must move for a pass on this layout: a write
    pass's partial-sector stores are read-modify-written (2x the sector bytes); a
    stencil reads 64-byte halves and writes whole sectors."""
    w = write_bytes(r, c)
    if kind == 0:
        return 2 * w
    return w + stencil_read_bytes_fetch(r, c, kind == 2)


def pass_bytes(r: int, c: int, kind: int) -> int:
    """Minimum DRAM bytes (read + write) of one pass: kind 0 write, 1 NSUM4, 2 NSUM8."""
    w = write_bytes(r, c)
    if kind == 0:
        return w
    return w + stencil_read_bytes(r, c, kind == 2)


def element_bytes(r: int, c: int, kind: int) -> int:
    """c bytes written per gasket cell (+ c read for stencils): not reachable on this layout."""
    return 3**r * c * (1 if kind == 0 else 2)
