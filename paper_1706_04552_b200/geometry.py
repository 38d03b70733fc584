"""Host-side gasket geometry and lambda planner (pure integer arithmetic).

Re-exported under the reference's module names by ``core``, ``blockmap`` and
``intra`` so ``from paper_1706_04552_b200.core import FractalSpec`` works like
``from gasketmap.core import FractalSpec``.  Only O(r)- or O(rho^2)-sized
planning arithmetic lives here; every per-block / per-cell computation runs in
the sm_100a library (``device.py``, ``backends.py``).

Reference anchors (``/root/reference/pkg/src/gasketmap``):
  core.py:19-22 (limits), :44-56 (scale_level, volume), :59-61 (Hausdorff),
  :64-72 (packing_dims), :75-81 (is_member), :84-102 (mask / enumeration),
  :105-127 (FractalSpec); blockmap.py:34-88 (block_region, region_offset,
  reduction_depth, map_block), :111-120 (suggested_block_threads), :169-195
  (corrupted_map_fn); intra.py:25-91 (strategies, tables, local cells).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Callable, NamedTuple, Optional

import numpy as np

MAX_LEVEL = 40  # 3**40 < 2**64: every count is an exact machine integer
ORACLE_MAX_EDGE = 1 << 13  # dense host scans stop here (device paths go further)
MAX_TABLE_EDGE = 1 << 10


class Coord2(NamedTuple):
    x: int
    y: int


class OrthotopeDims(NamedTuple):
    width: int
    height: int


class MapResult(NamedTuple):
    coord: Coord2
    depth: int


class BijectionReport(NamedTuple):
    ok: bool
    witness: Optional[Coord2]
    image_size: int


# ---------------------------------------------------------------------------
# levels, sizes, membership
# ---------------------------------------------------------------------------

def _level_ok(r: int) -> int:
    if r < 0 or r > MAX_LEVEL:
        raise ValueError(f"scale level must be in [0, {MAX_LEVEL}], got {r}")
    return r


def _is_pow2(v: int) -> bool:
    return v >= 1 and (v & (v - 1)) == 0


def scale_level(n: int) -> int:
    if not _is_pow2(n):
        raise ValueError(f"edge length must be a power of two >= 1, got {n}")
    return _level_ok(n.bit_length() - 1)


def volume(r: int) -> int:
    return 3 ** _level_ok(r)


def hausdorff_exponent() -> float:
    return math.log2(3.0)


def packing_dims(r: int) -> OrthotopeDims:
    """Packed rectangle of level r: width 3^floor(r/2) (even levels, omega_x),
    height 3^ceil(r/2) (odd levels, omega_y)."""
    _level_ok(r)
    half = r >> 1
    return OrthotopeDims(3 ** half, 3 ** (r - half))


def is_member(t, n: int) -> bool:
    scale_level(n)
    x, y = t
    if x < 0 or y < 0 or x >= n or y >= n:
        raise ValueError(f"coordinate {t!r} outside the {n}x{n} grid")
    return not (x & (n - 1 - y))


def member_mask(n: int) -> np.ndarray:
    """Dense boolean membership mask (host planning helper, edge <= 2^13)."""
    scale_level(n)
    if n > ORACLE_MAX_EDGE:
        raise ValueError(f"edge {n} too large for a dense scan (max {ORACLE_MAX_EDGE})")
    cols = np.arange(n, dtype=np.int64)
    return np.bitwise_and(cols[np.newaxis, :], (n - 1) - cols[:, np.newaxis]) == 0


def enumerate_cells(n: int) -> list[Coord2]:
    rows, cols = np.nonzero(member_mask(n))
    return [Coord2(int(c), int(r)) for r, c in zip(rows, cols)]


@dataclass(frozen=True)
class FractalSpec:
    """n x n cell grid tiled by rho x rho blocks; r = log2 n, n_b = n/rho, r_b = log2 n_b."""

    n: int
    rho: int = 1
    r: int = field(init=False)
    n_b: int = field(init=False)
    r_b: int = field(init=False)

    def __post_init__(self) -> None:
        level = scale_level(self.n)
        if not _is_pow2(self.rho):
            raise ValueError(f"block edge must be a power of two >= 1, got {self.rho}")
        if self.rho > self.n:
            raise ValueError(f"block edge {self.rho} exceeds grid edge {self.n}")
        k = self.rho.bit_length() - 1
        object.__setattr__(self, "r", level)
        object.__setattr__(self, "n_b", self.n >> k)
        object.__setattr__(self, "r_b", level - k)


# ---------------------------------------------------------------------------
# lambda(omega) scalar pieces (Eqs. 4-10)
# ---------------------------------------------------------------------------

def block_region(omega, mu: int) -> int:
    """beta_mu: base-3 digit (mu-1)//2 of omega.y for odd mu, mu//2-1 of omega.x for even mu."""
    if mu < 1:
        raise ValueError(f"scale-level index must be >= 1, got {mu}")
    axis_value = omega[1] if mu % 2 else omega[0]
    return (axis_value // 3 ** ((mu - 1) // 2)) % 3


def region_offset(region: int, mu: int) -> tuple[int, int]:
    if region not in (0, 1, 2):
        raise ValueError(f"region index must be 0, 1 or 2, got {region}")
    if mu < 1:
        raise ValueError(f"scale-level index must be >= 1, got {mu}")
    edge = 1 << (mu - 1)
    right = region >> 1
    return (right * edge, (region - right) * edge)


def reduction_depth(r_b: int) -> int:
    """ceil(log2(max(r_b, 1))): tree-reduction steps over r_b per-level offsets."""
    if r_b < 0:
        raise ValueError(f"scale level must be >= 0, got {r_b}")
    return (max(r_b, 1) - 1).bit_length()


def _lambda_bits(wx: int, wy: int, r_b: int) -> tuple[int, int]:
    """Closed form: each level sets one bit per axis (digit!=0 -> y, digit==2 -> x)."""
    lx = ly = 0
    for mu in range(1, r_b + 1):
        if mu & 1:
            wy, digit = divmod(wy, 3)
        else:
            wx, digit = divmod(wx, 3)
        bit = 1 << (mu - 1)
        if digit:
            ly |= bit
            if digit == 2:
                lx |= bit
    return lx, ly


def map_block(omega, r_b: int) -> MapResult:
    width, height = packing_dims(r_b)
    wx, wy = omega
    if not (0 <= wx < width and 0 <= wy < height):
        raise ValueError(f"block {omega!r} outside the {width}x{height} rectangle of level {r_b}")
    return MapResult(Coord2(*_lambda_bits(wx, wy, r_b)), reduction_depth(r_b))


def suggested_block_threads(n: int) -> int:
    r = scale_level(n)
    if r < 2:
        raise ValueError(f"edge length must be >= 4, got {n}")
    return max(1, math.ceil(r / math.log2(r)))


def corrupted_map_fn(defect: str) -> Callable[[tuple[int, int], int], MapResult]:
    """Mutation hooks: 'parity' swaps the axis feeding each level, 'divisor'
    reads one base-3 place too high, 'offset' doubles the region edge."""
    if defect not in ("parity", "divisor", "offset"):
        raise ValueError(f"unknown defect {defect!r}")
    swap = defect == "parity"
    place_shift = 1 if defect == "divisor" else 0
    edge_shift = 1 if defect == "offset" else 0

    def broken(omega, r_b: int) -> MapResult:
        wx, wy = omega
        x = y = 0
        for mu in range(1, r_b + 1):
            odd = mu % 2 == 1
            src = (wx if odd else wy) if swap else (wy if odd else wx)
            region = (src // 3 ** ((mu + 1) // 2 - 1 + place_shift)) % 3
            edge = 1 << (mu - 1 + edge_shift)
            x += (region // 2) * edge
            y += (region - region // 2) * edge
        return MapResult(Coord2(x, y), reduction_depth(r_b))

    return broken


# ---------------------------------------------------------------------------
# intra-block strategies (§3.4, intra.py)
# ---------------------------------------------------------------------------

class IntraStrategy(enum.Enum):
    UNROLL = "unroll"
    TABLE = "table"
    SUBBOX = "subbox"
    TUNED = "tuned"  # B200 row-segment kernel: same cell set, HBM-shaped thread layout


#: the reference's three strategies (what its sweeps iterate over)
PAPER_STRATEGIES = (IntraStrategy.UNROLL, IntraStrategy.TABLE, IntraStrategy.SUBBOX)


@dataclass(frozen=True)
class LookupTable:
    entries: tuple[Coord2, ...]
    rho: int


def unroll_thread_map(t, rho: int) -> Coord2:
    return map_block(t, scale_level(rho)).coord


def build_lookup_table(rho: int) -> LookupTable:
    scale_level(rho)
    if rho > MAX_TABLE_EDGE:
        raise ValueError(f"lookup table capped at edge {MAX_TABLE_EDGE}, got {rho}")
    return LookupTable(entries=tuple(enumerate_cells(rho)), rho=rho)


def subbox_thread_map(t, rho: int) -> Optional[Coord2]:
    x, y = t
    if x < 0 or y < 0 or x >= rho or y >= rho:
        raise ValueError(f"thread {t!r} outside the {rho}x{rho} box")
    return None if x & (rho - 1 - y) else Coord2(x, y)


def threads_per_block(strategy: IntraStrategy, rho: int) -> int:
    if strategy is IntraStrategy.SUBBOX:
        return rho * rho
    if strategy is IntraStrategy.TUNED:
        # one thread per 16-byte row segment of an int8 tile (the headline cell
        # width); the kernel is persistent, so this is work items, not a CUDA block
        return rho * max(1, rho // 16)
    return volume(scale_level(rho))


def local_cells(strategy: IntraStrategy, rho: int) -> list[Coord2]:
    """The edge-rho tile's gasket cells (row-major) -- identical for every strategy."""
    k = scale_level(rho)
    if strategy is IntraStrategy.TABLE:
        return list(build_lookup_table(rho).entries)
    if strategy in (IntraStrategy.SUBBOX, IntraStrategy.TUNED):
        return [Coord2(x, y) for y in range(rho) for x in range(rho) if not (x & (rho - 1 - y))]
    width, height = packing_dims(k)
    cells = (unroll_thread_map((tx, ty), rho) for ty in range(height) for tx in range(width))
    return sorted(cells, key=lambda c: (c.y, c.x))
