"""CPU oracle for the lambda(omega) gasket hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker or the timed CPU baseline.  The product package
(``paper_1706_04552_b200``) never imports it and has no CPU fallback.

The arithmetic lives in ``gasket_oracle.c`` (OpenMP C restatement of the
reference numba kernels, each function citing its reference file:line).  This
module is a thin ctypes layer plus numpy restatements of the host-side helpers
the reference uses to build plans (``core.member_mask``, ``intra.local_cells``).

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against ``tests/golden/*`` (generated from the live reference by
``tests/golden/make_golden.py``) and, when ``/root/reference`` is mounted,
``tests/test_oracle_vs_reference.py`` checks it against the reference itself.
The 8-neighbour kernel (KIND_NSUM8) has no reference implementation: it is our
labelled extension (parity pinned by construction through the shared NSUM4
code path only).
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libgasket_oracle.so"

KIND_CONST = 0
KIND_NSUM4 = 1
KIND_NSUM8 = 2
STRAT_UNROLL = 0
STRAT_TABLE = 1
STRAT_SUBBOX = 2

SUPPORTED_DTYPES = (np.int8, np.uint8, np.int16, np.uint16, np.int32, np.uint32, np.int64)

_lib = None
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> Path:
    """Compile gasket_oracle.c with gcc (the checker, not the product)."""
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "gasket_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-s", "-B" if force else "all"], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, i32, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
        L.go_max_threads.restype = c_int
        L.go_map_blocks.argtypes = [_i64p, _i64p, i64, c_int, _i64p, _i64p, c_int]
        L.go_map_rectangle.argtypes = [c_int, _i64p, _i64p, c_int]
        L.go_run_bounding_box.argtypes = [vp, vp, i64, c_int, i64, c_int, i32, c_int]
        L.go_run_bounding_box.restype = c_int
        L.go_run_block_space.argtypes = [vp, vp, i64, c_int, i64, c_int, c_int, _i64p, _i64p, i64,
                                         c_int, i32, c_int]
        L.go_run_block_space.restype = c_int
        L.go_fill_hash.argtypes = [vp, i64, c_int, ctypes.c_uint64, c_int, c_int]
        L.go_checksum.argtypes = [vp, i64, c_int, c_int]
        L.go_steps_band.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(i32), c_int, i64, c_int, ctypes.c_uint64,
                                    c_int, c_int, i32, i64, i64, c_int]
        L.go_steps_band.restype = c_int
        L.go_checksum.restype = ctypes.c_uint64
        L.go_coverage_blocks.argtypes = [_i64p, _i64p, i64, _i64p, _i64p, i64, i64, i64, _i64p]
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().go_max_threads())


def _p64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def _check_grid(a: np.ndarray) -> int:
    if a.ndim != 2 or a.shape[0] != a.shape[1] or not a.flags.c_contiguous:
        raise ValueError("oracle grids must be square C-contiguous 2-D arrays")
    if a.dtype.type not in SUPPORTED_DTYPES:
        raise ValueError(f"unsupported cell dtype {a.dtype}")
    return a.dtype.itemsize


# ---------------------------------------------------------------------------
# core.py restatements (host helpers)
# ---------------------------------------------------------------------------

def packing_dims(r: int) -> tuple[int, int]:
    """core.py:64-72."""
    return 3 ** (r // 2), 3 ** ((r + 1) // 2)


def member_mask(n: int) -> np.ndarray:
    """core.py:84-91 (no size cap here: the oracle is the checker)."""
    xs = np.arange(n, dtype=np.int64)
    return (xs[None, :] & (n - 1 - xs)[:, None]) == 0


def enumerate_cells(n: int) -> list[tuple[int, int]]:
    """core.py:94-102 -- row-major gasket cells."""
    ys, xs = np.nonzero(member_mask(n))
    return [(int(x), int(y)) for x, y in zip(xs, ys)]


def map_block_scalar(wx: int, wy: int, r_b: int) -> tuple[int, int]:
    """blockmap.py:34-60, 70-88 (pure-Python loop; small cases only)."""
    x = y = 0
    for mu in range(1, r_b + 1):
        picked = wx * ((mu + 1) % 2) + wy * (mu % 2)
        region = (picked // 3 ** ((mu + 1) // 2 - 1)) % 3
        dx = region // 2
        step = 1 << (mu - 1)
        x += dx * step
        y += (region - dx) * step
    return x, y


def local_cells(strategy: int, rho: int) -> tuple[np.ndarray, np.ndarray]:
    """intra.py:76-91 + backends.py:113-118 -- block-local cells, row-major."""
    k = rho.bit_length() - 1
    if strategy == STRAT_TABLE:
        cells = enumerate_cells(rho)
    elif strategy == STRAT_SUBBOX:
        cells = [(x, y) for y in range(rho) for x in range(rho) if not (x & (rho - 1 - y))]
    else:
        w, h = packing_dims(k)
        cells = sorted((map_block_scalar(tx, ty, k) for ty in range(h) for tx in range(w)),
                       key=lambda c: (c[1], c[0]))
    lx = np.fromiter((c[0] for c in cells), dtype=np.int64, count=len(cells))
    ly = np.fromiter((c[1] for c in cells), dtype=np.int64, count=len(cells))
    return lx, ly


# ---------------------------------------------------------------------------
# kernels (C)
# ---------------------------------------------------------------------------

def map_blocks(wx: np.ndarray, wy: np.ndarray, r_b: int, threads: int = 0):
    """blockmap.py:91-108."""
    wx = np.ascontiguousarray(wx, dtype=np.int64)
    wy = np.ascontiguousarray(wy, dtype=np.int64)
    if wx.shape != wy.shape:
        raise ValueError("wx and wy must have the same shape")
    lx = np.empty_like(wx)
    ly = np.empty_like(wy)
    lib().go_map_blocks(_p64(wx), _p64(wy), wx.size, r_b, _p64(lx), _p64(ly), threads)
    return lx, ly


def map_rectangle(r_b: int, threads: int = 0):
    """lambda over the whole packed rectangle in b = wy*W + wx order."""
    w, h = packing_dims(r_b)
    lx = np.empty(w * h, dtype=np.int64)
    ly = np.empty(w * h, dtype=np.int64)
    lib().go_map_rectangle(r_b, _p64(lx), _p64(ly), threads)
    return lx, ly


def run_bounding_box(grid: np.ndarray, src: np.ndarray, rho: int, kind: int, param: int,
                     threads: int = 0) -> None:
    """backends.py:225-231 / 143-156."""
    c = _check_grid(grid)
    if src.shape != grid.shape or src.dtype != grid.dtype or not src.flags.c_contiguous:
        raise ValueError("src must match grid")
    rc = lib().go_run_bounding_box(grid.ctypes.data, src.ctypes.data, grid.shape[0], c, rho, kind,
                                   int(np.int32(param)), threads)
    if rc:
        raise ValueError("bad cell width")


def run_block_space(grid: np.ndarray, src: np.ndarray, rho: int, r_b: int, strategy: int,
                    local_x: np.ndarray | None, local_y: np.ndarray | None, kind: int, param: int,
                    threads: int = 0) -> None:
    """backends.py:234-272 / 158-222."""
    c = _check_grid(grid)
    if src.shape != grid.shape or src.dtype != grid.dtype or not src.flags.c_contiguous:
        raise ValueError("src must match grid")
    if local_x is None or strategy != STRAT_TABLE:
        local_x = local_y = np.zeros(1, dtype=np.int64)
    tx = np.ascontiguousarray(local_x, dtype=np.int64)
    ty = np.ascontiguousarray(local_y, dtype=np.int64)
    rc = lib().go_run_block_space(grid.ctypes.data, src.ctypes.data, grid.shape[0], c, rho, r_b,
                                  strategy, _p64(tx), _p64(ty), tx.size, kind,
                                  int(np.int32(param)), threads)
    if rc:
        raise ValueError("bad cell width")


def fill_hash(n: int, dtype, seed: int, mode: int = 0, threads: int = 0) -> np.ndarray:
    """splitmix64(seed ^ (y<<32 | x)) truncated to the cell width; mode 1 zeroes off-gasket cells."""
    a = np.empty((n, n), dtype=dtype)
    lib().go_fill_hash(a.ctypes.data, n, a.dtype.itemsize, seed & (2**64 - 1), mode, threads)
    return a


def steps_band(n: int, dtype, seed: int, mode: int, kind: int, param: int, y0: int, y1: int,
               steps, threads: int = 0) -> list[np.ndarray]:
    """Rows [y0, y1) of fill_hash(n, dtype, seed, mode) after each count in ``steps`` of
    engine.launch NEIGHBOR_SUM steps (engine.py:201 snapshot semantics, _cell_value
    backends.py:127-141 on the gasket cells, backends.py:155-156) -- the band restatement
    in gasket_oracle.c, for grids too large to hold whole on the host."""
    steps = [int(s) for s in steps]
    outs = [np.empty((y1 - y0, n), dtype=dtype) for _ in steps]
    ptrs = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    st = (ctypes.c_int32 * len(steps))(*steps)
    rc = lib().go_steps_band(ptrs, st, len(steps), n, np.dtype(dtype).itemsize, seed & (2**64 - 1), mode, kind,
                             int(np.int32(param)), y0, y1, threads)
    if rc == -2:
        raise MemoryError("steps_band window")
    if rc:
        raise ValueError("steps_band: bad arguments")
    return outs


def checksum(a: np.ndarray, threads: int = 0) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().go_checksum(a.ctypes.data, a.size, a.dtype.itemsize, threads))


def coverage_counts(bx: np.ndarray, by: np.ndarray, lx: np.ndarray, ly: np.ndarray, rho: int,
                    n: int) -> np.ndarray:
    """engine.py:245-251 counting leg."""
    counts = np.zeros((n, n), dtype=np.int64)
    bx, by, lx, ly = (np.ascontiguousarray(v, dtype=np.int64) for v in (bx, by, lx, ly))
    lib().go_coverage_blocks(_p64(bx), _p64(by), bx.size, _p64(lx), _p64(ly), lx.size, rho, n,
                             counts.ctypes.data_as(_i64p))
    return counts


def nsum_reference_numpy(grid: np.ndarray, src: np.ndarray, param: int, eight: bool) -> None:
    """Independent numpy restatement of the neighbour-sum write over all gasket
    cells (backends.py:67-80 generalised to any int width and to 8 neighbours),
    used to cross-check the C oracle in tests.  Mutates grid."""
    n = grid.shape[0]
    bits = grid.dtype.itemsize * 8
    mask = member_mask(n)
    s = src.astype(np.int64).astype(np.uint64)
    total = np.full((n, n), np.uint64(np.int64(np.int32(param)).astype(np.uint64)), dtype=np.uint64)
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    if eight:
        offs += [(1, 1), (1, -1), (-1, 1), (-1, -1)]
    pad = np.zeros((n + 2, n + 2), dtype=np.uint64)
    pad[1:-1, 1:-1] = s
    for dx, dy in offs:
        total += pad[1 + dy:1 + dy + n, 1 + dx:1 + dx + n]
    if bits < 64:
        total &= np.uint64((1 << bits) - 1)
    vals = total.astype(np.dtype(f"u{grid.dtype.itemsize}")).view(grid.dtype)
    grid[mask] = vals[mask]


__all__ = [
    "KIND_CONST", "KIND_NSUM4", "KIND_NSUM8", "STRAT_UNROLL", "STRAT_TABLE", "STRAT_SUBBOX",
    "build", "lib", "max_threads", "packing_dims", "member_mask", "enumerate_cells",
    "map_block_scalar", "local_cells", "map_blocks", "map_rectangle", "run_bounding_box",
    "run_block_space", "fill_hash", "steps_band", "checksum", "coverage_counts", "nsum_reference_numpy",
]
