"""ctypes binding of libgasket_b200.so (include/gasket_b200.h).

The library is the product: there is no CPU fallback.  If the in-tree
``_lib/libgasket_b200.so`` is missing this module raises on first use
(run ``python -m paper_1706_04552_b200._build`` or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from . import _build

import os

# GASKET_B200_LIB: load another build of the same ABI (A/B kernel experiments)
LIB_PATH: Path = Path(os.environ["GASKET_B200_LIB"]) if os.environ.get("GASKET_B200_LIB") else _build.LIB

GM_OK, GM_EINVAL, GM_ECUDA, GM_ENOMEM = 0, 1, 2, 3

KIND_CONST, KIND_NSUM4, KIND_NSUM8, KIND_COUNT = 0, 1, 2, 3
STRAT_UNROLL, STRAT_TABLE, STRAT_SUBBOX, STRAT_TUNED = 0, 1, 2, 3
MAP_BB, MAP_LAMBDA, MAP_BB_EXIT, MAP_BB_VEC = 0, 1, 2, 3
FLAG_OMEGA_ORDER, FLAG_DST_FROM_SRC, FLAG_EXPLICIT_RMW, FLAG_WHOLE_LINES, FLAG_HOST_ROWS = 1, 2, 4, 8, 16
FLAG_ROWMAJOR, FLAG_CHUNKED, FLAG_NO_TMA, FLAG_FORCE_TMA = 32, 64, 128, 256
FLAG_FETCH_LINE, FLAG_FETCH64, FLAG_STENCIL_V1, FLAG_STAGES2 = 512, 1024, 2048, 4096
FLAG_PROBE_NOSTORE, FLAG_PROBE_NOLOAD, FLAG_PROBE_NOCOMPUTE = 8192, 16384, 32768
FLAG_DIGIT_ORDER, FLAG_STORE_CS, FLAG_BAND_MAJOR = 65536, 131072, 262144
FLAG_PREFETCH_AHEAD, FLAG_FETCH_MIXED, FLAG_FETCH_HALF, FLAG_FETCH256 = 524288, 1048576, 2097152, 4194304
FLAG_TWO_STEPS = 8388608
FLAG_FOUR_STEPS = 16777216
FLAG_SIX_STEPS = 33554432
FLAG_ZERO_BACKGROUND, FLAG_GRID_ROWS = 67108864, 536870912
FLAG_WRITE_HALVES, FLAG_WRITE_LINES, FLAG_WRITE_SWEEP = 134217728, 268435456, 1073741824
FLAG_STATIC_SCHEDULE = 4096  # write pass only (the stencil reads the same bit as FLAG_STAGES2)


class GmCfg(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("rho", ctypes.c_int32),
        ("mapping", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("cell_bytes", ctypes.c_int32),
        ("param", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib: ctypes.CDLL | None = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64

_SIGS = {
    "gm_run_bounding_box": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp],
    "gm_run_block_space": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _vp],
    "gm_launch": [ctypes.POINTER(GmCfg), _vp, _vp, _vp, _vp, _i32, _vp],
    "gm_map_blocks": [_vp, _vp, _i64, _i32, _vp, _vp, _vp],
    "gm_map_rectangle": [_i32, _vp, _vp, _vp],
    "gm_coverage": [ctypes.POINTER(GmCfg), _vp, _vp, _vp, _i32, _vp],
    "gm_coverage_blocks": [_vp, _vp, _i64, _vp, _vp, _i32, _i32, _i64, _vp, _vp],
    "gm_bijection_check": [_vp, _vp, _i64, _i64, _vp, _vp, _vp],
    "gm_snapshot_stencil": [_vp, _vp, _i64, _i32, _vp],
    "gm_writeback_tiles": [_vp, _vp, _vp, _i64, _i32, _vp],
    "gm_fill_hash": [_vp, _i64, _i32, _u64, _i32, _vp],
    "gm_checksum": [_vp, _i64, _i32, _vp, _vp],
    "gm_count_equal": [_vp, _vp, _i64, _i32, _vp, _vp],
    "gm_l2_flush": [_vp, _i64, _vp, _vp],
    "gm_host_map": [_vp, _i64, _i32, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int32)],
    "gm_host_unmap": [_vp],
    "gm_set_l2_fetch_granularity": [_i32],
    "gm_run_part": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_gather_cells": [_vp, _i32, _vp, _i64, _vp, _vp],
    "gm_scatter_cells": [_vp, _i32, _vp, _i64, _vp, _vp],
    "gm_tile_order": [_i32, _i32, _vp, _i64],
    "gm_ca_step2": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp],
    "gm_ca_steps": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp],
    "gm_run_part2": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_run_part_steps": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_run_part_peer": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp, _u64,
                         _u64, _vp],
    "gm_dev_alloc": [_i64, ctypes.POINTER(ctypes.c_void_p)],
    "gm_dev_free": [_vp],
    "gm_ipc_get_handle": [_vp, _vp],
    "gm_ipc_open_handle": [_vp, ctypes.POINTER(ctypes.c_void_p)],
    "gm_ipc_close": [_vp],
    "gm_peer_halo_put": [_vp, _vp, _vp, _i64, _i32, _vp, _i32, _i32, _u64, _vp],
    "gm_peer_halo_put_to": [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _i32, _u64, _vp],
    "gm_run_part_tiled": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp, _i64,
                          _vp, _u64, _u64, _vp, _vp],
    "gm_copy_cells": [_vp, _vp, _i32, _vp, _vp, _i64, _vp],
    "gm_fill_hash_window": [_vp, _i64, _i64, _i32, _i64, _i64, _i64, _i64, _u64, _i32, _vp],
    "gm_peer_halo_wait": [_vp, _i32, _i32, _u64, _u64, _vp, _vp],
    "gm_ca_edge_bytes": [_i64, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_int64)],
    "gm_ca_edge_build": [_vp, _vp, _i64, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp, _i64, _vp],
    "gm_ca_run": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp],
    "gm_border_bytes": [_i64, _i32, ctypes.POINTER(ctypes.c_int64)],
    "gm_coverage_check": [_vp, _i64, _vp, _vp, _vp, _i64, _vp],
    "gm_snapshot_stencil_range": [_vp, _vp, _i64, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_writeback_tiles_range": [_vp, _vp, _vp, _i64, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_run_tiles": [_vp, _vp, _i64, _i32, _i32, _i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp],
    "gm_run_inplace": [_vp, _vp, _i64, _i32, _i32, _i32, _vp],
}

# Every symbol include/gasket_b200.h declares (checked by tests/test_native_abi.py).
EXPORTED = tuple(_SIGS) + ("gm_launch_count", "gm_last_error", "gm_version")


class GasketError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load the sm_100a library; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise GasketError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -m paper_1706_04552_b200._build); there is no CPU fallback")
        L = ctypes.CDLL(str(LIB_PATH))
        ab_build = bool(os.environ.get("GASKET_B200_LIB"))
        for name, args in _SIGS.items():
            if ab_build and not hasattr(L, name):
                continue  # an older build under A/B comparison: entry points it predates stay unbound
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.gm_launch_count.restype = ctypes.c_uint64
        L.gm_launch_count.argtypes = []
        L.gm_last_error.restype = ctypes.c_char_p
        L.gm_last_error.argtypes = []
        L.gm_version.restype = ctypes.c_char_p
        L.gm_version.argtypes = []
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a GM_E* return code onto the reference's exception types."""
    if rc == GM_OK:
        return
    msg = lib().gm_last_error().decode(errors="replace")
    if rc == GM_EINVAL:
        raise ValueError(msg)
    raise GasketError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().gm_launch_count())


def version() -> str:
    return lib().gm_version().decode()


def ca_edge_bytes(n: int, cell_bytes: int, level: int = -1, sg_begin: int = 0, sg_end: int = 0) -> int:
    """Size of the static left-edge cache of a CA run (gm_ca_edge_bytes)."""
    out = ctypes.c_int64(0)
    check(lib().gm_ca_edge_bytes(n, cell_bytes, level, sg_begin, sg_end, ctypes.byref(out)))
    return int(out.value)


def border_bytes(n: int, cell_bytes: int) -> int:
    """Size of the border-cell buffer of an in-place neighbour-sum launch (gm_border_bytes)."""
    out = ctypes.c_int64(0)
    check(lib().gm_border_bytes(n, cell_bytes, ctypes.byref(out)))
    return int(out.value)


def tile_order(q: int, level: int = 0):
    """The tuned kernels' tile visiting order (gm_tile_order): (bx, by) int64 arrays."""
    import numpy as np

    out = np.zeros(3**q, dtype=np.uint32)
    check(lib().gm_tile_order(q, level, out.ctypes.data, out.size))
    return (out & 0xFFFF).astype(np.int64), (out >> 16).astype(np.int64)
