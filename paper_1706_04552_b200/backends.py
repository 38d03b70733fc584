"""The drop-in boundary: ``run_bounding_box`` / ``run_block_space`` on the B200.

Same call signatures, integer tags and conventions as the reference plugin
point (``gasketmap/backends.py:225-272``; tags ``:30-34``; backend selection
``:20, 39-59``), but every launch goes through the C ABI of
``libgasket_b200.so`` (include/gasket_b200.h).  There is exactly one backend,
the sm_100a library; asking for the reference's CPU backends raises instead of
silently falling back.

Grids may be
  * CUDA tensors (int8/uint8/int16/uint16/int32/uint32/int64, n x n,
    contiguous): launched asynchronously on the current torch stream, or
  * numpy arrays: synchronous, like the reference (see device.py for the
    "copy" and "mapped" host transports).
``grid`` is mutated in place and only gasket cells are written; ``src`` is the
pre-launch snapshot.  If a neighbour-sum launch passes ``src`` aliasing
``grid`` (racy in the reference) it is snapshotted first, which is exactly the
``engine.launch`` semantics (engine.py:201).
"""

from __future__ import annotations

import os
from typing import Any, Optional

import numpy as np
import torch

from . import device, native
from .geometry import IntraStrategy, local_cells, packing_dims, scale_level

BACKEND_ENV = "GASKETMAP_BACKEND"
BACKEND = "cuda"
HAVE_NUMBA = False  # kept for import compatibility: no CPU kernels exist here

KERNEL_CONST = native.KIND_CONST
KERNEL_NEIGHBOR_SUM = native.KIND_NSUM4
KERNEL_NEIGHBOR_SUM8 = native.KIND_NSUM8
STRAT_UNROLL = native.STRAT_UNROLL
STRAT_TABLE = native.STRAT_TABLE
STRAT_SUBBOX = native.STRAT_SUBBOX
STRAT_TUNED = native.STRAT_TUNED

_STRAT_TAG = {
    IntraStrategy.UNROLL: STRAT_UNROLL,
    IntraStrategy.TABLE: STRAT_TABLE,
    IntraStrategy.SUBBOX: STRAT_SUBBOX,
    IntraStrategy.TUNED: STRAT_TUNED,
}

_EMPTY = np.empty(0, dtype=np.int64)


def resolve_backend(name: str | None = None) -> str:
    """'auto' / 'cuda' (or the env flag) -> 'cuda'.  The CPU backends do not exist here."""
    choice = (name or os.environ.get(BACKEND_ENV, "") or "auto").strip().lower()
    if choice in ("auto", "cuda", "b200", "sm_100a"):
        return BACKEND
    if choice in ("numba", "numpy"):
        raise RuntimeError(
            f"{choice} backend requested, but this package runs the gasket kernels only on the "
            "B200 (sm_100a); there is no CPU backend")
    raise ValueError(f"unknown backend {choice!r} (expected cuda or auto)")


def set_workers(workers: int | None) -> None:
    """Accepted for API compatibility; device launches size themselves to the SMs."""
    return None


def local_cell_arrays(strategy: IntraStrategy, rho: int) -> tuple[np.ndarray, np.ndarray]:
    cells = local_cells(strategy, rho)
    lx = np.array([c.x for c in cells], dtype=np.int64)
    ly = np.array([c.y for c in cells], dtype=np.int64)
    return lx, ly


# ---------------------------------------------------------------------------
# argument plumbing
# ---------------------------------------------------------------------------

_table_cache: dict[tuple, tuple[torch.Tensor, torch.Tensor]] = {}


def _device_table(local_x, local_y, rho: int) -> tuple[int, int, int]:
    """Upload a TABLE lookup table once (cached by content); returns (px, py, count)."""
    lx = np.ascontiguousarray(local_x, dtype=np.int64).reshape(-1)
    ly = np.ascontiguousarray(local_y, dtype=np.int64).reshape(-1)
    if lx.shape != ly.shape:
        raise ValueError("local_x and local_y must have the same length")
    if lx.size and (lx.min() < 0 or ly.min() < 0 or lx.max() >= rho or ly.max() >= rho):
        raise ValueError(f"lookup table entries must lie inside the {rho}x{rho} tile")
    key = (torch.cuda.current_device(), rho, lx.tobytes(), ly.tobytes())
    hit = _table_cache.get(key)
    if hit is None:
        hit = (torch.from_numpy(lx.astype(np.int32)).cuda(), torch.from_numpy(ly.astype(np.int32)).cuda())
        if len(_table_cache) > 64:
            _table_cache.clear()
        _table_cache[key] = hit
    # a table dropped from the cache later must outlive the launches that read it
    cur = torch.cuda.current_stream()
    hit[0].record_stream(cur)
    hit[1].record_stream(cur)
    return int(hit[0].data_ptr()), int(hit[1].data_ptr()), int(lx.size)


def _param32(param) -> int:
    return int(np.int32(param))  # OverflowError for out-of-range, like np.int32(param) at backends.py:229


def _strategy_tag(strategy) -> int:
    if isinstance(strategy, IntraStrategy):
        return _STRAT_TAG[strategy]
    tag = int(strategy)
    if tag not in (STRAT_UNROLL, STRAT_TABLE, STRAT_SUBBOX, STRAT_TUNED):
        raise ValueError(f"unknown intra-block strategy {strategy!r}")
    return tag


def _shares_memory(a: Any, b: Any) -> bool:
    if a is b:
        return True
    if isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor):
        return a.data_ptr() == b.data_ptr()
    if isinstance(a, np.ndarray) and isinstance(b, np.ndarray):
        return np.shares_memory(a, b)
    return False


def _same_array(a: Any, b: Any) -> bool:
    """Both numpy arrays over exactly the same memory (same start, shape and strides)."""
    return (isinstance(a, np.ndarray) and isinstance(b, np.ndarray) and a.ctypes.data == b.ctypes.data
            and a.shape == b.shape and a.strides == b.strides)


def _run(grid: Any, src: Any, kind: int, launch, *, mapped_ok: bool, inplace: Optional[Any] = None,
         banded: Optional[Any] = None) -> None:
    """Route one launch: device tensors directly, numpy through a host transport.

    ``launch(grid_ptr, src_ptr, n, cell_bytes, stream, extra_flags)`` issues the C-ABI call.
    In the mapped (zero-copy) transport the kernel is asked for whole-sector
    writes (``FLAG_EXPLICIT_RMW``): PCIe cannot carry byte-masked partial lines
    efficiently, so partial sectors are read, blended and written back whole.

    ``inplace(grid)``: the in-place form of a neighbour-sum launch whose src is the grid
    itself (device.run_inplace, the tuned kernel only); otherwise such a launch reads a
    masked snapshot of the grid (engine.py:201).  ``banded(dst, snap, n, c, t0, t1,
    stream)``: the tuned step over a tile range, for the banded staged host path."""
    device.require_cuda()
    n = device.check_square(grid)
    c = device.cell_bytes_of(grid)
    reads_src = kind in (KERNEL_NEIGHBOR_SUM, KERNEL_NEIGHBOR_SUM8)
    if src is None:
        src = grid
    if reads_src:
        if tuple(src.shape) != tuple(grid.shape) or device.cell_bytes_of(src) != c:
            raise ValueError("src must have the grid's shape and dtype")
    stream = device.stream_handle()

    if device.is_device(grid):
        src_dev = src
        if reads_src:
            if not device.is_device(src):
                src_dev = torch.from_numpy(np.ascontiguousarray(src)).to(grid.device, non_blocking=True)
            elif _shares_memory(src, grid):
                if (inplace is not None and src.data_ptr() == grid.data_ptr() and src.stride() == grid.stride()
                        and device.inplace_ok(n, c)):
                    inplace(grid)  # engine.py:201's semantics, the snapshot reduced to tile borders
                    return
                src_dev = device.stencil_snapshot(grid)  # engine.py:201's snapshot, masked
                # the grid and its snapshot agree off the gasket: stencils may blend from src
                launch(device.data_ptr(grid), device.data_ptr(src_dev), n, c, stream, native.FLAG_DST_FROM_SRC)
                return
            else:
                device.check_square(src, "src")
        launch(device.data_ptr(grid), device.data_ptr(src_dev) if reads_src else 0, n, c, stream, 0)
        return

    if not isinstance(grid, np.ndarray):
        raise TypeError(f"grid must be a CUDA tensor or a numpy array, got {type(grid).__name__}")
    if not grid.flags.writeable:
        raise ValueError("grid is read-only")
    mode = device.host_transport()
    if (mode == "mapped" and mapped_ok and reads_src and _same_array(src, grid)
            and device.staged_writeback_ok(n, c)):
        # engine.launch semantics on a host grid (src is the grid: its pre-launch snapshot):
        # stage only what the launch reads (the member tiles' windows) into the device,
        # run the tuned kernel there, write the tiles' own lines back whole -- the host
        # sees whole-line traffic for the dilated gasket instead of 16-byte pieces
        tdtype = device._torch_dtype(grid.dtype)
        # (scratch per stream: host calls made from several threads on their own streams)
        snap = device.scratch.get(f"host_snap:{stream}", n * n, tdtype).view(n, n)
        dst = device.scratch.get(f"host_dst:{stream}", n * n, tdtype).view(n, n)
        with device.MappedHost(grid) as gptr:
            if banded is not None and c in (1, 2, 4):
                # in bands of block rows: band b's write-back (device -> host) runs on a side
                # stream next to band b+2's snapshot (host -> device), the two PCIe directions
                # at once.  Band b+1's snapshot precedes band b's step and write-back: it holds
                # the rows band b reads below itself and the pre-launch values band b's
                # write-back would overwrite.
                bands = device.staged_bands(n, c)
                main, side = torch.cuda.current_stream(), device.side_stream()
                side.wait_stream(main)
                sh = device.stream_handle(side)
                native.call("gm_snapshot_stencil_range", snap.data_ptr(), gptr, n, c, *bands[0], stream)
                for b, (t0, t1) in enumerate(bands):
                    if b + 1 < len(bands):
                        native.call("gm_snapshot_stencil_range", snap.data_ptr(), gptr, n, c, *bands[b + 1], stream)
                    banded(dst.data_ptr(), snap.data_ptr(), n, c, t0, t1, stream)
                    ev = torch.cuda.Event()
                    ev.record(main)
                    side.wait_event(ev)
                    native.call("gm_writeback_tiles_range", gptr, dst.data_ptr(), snap.data_ptr(), n, c, t0, t1, sh)
                main.wait_stream(side)
            else:
                native.call("gm_snapshot_stencil", snap.data_ptr(), gptr, n, c, stream)
                launch(dst.data_ptr(), snap.data_ptr(), n, c, stream, native.FLAG_DST_FROM_SRC)
                native.call("gm_writeback_tiles", gptr, dst.data_ptr(), snap.data_ptr(), n, c, stream)
            torch.cuda.current_stream().synchronize()
        return
    if mode == "mapped" and mapped_ok and not (reads_src and _shares_memory(src, grid)):
        src_host = np.ascontiguousarray(src) if reads_src else None
        with device.MappedHost(grid) as gptr:
            if src_host is None:
                launch(gptr, 0, n, c, stream, device.host_flags())
            else:
                with device.MappedHost(src_host) as sptr:
                    launch(gptr, sptr, n, c, stream, device.host_flags())
            torch.cuda.current_stream().synchronize()
        return

    tdtype = device._torch_dtype(grid.dtype)
    dev_grid = device.scratch.get(f"host_grid:{stream}", n * n, tdtype).view(n, n)
    host_grid = torch.from_numpy(grid)
    dev_grid.copy_(host_grid, non_blocking=True)
    src_ptr = 0
    if reads_src:
        if _shares_memory(src, grid):
            dev_src = device.stencil_snapshot(dev_grid)
        else:
            dev_src = device.scratch.get(f"host_src:{stream}", n * n, tdtype).view(n, n)
            dev_src.copy_(torch.from_numpy(np.ascontiguousarray(src)), non_blocking=True)
        src_ptr = dev_src.data_ptr()
    launch(dev_grid.data_ptr(), src_ptr, n, c, stream, 0)
    host_grid.copy_(dev_grid, non_blocking=True)
    torch.cuda.current_stream().synchronize()


# ---------------------------------------------------------------------------
# the reference plugin API
# ---------------------------------------------------------------------------

def run_bounding_box(grid, src, rho: int, kind: int, param: int, backend: str = BACKEND, *,
                     early_exit: bool = False, vectorized: bool = False) -> None:
    """backends.py:225-231: identity map over n_b x n_b blocks of rho x rho threads,
    each thread testing x & (n-1-y) (``early_exit``: whole tiles off the gasket exit first).

    ``vectorized``: the bounding box written like the tuned lambda kernels, the competent
    BB baseline of the lambda-vs-BB speed-up (rho does not shape this launch) -- the write
    pass as one lane per 16-byte segment of all n x n cells with the tuned kernels' stores,
    neighbour sums as the tuned tile stencil over every tile of the grid, tiles off the
    gasket exiting after one membership test."""
    resolve_backend(backend)
    p = _param32(param)
    kind = int(kind)
    variant = 2 if vectorized else (1 if early_exit else 0)

    def launch(gp, sp, n, c, stream, extra_flags):
        native.call("gm_run_bounding_box", gp, sp, n, c, int(rho), kind, p, variant, stream)

    _run(grid, src, kind, launch, mapped_ok=False)


def run_block_space(grid, src, rho: int, r_b: int, strategy, local_x: Optional[np.ndarray] = None,
                    local_y: Optional[np.ndarray] = None, kind: int = KERNEL_CONST, param: int = 1,
                    backend: str = BACKEND, *, flags: int = 0, assume_zero_background: bool = False) -> None:
    """backends.py:234-272: lambda over the packed rectangle of level r_b, then the
    intra-block strategy.  ``local_x/local_y`` are the TABLE lookup table
    (ignored by the other strategies, as in the numba leg).

    ``assume_zero_background`` (tuned constant write pass only, off by default): the
    caller asserts that every off-gasket cell of ``grid`` is 0 -- the paper's
    zero-filled matrix and the reference bench's ``make_grid``
    zeros re-written in place (engine.py:88-90, bench.py:145-150).  The kernel then
    stores every touched 32-byte sector whole (gasket cells = param, the rest 0),
    which leaves the same grid without the DRAM read-modify-write of partial
    sectors.  On a grid with a nonzero background the off-gasket cells of touched
    sectors would be zeroed, so it is never implied."""
    resolve_backend(backend)
    tag = _strategy_tag(strategy)
    p = _param32(param)
    kind = int(kind)
    if assume_zero_background:
        if kind != KERNEL_CONST or tag != STRAT_TUNED:
            raise ValueError("assume_zero_background applies to the tuned constant write pass only")
        flags = int(flags) | native.FLAG_ZERO_BACKGROUND
    packing_dims(int(r_b))  # level range check
    tx = ty = 0
    ntab = 0
    if tag == STRAT_TABLE:
        if local_x is None or local_y is None:
            local_x, local_y = local_cell_arrays(IntraStrategy.TABLE, int(rho))
        device.require_cuda()
        tx, ty, ntab = _device_table(local_x, local_y, int(rho))

    def launch(gp, sp, n, c, stream, extra_flags):
        native.call("gm_run_block_space", gp, sp, n, c, int(rho), int(r_b), tag, tx, ty, ntab, kind, p,
                    int(flags) | extra_flags, stream)

    inplace = banded = None
    if tag == STRAT_TUNED and kind in (KERNEL_NEIGHBOR_SUM, KERNEL_NEIGHBOR_SUM8):
        inplace = lambda g: device.run_inplace(g, kind, p)  # noqa: E731

        def banded(gp, sp, n, c, t0, t1, stream):
            native.call("gm_run_tiles", gp, sp, n, c, kind, p, int(flags) | native.FLAG_DST_FROM_SRC, t0, t1, stream)
    _run(grid, src, kind, launch, mapped_ok=(tag == STRAT_TUNED), inplace=inplace, banded=banded)


__all__ = [
    "BACKEND_ENV", "HAVE_NUMBA", "KERNEL_CONST", "KERNEL_NEIGHBOR_SUM", "KERNEL_NEIGHBOR_SUM8",
    "STRAT_UNROLL", "STRAT_TABLE", "STRAT_SUBBOX", "STRAT_TUNED", "resolve_backend", "set_workers",
    "local_cell_arrays", "run_bounding_box", "run_block_space", "scale_level",
]
