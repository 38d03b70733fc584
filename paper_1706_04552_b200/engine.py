"""Launch engine: LaunchConfig -> prepare -> LaunchPlan.run, work counters, coverage audit.

Mirrors the reference engine API (``gasketmap/engine.py``: enums :25-41,
LaunchConfig :44-54, WorkMetrics :57-65, CoverageReport/Error :68-85,
make_grid :88-90, work_counts :93-137, LaunchPlan/prepare/launch :146-211,
verify_coverage :214-258) on top of the sm_100a library.  Differences, all
additive: a block-early-exit BB mapping, the TUNED strategy, the 8-neighbour
kernel, device-resident grids (``make_grid`` returns a CUDA tensor), and a
coverage audit that counts the writes of the real kernels on the GPU.
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import torch

from . import backends, device, native
from .geometry import (
    ORACLE_MAX_EDGE,
    Coord2,
    FractalSpec,
    IntraStrategy,
    MapResult,
    packing_dims,
    reduction_depth,
    threads_per_block,
    volume,
)


class Mapping(enum.Enum):
    BOUNDING_BOX = "bb"
    BLOCK_SPACE = "blockspace"
    BOUNDING_BOX_EXIT = "bb-exit"  # BB whose off-gasket tiles exit before any per-thread test
    BOUNDING_BOX_VEC = "bb-vec"  # BB written like the tuned kernels (16-byte segments / every tile of the grid)


class KernelKind(enum.Enum):
    CONST = "const"
    NEIGHBOR_SUM = "neighbor-sum"
    NEIGHBOR_SUM8 = "neighbor-sum8"  # Moore neighbourhood (our extension)


_KIND_TAG = {KernelKind.CONST: backends.KERNEL_CONST, KernelKind.NEIGHBOR_SUM: backends.KERNEL_NEIGHBOR_SUM,
             KernelKind.NEIGHBOR_SUM8: backends.KERNEL_NEIGHBOR_SUM8}
_BB_MAPPINGS = (Mapping.BOUNDING_BOX, Mapping.BOUNDING_BOX_EXIT, Mapping.BOUNDING_BOX_VEC)


@dataclass(frozen=True)
class CellKernel:
    """Write ``param``, or ``param`` plus the 4- (8-) neighbour sum of the pre-launch
    snapshot with out-of-grid neighbours reading 0; results wrap to the cell width."""

    kind: KernelKind = KernelKind.CONST
    param: int = 1


@dataclass(frozen=True)
class LaunchConfig:
    spec: FractalSpec
    mapping: Mapping
    strategy: Optional[IntraStrategy] = None
    kernel: CellKernel = CellKernel()
    verify_coverage: bool = False

    def __post_init__(self) -> None:
        if self.mapping is Mapping.BLOCK_SPACE and self.strategy is None:
            raise ValueError("block-space launches need an intra-block strategy")


@dataclass
class WorkMetrics:
    blocks_launched: int
    threads_launched: int
    threads_useful: int
    map_ops: int
    reduction_depth: int
    simulated_cost: int
    wall_ns: float = 0.0


@dataclass
class CoverageReport:
    counts: object  # numpy int64 (n, n) for n <= 2^13, else a CUDA int32 tensor
    duplicates: list[Coord2]
    misses: list[Coord2]

    @property
    def exact(self) -> bool:
        return not (self.duplicates or self.misses)


class CoverageError(RuntimeError):
    def __init__(self, report: CoverageReport):
        super().__init__(
            f"coverage violated: {len(report.duplicates)} over-written, {len(report.misses)} missed")
        self.report = report


def make_grid(n: int, dtype: torch.dtype = torch.int32) -> torch.Tensor:
    """Zeroed n x n device grid (int32 cells by default, like the reference)."""
    device.require_cuda()
    return torch.zeros((n, n), dtype=dtype, device="cuda")


# ---------------------------------------------------------------------------
# the cost model (engine.py:93-137), extended to the TUNED strategy
# ---------------------------------------------------------------------------

def _intra_ops(strategy: IntraStrategy, rho: int) -> int:
    if rho == 1:
        return 0  # one thread per block: every strategy is the identity
    k = rho.bit_length() - 1
    per_strategy = {
        IntraStrategy.UNROLL: volume(k) * k,   # each of 3^k threads re-sums k offsets
        IntraStrategy.TABLE: volume(k),        # one table read per thread
        IntraStrategy.SUBBOX: rho * rho,       # one membership test per boxed thread
        IntraStrategy.TUNED: threads_per_block(IntraStrategy.TUNED, rho),  # one test per row segment
    }
    return per_strategy[strategy]


def work_counts(spec: FractalSpec, mapping: Mapping, strategy: Optional[IntraStrategy] = None) -> WorkMetrics:
    useful = volume(spec.r)
    if mapping in _BB_MAPPINGS:
        blocks = spec.n_b * spec.n_b
        threads = blocks * spec.rho * spec.rho
        return WorkMetrics(blocks, threads, useful, threads, 0, threads + useful)
    if strategy is None:
        raise ValueError("block-space launches need an intra-block strategy")
    blocks = volume(spec.r_b)
    threads = blocks * threads_per_block(strategy, spec.rho)
    ops = blocks * (spec.r_b + _intra_ops(strategy, spec.rho))
    return WorkMetrics(blocks, threads, useful, ops, reduction_depth(spec.r_b), ops + useful)


def simulated_cost(spec: FractalSpec, mapping: Mapping, strategy: Optional[IntraStrategy] = None) -> int:
    return work_counts(spec, mapping, strategy).simulated_cost


# ---------------------------------------------------------------------------
# plans
# ---------------------------------------------------------------------------

@dataclass
class LaunchPlan:
    """A configuration bound to the device library; the TABLE lookup table is
    built (and uploaded) once, lambda is recomputed on every run."""

    config: LaunchConfig
    backend: str
    local_x: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    local_y: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    flags: int = 0

    def run(self, grid, src) -> None:
        cfg = self.config
        tag = _KIND_TAG[cfg.kernel.kind]
        if cfg.mapping in _BB_MAPPINGS:
            backends.run_bounding_box(grid, src, cfg.spec.rho, tag, cfg.kernel.param, self.backend,
                                      early_exit=cfg.mapping is Mapping.BOUNDING_BOX_EXIT,
                                      vectorized=cfg.mapping is Mapping.BOUNDING_BOX_VEC)
        else:
            backends.run_block_space(grid, src, cfg.spec.rho, cfg.spec.r_b, cfg.strategy, self.local_x,
                                     self.local_y, tag, cfg.kernel.param, self.backend, flags=self.flags)


def prepare(config: LaunchConfig, backend: Optional[str] = None) -> LaunchPlan:
    plan = LaunchPlan(config, backends.resolve_backend(backend))
    if config.mapping is Mapping.BLOCK_SPACE and config.strategy is IntraStrategy.TABLE:
        plan.local_x, plan.local_y = backends.local_cell_arrays(config.strategy, config.spec.rho)
    return plan


def _is_int32(grid) -> bool:
    if isinstance(grid, torch.Tensor):
        return grid.dtype == torch.int32
    return isinstance(grid, np.ndarray) and grid.dtype == np.int32


def launch(config: LaunchConfig, grid, backend: Optional[str] = None) -> WorkMetrics:
    """One launch, mutating ``grid``; returns the work counters and the device time."""
    n = config.spec.n
    if tuple(grid.shape) != (n, n) or not _is_int32(grid):
        raise ValueError(f"grid must be int32 of shape ({n}, {n}), got {grid.dtype} {tuple(grid.shape)}")
    plan = prepare(config, backend)
    neighbour = config.kernel.kind is not KernelKind.CONST
    if neighbour:
        # engine.py:201 (src = grid.copy()).  The launch gets src = grid and the backend keeps
        # the semantics: on the device the tuned kernel runs in place with a snapshot of the
        # tiles' border cells only (device.run_inplace), the other strategies read a masked
        # snapshot of the cells they read (device.stencil_snapshot); a host grid takes the
        # staged path (masked snapshot over PCIe, device step, write-back) instead of a
        # grid-sized host copy
        src = grid
        # grid and its snapshot agree off the gasket: stencils may blend from src
        plan.flags |= native.FLAG_DST_FROM_SRC
    else:
        src = grid
    if isinstance(grid, torch.Tensor):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        plan.run(grid, src)
        stop.record()
        stop.synchronize()
        wall = start.elapsed_time(stop) * 1e6
    else:
        t0 = time.perf_counter_ns()
        plan.run(grid, src)
        wall = float(time.perf_counter_ns() - t0)
    metrics = work_counts(config.spec, config.mapping, config.strategy)
    metrics.wall_ns = float(wall)
    if config.verify_coverage:
        report = verify_coverage(config)
        if not report.exact:
            raise CoverageError(report)
    return metrics


# ---------------------------------------------------------------------------
# coverage audit on the device
# ---------------------------------------------------------------------------

def _coverage_counts(config: LaunchConfig, map_fn) -> torch.Tensor:
    spec = config.spec
    n = spec.n
    counts = torch.zeros((n, n), dtype=torch.int32, device="cuda")
    stream = device.stream_handle()
    strategy = config.strategy or IntraStrategy.SUBBOX
    if map_fn is None:
        cfg = native.GmCfg()
        cfg.n, cfg.rho, cfg.cell_bytes = n, spec.rho, 4
        cfg.kind = native.KIND_COUNT
        if config.mapping in _BB_MAPPINGS:
            # (the vectorised BB covers exactly the cells of the literal one: audited as that)
            cfg.mapping = native.MAP_BB_EXIT if config.mapping is Mapping.BOUNDING_BOX_EXIT else native.MAP_BB
            cfg.strategy = native.STRAT_SUBBOX
            tx = ty = ntab = 0
        else:
            cfg.mapping = native.MAP_LAMBDA
            cfg.strategy = backends._strategy_tag(strategy)
            tx = ty = ntab = 0
            if strategy is IntraStrategy.TABLE:
                lx, ly = backends.local_cell_arrays(strategy, spec.rho)
                tx, ty, ntab = backends._device_table(lx, ly, spec.rho)
        native.check(native.lib().gm_coverage(cfg, counts.data_ptr(), tx, ty, ntab, stream))
        return counts
    width, height = packing_dims(spec.r_b)
    coords = [map_fn((wx, wy), spec.r_b).coord for wy in range(height) for wx in range(width)]
    bx = torch.tensor([c[0] for c in coords], dtype=torch.int64, device="cuda")
    by = torch.tensor([c[1] for c in coords], dtype=torch.int64, device="cuda")
    lx, ly = backends.local_cell_arrays(strategy, spec.rho)
    tlx = torch.from_numpy(lx.astype(np.int32)).cuda()
    tly = torch.from_numpy(ly.astype(np.int32)).cuda()
    native.call("gm_coverage_blocks", bx.data_ptr(), by.data_ptr(), bx.numel(), tlx.data_ptr(), tly.data_ptr(),
                tlx.numel(), spec.rho, n, counts.data_ptr(), stream)
    return counts


def _coverage_compare(counts: torch.Tensor, n: int) -> tuple[list, list]:
    """Duplicates and misses of the counters (engine.py:252-258), row-major like the
    reference's np.argwhere: one device pass (gm_coverage_check) that counts them, and a
    second that collects their indices when there are any -- no n^2 temporaries."""
    if n == 1:
        c = int(counts.reshape(-1)[0].item())
        return ([Coord2(0, 0)] if c > 1 else []), ([Coord2(0, 0)] if c == 0 else [])
    stream = device.stream_handle()
    totals = torch.zeros(2, dtype=torch.int64, device="cuda")
    native.call("gm_coverage_check", counts.data_ptr(), n, totals.data_ptr(), None, None, 0, stream)
    nd, nm = (int(v) for v in totals.cpu().tolist())
    if nd == 0 and nm == 0:
        return [], []
    cap = max(nd, nm)
    di = torch.empty(cap, dtype=torch.int64, device="cuda")
    mi = torch.empty(cap, dtype=torch.int64, device="cuda")
    native.call("gm_coverage_check", counts.data_ptr(), n, totals.data_ptr(), di.data_ptr(), mi.data_ptr(), cap,
                stream)
    out = []
    for idx, k in ((di, nd), (mi, nm)):
        lin = torch.sort(idx[:k]).values.cpu().numpy()
        out.append([Coord2(int(i % n), int(i // n)) for i in lin])
    return out[0], out[1]


def verify_coverage(config: LaunchConfig,
                    map_fn: Optional[Callable[[tuple[int, int], int], MapResult]] = None) -> CoverageReport:
    """Per-cell write counters of the launch shape; duplicates = cells written more
    often than their membership allows, misses = gasket cells never written."""
    device.require_cuda()
    n = config.spec.n
    counts = _coverage_counts(config, map_fn)
    dups, miss = _coverage_compare(counts, n)
    out = counts.cpu().numpy().astype(np.int64) if n <= ORACLE_MAX_EDGE else counts
    return CoverageReport(counts=out, duplicates=dups, misses=miss)
