"""Sweep harness over (scale level, block edge, mapping, strategy) on the B200.

Same CSV schema, record type, skip statuses and atomic write as the reference
(``gasketmap/bench.py``: CSV_HEADER :25-29, SweepConfig :35-46, BenchRecord
:49-66, formatting :69-93, write/read :96-139, _time_plan :142-154,
run_sweep :166-232).  Timing is on the device: each sub-average brackets
``inner`` back-to-back launches with CUDA events on the launching stream,
after one warm-up launch, and the L2 is flushed (a read of 4x its size)
before every sub-average so no sub-average starts with the grid cached.
Extras: ``dtype`` (the reference sweeps int32 only), a device memory budget,
and a ``time_budget_s`` per row that shrinks ``outer`` for rows whose single
launch is slow (recorded in the row's status as ``ok-reps=<outer>x<inner>``).
"""

from __future__ import annotations

import math
import os
import statistics
import tempfile
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import torch

from .engine import LaunchConfig, LaunchPlan, Mapping, make_grid, prepare, work_counts
from .geometry import FractalSpec, IntraStrategy, PAPER_STRATEGIES
from . import device

CSV_HEADER = (
    "mapping,strategy,r,n,rho,blocks_launched,threads_launched,threads_useful,"
    "map_ops,reduction_depth,simulated_cost,wall_ns_mean,wall_ns_stderr,"
    "cost_ratio,speedup,status"
)

DEFAULT_RHO_SET = (1, 2, 4, 8, 16, 32)
DEFAULT_MEM_LIMIT = 256 * 1024 * 1024  # the reference's default grid budget


@dataclass
class SweepConfig:
    r_min: int = 0
    r_max: int = 16
    rho_set: Sequence[int] = DEFAULT_RHO_SET
    mappings: Sequence[Mapping] = (Mapping.BOUNDING_BOX, Mapping.BLOCK_SPACE)
    strategies: Sequence[IntraStrategy] = PAPER_STRATEGIES
    reps: tuple[int, int] = (100, 10)
    out: Path = Path("bench.csv")
    workers: Optional[int] = None
    backend: Optional[str] = None
    mem_limit_bytes: int = DEFAULT_MEM_LIMIT
    dtype: torch.dtype = torch.int32
    flush_l2: bool = True
    time_budget_s: Optional[float] = None
    max_launch_s: Optional[float] = None  # skip rows predicted slower than this ("skipped-time")


@dataclass
class BenchRecord:
    mapping: str
    strategy: str
    r: int
    n: int
    rho: int
    blocks_launched: int = 0
    threads_launched: int = 0
    threads_useful: int = 0
    map_ops: int = 0
    reduction_depth: int = 0
    simulated_cost: int = 0
    wall_ns_mean: Optional[float] = None
    wall_ns_stderr: Optional[float] = None
    cost_ratio: Optional[float] = None
    speedup: Optional[float] = None
    status: str = "ok"


def _num(v: Optional[float]) -> str:
    return "" if v is None else format(v, ".6g")


def record_to_row(rec: BenchRecord) -> str:
    ints = (rec.r, rec.n, rec.rho, rec.blocks_launched, rec.threads_launched, rec.threads_useful,
            rec.map_ops, rec.reduction_depth, rec.simulated_cost)
    floats = (rec.wall_ns_mean, rec.wall_ns_stderr, rec.cost_ratio, rec.speedup)
    return ",".join([rec.mapping, rec.strategy, *map(str, ints), *map(_num, floats), rec.status])


def write_csv(records: Sequence[BenchRecord], path: Path | str) -> None:
    """Atomic: write a temp file in the target directory, then rename over the target."""
    path = Path(path)
    body = "\n".join([CSV_HEADER, *(record_to_row(r) for r in records)]) + "\n"
    fd, tmp = tempfile.mkstemp(dir=path.parent or Path("."), suffix=".tmp")
    try:
        with os.fdopen(fd, "w", newline="\n") as fh:
            fh.write(body)
        os.replace(tmp, path)
    except BaseException:
        os.unlink(tmp)
        raise


def _opt_float(s: str) -> Optional[float]:
    return float(s) if s else None


def read_csv(path: Path | str) -> list[BenchRecord]:
    lines = [ln for ln in Path(path).read_text().split("\n") if ln]
    if lines[0] != CSV_HEADER:
        raise ValueError(f"unexpected CSV header: {lines[0]!r}")
    out = []
    for ln in lines[1:]:
        f = ln.split(",")
        out.append(BenchRecord(f[0], f[1], *(int(v) for v in f[2:11]), *(_opt_float(v) for v in f[11:15]), f[15]))
    return out


_flusher: Optional[device.L2Flusher] = None


def _flush() -> None:
    global _flusher
    if _flusher is None:
        _flusher = device.L2Flusher()
    _flusher()


def _time_plan(plan: LaunchPlan, grid, reps: tuple[int, int], flush_l2: bool = True,
               time_budget_s: Optional[float] = None) -> tuple[float, float, tuple[int, int]]:
    """Mean and standard error (ns) over ``outer`` sub-averages of ``inner`` launches."""
    outer, inner = reps
    plan.run(grid, grid)  # warm-up (also loads the module and the lookup table)
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    subs: list[float] = []
    deadline = None
    for i in range(outer):
        if flush_l2:
            _flush()
        start.record()
        for _ in range(inner):
            plan.run(grid, grid)
        stop.record()
        stop.synchronize()
        subs.append(start.elapsed_time(stop) * 1e6 / inner)
        if time_budget_s is not None:
            if deadline is None:
                per_sub = subs[0] * inner / 1e9
                keep = max(2, min(outer, int(time_budget_s / max(per_sub, 1e-9))))
                deadline = keep
            if len(subs) >= deadline:
                break
    mean = statistics.fmean(subs)
    stderr = statistics.stdev(subs) / math.sqrt(len(subs)) if len(subs) > 1 else 0.0
    return mean, stderr, (len(subs), inner)


def _combos(cfg: SweepConfig) -> list[tuple[Mapping, Optional[IntraStrategy]]]:
    out: list[tuple[Mapping, Optional[IntraStrategy]]] = []
    for m in cfg.mappings:
        if m is Mapping.BLOCK_SPACE:
            out.extend((m, s) for s in cfg.strategies)
        else:
            out.append((m, None))
    # BB rows first: lambda rows report their speedup against the BB row
    out.sort(key=lambda c: 0 if c[0] is Mapping.BOUNDING_BOX else 1)
    return out


def run_sweep(cfg: SweepConfig) -> list[BenchRecord]:
    device.require_cuda()
    cell = torch.empty(0, dtype=cfg.dtype).element_size()
    records: list[BenchRecord] = []
    combos = _combos(cfg)
    last_ns: dict = {}
    last_threads: dict = {}
    for r in range(cfg.r_min, cfg.r_max + 1):
        n = 1 << r
        for rho in cfg.rho_set:
            status = None
            if rho > n:
                status = "skipped-shape"
            elif n * n * cell > cfg.mem_limit_bytes:
                status = "skipped-mem"
            if status:
                records.extend(BenchRecord(m.value, s.value if s else "none", r, n, rho, status=status)
                               for m, s in combos)
                continue
            spec = FractalSpec(n=n, rho=rho)
            grid = make_grid(n, cfg.dtype)
            bb_cost = work_counts(spec, Mapping.BOUNDING_BOX).simulated_cost
            bb_mean: Optional[float] = None
            for mapping, strat in combos:
                counts = work_counts(spec, mapping, strat)
                key = (mapping, strat, rho)
                if cfg.max_launch_s is not None and key in last_ns:
                    # launch time grows with the launched threads: predict from the previous level
                    grow = counts.threads_launched / max(1, last_threads[key])
                    if last_ns[key] * grow > cfg.max_launch_s * 1e9:
                        records.append(BenchRecord(mapping.value, strat.value if strat else "none", r, n, rho,
                                                   status="skipped-time"))
                        last_ns[key] *= grow
                        last_threads[key] = counts.threads_launched
                        continue
                plan = prepare(LaunchConfig(spec=spec, mapping=mapping, strategy=strat), cfg.backend)
                mean, stderr, used = _time_plan(plan, grid, cfg.reps, cfg.flush_l2, cfg.time_budget_s)
                last_ns[key], last_threads[key] = mean, counts.threads_launched
                is_bb = mapping is Mapping.BOUNDING_BOX
                if is_bb:
                    bb_mean = mean
                rec = BenchRecord(
                    mapping.value, strat.value if strat else "none", r, n, rho,
                    counts.blocks_launched, counts.threads_launched, counts.threads_useful, counts.map_ops,
                    counts.reduction_depth, counts.simulated_cost, mean, stderr,
                    None if is_bb else bb_cost / counts.simulated_cost,
                    None if is_bb or not bb_mean else bb_mean / mean,
                    "ok" if tuple(used) == tuple(cfg.reps) else f"ok-reps={used[0]}x{used[1]}",
                )
                records.append(rec)
            del grid
            torch.cuda.empty_cache()
    return records


def crossover(records: Sequence[BenchRecord]) -> dict:
    """The lambda-vs-BB speed-up curve of a sweep and its crossover n0 (the paper's Fig. 7
    reading): per rho, speedup(r) = BB time / best paper-literal lambda
    time (SUBBOX / TABLE / UNROLL) and BB / best of any lambda row; n0 = the smallest n
    from which the paper-literal speed-up stays > 1.  Also best-vs-best over every rho."""
    table: dict = {}
    for rec in records:
        if not rec.status.startswith("ok") or rec.wall_ns_mean is None:
            continue
        row = table.setdefault(rec.rho, {}).setdefault(rec.r, {})
        row["bb" if rec.mapping == Mapping.BOUNDING_BOX.value else rec.strategy] = rec.wall_ns_mean
    literal = ("subbox", "table", "unroll")
    per_rho = {}
    for rho, rows in sorted(table.items()):
        curve = {}
        for r, row in sorted(rows.items()):
            lit = [v for k, v in row.items() if k in literal]
            if "bb" not in row or not lit:
                continue
            curve[r] = {"paper_literal": row["bb"] / min(lit),
                        "best": row["bb"] / min(v for k, v in row.items() if k != "bb")}
        n0 = next((1 << r for r in sorted(curve) if all(curve[q]["paper_literal"] > 1 for q in curve if q >= r)), None)
        per_rho[str(rho)] = {"n0_paper_literal": n0, "speedup_by_r": curve}
    best = {}
    for r in sorted({r for rows in table.values() for r in rows}):
        bb = [rows[r]["bb"] for rows in table.values() if r in rows and "bb" in rows[r]]
        lam = [v for rows in table.values() if r in rows for k, v in rows[r].items() if k in literal]
        if bb and lam:
            best[r] = min(bb) / min(lam)
    n0_best = next((1 << r for r in sorted(best) if all(best[q] > 1 for q in best if q >= r)), None)
    return {"per_rho": per_rho, "best_vs_best_paper_literal_by_r": best, "n0_best_vs_best": n0_best}

