#!/usr/bin/env python
"""Headline benchmark: lambda(omega) gasket passes on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload write16|write16-i32|write17|stencil16|stencil16-i32-nsum4|
                                stencil17|stencil17-nsum4|part15|part18]
                    [--halo collective|peer|peer-fused] [--temporal 1|2|4|6]   (part* workloads)
                    [--no-sweep] [--no-e2e] [--no-cpu] [--nsweep]

Default workload (BASELINE configs[1]): the n = 2^16 write pass ("write a
constant value on all the elements") on int8 cells, lambda
map, tuned strategy.  One step = one launch over the whole gasket
(3^16 = 43,046,721 cells).  Each timed step is bracketed by CUDA events on
the launching stream, and the L2 is flushed (a 4x-L2 read) before every step,
outside the events.  value = gasket cells/s over all ranks (every rank runs
its own independent grid: weak scaling, no collective on the data path).

Extras on the same JSON line: the rho sweep of lambda vs bounding box at the
headline size (paper-literal SUBBOX/TABLE/UNROLL and tuned lambda, paper-
literal and block-early-exit BB) with the best-vs-best speedup and the useful-
thread fractions; `roofline` (sector-minimum bytes / event time vs the measured
HBM peak, plus `hw_model`: the bytes this memory system must move); for the
stencils `multi_step` (the CA driver, 1 / 2 / 4 / 6 fused steps per launch); `cpu_baseline`
(the C/OpenMP port of the reference numba kernels, all host threads, bounded
sample); `e2e` (the reference-facing call with host numpy buffers); `clocks`
(NVML sampled during the timed region); `gpu_launches`.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port of backends.py:143-222, the reference itself being pure
Python/numba that does not travel to the GPU box) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (r, cell dtype name, kind, rho, description)
    "write16": (16, "int8", 0, 32, "n=2^16 gasket write pass (const 1), int8 cells, lambda map"),
    "write16-i32": (16, "int32", 0, 32, "n=2^16 gasket write pass (const 1), int32 cells, lambda map"),
    "write17": (17, "int8", 0, 32, "n=2^17 gasket write pass (const 1), int8 cells, lambda map"),
    "stencil16": (16, "int8", 2, 64, "n=2^16 8-neighbour CA step, int8 states, lambda map"),
    "stencil16-i32-nsum4": (16, "int32", 1, 64, "n=2^16 4-neighbour CA step, int32 states (the reference's dtype), lambda map"),
    "stencil17": (17, "int8", 2, 64, "n=2^17 8-neighbour CA step, int8 states, lambda map"),
    "stencil17-nsum4": (17, "int8", 1, 64, "n=2^17 4-neighbour CA step, int8 states, lambda map"),
    "part15": (15, "int8", 2, 0, "n=2^15 8-neighbour CA step, int8 states, level-5 sub-gasket partition (functional "
                                 "check of the multi-rank path)"),
    "part18": (18, "int8", 2, 0, "n=2^18 8-neighbour CA step, int8 states, level-5 sub-gasket partition over "
                                 "the ranks, NCCL all_gather of the changing halo cells"),
}
PART_LEVEL = 5
# measured floor of each pass's exact DRAM access set moved in address order (the best
# this memory system does with those accesses; scripts/probe_rmw.cu, profiles/r1_probes.md)
PATTERN_CEILING_US = {"write16": 81.9, "stencil17": 344.0}
FALLBACK_HBM_GBS = 6650.0


def _metric(workload: str) -> str:
    """The metric string both arms print (BASELINE.json metric, this workload)."""
    r, _, _, _, desc = WORKLOADS[workload]
    what = desc.split(',')[1].strip() if ',' in desc else ''
    return "gasket cells/s (lambda map), n=2^%d %s; lambda-vs-BB speedup and %% HBM roofline alongside" % (r, what)


def _config(workload: str, rho: int, world: int, partitioned: bool) -> dict:
    """The workload description both arms print.  The tuned kernels do not take the
    paper's block size rho: their blocks are 128-byte-line tiles (128 / cell-bytes cells
    square); rho shapes only the paper-literal launches of the sweep."""
    r, dname, kind, _, desc = WORKLOADS[workload]
    c = {"int8": 1, "int16": 2, "int32": 4, "int64": 8}[dname]
    tile = 128 // c
    return {"workload": workload, "description": desc, "n": 1 << r, "mapping": "lambda",
            "strategy": "tuned",
            "blocks": (f"lambda tiles of {tile}x{tile} cells (one 128-byte line per row), lambda(omega) "
                       f"computed per tile on the warp (one lane per level, two ballots)" if kind == 0 else
                       f"lambda tiles of {tile}x{tile} cells in row-major tile order"),
            "kind": ["const", "nsum4", "nsum8"][kind], "cells_per_step": 3**r,
            "parallelism": (f"subgasket-partition{world} (level {PART_LEVEL})" if partitioned
                            else f"replicas{world}" if world > 1 else "single"),
            "l2": ("not flushed: every step touches several times the 126 MB L2 (the write pass's member "
                   "lines alone are 2.6x L2 at n=2^16), and the K timed steps run back to back between two "
                   "events, so each step's dirty-line write-back lands inside the timed region")}


def _host_threads() -> int:
    """All the host cores this process may use (torchrun sets OMP_NUM_THREADS=1 for its
    workers; the CPU arms pass the count explicitly so they still use every core)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML in-process sampler)
# ---------------------------------------------------------------------------

_REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle", 0x2: "applications_clocks_setting"}


class ClockSampler:
    def __init__(self, index: int, period_s: float = 0.005) -> None:
        self.index, self.period = index, period_s
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        self.error = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append((int(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             int(get_reasons(h))))
                    except Exception as e:  # pragma: no cover
                        self.error = repr(e)
                    time.sleep(self.period)

            self._thr = threading.Thread(target=loop, daemon=True)
            self._thr.start()
        except Exception as e:  # pragma: no cover
            self.error = repr(e)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "error": self.error}
        mhz = [s[0] for s in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = sorted(v for k, v in _REASONS.items() if bits & k and v != "gpu_idle")
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(mhz), "sm_mhz_min": min(mhz)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def _dist_init(ngpus: int):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("GASKET_BENCH_SHARED_GPU") == "1":
            # functional test of the multi-rank path on a one-GPU box: every rank on
            # cuda:0, gloo for the host plumbing (numbers are time-sliced, not a bench)
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
            return world, rank, 0
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return world, rank, local


def _barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _traffic_from_profiles(workload: str) -> tuple[float | None, str | None]:
    """(DRAM bytes per launch, where they were measured): ncu cannot run inside the timed
    process, so `traffic` comes from the committed capture of the same kernel."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        d = json.loads(p.read_text())[workload]
        return float(d["dram_bytes_per_launch"]), d.get("source")
    except Exception:
        return None, None


def _make_step(workload: str, grid, src, rho: int, flags: int, edge=None):
    """One timed step.  Write pass: backends.run_block_space(grid, grid, ...).  CA step:
    ping-pong between two buffers that agree off the gasket -- through gm_ca_run with the
    static left-edge cache when `edge` is given (the CA driver's single step, ca.CARunner),
    else through the drop-in backends.run_block_space(..., flags=DST_FROM_SRC)."""
    from paper_1706_04552_b200 import backends, device, native
    from paper_1706_04552_b200.geometry import IntraStrategy

    r, _, kind, _, _ = WORKLOADS[workload]
    r_b = r - (rho.bit_length() - 1)
    bufs = [grid, src]
    state = {"i": 0}

    def step():
        if kind == 0:
            backends.run_block_space(grid, grid, rho, r_b, IntraStrategy.TUNED, kind=0, param=1)
            return
        # CA ping-pong: read bufs[i], write bufs[1-i]; both agree off the gasket
        i = state["i"]
        if edge is not None:
            native.call("gm_ca_run", bufs[1 - i].data_ptr(), bufs[i].data_ptr(), 1 << r, grid.element_size(), kind,
                        1, 1, edge.data_ptr(), 0, device.stream_handle())
        else:
            backends.run_block_space(bufs[1 - i], bufs[i], rho, r_b, IntraStrategy.TUNED, kind=kind, param=1,
                                     flags=flags)
        state["i"] = 1 - i

    return step


_STEP_LAUNCHES = [0]  # our kernels launched between the events of the last _time_steps call


def _time_steps(step, flusher, steps: int) -> list[float]:
    import torch

    from paper_1706_04552_b200 import native

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    _STEP_LAUNCHES[0] = 0
    for a, b in ev:
        flusher()  # (its own kernel, outside the events: not counted)
        a.record()
        k0 = native.launch_count()
        step()
        _STEP_LAUNCHES[0] += native.launch_count() - k0
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def _sweep(r: int, dtype, flusher, budget_s: float = 3.0) -> dict:
    """rho sweep at the headline size: lambda (literal strategies + tuned) vs BB."""
    import torch

    from paper_1706_04552_b200 import backends
    from paper_1706_04552_b200.geometry import IntraStrategy

    n = 1 << r
    cells = 3**r
    grid = torch.zeros((n, n), dtype=dtype, device="cuda")
    out: dict = {}

    def timed(fn) -> float:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        one = time.perf_counter() - t0
        reps = int(max(2, min(20, budget_s / max(one, 1e-6))))
        ts = _time_steps(fn, flusher, reps)
        return statistics.fmean(ts)

    for rho in (1, 2, 4, 8, 16, 32):
        r_b = r - (rho.bit_length() - 1)
        row = {}
        row["bb"] = timed(lambda: backends.run_bounding_box(grid, grid, rho, 0, 1))
        row["bb-exit"] = timed(lambda: backends.run_bounding_box(grid, grid, rho, 0, 1, early_exit=True))
        for s in (IntraStrategy.SUBBOX, IntraStrategy.TABLE, IntraStrategy.UNROLL, IntraStrategy.TUNED):
            row[s.value] = timed(lambda: backends.run_block_space(grid, grid, rho, r_b, s, kind=0, param=1))
        out[str(rho)] = {k: {"ms": round(v, 5), "cells_per_s": cells / (v * 1e-3)} for k, v in row.items()}
    # the vectorised bounding box (rho does not shape it): the competent BB baseline
    bbv = timed(lambda: backends.run_bounding_box(grid, grid, 32, 0, 1, vectorized=True))
    del grid
    torch.cuda.empty_cache()

    def best(keys):
        return min(((float(out[rho][k]["ms"]), rho, k) for rho in out for k in keys))

    bb = best(["bb"])
    bbx = best(["bb", "bb-exit"])
    lit = best(["subbox", "table", "unroll"])
    tun = best(["subbox", "table", "unroll", "tuned"])
    summary = {
        "best_bb_paper": {"rho": bb[1], "ms": bb[0]},
        "best_bb_any": {"rho": bbx[1], "variant": bbx[2], "ms": bbx[0]},
        "best_lambda_paper": {"rho": lit[1], "strategy": lit[2], "ms": lit[0]},
        "best_lambda_any": {"rho": tun[1], "strategy": tun[2], "ms": tun[0]},
        "speedup_paper_literal_best_vs_best": bb[0] / lit[0],
        "speedup_best_lambda_vs_best_bb_paper": bb[0] / tun[0],
        "speedup_best_lambda_vs_best_bb_any": bbx[0] / tun[0],
        "speedup_rho32_subbox_vs_bb": float(out["32"]["bb"]["ms"]) / float(out["32"]["subbox"]["ms"]),
        "speedup_rho1_subbox_vs_bb": float(out["1"]["bb"]["ms"]) / float(out["1"]["subbox"]["ms"]),
        "bb_vectorised_ms": bbv,
        "speedup_tuned_lambda_vs_bb_vectorised": bbv / tun[0],
        "bb_vectorised_note": ("the bounding box written like the tuned kernels (one lane per 16-byte segment "
                               "of all n^2 cells, the same stores): lambda's gain over a competent BB"),
    }
    # fraction of launched threads that land on gasket cells (engine.work_counts;
    # the tuned kernel launches warps over whole 128-byte tile rows, so its figure is per
    # touched word rather than per thread)
    from paper_1706_04552_b200.engine import Mapping, work_counts
    from paper_1706_04552_b200.geometry import FractalSpec

    useful = {}
    for rho in (1, 2, 4, 8, 16, 32):
        spec = FractalSpec(n=n, rho=rho)
        row = {"bb": work_counts(spec, Mapping.BOUNDING_BOX).threads_useful
               / work_counts(spec, Mapping.BOUNDING_BOX).threads_launched}
        for s in (IntraStrategy.SUBBOX, IntraStrategy.TABLE, IntraStrategy.UNROLL):
            w = work_counts(spec, Mapping.BLOCK_SPACE, s)
            row[s.value] = w.threads_useful / w.threads_launched
        k3 = 3 ** (rho.bit_length() - 1)  # TABLE / UNROLL threads per block: lanes used of the launched warps
        row["table_unroll_lane_utilisation"] = k3 / (32 * -(-k3 // 32))
        useful[str(rho)] = row
    return {"per_rho_ms": {rho: {k: v["ms"] for k, v in row.items()} for rho, row in out.items()},
            "summary": summary, "useful_thread_fraction": useful}


def _stencil_vs_bb(r: int, tdt, kind: int, flusher, budget_s: float = 2.0) -> dict:
    """BASELINE config 3's "lambda vs BB" for the neighbour-sum step: the paper's
    bounding-box kernel (and its block-exit variant) against the paper-literal lambda
    strategies and the tuned lambda step, every one a full step dst <- step(src)
    (backends.run_bounding_box / run_block_space, flushed launches)."""
    import torch

    from paper_1706_04552_b200 import backends, device
    from paper_1706_04552_b200.geometry import IntraStrategy

    n = 1 << r
    src = device.fill_hash(n, tdt, 1, 0)
    dst = src.clone()

    def timed(fn) -> float:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        one = time.perf_counter() - t0
        reps = int(max(2, min(10, budget_s / max(one, 1e-6))))
        return statistics.fmean(_time_steps(fn, flusher, reps))

    row = {}
    for rho in (16, 32):
        r_b = r - (rho.bit_length() - 1)
        row[f"bb rho={rho}"] = timed(lambda: backends.run_bounding_box(dst, src, rho, kind, 1))
        row[f"bb-exit rho={rho}"] = timed(lambda: backends.run_bounding_box(dst, src, rho, kind, 1, early_exit=True))
        for st in (IntraStrategy.SUBBOX, IntraStrategy.TABLE):
            lx, ly = backends.local_cell_arrays(st, rho) if st == IntraStrategy.TABLE else (None, None)
            row[f"lambda {st.value} rho={rho}"] = timed(
                lambda: backends.run_block_space(dst, src, rho, r_b, st, lx, ly, kind=kind, param=1))
    row["lambda tuned"] = timed(lambda: backends.run_block_space(dst, src, 64, r - 6, IntraStrategy.TUNED, kind=kind,
                                                                 param=1))
    # the bounding box written like the tuned kernel (the same tile stencil over every tile of
    # the grid, tiles off the gasket exiting): lambda's gain over a competent BB
    row["bb vectorised"] = timed(lambda: backends.run_bounding_box(dst, src, 32, kind, 1, vectorized=True))
    del src, dst
    torch.cuda.empty_cache()
    bb = min(v for k, v in row.items() if k.startswith("bb rho"))
    bbx = min(v for k, v in row.items() if k.startswith("bb") and "vectorised" not in k)
    lit = min(v for k, v in row.items() if k.startswith("lambda") and "tuned" not in k)
    return {"ms": {k: round(v, 4) for k, v in row.items()},
            "speedup_paper_literal_best_vs_best": bb / lit,
            "speedup_tuned_lambda_vs_best_bb_paper": bb / row["lambda tuned"],
            "speedup_tuned_lambda_vs_best_bb_any": bbx / row["lambda tuned"],
            "speedup_tuned_lambda_vs_bb_vectorised": row["bb vectorised"] / row["lambda tuned"],
            "note": "single launches after an L2 flush, the drop-in semantics (off-gasket cells of dst kept)"}


def _multi_step(r: int, tdt, kind: int, flusher, steps: int = 48) -> dict:
    """The multi-step CA driver (ca.CARunner): single-step launches vs 2 or 4 fused steps
    per launch (temporal blocking, stencil_tb.cu), CUDA graphs, L2 flushed once before
    the run.  Not the headline: `value` above is one step = one pass."""
    import torch

    from paper_1706_04552_b200 import ca, device

    n = 1 << r
    out = {"steps": steps, "l2": "flushed once before the run (the state never fits L2)"}
    for temporal in (1, 2, 4, 6):
        if temporal == 6 and torch.empty((), dtype=tdt).element_size() == 4:
            continue  # (4-byte cells: at most 4 fused steps)
        g = device.fill_hash(n, tdt, 1, 0)
        run = ca.CARunner(g, kind=kind, param=1, use_graph=True, temporal=temporal)
        run.run(4 * temporal)  # warm-up + graph capture (a graph replay covers 2 * temporal steps)
        torch.cuda.synchronize()
        flusher()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run.run(steps)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / steps
        out[f"temporal{temporal}"] = {"ms_per_step": ms, "cells_per_s": 3**r / (ms * 1e-3),
                                      "steps_per_launch": temporal}
        del run, g
        torch.cuda.empty_cache()
    out["speedup_fused"] = out["temporal1"]["ms_per_step"] / out["temporal2"]["ms_per_step"]
    for t in (4, 6):
        if f"temporal{t}" in out:
            out[f"speedup_fused{t}"] = out["temporal1"]["ms_per_step"] / out[f"temporal{t}"]["ms_per_step"]
    # work-equivalent roofline: the §8d bytes of one single step per fused step time (the
    # fused pass moves about one step's bytes per two steps, so this can exceed what the
    # memory system moves; labelled "effective", not the kernel's own roofline)
    from paper_1706_04552_b200 import roofline as R

    peak, _ = _peaks()
    c = torch.empty((), dtype=tdt).element_size()
    for t in [k for k in ("temporal2", "temporal4", "temporal6") if k in out]:
        out[t]["effective_frac"] = R.pass_bytes(r, c, kind) / (out[t]["ms_per_step"] * 1e-3) / 1e9 / peak
    return out


def _time_b2b(step, steps: int) -> float:
    """ms per step of `steps` steps back to back between two CUDA events on the launching
    stream (synchronised on both sides; no L2 flush: the inputs exceed L2)."""
    import torch

    from paper_1706_04552_b200 import native

    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0 = native.launch_count()
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    _STEP_LAUNCHES[0] = native.launch_count() - k0
    return a.elapsed_time(b) / steps


def _zero_background(r: int, tdt, flusher, steps: int = 20) -> dict:
    """The opt-in zero-background write pass (assume_zero_background=True: the paper's
    zero-filled matrix; the reference bench's make_grid zeros,
    engine.py:88-90): touched 32-byte sectors stored whole, no DRAM read-modify-write.
    Same cells and values as the headline on that grid (tests/test_baseline_sizes.py)."""
    import torch

    from paper_1706_04552_b200 import backends, native
    from paper_1706_04552_b200 import roofline as R
    from paper_1706_04552_b200.geometry import IntraStrategy

    n = 1 << r
    c = torch.empty((), dtype=tdt).element_size()
    grid = torch.zeros((n, n), dtype=tdt, device="cuda")
    peak, _ = _peaks()
    alg = R.write_bytes(r, c)
    out = {}
    # the default schedule: grid rows for 1- and 2-byte cells, the address sweep for wider ones
    for name, flags in (("default (grid rows for 1-2-byte cells, address sweep for 4-8)", 0),
                        ("grid rows", native.FLAG_GRID_ROWS), ("lambda tiles", native.FLAG_DIGIT_ORDER),
                        ("address sweep", native.FLAG_WRITE_SWEEP)):
        def step():
            backends.run_block_space(grid, grid, 32, r - 5, IntraStrategy.TUNED, kind=0, param=1, flags=flags,
                                     assume_zero_background=True)

        for _ in range(3):
            step()
        ms = _time_b2b(step, steps)
        fl_ms = statistics.fmean(_time_steps(step, flusher, 10))
        out[name] = {"ms_per_step": ms, "cells_per_s": 3**r / (ms * 1e-3), "frac": alg / (ms * 1e-3) / 1e9 / peak,
                     "flushed_ms_per_launch": fl_ms}
    del grid
    torch.cuda.empty_cache()
    best = min(out, key=lambda k: out[k]["ms_per_step"])
    return {"api": "backends.run_block_space(..., assume_zero_background=True)", "best": best,
            "frac": out[best]["frac"], "value": out[best]["cells_per_s"], "schedules": out,
            "bytes": alg, "note": "off-gasket cells must be 0 (opt-in); no DRAM reads"}


def _staged_bytes(r: int, c: int, s64: int) -> tuple[int, int]:
    """Host bytes of the staged mapped stencil (gm_snapshot_stencil + gm_writeback_tiles),
    in the 64-byte units PCIe moves.  Per member tile: its TT rows, plus rows -1 / TT when
    the tile above / below is not a member.  s64 == 0 (64-byte aligned grid): the line, the
    unit left of it unless the left tile is a member, the unit right of it on rows TT-2..TT
    unless the right tile is a member; written back: the TT lines.  s64 != 0 (a numpy grid
    off a 64-byte boundary): the three host units covering [-16, 144) of each row, less the
    last on the tile's own rows when the right tile is a member (it reads / writes that
    unit); written back: the same units of the TT rows."""
    tt = 128 // c
    nb = (1 << r) // tt
    h2d = d2h = 0

    def member(x, y):
        return 0 <= x < nb and 0 <= y < nb and (x & ~y) == 0

    for Y in range(nb):
        X = Y
        while True:  # subsets of Y
            lm, rm = member(X - 1, Y) or X == 0, member(X + 1, Y) or X == nb - 1
            extra = int(Y > 0 and not member(X, Y - 1)) + int(Y < nb - 1 and not member(X, Y + 1))
            if s64 == 0:
                side = 0 if lm else 64
                h2d += tt * (128 + side) + (0 if rm else 2 * 64)
                h2d += int(Y > 0 and not member(X, Y - 1)) * (128 + side)
                h2d += int(Y < nb - 1 and not member(X, Y + 1)) * (128 + side + (0 if rm else 64))
                d2h += tt * 128
            else:
                own = 128 if (member(X + 1, Y)) else 192
                h2d += tt * own + extra * 192
                d2h += tt * own
            if X == 0:
                break
            X = (X - 1) & Y
    return h2d, d2h


def _e2e(workload: str, rho: int, steps: int, transports: tuple = ("mapped", "mapped-pinned", "copy")) -> dict:
    """The reference-facing call (backends.run_block_space on host numpy grids).

    "mapped": a plain pageable numpy grid (what the reference's make_grid returns,
    engine.py:88-90); the first call registers it (cudaHostRegister, kept until the
    array dies: device.pinned) and is reported on its own, the timed steps reuse the
    mapping.  "mapped-pinned": the same on a torch pin_memory grid.  "copy": whole-grid
    H2D / D2H through a device buffer."""
    import numpy as np
    import torch

    from paper_1706_04552_b200 import backends, device
    from paper_1706_04552_b200.geometry import IntraStrategy

    r, dname, kind, _, _ = WORKLOADS[workload]
    n = 1 << r
    c = np.dtype(dname).itemsize
    rho = 32
    r_b = r - (rho.bit_length() - 1)
    tdt = getattr(torch, dname)
    init = device.fill_hash(n, tdt, 1, 0).cpu().numpy() if kind != 0 else None
    res = {}
    for transport in transports:
        if transport == "mapped-pinned":
            host = torch.zeros((n, n), dtype=tdt, pin_memory=True)
            g = host.numpy()
        else:
            g = np.zeros((n, n), dtype=np.dtype(dname))
        if init is not None:
            g[...] = init
        os.environ[device.HOST_TRANSPORT_ENV] = "copy" if transport == "copy" else "mapped"
        # neighbour sums: engine.launch semantics (src is the grid's pre-launch snapshot),
        # which the staged mapped path serves (masked snapshot -> device kernel -> write-back)
        call = (lambda: backends.run_block_space(g, g, rho, r_b, IntraStrategy.TUNED, kind=kind, param=1))
        t0 = time.perf_counter()
        call()  # first call ("mapped": registers and maps the pageable buffer once)
        first = time.perf_counter() - t0
        k = steps if transport != "copy" else max(2, min(steps, 3))
        t0 = time.perf_counter()
        for _ in range(k):
            call()
        dt = (time.perf_counter() - t0) / k
        if transport != "copy":
            # zero-copy: only what the kernel touches crosses PCIe.  Write pass (row-ordered
            # schedule): the 64-byte halves holding gasket cells are read (unless all their
            # cells are gasket cells) and written back whole.  Stencils: the staged windows.
            if kind == 0:
                # (64-byte halves of the grid; on a numpy grid 16 bytes off a 64-byte boundary
                # the kernel moves the host units covering them instead -- about as many)
                kh = (64 // c).bit_length() - 1
                halves = (1 << kh) * 3 ** (r - kh)
                full = 3 ** (r - kh)  # halves made only of gasket cells need no read
                h2d, d2h = (halves - full) * 64, halves * 64
            else:
                h2d, d2h = _staged_bytes(r, c, 0 if transport == "mapped-pinned" else 16)
        else:
            h2d = n * n * c
            d2h = n * n * c
        res[transport] = {"s_per_step": dt, "cells_per_s": 3**r / dt, "h2d_bytes_per_step": int(h2d),
                          "d2h_bytes_per_step": int(d2h), "steps": k, "first_call_s": first}
        del g
        if transport == "mapped-pinned":
            del host
    os.environ.pop(device.HOST_TRANSPORT_ENV, None)
    device.pinned.clear()
    head = res["mapped"] if "mapped" in res else min(res.values(), key=lambda v: v["s_per_step"])
    return {"value": head["cells_per_s"], "unit": "cells/s", "h2d_bytes_per_step": head["h2d_bytes_per_step"],
            "d2h_bytes_per_step": head["d2h_bytes_per_step"], "transport": "mapped (pageable numpy grid)",
            "api": "backends.run_block_space(numpy grid, numpy grid, ...)",
            "timer": "host wall clock around the synchronous call; first call (buffer registration) reported "
                     "separately as variants.mapped.first_call_s",
            "variants": res}


def _cpu_baseline(workload: str, budget_s: float = 12.0) -> dict:
    """The reference algorithm on the host cores (oracle = C/OpenMP port of the numba kernels)."""
    import numpy as np

    import oracle

    r, dname, kind, _, _ = WORKLOADS[workload]
    if r >= 17:
        r_s = 16  # bounded sample: one 2^16 tile-equivalent of the same pass
    else:
        r_s = r
    n = 1 << r_s
    rho = 16
    g = np.zeros((n, n), dtype=np.dtype(dname))
    T = _host_threads()
    src = oracle.fill_hash(n, np.dtype(dname), 1, 0, threads=T) if kind else g
    lx, ly = oracle.local_cells(oracle.STRAT_TABLE, rho)
    oracle.run_block_space(g, src, rho, r_s - 4, oracle.STRAT_TABLE, lx, ly, kind, 1, threads=T)  # warm
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        oracle.run_block_space(g, src, rho, r_s - 4, oracle.STRAT_TABLE, lx, ly, kind, 1, threads=T)
        times.append(time.perf_counter() - t0)
    mean = statistics.fmean(times)
    return {"value": 3**r_s / mean, "unit": "cells/s", "cores": T, "kind": "port",
            "sample": f"{len(times)} x lambda TABLE rho=16 pass over n=2^{r_s} {dname} "
                      f"({['write', 'nsum4', 'nsum8'][kind]}), oracle/gasket_oracle.c (OpenMP)",
            "s_per_pass": mean}


def run_ours(args) -> None:
    import numpy as np
    import torch

    from paper_1706_04552_b200 import device, native
    from paper_1706_04552_b200 import roofline as R

    world, rank, local = _dist_init(args.gpus)
    workload = args.workload
    r, dname, kind, rho, desc = WORKLOADS[workload]
    if args.rho:
        rho = args.rho
    n = 1 << r
    c = np.dtype(dname).itemsize
    tdt = getattr(torch, dname)
    native.lib()
    flusher = device.L2Flusher()

    part = None
    if workload.startswith("part"):
        import torch.distributed as dist

        from paper_1706_04552_b200 import partition as P

        # --temporal 2|4|6: every timed step is one fused launch of that many CA steps
        # (gm_run_part_steps) with one exchange of the depth-2|4|6 halo; the line then
        # reports per-CA-step figures
        plan = P.PartitionPlan(n, PART_LEVEL, world, eight=kind == 2, depth=args.temporal)
        group = dist.group.WORLD if world > 1 else None
        if args.storage == "tiled":
            # each rank holds only its sub-gaskets, each a block with a ring (TiledLayout)
            peer = world > 1 and args.halo in ("peer", "peer-fused")
            part = P.TiledCA(plan, rank, kind, 1, dtype=tdt, seed=1, group=group,
                             halo="peer" if peer else "collective", fused=args.halo == "peer-fused" and peer)
        elif world > 1 and args.halo in ("peer", "peer-fused"):
            # halo over peer memory (CUDA IPC + release/acquire flags): no collective per step
            def fill(t):
                native.call("gm_fill_hash", t.data_ptr(), n, c, 1, 0, device.stream_handle())

            part = P.PartitionedCA(plan, rank, torch.empty((n, n), dtype=tdt, device="meta"), kind, 1,
                                   group=group, halo="peer", init_fill=fill, fused=args.halo == "peer-fused")
        else:
            init = device.fill_hash(n, tdt, 1, 0)  # every rank holds the same initial state
            part = P.PartitionedCA(plan, rank, init, kind, 1, group=group, adopt_init=True)
            del init
        torch.cuda.empty_cache()
        if world == 1 and args.storage != "tiled":
            step = lambda: (part.compute(), part.finish())  # noqa: E731  (no peers: nothing to exchange)
        else:
            step = part.step  # (tiled, one rank: the blocks' own ring copies every round)
        grid = src = edge = None
    else:
        grid = torch.zeros((n, n), dtype=tdt, device="cuda")
        src = edge = None
        flags = 0
        if kind != 0:
            src = device.fill_hash(n, tdt, 1 + rank, 0)
            grid.copy_(src)
            flags = native.FLAG_DST_FROM_SRC
            if c in (1, 2, 4):  # the CA driver's step: static left-edge cache (edge.cu)
                edge = torch.empty(native.ca_edge_bytes(n, c), dtype=torch.uint8, device="cuda")
                native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, c, -1, 0, 0, None, 0,
                            device.stream_handle())
        step = _make_step(workload, grid, src, rho, flags, edge=edge)
    torch.cuda.synchronize()
    t_warm = time.perf_counter()
    for _ in range(args.warmup):
        flusher()
        step()
    torch.cuda.synchronize()
    t_warm = (time.perf_counter() - t_warm) / max(1, args.warmup)
    # the same steps for ~60 ms right before the timed region, so that the clock sampler sees
    # the GPU under this load (the timed region itself lasts only milliseconds).  A fixed step
    # count, the same on every rank: each step of a partitioned run is a collective / a peer
    # epoch, so ranks must run exactly as many steps as each other
    busy_steps = int(_max_over_ranks(float(min(2000, max(8, int(0.06 / max(t_warm, 1e-6)) + 1))), world))

    _barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(busy_steps):
            step()
            if i % 8 == 7:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        _barrier(world)
        t_wall0 = time.perf_counter()
        per = _time_b2b(step, args.steps)
        t_wall = time.perf_counter() - t_wall0
    torch.cuda.synchronize()
    _barrier(world)
    launches = _STEP_LAUNCHES[0]  # inside the timed (event-bracketed) region only
    ms = [per] * args.steps
    total_ms = _max_over_ranks(per * args.steps, world)
    ms_per_step = total_ms / args.steps
    # the same launch after an L2 flush (outside the events): the cold-L2 single-launch time
    flushed = statistics.fmean(_time_steps(step, flusher, min(args.steps, 10)))
    ca_steps = args.temporal if part is not None else 1  # CA steps per timed step
    if ca_steps > 1:
        ms = [t / ca_steps for t in ms]
        ms_per_step /= ca_steps
    cells = 3**r
    value = (1 if part is not None else world) * cells / (ms_per_step * 1e-3)

    peak, peak_src = _peaks()
    alg_bytes = R.pass_bytes(r, c, kind)
    achieved = alg_bytes / (statistics.fmean(ms) * 1e-3) / 1e9
    traffic, traffic_src = _traffic_from_profiles(workload)
    line = {
        "metric": _metric(workload),
        "value": value,
        "unit": "cells/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if part is not None else "weak",
        "vs_baseline": None,
        "dtype": dname,
        "data": "synthetic (zero grid, param=1)" if kind == 0 else "synthetic (splitmix64 hash states, all cells)",
        "config": _config(workload, rho, world, part is not None),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_model": "exact 32-byte-sector minimum on the dense row-major grid (SURVEY §8d)",
                     "element_bytes_frac": R.element_bytes(r, c, kind) / (statistics.fmean(ms) * 1e-3) / 1e9 / peak,
                     # what DRAM must move on this layout (roofline.hw_bytes): a write pass's
                     # partial-sector stores cost a DRAM read of the sector (ECC RMW,
                     # scripts/probe_partial.cu); a stencil's reads come in 64-byte halves at
                     # best (scripts/probe_fetch.cu).  Explains the gap, not the headline frac.
                     "hw_model": {"bytes": R.hw_bytes(r, c, kind),
                                  "note": ("sector writes + forced RMW re-read" if kind == 0 else
                                           "64-byte-half reads of the dilated gasket + sector writes"),
                                  "frac": R.hw_bytes(r, c, kind) / (statistics.fmean(ms) * 1e-3) / 1e9 / peak}},
        "clocks": dict(clk.summary(), window="the last ~60 ms of warm-up (same steps) and the timed region"),
        "gpu_launches": int(launches),
        "flushed_ms_per_launch": flushed / (args.temporal if part is not None else 1),
        "timed_region_wall_s": t_wall,
    }
    if workload in PATTERN_CEILING_US and part is None:
        fl = PATTERN_CEILING_US[workload]
        line["roofline"]["pattern_ceiling"] = {
            "us": fl, "frac": fl * 1e-3 / statistics.fmean(ms),
            "note": "the same DRAM accesses in address order (scripts/probe_rmw.cu); frac = ceiling / measured"}
    if part is None and kind != 0 and edge is not None:
        # the same CA step through the drop-in call (no edge cache): the reference-shaped launch
        drop = _make_step(workload, grid, src, rho, flags)
        for _ in range(3):
            drop()
        ms_drop = _time_b2b(drop, args.steps)
        line["config"]["step"] = ("CA step src -> dst through gm_ca_run (ca.CARunner's single step) with the static "
                                  "left-edge cache (edge.cu), ping-pong buffers")
        line["drop_in_step"] = {"ms_per_step": ms_drop, "cells_per_s": cells / (ms_drop * 1e-3),
                                "frac": alg_bytes / (ms_drop * 1e-3) / 1e9 / peak,
                                "api": "backends.run_block_space(dst, src, ..., flags=FLAG_DST_FROM_SRC), no edge cache"}
        line["roofline"]["edge_cache_note"] = (
            "the CA step stages the off-gasket cells left of member tiles whose left neighbour tile holds no gasket "
            "cell from a dense cache built once per run, so it reads fewer DRAM lines than the single-launch "
            "sector model counts; frac keeps the single-launch bytes (drop_in_step.frac: the same bytes, no cache)")
    if part is not None:
        line["config"]["halo_bytes_per_step"] = part.halo_bytes_per_step if world > 1 else 0
        line["config"]["halo"] = (args.halo if world > 1 else "none (one rank)")
        line["config"]["storage"] = args.storage
        if args.storage == "tiled":
            line["config"]["storage_bytes_per_rank"] = part.storage_bytes
            line["config"]["storage_note"] = ("the rank's level-5 sub-gaskets as ringed blocks, two ping-pong "
                                              "buffers (the dense layout: two n x n grids per rank)")
        if ca_steps > 1:
            line["config"]["ca_steps_per_launch"] = ca_steps
            line["config"]["timing"] = (f"{ca_steps} fused CA steps per timed launch; ms_per_step and value are per "
                                        f"CA step; roofline fracs are work-equivalent (one step's bytes per step)")
        if args.project and world == 1:
            proj = _project_tiled if args.storage == "tiled" else _project
            line["projection"] = [proj(part, int(w), ms_per_step * ca_steps, ca_steps, flusher)
                                  for w in args.project.split(",")]
        if hasattr(part, "close"):
            part.close()
        line["config"]["subgasket_ranges"] = part.plan.ranges
        del part
    del grid, src, edge
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not workload.startswith("part"):
        if not args.no_sweep and kind == 0:
            line["sweep"] = _sweep(r, tdt, flusher)
        if kind == 0:
            line["zero_background"] = _zero_background(r, tdt, flusher, steps=args.steps)
        if kind != 0 and c in (1, 2, 4):
            line["multi_step"] = _multi_step(r, tdt, kind, flusher)
        if kind != 0 and not args.no_sweep:
            line["lambda_vs_bb"] = _stencil_vs_bb(r, tdt, kind, flusher)
        if not args.no_e2e:
            line["e2e"] = _e2e(workload, rho, steps=max(3, min(args.steps, 10)))
        if not args.no_cpu:
            line["cpu_baseline"] = _cpu_baseline(workload)
    if world > 1 and not workload.startswith("part") and kind == 0 and not args.no_e2e:
        # every rank drives its own GPU from its own pinned host grid over its own PCIe
        # link (mapped transport), concurrently; the job's e2e = all ranks' cells / the
        # slowest rank's time per step
        _barrier(world)
        mine = _e2e(workload, rho, steps=max(3, min(args.steps, 10)), transports=("mapped",))
        worst = _max_over_ranks(mine["variants"]["mapped"]["s_per_step"], world)
        line["e2e"] = {"value": world * 3**r / worst, "unit": "cells/s",
                       "h2d_bytes_per_step": world * mine["h2d_bytes_per_step"],
                       "d2h_bytes_per_step": world * mine["d2h_bytes_per_step"], "transport": "mapped",
                       "api": "backends.run_block_space(numpy), one host grid per rank",
                       "timer": "host wall clock around the synchronous call, max over ranks"}
    if rank == 0:
        if "e2e" not in line:
            line["e2e"] = None
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _project(part, world: int, ms_launch_1: float, ca_steps: int, flusher, reps: int = 10) -> dict:
    """Multi-GPU projection on one GPU: time each of `world` ranks' sub-gasket ranges
    (PartitionPlan(world)) alone, on the full-size buffers, without the halo exchange.
    The slowest rank bounds an N-GPU step from below; the exchange adds a few hundred
    bytes of NVLink traffic per step (latency).  Not a scaling measurement."""
    import torch

    from paper_1706_04552_b200 import partition as P

    plan = P.PartitionPlan(part.plan.n, part.plan.level, world, eight=part.plan.eight, depth=part.plan.depth)
    per_rank = []
    for lo, hi in plan.ranges:
        part.step_fn(part.b, part.a, lo, hi)
        # back to back, like the one-GPU line it is compared with
        per_rank.append(_time_b2b(lambda: part.step_fn(part.b, part.a, lo, hi), reps * 5) / ca_steps)
    slots, width = plan.exchange_slots()
    worst = max(per_rank)
    return {"world": world, "per_rank_ms_per_step": per_rank, "max_rank_ms_per_step": worst,
            "speedup_vs_one_gpu": ms_launch_1 / ca_steps / worst,
            "halo_cells_per_rank_per_exchange": [int(len(x)) for x in slots],
            "note": ("each rank's sub-gasket range timed alone on one GPU, no exchange: a compute-only "
                     "bound on the N-GPU step, not a scaling measurement")}


def _project_tiled(part, world: int, ms_launch_1: float, ca_steps: int, flusher, reps: int = 10) -> dict:
    """_project on tiled storage: each of `world` ranks built alone (its own blocks, rings
    loaded from the synthetic grid) and timed for one round -- its launch plus its own ring
    copies, no peer traffic.  A compute-only bound on the N-GPU step."""
    import torch

    from paper_1706_04552_b200 import partition as P

    plan = P.PartitionPlan(part.plan.n, part.plan.level, world, eight=part.plan.eight, depth=part.plan.depth)
    per_rank, storage = [], []
    for r in range(world):
        ca = P.TiledCA(plan, r, part.kind, part.param, dtype=part.a.dtype, seed=1,
                       loopback=P.LoopbackGroup(world))
        storage.append(ca.storage_bytes)

        def one():
            ca.compute()
            ca._coll.complete(ca.b)  # (own ring copies; the loopback values of the others are stale)
            ca.finish()

        ca._coll.post(ca.b)  # one contribution so complete() has a gathered buffer
        for _ in range(3):
            one()
        # back to back, like the one-GPU line it is compared with
        per_rank.append(_time_b2b(one, reps * 5) / ca_steps)
        del ca
        torch.cuda.empty_cache()
    worst = max(per_rank)
    return {"world": world, "per_rank_ms_per_step": per_rank, "max_rank_ms_per_step": worst,
            "speedup_vs_one_gpu": ms_launch_1 / ca_steps / worst, "storage_bytes_per_rank": storage,
            "note": ("each rank's blocks built and timed alone on one GPU (launch + own ring copies, no peer "
                     "traffic): a compute-only bound on the N-GPU step, not a scaling measurement")}


def run_reference(args) -> None:
    """Reference arm: the reference algorithm's CPU path (C/OpenMP port of its
    numba kernels, all host threads), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np

    import oracle

    workload = args.workload
    r, dname, kind, _, desc = WORKLOADS[workload]
    # bounded sample: one pass at n=2^16 for 2^17 workloads (cells/s is size-independent here)
    r_s = min(r, 16)
    n = 1 << r_s
    rho = 16  # the reference's best lambda configuration on CPU
    g = np.zeros((n, n), dtype=np.dtype(dname))
    T = _host_threads()
    src = oracle.fill_hash(n, np.dtype(dname), 1, 0, threads=T) if kind else g
    lx, ly = oracle.local_cells(oracle.STRAT_TABLE, rho)
    for _ in range(max(1, args.warmup)):
        oracle.run_block_space(g, src, rho, r_s - 4, oracle.STRAT_TABLE, lx, ly, kind, 1, threads=T)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run_block_space(g, src, rho, r_s - 4, oracle.STRAT_TABLE, lx, ly, kind, 1, threads=T)
        times.append(time.perf_counter() - t0)
    sec = statistics.fmean(times)
    value = 3**r_s / sec
    line = {
        "impl": "reference",
        "metric": _metric(workload),
        "value": value,
        "unit": "cells/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sec * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dname,
        "data": "synthetic",
        "config": _config(workload, WORKLOADS[workload][3], world, workload.startswith("part")),
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": T, "kind": "port",
                         "sample": f"one lambda TABLE rho=16 pass over n=2^{r_s} {dname} per step "
                                   f"(oracle/gasket_oracle.c, the reference's numba kernel restated; cells/s is "
                                   f"size-independent for this pass)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_nsweep(args) -> None:
    """BASELINE config 4: n = 2^8..2^18 write pass (int8) on one B200, lambda vs BB for every
    rho, rows in the reference CSV schema (bench.py:25-29), crossover n0 per rho."""
    import torch

    from paper_1706_04552_b200 import bench as B
    from paper_1706_04552_b200.engine import Mapping
    from paper_1706_04552_b200.geometry import IntraStrategy

    torch.cuda.set_device(0)
    strategies = (IntraStrategy.SUBBOX, IntraStrategy.TABLE, IntraStrategy.UNROLL, IntraStrategy.TUNED)
    cfg = B.SweepConfig(r_min=args.r_min, r_max=args.r_max, strategies=strategies, reps=(10, 10),
                        mappings=(Mapping.BOUNDING_BOX, Mapping.BLOCK_SPACE), dtype=torch.int8,
                        mem_limit_bytes=100 * 2**30, time_budget_s=2.0, max_launch_s=3.0)
    recs = B.run_sweep(cfg)
    out = Path(args.nsweep_out)
    out.parent.mkdir(parents=True, exist_ok=True)
    B.write_csv(recs, out)
    cross = B.crossover(recs)
    summary, best, n0_best = cross["per_rho"], cross["best_vs_best_paper_literal_by_r"], cross["n0_best_vs_best"]
    print(json.dumps({"nsweep_csv": str(out), "rows": len(recs), "per_rho": summary,
                      "best_vs_best_paper_literal_by_r": best, "n0_best_vs_best": n0_best}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="write16")
    ap.add_argument("--rho", type=int, default=None)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--nsweep", action="store_true", help="BASELINE config 4: n sweep + crossover n0, CSV")
    ap.add_argument("--temporal", type=int, choices=(1, 2, 4, 6), default=1,
                    help="part* workloads: CA steps fused per launch and per halo exchange")
    ap.add_argument("--project", default="",
                    help="part* workloads on one GPU, e.g. 2,4,8: also time each of N ranks' sub-gasket ranges "
                         "alone (compute-only bound of an N-GPU step; 'projection' in the line)")
    ap.add_argument("--halo", choices=("collective", "peer", "peer-fused"), default="collective",
                    help="part* workloads, N>1: NCCL all_gather of the halo cells, peer-memory puts (CUDA IPC), "
                         "or the peer exchange fused into the step kernel (any --temporal)")
    ap.add_argument("--storage", choices=("tiled", "dense"), default="tiled",
                    help="part* workloads: per-rank sub-gasket blocks with a ring (tiled) or two n x n grids per "
                         "rank (dense)")
    ap.add_argument("--r-min", type=int, default=8)
    ap.add_argument("--r-max", type=int, default=18)
    ap.add_argument("--nsweep-out", default="gpurun_out/nsweep.csv")
    args = ap.parse_args()
    if args.nsweep:
        run_nsweep(args)
        return
    if args.impl == "reference":
        args.steps = args.steps or 10
        args.warmup = args.warmup if args.warmup is not None else 3
        run_reference(args)
    else:
        args.steps = args.steps or 500
        args.warmup = max(3, args.warmup if args.warmup is not None else 10)
        run_ours(args)


if __name__ == "__main__":
    main()
