"""Generate golden fixtures by running the LIVE reference (gasketmap) in this container.

Usage (container only; /root/reference does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` and ``tests/golden/golden.json``.  Every
value is produced by the reference's own public functions (core, blockmap,
intra, backends.run_* numba leg, engine, bench.record_to_row); synthetic
inputs use a numpy splitmix64 written here, independently of oracle/.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GASKET_REFERENCE", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
K = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def hash_grid(n: int, dtype, seed: int, mode: int = 0) -> np.ndarray:
    ys, xs = np.meshgrid(np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64), indexing="ij")
    v = splitmix64(np.uint64(seed) ^ ((ys << np.uint64(32)) | xs))
    if mode == 1:
        v[(xs.astype(np.int64) & (n - 1 - ys.astype(np.int64))) != 0] = 0
    width = np.dtype(dtype).itemsize
    if width < 8:
        v = v & np.uint64((1 << (8 * width)) - 1)
    return v.astype(np.dtype(f"u{width}")).view(dtype)


def checksum(a: np.ndarray) -> int:
    flat = np.ascontiguousarray(a).reshape(-1)
    v = flat.view(np.dtype(f"u{flat.dtype.itemsize}")).astype(np.uint64)
    i = np.arange(flat.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        w = (np.uint64(2) * i + np.uint64(1)) * K
        return int(np.sum(w * v, dtype=np.uint64))


def main() -> None:
    sys.path.insert(0, str(REF))
    from gasketmap import backends, bench, blockmap, core, engine, intra  # noqa: E402

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": str(REF), "generator": "tests/golden/make_golden.py"}

    # -- core (core.py) ---------------------------------------------------
    meta["volume"] = {str(r): core.volume(r) for r in range(0, 41)}
    meta["packing_dims"] = {str(r): list(core.packing_dims(r)) for r in range(0, 41)}
    meta["scale_level"] = {str(1 << r): core.scale_level(1 << r) for r in range(0, 41)}
    meta["hausdorff"] = core.hausdorff_exponent()
    for n in (1, 2, 4, 8, 16, 64, 256):
        arrays[f"member_mask_{n}"] = core.member_mask(n)
    meta["spec"] = [
        {"n": n, "rho": rho, "r": s.r, "n_b": s.n_b, "r_b": s.r_b}
        for n in (1, 2, 8, 64, 1 << 16, 1 << 20)
        for rho in (1, 2, 4, 32)
        if rho <= n
        for s in [core.FractalSpec(n=n, rho=rho)]
    ]

    # -- lambda (blockmap.py:91-108) -------------------------------------
    for r_b in range(0, 10):
        w, h = core.packing_dims(r_b)
        idx = np.arange(w * h, dtype=np.int64)
        lx, ly = blockmap.map_blocks_array(idx % w, idx // w, r_b)
        arrays[f"lambda_lx_{r_b}"] = lx.astype(np.int32)
        arrays[f"lambda_ly_{r_b}"] = ly.astype(np.int32)
    lam_ck = {}
    for r_b in range(10, 17):
        w, h = core.packing_dims(r_b)
        idx = np.arange(w * h, dtype=np.int64)
        lx, ly = blockmap.map_blocks_array(idx % w, idx // w, r_b)
        lam_ck[str(r_b)] = [checksum(lx), checksum(ly)]
    meta["lambda_checksum"] = lam_ck
    rng = np.random.default_rng(1706)
    wx = rng.integers(-10_000, 3**12, size=4096, dtype=np.int64)
    wy = rng.integers(-10_000, 3**12, size=4096, dtype=np.int64)
    arrays["lambda_rand_wx"], arrays["lambda_rand_wy"] = wx, wy
    for r_b in (0, 1, 7, 20, 33):
        lx, ly = blockmap.map_blocks_array(wx, wy, r_b)
        arrays[f"lambda_rand_lx_{r_b}"], arrays[f"lambda_rand_ly_{r_b}"] = lx, ly
    meta["map_block"] = [
        {"omega": [wx_, wy_], "r_b": rb, "coord": list(blockmap.map_block((wx_, wy_), rb).coord),
         "depth": blockmap.map_block((wx_, wy_), rb).depth}
        for rb, wx_, wy_ in [(0, 0, 0), (2, 2, 0), (3, 2, 8), (5, 4, 20), (10, 200, 100), (16, 6000, 6500)]
    ]
    meta["block_region"] = [[w_, mu, blockmap.block_region(w_, mu)] for w_ in [(0, 0), (2, 0), (2, 5), (7, 11)]
                            for mu in (1, 2, 3, 4)]
    meta["reduction_depth"] = {str(r): blockmap.reduction_depth(r) for r in range(0, 33)}
    meta["suggested_block_threads"] = {str(1 << r): blockmap.suggested_block_threads(1 << r) for r in range(2, 41)}
    bij = {}
    for defect in (None, "parity", "divisor", "offset"):
        fn = None if defect is None else blockmap.corrupted_map_fn(defect)
        for r_b in range(0, 9):
            rep = blockmap.verify_bijection(r_b, fn)
            bij[f"{defect}_{r_b}"] = [rep.ok, None if rep.witness is None else list(rep.witness), rep.image_size]
    meta["verify_bijection"] = bij

    # -- intra (intra.py) ------------------------------------------------
    loc = {}
    for strat in intra.IntraStrategy:
        for rho in (1, 2, 4, 8, 16, 32, 64):
            cells = intra.local_cells(strat, rho)
            loc[f"{strat.value}_{rho}"] = checksum(np.array([[c.x, c.y] for c in cells], dtype=np.int64))
    meta["local_cells_checksum"] = loc
    meta["threads_per_block"] = {f"{s.value}_{rho}": intra.threads_per_block(s, rho)
                                 for s in intra.IntraStrategy for rho in (1, 2, 4, 8, 16, 32, 64)}

    # -- engine.work_counts (engine.py:109-137) --------------------------
    wc = []
    for n in (1, 2, 16, 64, 256, 1 << 13, 1 << 16, 1 << 18):
        for rho in (1, 2, 4, 8, 16, 32):
            if rho > n:
                continue
            spec = core.FractalSpec(n=n, rho=rho)
            combos = [(engine.Mapping.BOUNDING_BOX, None)] + [(engine.Mapping.BLOCK_SPACE, s) for s in intra.IntraStrategy]
            for mp, st in combos:
                m = engine.work_counts(spec, mp, st)
                wc.append({"n": n, "rho": rho, "mapping": mp.value, "strategy": st.value if st else None,
                           "counts": [m.blocks_launched, m.threads_launched, m.threads_useful, m.map_ops,
                                      m.reduction_depth, m.simulated_cost]})
    meta["work_counts"] = wc

    # -- kernels via the reference's own backends (numba leg) ------------
    backend = backends.resolve_backend("numba")
    strat_tags = {intra.IntraStrategy.UNROLL: 0, intra.IntraStrategy.TABLE: 1, intra.IntraStrategy.SUBBOX: 2}
    kern = []
    for dtype in (np.int8, np.uint8, np.int16, np.int32, np.int64):
        for n in (1, 2, 4, 8, 32, 64, 256):
            for rho in (1, 2, 4, 8, 16, 32):
                if rho > n:
                    continue
                spec = core.FractalSpec(n=n, rho=rho)
                for kind, param in ((0, 7), (0, -3), (1, 1), (1, 2**31 - 1)):
                    for seed in (0, 1):
                        if kind == 0 and seed == 1:
                            continue
                        src = hash_grid(n, dtype, seed, mode=0)
                        rows = {"dtype": np.dtype(dtype).name, "n": n, "rho": rho, "kind": kind, "param": param,
                                "seed": seed, "src_checksum": checksum(src)}
                        g = src.copy()
                        backends.run_bounding_box(g, src.copy(), rho, kind, param, backend)
                        rows["bb"] = checksum(g)
                        for strat, tag in strat_tags.items():
                            lx, ly = backends.local_cell_arrays(strat, rho)
                            g = src.copy()
                            backends.run_block_space(g, src.copy(), rho, spec.r_b, strat, lx, ly, kind, param, backend)
                            rows[strat.value] = checksum(g)
                        if n <= 32 and dtype in (np.int8, np.int32) and seed == 0:
                            arrays[f"grid_{np.dtype(dtype).name}_{n}_{rho}_{kind}_{param}"] = g
                        kern.append(rows)
    meta["kernels"] = kern

    # n = 2^12 int8 / int32 NSUM4 + CONST via numba, one rho per strategy (larger-n anchor).
    big = []
    for dtype in (np.int8, np.int32):
        n = 1 << 12
        src = hash_grid(n, dtype, 7, mode=1)
        for kind, param in ((0, 1), (1, 1)):
            for rho in (4, 32):
                spec = core.FractalSpec(n=n, rho=rho)
                g = src.copy()
                lx, ly = backends.local_cell_arrays(intra.IntraStrategy.TABLE, rho)
                backends.run_block_space(g, src.copy(), rho, spec.r_b, intra.IntraStrategy.TABLE, lx, ly, kind, param, backend)
                g2 = src.copy()
                backends.run_bounding_box(g2, src.copy(), rho, kind, param, backend)
                assert np.array_equal(g, g2)
                big.append({"dtype": np.dtype(dtype).name, "n": n, "rho": rho, "kind": kind, "param": param,
                            "seed": 7, "mode": 1, "src_checksum": checksum(src), "out": checksum(g)})
    meta["kernels_big"] = big

    # -- engine.launch SPEC examples -------------------
    ex = []
    for n, rho, mp, st, kind, param in [
        (1, 1, "bb", None, "const", 7), (1, 1, "blockspace", "subbox", "const", 7),
        (8, 2, "blockspace", "subbox", "const", 7), (64, 8, "bb", None, "const", 1),
        (64, 8, "blockspace", "subbox", "const", 1), (64, 8, "blockspace", "table", "neighbor-sum", 3),
        (16, 4, "blockspace", "unroll", "neighbor-sum", -5),
    ]:
        spec = core.FractalSpec(n=n, rho=rho)
        cfg = engine.LaunchConfig(spec=spec, mapping=engine.Mapping(mp),
                                  strategy=intra.IntraStrategy(st) if st else None,
                                  kernel=engine.CellKernel(engine.KernelKind(kind), param))
        g = hash_grid(n, np.int32, 3, mode=0) if kind != "const" else engine.make_grid(n)
        m = engine.launch(cfg, g, backend)
        ex.append({"n": n, "rho": rho, "mapping": mp, "strategy": st, "kind": kind, "param": param,
                   "grid": checksum(g), "set_cells": int((g == param).sum()),
                   "metrics": [m.blocks_launched, m.threads_launched, m.threads_useful, m.map_ops,
                               m.reduction_depth, m.simulated_cost]})
    meta["launch_examples"] = ex

    # -- verify_coverage (engine.py:214-258) incl. corrupted maps --------
    cov = []
    for defect in (None, "parity", "divisor", "offset"):
        for n, rho, st in ((8, 1, "subbox"), (64, 4, "table"), (32, 2, "unroll"), (16, 16, "subbox")):
            spec = core.FractalSpec(n=n, rho=rho)
            cfg = engine.LaunchConfig(spec=spec, mapping=engine.Mapping.BLOCK_SPACE, strategy=intra.IntraStrategy(st))
            fn = None if defect is None else blockmap.corrupted_map_fn(defect)
            rep = engine.verify_coverage(cfg, fn)
            cov.append({"defect": defect, "n": n, "rho": rho, "strategy": st, "exact": rep.exact,
                        "counts": checksum(rep.counts), "dups": [list(c) for c in rep.duplicates[:50]],
                        "ndups": len(rep.duplicates), "misses": [list(c) for c in rep.misses[:50]],
                        "nmisses": len(rep.misses)})
    meta["coverage"] = cov

    # -- bench CSV formatting (bench.py:25-29, 69-93) --------------------
    recs = [bench.BenchRecord("bb", "none", 4, 16, 2, 64, 256, 81, 256, 0, 337, 1234.5678, 12.3456789, None, None, "ok"),
            bench.BenchRecord("blockspace", "table", 16, 65536, 16, 3**12, 3**16, 3**16, 3**12 * 93, 4, 123,
                              7.7e7, 1.1e5, 3.16049382716, 6.0e0, "ok"),
            bench.BenchRecord("blockspace", "subbox", 3, 8, 16, status="skipped-shape")]
    meta["csv_header"] = bench.CSV_HEADER
    meta["csv_rows"] = [bench.record_to_row(r) for r in recs]

    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT / "golden.npz", (OUT / "golden.npz").stat().st_size, "bytes;",
          OUT / "golden.json", (OUT / "golden.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
