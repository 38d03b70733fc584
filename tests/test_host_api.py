"""Host-side API parity with the reference (CPU only): geometry, cost model,
CSV schema, backend selection and the error messages of the reference."""

import numpy as np
import pytest

from paper_1706_04552_b200 import geometry as G
from tests.golden.make_golden import checksum


def test_core_tables(golden):
    meta, arr = golden
    for r, v in meta["volume"].items():
        assert G.volume(int(r)) == v
    for r, d in meta["packing_dims"].items():
        assert list(G.packing_dims(int(r))) == d
    for n, r in meta["scale_level"].items():
        assert G.scale_level(int(n)) == r
    assert G.hausdorff_exponent() == meta["hausdorff"]
    for n in (1, 2, 4, 8, 16, 64, 256):
        assert np.array_equal(G.member_mask(n), arr[f"member_mask_{n}"])
    for s in meta["spec"]:
        spec = G.FractalSpec(n=s["n"], rho=s["rho"])
        assert (spec.r, spec.n_b, spec.r_b) == (s["r"], s["n_b"], s["r_b"])


def test_lambda_scalars(golden):
    meta, _ = golden
    for ex in meta["map_block"]:
        res = G.map_block(tuple(ex["omega"]), ex["r_b"])
        assert list(res.coord) == ex["coord"] and res.depth == ex["depth"]
    for (w, mu, beta) in meta["block_region"]:
        assert G.block_region(tuple(w), mu) == beta
    for r, d in meta["reduction_depth"].items():
        assert G.reduction_depth(int(r)) == d
    for n, t in meta["suggested_block_threads"].items():
        assert G.suggested_block_threads(int(n)) == t


def _scan_witness(fn, r_b):
    """The reference's scalar scan (blockmap.py:144-156) over a map_fn, host side."""
    w, h = G.packing_dims(r_b)
    n_b = 1 << r_b
    seen = set()
    for wy in range(h):
        for wx in range(w):
            cx, cy = fn((wx, wy), r_b).coord
            bad = not (0 <= cx < n_b and 0 <= cy < n_b) or (cx & (n_b - 1 - cy)) != 0 or (cx, cy) in seen
            if bad:
                return [False, [wx, wy], len(seen)]
            seen.add((cx, cy))
    return [len(seen) == 3**r_b, None, len(seen)]


def test_corrupted_maps_match_reference(golden):
    meta, _ = golden
    for key, want in meta["verify_bijection"].items():
        defect, r_b = key.rsplit("_", 1)
        if defect == "None" or int(r_b) > 6:
            continue
        assert _scan_witness(G.corrupted_map_fn(defect), int(r_b)) == want, key


def test_local_cells_and_threads(golden):
    meta, _ = golden
    for key, ck in meta["local_cells_checksum"].items():
        strat, rho = key.split("_")
        cells = G.local_cells(G.IntraStrategy(strat), int(rho))
        assert checksum(np.array([[c.x, c.y] for c in cells], dtype=np.int64)) == ck
    for key, t in meta["threads_per_block"].items():
        strat, rho = key.split("_")
        assert G.threads_per_block(G.IntraStrategy(strat), int(rho)) == t
    # the TUNED strategy covers the same cell set
    for rho in (1, 2, 4, 8, 16, 32, 64):
        assert G.local_cells(G.IntraStrategy.TUNED, rho) == G.local_cells(G.IntraStrategy.SUBBOX, rho)


def test_work_counts(golden):
    from paper_1706_04552_b200 import engine

    meta, _ = golden
    for row in meta["work_counts"]:
        spec = G.FractalSpec(n=row["n"], rho=row["rho"])
        st = G.IntraStrategy(row["strategy"]) if row["strategy"] else None
        m = engine.work_counts(spec, engine.Mapping(row["mapping"]), st)
        assert [m.blocks_launched, m.threads_launched, m.threads_useful, m.map_ops, m.reduction_depth,
                m.simulated_cost] == row["counts"], row


def test_acceptance_cost_ratio_monotone():
    """SPEC.md AC8: BB/lambda simulated cost at rho=16 strictly increasing for n=2^8..2^13, > 1."""
    from paper_1706_04552_b200 import engine

    prev = 0.0
    for r in range(8, 14):
        spec = G.FractalSpec(n=1 << r, rho=16)
        ratio = engine.simulated_cost(spec, engine.Mapping.BOUNDING_BOX) / engine.simulated_cost(
            spec, engine.Mapping.BLOCK_SPACE, G.IntraStrategy.SUBBOX)
        assert ratio > prev and ratio > 1
        prev = ratio


def test_csv_schema(golden, tmp_path):
    from paper_1706_04552_b200 import bench

    meta, _ = golden
    assert bench.CSV_HEADER == meta["csv_header"]
    recs = [bench.BenchRecord("bb", "none", 4, 16, 2, 64, 256, 81, 256, 0, 337, 1234.5678, 12.3456789, None, None, "ok"),
            bench.BenchRecord("blockspace", "table", 16, 65536, 16, 3**12, 3**16, 3**16, 3**12 * 93, 4, 123,
                              7.7e7, 1.1e5, 3.16049382716, 6.0e0, "ok"),
            bench.BenchRecord("blockspace", "subbox", 3, 8, 16, status="skipped-shape")]
    assert [bench.record_to_row(r) for r in recs] == meta["csv_rows"]
    p = tmp_path / "x.csv"
    bench.write_csv(recs, p)
    back = bench.read_csv(p)
    assert [bench.record_to_row(r) for r in back] == meta["csv_rows"]


def test_reference_error_messages():
    with pytest.raises(ValueError, match="edge length must be a power of two >= 1, got 6"):
        G.scale_level(6)
    with pytest.raises(ValueError, match="block edge 16 exceeds grid edge 8"):
        G.FractalSpec(n=8, rho=16)
    with pytest.raises(ValueError, match="block edge must be a power of two >= 1, got 3"):
        G.FractalSpec(n=8, rho=3)
    with pytest.raises(ValueError, match=r"scale level must be in \[0, 40\], got 41"):
        G.volume(41)
    with pytest.raises(ValueError, match="outside the 3x9 rectangle"):
        G.map_block((3, 0), 3)
    with pytest.raises(ValueError, match="unknown defect"):
        G.corrupted_map_fn("nope")


def test_error_messages_equal_live_reference(reference):
    from gasketmap import blockmap as rb
    from gasketmap import core as rc

    cases = [(G.scale_level, rc.scale_level, (6,)), (G.volume, rc.volume, (41,)),
             (G.map_block, rb.map_block, ((3, 0), 3)), (G.region_offset, rb.region_offset, (3, 1)),
             (G.block_region, rb.block_region, ((1, 1), 0)), (G.suggested_block_threads, rb.suggested_block_threads, (2,)),
             (G.subbox_thread_map, None, ((9, 0), 8)), (G.is_member, rc.is_member, ((9, 0), 8))]
    for ours, theirs, args in cases:
        if theirs is None:
            continue
        with pytest.raises(ValueError) as a:
            ours(*args)
        with pytest.raises(ValueError) as b:
            theirs(*args)
        assert str(a.value) == str(b.value)


def test_backend_resolution(monkeypatch):
    from paper_1706_04552_b200 import backends

    assert backends.resolve_backend(None) == "cuda"
    assert backends.resolve_backend("auto") == "cuda"
    monkeypatch.setenv("GASKETMAP_BACKEND", "numpy")
    with pytest.raises(RuntimeError):
        backends.resolve_backend(None)
    with pytest.raises(ValueError):
        backends.resolve_backend("fortran")


def test_launch_config_validation():
    from paper_1706_04552_b200 import engine

    with pytest.raises(ValueError, match="block-space launches need an intra-block strategy"):
        engine.LaunchConfig(spec=G.FractalSpec(8, 2), mapping=engine.Mapping.BLOCK_SPACE)


def test_staged_bands_cover_whole_block_rows():
    """The banded staged host path's tile ranges (device.staged_bands): consecutive, covering
    every member tile of the row-major order exactly once, each a run of whole block rows
    (block row Y holds 2^popcount(Y) tiles), about equal in size."""
    import numpy as np

    from paper_1706_04552_b200 import device, native

    for n, c in ((128, 1), (256, 1), (1 << 12, 1), (1 << 12, 2), (1 << 11, 4), (1 << 17, 1)):
        q = (n // (128 // c)).bit_length() - 1
        bands = device.staged_bands(n, c)
        assert bands[0][0] == 0 and bands[-1][1] == 3**q
        assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
        starts = set(np.concatenate([[0], np.cumsum([1 << bin(y).count("1") for y in range(1 << q)])]).tolist())
        assert all(t0 in starts and t1 in starts for t0, t1 in bands)
        if q >= 5:
            _, by = native.tile_order(q, 0)
            assert np.all(np.diff(by) >= 0)  # the row-major order: block rows ascending
            sizes = [t1 - t0 for t0, t1 in bands]
            assert len(bands) >= 4 and max(sizes) <= 2 * 3**q / len(bands)
