"""Pin the CPU oracle (oracle/) to golden vectors generated from the live reference.

CPU-only (no GPU): these tests establish that the checker used by the GPU
parity tests computes exactly what the reference computes.
"""

import numpy as np
import pytest

from tests.golden.make_golden import checksum as np_checksum
from tests.golden.make_golden import hash_grid as np_hash_grid

STRATS = {"unroll": 0, "table": 1, "subbox": 2}


def test_checksum_and_hash_match_numpy(oracle):
    for dtype in (np.int8, np.int16, np.int32, np.int64, np.uint8):
        for n in (1, 8, 64):
            for mode in (0, 1):
                a = oracle.fill_hash(n, dtype, 12345, mode)
                b = np_hash_grid(n, dtype, 12345, mode)
                assert np.array_equal(a, b)
                assert oracle.checksum(a) == np_checksum(a)


def test_lambda_rectangle_exhaustive(oracle, golden):
    meta, arr = golden
    for r_b in range(0, 10):
        lx, ly = oracle.map_rectangle(r_b)
        assert np.array_equal(lx, arr[f"lambda_lx_{r_b}"]), r_b
        assert np.array_equal(ly, arr[f"lambda_ly_{r_b}"]), r_b
    for r_b in range(10, 15):
        lx, ly = oracle.map_rectangle(r_b)
        assert [oracle.checksum(lx), oracle.checksum(ly)] == meta["lambda_checksum"][str(r_b)], r_b


def test_lambda_arbitrary_coords(oracle, golden):
    """map_blocks_array on out-of-rectangle and negative inputs (floor semantics)."""
    _, arr = golden
    wx, wy = arr["lambda_rand_wx"], arr["lambda_rand_wy"]
    for r_b in (0, 1, 7, 20, 33):
        lx, ly = oracle.map_blocks(wx, wy, r_b)
        assert np.array_equal(lx, arr[f"lambda_rand_lx_{r_b}"])
        assert np.array_equal(ly, arr[f"lambda_rand_ly_{r_b}"])


def test_map_block_scalar(oracle, golden):
    meta, _ = golden
    for ex in meta["map_block"]:
        assert list(oracle.map_block_scalar(*ex["omega"], ex["r_b"])) == ex["coord"]


def test_member_mask(oracle, golden):
    _, arr = golden
    for n in (1, 2, 4, 8, 16, 64, 256):
        assert np.array_equal(oracle.member_mask(n), arr[f"member_mask_{n}"])


def test_local_cells(oracle, golden):
    meta, _ = golden
    for key, ck in meta["local_cells_checksum"].items():
        strat, rho = key.split("_")
        lx, ly = oracle.local_cells(STRATS[strat], int(rho))
        assert oracle.checksum(np.stack([lx, ly], axis=1)) == ck, key


def _run_all(oracle, src, rho, kind, param):
    n = src.shape[0]
    r_b = (n // rho).bit_length() - 1
    out = {}
    g = src.copy()
    oracle.run_bounding_box(g, src.copy(), rho, kind, param)
    out["bb"] = g
    for name, tag in STRATS.items():
        lx, ly = oracle.local_cells(tag, rho)
        g = src.copy()
        oracle.run_block_space(g, src.copy(), rho, r_b, tag, lx, ly, kind, param)
        out[name] = g
    return out


def test_kernels_vs_reference_golden(oracle, golden):
    meta, arr = golden
    for row in meta["kernels"]:
        dtype = np.dtype(row["dtype"])
        src = oracle.fill_hash(row["n"], dtype, row["seed"], 0)
        assert oracle.checksum(src) == row["src_checksum"]
        outs = _run_all(oracle, src, row["rho"], row["kind"], row["param"])
        for name, g in outs.items():
            assert oracle.checksum(g) == row[name], (row, name)
        key = f"grid_{dtype.name}_{row['n']}_{row['rho']}_{row['kind']}_{row['param']}"
        if key in arr.files and row["seed"] == 0:
            assert np.array_equal(outs["unroll"], arr[key])


def test_kernels_big_vs_reference_golden(oracle, golden):
    meta, _ = golden
    for row in meta["kernels_big"]:
        src = oracle.fill_hash(row["n"], np.dtype(row["dtype"]), row["seed"], row["mode"])
        assert oracle.checksum(src) == row["src_checksum"]
        g = src.copy()
        lx, ly = oracle.local_cells(1, row["rho"])
        r_b = (row["n"] // row["rho"]).bit_length() - 1
        oracle.run_block_space(g, src.copy(), row["rho"], r_b, 1, lx, ly, row["kind"], row["param"])
        assert oracle.checksum(g) == row["out"]


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32, np.int64])
@pytest.mark.parametrize("eight", [False, True])
def test_nsum_numpy_crosscheck(oracle, dtype, eight):
    """C oracle vs an independent numpy restatement (NSUM4 and our NSUM8 extension)."""
    for n in (1, 2, 16, 128):
        src = oracle.fill_hash(n, dtype, 99, 0)
        a = oracle.fill_hash(n, dtype, 5, 0)
        b = a.copy()
        oracle.run_bounding_box(a, src, 1, 2 if eight else 1, -77)
        oracle.nsum_reference_numpy(b, src, -77, eight)
        assert np.array_equal(a, b)


def test_coverage_counts_golden(oracle, golden):
    meta, _ = golden
    for row in meta["coverage"]:
        if row["defect"] is not None:
            continue
        n, rho = row["n"], row["rho"]
        r_b = (n // rho).bit_length() - 1
        bx, by = oracle.map_rectangle(r_b)
        lx, ly = oracle.local_cells(STRATS[row["strategy"]], rho)
        counts = oracle.coverage_counts(bx, by, lx, ly, rho, n)
        assert oracle.checksum(counts) == row["counts"]


def test_mutations_break_elementwise_lambda(oracle):
    """SURVEY §4 blind spot: 'parity' survives verify_bijection at even r_b, but
    every corrupted map differs from lambda element-wise at every r_b >= 1."""
    from paper_1706_04552_b200.geometry import corrupted_map_fn, packing_dims

    for defect in ("parity", "divisor", "offset"):
        fn = corrupted_map_fn(defect)
        for r_b in range(1, 8):
            w, h = packing_dims(r_b)
            lx, ly = oracle.map_rectangle(r_b)
            got = [fn((b % w, b // w), r_b).coord for b in range(w * h)]
            assert any((gx, gy) != (int(x), int(y)) for (gx, gy), x, y in zip(got, lx, ly)), (defect, r_b)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32, np.int64])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_steps_band_equals_full_grid_steps(oracle, dtype, kind):
    """The row-band restatement (go_steps_band, used by the GPU tests at n = 2^17 / 2^18
    where whole grids do not fit the host) == repeated full-grid oracle steps (the
    golden-pinned bb_* kernel, each step reading the previous state: engine.py:201),
    for every band placement: touching the top/bottom grid edge, interior, whole grid."""
    for n in (1, 2, 16, 64, 256):
        for mode in (0, 1):
            states = [oracle.fill_hash(n, dtype, 77, mode)]
            for _ in range(7):
                nxt = states[-1].copy()
                oracle.run_bounding_box(nxt, states[-1], 1, kind, -5)
                states.append(nxt)
            bands = {(0, n), (0, max(1, n // 4)), (n - max(1, n // 4), n), (n // 3, max(n // 3 + 1, n // 2))}
            for y0, y1 in bands:
                steps = [0, 1, 2, 4, 6, 7]
                outs = oracle.steps_band(n, dtype, 77, mode, kind, -5, y0, y1, steps)
                for s, o in zip(steps, outs):
                    assert np.array_equal(o, states[s][y0:y1]), (n, mode, y0, y1, s)
