"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle.

Bit-exact for every integer result: index sets element-wise, grids cell by
cell at sizes the oracle finishes in seconds, and -- at the BASELINE sizes --
checksums against the oracle plus size-independent properties (every
strategy agrees with every other, writes land exactly on the gasket, wrap
arithmetic is linear).
"""

import itertools

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DTYPES = {np.int8: torch.int8, np.int16: torch.int16, np.int32: torch.int32, np.int64: torch.int64,
          np.uint8: torch.uint8}
KINDS = (0, 1, 2)  # CONST, NSUM4, NSUM8 (ours)
# every result-preserving kernel variant of the tuned strategy (include/gasket_b200.h):
# omega order, explicit RMW (+ whole lines), host-row schedule, row-major/chunked,
# cp.async/TMA staging, whole-line fetch, L2 touch, stencil v1, 2-deep ring, digit order
TUNED_FLAGS = (0, 1, 4, 12, 16, 32, 96, 128, 256, 512, 1024, 2048, 2048 | 65536, 2048 | 128, 4096, 65536,
               4 | 512, 65536 | 4096, 2097152, 2097152 | 1048576)


def _to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(a.copy()).cuda()


def _strategies(gm):
    S = gm.geometry.IntraStrategy
    return [S.UNROLL, S.TABLE, S.SUBBOX, S.TUNED]


# ---------------------------------------------------------------------------
# lambda index sets
# ---------------------------------------------------------------------------

def test_lambda_rectangle_elementwise(gpu, oracle):
    for r_b in range(0, 17):
        lx, ly = gpu.device.map_rectangle(r_b)
        ox, oy = oracle.map_rectangle(r_b)
        assert np.array_equal(lx.cpu().numpy(), ox), r_b
        assert np.array_equal(ly.cpu().numpy(), oy), r_b


def test_lambda_rectangle_golden_checksums(gpu, golden):
    meta, _ = golden
    for r_b, (cx, cy) in meta["lambda_checksum"].items():
        lx, ly = gpu.device.map_rectangle(int(r_b))
        assert gpu.device.checksum(lx) == cx and gpu.device.checksum(ly) == cy, r_b


def test_lambda_sampled_levels_17_18(gpu, oracle):
    rng = np.random.default_rng(17)
    for r_b in (17, 18, 19, 20):
        w, h = oracle.packing_dims(r_b)
        idx = rng.integers(0, w * h, size=200_000, dtype=np.int64)
        lx, ly = gpu.device.map_rectangle(r_b)
        ox, oy = oracle.map_blocks(idx % w, idx // w, r_b)
        t = torch.from_numpy(idx).cuda()
        assert np.array_equal(lx[t].cpu().numpy(), ox)
        assert np.array_equal(ly[t].cpu().numpy(), oy)
        del lx, ly


def test_map_blocks_array_arbitrary_inputs(gpu, golden):
    _, arr = golden
    wx, wy = arr["lambda_rand_wx"], arr["lambda_rand_wy"]
    for r_b in (0, 1, 7, 20, 33):
        lx, ly = gpu.blockmap.map_blocks_array(wx, wy, r_b)
        assert lx.dtype == np.int64
        assert np.array_equal(lx, arr[f"lambda_rand_lx_{r_b}"])
        assert np.array_equal(ly, arr[f"lambda_rand_ly_{r_b}"])
    # device in, device out
    lx, ly = gpu.blockmap.map_blocks_array(torch.from_numpy(wx).cuda(), torch.from_numpy(wy).cuda(), 7)
    assert lx.is_cuda and np.array_equal(lx.cpu().numpy(), arr["lambda_rand_lx_7"])


def test_verify_bijection_matches_reference(gpu, golden):
    meta, _ = golden
    bm = gpu.blockmap
    for key, (ok, witness, size) in meta["verify_bijection"].items():
        defect, r_b = key.rsplit("_", 1)
        fn = None if defect == "None" else bm.corrupted_map_fn(defect)
        rep = bm.verify_bijection(int(r_b), fn)
        assert rep.ok == ok, key
        assert (None if rep.witness is None else list(rep.witness)) == witness, key
        assert rep.image_size == size, key
    for r_b in (13, 14, 15, 16):  # beyond the reference's host cap of 12
        assert bm.verify_bijection(r_b).ok


# ---------------------------------------------------------------------------
# grids: every mapping x strategy x kernel x dtype vs the oracle
# ---------------------------------------------------------------------------

def _oracle_result(oracle, grid0, src, rho, kind, param):
    g = grid0.copy()
    oracle.run_bounding_box(g, src, rho, kind, param)
    return g


def _gpu_all(gpu, grid0, src, rho, kind, param):
    """Yield (label, result) for every launch shape the device offers."""
    be = gpu.backends
    n = grid0.shape[0]
    r_b = (n // rho).bit_length() - 1
    sdev = _to_dev(src)
    for early in (False, True):
        g = _to_dev(grid0)
        be.run_bounding_box(g, sdev, rho, kind, param, early_exit=early)
        yield ("bb-exit" if early else "bb"), g
    for strat in _strategies(gpu):
        for flags in (TUNED_FLAGS if strat.value == "tuned" else (0,)):
            g = _to_dev(grid0)
            lx, ly = be.local_cell_arrays(strat, rho)
            be.run_block_space(g, sdev, rho, r_b, strat, lx, ly, kind, param, flags=flags)
            yield f"{strat.value}/f{flags}", g


@pytest.mark.parametrize("dtype", list(DTYPES))
def test_grids_small_exhaustive(gpu, oracle, dtype):
    for n in (1, 2, 4, 8, 16, 32, 64, 128):
        for rho in (1, 2, 4, 8, 16, 32, 64):
            if rho > n:
                continue
            for kind in KINDS:
                for param in (1, -3, 2**31 - 1):
                    grid0 = oracle.fill_hash(n, dtype, 11, 0)
                    src = oracle.fill_hash(n, dtype, 22, 0)
                    want = _oracle_result(oracle, grid0, src, rho, kind, param)
                    for label, got in _gpu_all(gpu, grid0, src, rho, kind, param):
                        ok = np.array_equal(got.cpu().numpy(), want)
                        assert ok, (np.dtype(dtype).name, n, rho, kind, param, label)


@pytest.mark.parametrize("dtype", [np.int8, np.int32])
@pytest.mark.parametrize("n", [1 << 10, 1 << 12, 1 << 13])
def test_grids_medium(gpu, oracle, dtype, n):
    """SURVEY §4 plan: n up to 2^13 x rho in {1..32} x every mapping/strategy x kernel."""
    for kind in KINDS:
        grid0 = oracle.fill_hash(n, dtype, 5, 1)
        src = oracle.fill_hash(n, dtype, 6, 0)
        want = _oracle_result(oracle, grid0, src, 8, kind, 7)
        ck = oracle.checksum(want)
        for rho in (1, 2, 4, 8, 16, 32, 128):
            for label, got in _gpu_all(gpu, grid0, src, rho, kind, 7):
                if n <= 1 << 10:
                    assert np.array_equal(got.cpu().numpy(), want), (n, rho, kind, label)
                else:
                    assert gpu.device.checksum(got) == ck, (n, rho, kind, label)


def test_golden_kernel_checksums_on_device(gpu, oracle, golden):
    """Reference (numba) checksums reproduced by the device kernels directly."""
    meta, _ = golden
    be = gpu.backends
    S = gpu.geometry.IntraStrategy
    for row in meta["kernels_big"]:
        dt = {"int8": torch.int8, "int32": torch.int32}[row["dtype"]]
        src = gpu.device.fill_hash(row["n"], dt, row["seed"], row["mode"])
        assert gpu.device.checksum(src) == row["src_checksum"]
        for strat in (S.TABLE, S.SUBBOX, S.TUNED, S.UNROLL):
            g = src.clone()
            be.run_block_space(g, src.clone(), row["rho"], (row["n"] // row["rho"]).bit_length() - 1, strat,
                               kind=row["kind"], param=row["param"])
            assert gpu.device.checksum(g) == row["out"], (row, strat)


# ---------------------------------------------------------------------------
# BASELINE sizes
# ---------------------------------------------------------------------------

# n = 2^16 / 2^17 / 2^18 against the oracle cell for cell: tests/test_baseline_sizes.py


def test_n16_int32_const_write_counts(gpu):
    """Write pass at 2^16 int32 on a sentinel background: exactly 3^16 cells change."""
    n = 1 << 16
    S = gpu.geometry.IntraStrategy
    for rho, strat in [(16, S.TUNED), (32, S.SUBBOX)]:
        g = torch.full((n, n), -5, dtype=torch.int32, device="cuda")
        gpu.backends.run_block_space(g, g, rho, 16 - rho.bit_length() + 1, strat, kind=0, param=7)
        assert int((g == 7).sum()) == 3**16
        assert int((g == -5).sum()) == n * n - 3**16
        del g


# ---------------------------------------------------------------------------
# engine API, coverage, host transports
# ---------------------------------------------------------------------------

def test_launch_examples_match_reference(gpu, golden):
    meta, _ = golden
    eng = gpu.engine
    from tests.golden.make_golden import hash_grid
    for ex in meta["launch_examples"]:
        spec = gpu.geometry.FractalSpec(n=ex["n"], rho=ex["rho"])
        cfg = eng.LaunchConfig(spec=spec, mapping=eng.Mapping(ex["mapping"]),
                               strategy=gpu.geometry.IntraStrategy(ex["strategy"]) if ex["strategy"] else None,
                               kernel=eng.CellKernel(eng.KernelKind(ex["kind"]), ex["param"]), verify_coverage=True)
        for as_device in (True, False):
            g = hash_grid(ex["n"], np.int32, 3, 0) if ex["kind"] != "const" else np.zeros((ex["n"],) * 2, np.int32)
            if as_device:
                g = torch.from_numpy(g).cuda()
            m = eng.launch(cfg, g)
            gn = g.cpu().numpy() if as_device else g
            from tests.golden.make_golden import checksum
            assert checksum(gn) == ex["grid"], ex
            assert [m.blocks_launched, m.threads_launched, m.threads_useful, m.map_ops, m.reduction_depth,
                    m.simulated_cost] == ex["metrics"]


def test_coverage_reports_match_reference(gpu, golden):
    meta, _ = golden
    eng = gpu.engine
    from tests.golden.make_golden import checksum
    for row in meta["coverage"]:
        spec = gpu.geometry.FractalSpec(n=row["n"], rho=row["rho"])
        cfg = eng.LaunchConfig(spec=spec, mapping=eng.Mapping.BLOCK_SPACE,
                               strategy=gpu.geometry.IntraStrategy(row["strategy"]))
        fn = None if row["defect"] is None else gpu.blockmap.corrupted_map_fn(row["defect"])
        rep = eng.verify_coverage(cfg, fn)
        assert rep.exact == row["exact"], row
        assert checksum(rep.counts) == row["counts"], row
        assert len(rep.duplicates) == row["ndups"] and len(rep.misses) == row["nmisses"]
        assert [list(c) for c in rep.duplicates[:50]] == row["dups"]
        assert [list(c) for c in rep.misses[:50]] == row["misses"]


def test_coverage_real_kernels_exact_large(gpu):
    eng = gpu.engine
    S = gpu.geometry.IntraStrategy
    for n, rho in ((1 << 12, 8), (1 << 14, 32), (1 << 14, 1)):
        spec = gpu.geometry.FractalSpec(n=n, rho=rho)
        for mapping, strat in [(eng.Mapping.BOUNDING_BOX, None), (eng.Mapping.BOUNDING_BOX_EXIT, None)] + \
                [(eng.Mapping.BLOCK_SPACE, s) for s in S]:
            rep = eng.verify_coverage(eng.LaunchConfig(spec=spec, mapping=mapping, strategy=strat))
            assert rep.exact, (n, rho, mapping, strat)


@pytest.mark.parametrize("transport", ["copy", "mapped"])
def test_numpy_host_path(gpu, oracle, monkeypatch, transport):
    monkeypatch.setenv("GASKET_HOST_TRANSPORT", transport)
    S = gpu.geometry.IntraStrategy
    for n, dtype, kind in itertools.product((64, 1024), (np.int8, np.int32), KINDS):
        grid0 = oracle.fill_hash(n, dtype, 1, 0)
        src = oracle.fill_hash(n, dtype, 2, 0)
        want = _oracle_result(oracle, grid0, src, 16, kind, 9)
        for strat in (S.TUNED, S.SUBBOX):
            g = grid0.copy()
            gpu.backends.run_block_space(g, src, 16, (n // 16).bit_length() - 1, strat, kind=kind, param=9)
            assert np.array_equal(g, want), (transport, n, dtype, kind, strat)
        g = grid0.copy()
        gpu.backends.run_bounding_box(g, src, 16, kind, 9)
        assert np.array_equal(g, want)


def test_mapped_write_pass_multi_chunk_rows(gpu, monkeypatch):
    """The host-mapped write pass (hostrows.cu) at sizes whose rows span several K-line
    work units: equal to the device write pass on the same grid, cell for cell."""
    from paper_1706_04552_b200 import device

    monkeypatch.setenv("GASKET_HOST_TRANSPORT", "mapped")
    S = gpu.geometry.IntraStrategy
    for n, dtype in ((1 << 14, torch.int8), (1 << 14, torch.int16), (1 << 13, torch.int32)):
        dev = device.fill_hash(n, dtype, 17, 0)
        host = torch.empty((n, n), dtype=dtype, pin_memory=True)
        host.copy_(dev.cpu())
        g = host.numpy()
        rho = 32
        r_b = (n // rho).bit_length() - 1
        gpu.backends.run_block_space(g, g, rho, r_b, S.TUNED, kind=0, param=-3)
        gpu.backends.run_block_space(dev, dev, rho, r_b, S.TUNED, kind=0, param=-3)
        assert torch.equal(torch.from_numpy(g).cuda(), dev), (n, str(dtype))


def test_src_alias_is_snapshotted(gpu, oracle):
    n = 256
    grid0 = oracle.fill_hash(n, np.int32, 4, 0)
    want = grid0.copy()
    oracle.run_bounding_box(want, grid0.copy(), 4, 1, 1)
    g = torch.from_numpy(grid0.copy()).cuda()
    gpu.backends.run_block_space(g, g, 4, 6, gpu.geometry.IntraStrategy.TUNED, kind=1, param=1)
    assert np.array_equal(g.cpu().numpy(), want)


def test_errors_are_loud(gpu):
    be = gpu.backends
    g = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        be.run_block_space(g, g, 128, 0, gpu.geometry.IntraStrategy.SUBBOX)
    with pytest.raises(ValueError):
        be.run_block_space(g, g, 8, 4, gpu.geometry.IntraStrategy.SUBBOX)  # r_b mismatch (64/8 = 2^3)
    with pytest.raises(ValueError):
        be.run_bounding_box(torch.zeros((64, 32), dtype=torch.int32, device="cuda"), None, 8, 0, 1)
    with pytest.raises(ValueError):
        be.run_bounding_box(torch.zeros((64, 64), dtype=torch.float32, device="cuda"), None, 8, 0, 1)
    with pytest.raises(RuntimeError):
        be.resolve_backend("numba")
    with pytest.raises(OverflowError):
        be.run_bounding_box(g, g, 8, 0, 2**31)


def test_launch_counter_moves(gpu):
    before = gpu.native.launch_count()
    g = torch.zeros((64, 64), dtype=torch.int8, device="cuda")
    gpu.backends.run_block_space(g, g, 8, 3, gpu.geometry.IntraStrategy.TUNED)
    torch.cuda.synchronize()
    assert gpu.native.launch_count() == before + 1


# ---------------------------------------------------------------------------
# multi-step CA driver (ping-pong + CUDA graph) and wide cells
# ---------------------------------------------------------------------------

def _oracle_steps(oracle, init, kind, param, steps):
    want = init.copy()
    for _ in range(steps):
        nxt = want.copy()
        oracle.run_bounding_box(nxt, want, 1, kind, param)
        want = nxt
    return want


@pytest.mark.parametrize("kind", [1, 2])
@pytest.mark.parametrize("temporal", [1, 2, 4, 6])
def test_ca_runner_matches_oracle_steps(gpu, oracle, kind, temporal):
    from paper_1706_04552_b200 import ca

    for dtype, n in ((np.int8, 512), (np.int8, 128), (np.int16, 256), (np.int32, 64), (np.int32, 32)):
        init = oracle.fill_hash(n, dtype, 13, 0)
        want7 = _oracle_steps(oracle, init, kind, 3, 7)
        want20 = _oracle_steps(oracle, want7, kind, 3, 13)
        for use_graph in (False, True):
            g = torch.from_numpy(init.copy()).cuda()
            runner = ca.CARunner(g, kind=kind, param=3, use_graph=use_graph, temporal=temporal)
            out = runner.run(3)
            out = runner.run(4)
            assert runner.steps_done == 7
            assert np.array_equal(out.cpu().numpy(), want7), (np.dtype(dtype).name, n, use_graph)
            # a longer run: graph replays of 2 * temporal steps plus a remainder
            out = runner.run(13)
            assert runner.steps_done == 20
            want = want20
            assert np.array_equal(out.cpu().numpy(), want), (np.dtype(dtype).name, n, use_graph)
        g = torch.from_numpy(init.copy()).cuda()
        ca.run_ca(g, 10, kind=kind, param=3, temporal=temporal)
        assert np.array_equal(g.cpu().numpy(), _oracle_steps(oracle, init, kind, 3, 10)), (np.dtype(dtype).name, n)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32])
@pytest.mark.parametrize("steps", [2, 4, 6])
def test_fused_steps_vs_oracle(gpu, oracle, dtype, steps):
    """gm_ca_steps (2 or 4 CA steps per pass) == that many oracle steps, cell by cell,
    incl. grid-edge tiles and a 2^12 grid; also on a CA state that is 0 off the gasket."""
    from paper_1706_04552_b200 import device, native

    n0 = 128 // np.dtype(dtype).itemsize
    if steps == 6 and np.dtype(dtype).itemsize == 4:  # the 6-cell cone outgrows a 4-cell halo chunk
        src = torch.zeros((n0, n0), dtype=torch.int32, device="cuda")
        with pytest.raises(ValueError):
            native.call("gm_ca_steps", src.clone().data_ptr(), src.data_ptr(), n0, 4, 2, 1, 6, 0,
                        device.stream_handle())
        return
    for n in (n0, 2 * n0, 4 * n0, 1 << 12):
        for mode in (0, 1):
            init = oracle.fill_hash(n, dtype, 41 + mode, mode)
            for kind in (1, 2):
                for param in (1, -7):
                    want = _oracle_steps(oracle, init, kind, param, steps)
                    src = torch.from_numpy(init.copy()).cuda()
                    dst = src.clone()
                    if steps == 2:
                        native.call("gm_ca_step2", dst.data_ptr(), src.data_ptr(), n, src.element_size(), kind, param,
                                    0, device.stream_handle())
                    else:
                        native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, src.element_size(), kind, param,
                                    steps, 0, device.stream_handle())
                    assert np.array_equal(dst.cpu().numpy(), want), (np.dtype(dtype).name, n, mode, kind, param)
                    assert np.array_equal(src.cpu().numpy(), init)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32])
@pytest.mark.parametrize("steps", [1, 2, 4, 6])
def test_ca_run_edge_cache_vs_oracle(gpu, oracle, dtype, steps):
    """gm_ca_run with the static left-edge cache (edge.cu) == the same run without it ==
    that many oracle steps, every cell: grid-edge tiles, interior tiles whose left
    neighbour tile is (not) a gasket tile, both kinds, both background modes."""
    from paper_1706_04552_b200 import device, native

    c = np.dtype(dtype).itemsize
    if steps == 6 and c == 4:
        return  # (the 6-cell cone outgrows a 4-cell halo chunk: gm_ca_run raises, as gm_ca_steps)
    n0 = 128 // c
    for n in (n0, 2 * n0, 8 * n0, 1 << 12):
        for mode in (0, 1):
            init = oracle.fill_hash(n, dtype, 51 + mode, mode)
            src = torch.from_numpy(init.copy()).cuda()
            edge = torch.empty(native.ca_edge_bytes(n, c), dtype=torch.uint8, device="cuda")
            native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, c, -1, 0, 0, None, 0,
                        device.stream_handle())
            for kind in (1, 2):
                want = _oracle_steps(oracle, init, kind, -3, steps)
                for e in (None, edge.data_ptr()):
                    dst = src.clone()
                    native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), n, c, kind, -3, steps, e, 0,
                                device.stream_handle())
                    assert np.array_equal(dst.cpu().numpy(), want), (np.dtype(dtype).name, n, mode, kind, e is None)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32])
def test_inplace_neighbour_sum_vs_oracle(gpu, oracle, dtype):
    """A neighbour-sum launch whose src is the grid (engine.launch semantics, engine.py:201)
    through the tuned kernel runs in place with a snapshot of the tiles' border cells only
    (gm_run_inplace): every cell equals the oracle's step from the pre-launch grid --
    grid-edge tiles, n from one tile to 2^12, both kinds, both background modes, and
    repeated launches (each reading the previous launch's result)."""
    be, S = gpu.backends, gpu.geometry.IntraStrategy
    c = np.dtype(dtype).itemsize
    n0 = 128 // c
    for n in (n0, 2 * n0, 8 * n0, 1 << 12):
        for mode in (0, 1):
            init = oracle.fill_hash(n, dtype, 61 + mode, mode)
            for kind in (1, 2):
                g = torch.from_numpy(init.copy()).cuda()
                want = init.copy()
                rho = min(64, n)
                for _ in range(3):
                    be.run_block_space(g, g, rho, (n // rho).bit_length() - 1, S.TUNED, kind=kind, param=-7)
                    nxt = want.copy()
                    oracle.run_bounding_box(nxt, want, 1, kind, -7)
                    want = nxt
                    assert np.array_equal(g.cpu().numpy(), want), (np.dtype(dtype).name, n, mode, kind)


def test_engine_launch_device_inplace_int32(gpu, oracle):
    """engine.launch NEIGHBOR_SUM on an int32 device grid (the reference's entry point):
    tuned (in place, border snapshot) and SUBBOX (masked snapshot) == the oracle."""
    from paper_1706_04552_b200 import engine
    from paper_1706_04552_b200.geometry import FractalSpec, IntraStrategy

    n = 1 << 11
    init = oracle.fill_hash(n, np.int32, 5, 0)
    want = init.copy()
    oracle.run_bounding_box(want, init, 1, 1, 3)
    for strat, rho in ((IntraStrategy.TUNED, 32), (IntraStrategy.SUBBOX, 16)):
        g = torch.from_numpy(init.copy()).cuda()
        cfg = engine.LaunchConfig(spec=FractalSpec(n=n, rho=rho), mapping=engine.Mapping.BLOCK_SPACE, strategy=strat,
                                  kernel=engine.CellKernel(engine.KernelKind.NEIGHBOR_SUM, 3))
        engine.launch(cfg, g)
        assert np.array_equal(g.cpu().numpy(), want), strat


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32, np.int64])
def test_vectorised_bounding_box_neighbour_sums(gpu, oracle, dtype):
    """run_bounding_box(vectorized=True) for neighbour sums -- the tuned tile stencil over
    every tile of the grid, tiles off the gasket exiting (8-byte cells and narrow grids: the
    literal bounding box) -- == the oracle, with the drop-in semantics (grid keeps its
    off-gasket cells) and on src aliasing grid."""
    be = gpu.backends
    c = np.dtype(dtype).itemsize
    for n in sorted({16, 128 // c, 4 * (128 // c), 1 << 11}):
        grid0 = oracle.fill_hash(n, dtype, 71, 0)
        src = oracle.fill_hash(n, dtype, 72, 0)
        for kind in (1, 2):
            want = _oracle_result(oracle, grid0, src, 8, kind, -2)
            g = _to_dev(grid0)
            be.run_bounding_box(g, _to_dev(src), min(32, n), kind, -2, vectorized=True)
            assert np.array_equal(g.cpu().numpy(), want), (np.dtype(dtype).name, n, kind)
            # src is the grid: engine.launch semantics (the snapshot path)
            want_a = _oracle_result(oracle, grid0, grid0, 8, kind, -2)
            g = _to_dev(grid0)
            be.run_bounding_box(g, g, min(32, n), kind, -2, vectorized=True)
            assert np.array_equal(g.cpu().numpy(), want_a), (np.dtype(dtype).name, n, kind, "alias")


def test_ca_run_rejects_bad_arguments(gpu):
    from paper_1706_04552_b200 import device, native

    g = torch.zeros((256, 256), dtype=torch.int8, device="cuda")
    h = g.clone()
    s = device.stream_handle()
    for steps in (0, 3, 8):
        with pytest.raises(ValueError):
            native.call("gm_ca_run", g.data_ptr(), h.data_ptr(), 256, 1, 2, 1, steps, None, 0, s)
    with pytest.raises(ValueError):  # CONST is not a CA step
        native.call("gm_ca_run", g.data_ptr(), h.data_ptr(), 256, 1, 0, 1, 1, None, 0, s)
    with pytest.raises(ValueError):  # src must not alias grid
        native.call("gm_ca_run", g.data_ptr(), g.data_ptr(), 256, 1, 2, 1, 1, None, 0, s)
    with pytest.raises(ValueError):  # 8-byte cells have no tiled kernel
        native.call("gm_ca_run", g.data_ptr(), h.data_ptr(), 32, 8, 2, 1, 1, None, 0, s)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32])
def test_dst_from_src_variants(gpu, oracle, dtype):
    """GM_FLAG_DST_FROM_SRC (grid == snapshot off the gasket: engine.launch / CA
    ping-pong) through every stencil kernel variant, including edge tiles."""
    be, S = gpu.backends, gpu.geometry.IntraStrategy
    n0 = 128 // np.dtype(dtype).itemsize  # one tile
    for n in (n0, 2 * n0, 8 * n0, 1 << 12):
        src = oracle.fill_hash(n, dtype, 31, 0)
        for kind in (1, 2):
            want = _oracle_result(oracle, src.copy(), src, 8, kind, -5)
            for flags in (2, 2 | 65536, 2 | 2048, 2 | 2048 | 128, 2 | 4096, 2 | 512, 2 | 64, 2 | 256, 2 | 2097152):
                g = _to_dev(src)
                r_b = (n // 8).bit_length() - 1
                be.run_block_space(g, _to_dev(src), 8, r_b, S.TUNED, kind=kind, param=-5, flags=flags)
                assert np.array_equal(g.cpu().numpy(), want), (np.dtype(dtype).name, n, kind, flags)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_int64_and_uint16_cells(gpu, oracle, kind):
    for dtype in (np.int64, np.uint16):
        for n in (64, 256):
            grid0 = oracle.fill_hash(n, dtype, 3, 0)
            src = oracle.fill_hash(n, dtype, 4, 0)
            want = _oracle_result(oracle, grid0, src, 8, kind, -9)
            for label, got in _gpu_all(gpu, grid0, src, 8, kind, -9):
                assert np.array_equal(got.cpu().numpy(), want), (np.dtype(dtype).name, n, label)


def test_whole_grid_tile_and_unit_grid(gpu, oracle):
    """rho == n (one block) and n == 1 (a single cell) for every mapping."""
    for n in (1, 2, 128):
        for kind in KINDS:
            grid0 = oracle.fill_hash(n, np.int8, 8, 0)
            src = oracle.fill_hash(n, np.int8, 9, 0)
            want = _oracle_result(oracle, grid0, src, n, kind, 5)
            for label, got in _gpu_all(gpu, grid0, src, n, kind, 5):
                assert np.array_equal(got.cpu().numpy(), want), (n, kind, label)


@pytest.mark.parametrize("dtype", [torch.int8, torch.int16, torch.int32])
@pytest.mark.parametrize("steps", [2, 4, 6])
def test_fused_steps_equal_single_steps_large(gpu, dtype, steps):
    """At sizes past the oracle's reach: gm_ca_steps == that many single-step launches,
    bit for bit."""
    from paper_1706_04552_b200 import device, native

    be, S = gpu.backends, gpu.geometry.IntraStrategy
    if steps == 6 and dtype == torch.int32:
        pytest.skip("6 fused steps need 1- or 2-byte cells")
    n = 1 << 15 if dtype == torch.int8 else 1 << 14
    for kind in (1, 2):
        src = device.fill_hash(n, dtype, 77, 0)
        a, b = src.clone(), src.clone()
        for _ in range(steps):
            be.run_block_space(b, a, 64, (n // 64).bit_length() - 1, S.TUNED, kind=kind, param=5,
                               flags=native.FLAG_DST_FROM_SRC)
            a, b = b, a
        fused = src.clone()
        native.call("gm_ca_steps", fused.data_ptr(), src.data_ptr(), n, src.element_size(), kind, 5, steps, 0,
                    device.stream_handle())
        assert torch.equal(fused, a), (dtype, kind)


def test_randomised_launches_vs_oracle(gpu, oracle):
    """Seeded fuzz over (n, rho, cell type, kernel, param, strategy, tuned flags) -- every
    launch cell-by-cell against the oracle."""
    rng = np.random.default_rng(20261017)
    be, S = gpu.backends, gpu.geometry.IntraStrategy
    dtypes = list(DTYPES)
    for _ in range(160):
        r = int(rng.integers(0, 11))
        n = 1 << r
        rho = 1 << int(rng.integers(0, r + 1))
        dtype = dtypes[int(rng.integers(0, len(dtypes)))]
        kind = int(rng.integers(0, 3))
        param = int(rng.integers(-(2**31), 2**31 - 1))
        grid0 = oracle.fill_hash(n, dtype, int(rng.integers(0, 1 << 30)), int(rng.integers(0, 2)))
        src = oracle.fill_hash(n, dtype, int(rng.integers(0, 1 << 30)), 0)
        want = _oracle_result(oracle, grid0, src, rho, kind, param)
        strat = [S.UNROLL, S.TABLE, S.SUBBOX, S.TUNED][int(rng.integers(0, 4))]
        flags = int(TUNED_FLAGS[int(rng.integers(0, len(TUNED_FLAGS)))]) if strat is S.TUNED else 0
        g = _to_dev(grid0)
        lx, ly = be.local_cell_arrays(strat, rho)
        be.run_block_space(g, _to_dev(src), rho, (n // rho).bit_length() - 1, strat, lx, ly, kind, param, flags=flags)
        assert np.array_equal(g.cpu().numpy(), want), (n, rho, np.dtype(dtype).name, kind, param, strat, flags)


def test_randomised_fused_steps_vs_oracle(gpu, oracle):
    """Seeded fuzz over the fused multi-step kernel (gm_ca_steps): grid size, cell type,
    kernel, param, steps per launch, CA-mode or random off-gasket state -- every launch
    cell by cell against that many oracle steps."""
    from paper_1706_04552_b200 import device, native

    rng = np.random.default_rng(20261018)
    for _ in range(40):
        dtype = [np.int8, np.uint8, np.int16, np.int32][int(rng.integers(0, 4))]
        c = np.dtype(dtype).itemsize
        n = (128 // c) << int(rng.integers(0, 4))  # one tile .. 8 tiles per edge
        kind = int(rng.integers(1, 3))
        steps = (2, 4, 6)[int(rng.integers(0, 3 if c <= 2 else 2))]
        param = int(rng.integers(-(2**31), 2**31 - 1))
        init = oracle.fill_hash(n, dtype, int(rng.integers(0, 1 << 30)), int(rng.integers(0, 2)))
        want = _oracle_steps(oracle, init, kind, param, steps)
        src = torch.from_numpy(init.copy()).cuda()
        dst = src.clone()
        native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, c, kind, int(np.int32(param)), steps, 0,
                    device.stream_handle())
        assert np.array_equal(dst.cpu().numpy(), want), (n, np.dtype(dtype).name, kind, steps, param)


def test_partitioned_fused_steps_random_ranges(gpu):
    """gm_run_part_steps over random sub-gasket ranges [lo, hi) of a random level: the
    cells of those sub-gaskets == the unpartitioned fused launch, everything else
    untouched (the launch reads a halo-complete copy: here the whole previous state)."""
    from paper_1706_04552_b200 import device, native
    from paper_1706_04552_b200 import partition as P

    rng = np.random.default_rng(7)
    n = 1 << 12
    for _ in range(12):
        kind = int(rng.integers(1, 3))
        steps = (2, 4, 6)[int(rng.integers(0, 3))]
        level = int(rng.integers(0, 6))  # sub-gaskets >= one 128-byte tile
        nsg = 3**level
        lo = int(rng.integers(0, nsg))
        hi = int(rng.integers(lo, nsg + 1))
        src = device.fill_hash(n, torch.int8, int(rng.integers(0, 1 << 30)), 0)
        full = src.clone()
        native.call("gm_ca_steps", full.data_ptr(), src.data_ptr(), n, 1, kind, 3, steps, 0, device.stream_handle())
        part = src.clone()
        native.call("gm_run_part_steps", part.data_ptr(), src.data_ptr(), n, 1, kind, 3, steps, 0, level, lo, hi,
                    device.stream_handle())
        m = n >> level
        mask = torch.zeros((n, n), dtype=torch.bool, device="cuda")
        for s in range(lo, hi):
            bx, by = P.subgasket_block(s, level)
            mask[by * m:(by + 1) * m, bx * m:(bx + 1) * m] = True
        assert torch.equal(part[mask], full[mask]), (kind, steps, level, lo, hi)
        assert torch.equal(part[~mask], src[~mask]), (kind, steps, level, lo, hi)


@pytest.mark.parametrize("dtype", [torch.int8, torch.int16, torch.int32, torch.int64])
def test_masked_snapshot_serves_every_stencil(gpu, dtype):
    """gm_snapshot_stencil (engine.launch's grid.copy(), masked): a snapshot buffer that
    holds garbage outside the copied windows gives every neighbour-sum kernel the same
    result as a full copy -- literal strategies, BB, the tuned kernel and its variants."""
    from paper_1706_04552_b200 import device, native

    be, S = gpu.backends, gpu.geometry.IntraStrategy
    c = torch.empty((), dtype=dtype).element_size()
    for n in (128 // c, 4 * (128 // c), 1 << 11):
        grid0 = device.fill_hash(n, dtype, 91, 0)
        snap = device.fill_hash(n, dtype, 92, 0)  # garbage outside the windows
        native.call("gm_snapshot_stencil", snap.data_ptr(), grid0.data_ptr(), n, c, device.stream_handle())
        for kind in (1, 2):
            for rho, strat, flags in ((8, S.TUNED, 2), (8, S.TUNED, 0), (8, S.SUBBOX, 0), (8, S.TABLE, 0),
                                      (16, S.UNROLL, 0), (8, S.TUNED, 2 | 2048), (8, S.TUNED, 2 | 4096)):
                if rho > n:
                    continue
                r_b = (n // rho).bit_length() - 1
                lx, ly = be.local_cell_arrays(strat, rho)
                want = grid0.clone()
                be.run_block_space(want, grid0.clone(), rho, r_b, strat, lx, ly, kind, 7, flags=flags)
                got = grid0.clone()
                be.run_block_space(got, snap, rho, r_b, strat, lx, ly, kind, 7, flags=flags)
                assert torch.equal(got, want), (n, str(dtype), kind, rho, strat, flags)
            want = grid0.clone()
            be.run_bounding_box(want, grid0.clone(), 8, kind, 7)
            got = grid0.clone()
            be.run_bounding_box(got, snap, 8, kind, 7)
            assert torch.equal(got, want), (n, str(dtype), kind, "bb")


def test_engine_launch_neighbour_sum_uses_masked_snapshot(gpu, oracle):
    """engine.launch (engine.py:193-211) on a device grid, NEIGHBOR_SUM: the result equals
    the oracle's step (the masked snapshot replaces the full grid.copy())."""
    eng = gpu.engine
    from paper_1706_04552_b200.geometry import FractalSpec

    for n, rho in ((256, 8), (1024, 16)):
        init = oracle.fill_hash(n, np.int32, 5, 0)
        want = init.copy()
        oracle.run_bounding_box(want, init, 1, oracle.KIND_NSUM4, 1)
        spec = FractalSpec(n=n, rho=rho)
        for strat in (gpu.geometry.IntraStrategy.TUNED, gpu.geometry.IntraStrategy.TABLE):
            g = torch.from_numpy(init.copy()).cuda()
            cfg = eng.LaunchConfig(spec=spec, mapping=eng.Mapping.BLOCK_SPACE, strategy=strat,
                                   kernel=eng.CellKernel(eng.KernelKind.NEIGHBOR_SUM, 1))
            eng.launch(cfg, g)
            assert np.array_equal(g.cpu().numpy(), want), (n, rho, strat)


@pytest.mark.parametrize("transport", ["mapped", "copy"])
def test_engine_launch_neighbour_sum_host_grid(gpu, oracle, monkeypatch, transport):
    """engine.launch NEIGHBOR_SUM on an int32 numpy grid: src is the grid itself and the
    backend keeps engine.py:201's snapshot semantics (the staged path for the tuned
    kernel, a device snapshot otherwise) -- the oracle's step for every mapping."""
    monkeypatch.setenv("GASKET_HOST_TRANSPORT", transport)
    eng = gpu.engine
    from paper_1706_04552_b200.geometry import FractalSpec

    S = gpu.geometry.IntraStrategy
    for n, rho in ((256, 8), (1024, 16)):
        init = oracle.fill_hash(n, np.int32, 15, 0)
        want = init.copy()
        oracle.run_bounding_box(want, init, 1, oracle.KIND_NSUM4, 2)
        spec = FractalSpec(n=n, rho=rho)
        for mapping, strat in ((eng.Mapping.BLOCK_SPACE, S.TUNED), (eng.Mapping.BLOCK_SPACE, S.TABLE),
                               (eng.Mapping.BOUNDING_BOX, None)):
            g = init.copy()
            cfg = eng.LaunchConfig(spec=spec, mapping=mapping, strategy=strat,
                                   kernel=eng.CellKernel(eng.KernelKind.NEIGHBOR_SUM, 2))
            eng.launch(cfg, g)
            assert np.array_equal(g, want), (transport, n, mapping, strat)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32, np.int64])
@pytest.mark.parametrize("pinned", [True, False])
def test_mapped_staged_neighbour_sum(gpu, oracle, monkeypatch, dtype, pinned):
    """Host-mapped numpy grid, src is the grid (engine.launch semantics): the staged path
    (masked snapshot -> device kernel -> whole-line write-back, gm_writeback_tiles; for
    1/2/4-byte cells in bands of block rows on two streams) ==
    the oracle's step, cell for cell, off-gasket cells untouched.  Pinned (torch
    pin_memory) and pageable (plain numpy, registered once by the pin cache) grids;
    int64 covers the grids whose stencil kernel does not store whole sectors (16 <= n <
    32), which must not take the staged path."""
    monkeypatch.setenv("GASKET_HOST_TRANSPORT", "mapped")
    S = gpu.geometry.IntraStrategy
    c = np.dtype(dtype).itemsize
    sizes = {128 // c, 2 * (128 // c), 4 * (128 // c), 1 << 12}
    if c == 1:
        sizes.add(1 << 14)  # (the banded path: 8 bands of whole block rows, 2 streams)
    for n in sorted(sizes):
        for kind in (1, 2):
            grid0 = oracle.fill_hash(n, dtype, 23 + kind, 0)
            want = grid0.copy()
            oracle.run_bounding_box(want, grid0.copy(), 1, kind, -4)
            g = torch.from_numpy(grid0.copy()).pin_memory().numpy() if pinned else grid0.copy()
            rho = min(64, n)
            for _ in range(2):  # the second call reuses the cached registration
                gpu.backends.run_block_space(g, g, rho, (n // rho).bit_length() - 1, S.TUNED, kind=kind, param=-4)
                assert np.array_equal(g, want), (n, np.dtype(dtype).name, kind, pinned)
                g[...] = grid0


def test_pin_cache_registers_once_and_releases(gpu, monkeypatch):
    """Pageable numpy grids are registered once per owning array and unregistered when
    the array is collected; views share the owner's registration."""
    import gc

    monkeypatch.setenv("GASKET_HOST_TRANSPORT", "mapped")
    dev = gpu.device
    dev.pinned.clear()
    n = 1 << 10
    g = np.zeros((n, n), dtype=np.int8)
    S = gpu.geometry.IntraStrategy
    gpu.backends.run_block_space(g, g, 32, 5, S.TUNED, kind=0, param=3)
    assert dev.pinned.pinned_bytes() == g.nbytes
    v = g[: n // 2]
    assert dev.pinned.pin(v) and dev.pinned.pinned_bytes() == g.nbytes
    y = np.arange(n).reshape(n, 1)
    x = np.arange(n).reshape(1, n)
    assert np.array_equal(g, np.where((x & (n - 1 - y)) == 0, 3, 0).astype(np.int8))
    del v, g
    gc.collect()
    assert dev.pinned.pinned_bytes() == 0


def test_mapped_staged_stencil_misaligned_host_grids(gpu, oracle, monkeypatch):
    """The staged neighbour-sum path (masked snapshot -> kernel -> write-back) on host grids
    16..112 bytes past a 64-byte boundary (the host-aligned windows of snapshot.cu):
    == the oracle step, the bytes around the array untouched."""
    monkeypatch.setenv("GASKET_HOST_TRANSPORT", "mapped")
    S = gpu.geometry.IntraStrategy
    for dtype in (np.int8, np.int16, np.int32):
        c = np.dtype(dtype).itemsize
        for n in (128 // c, 4 * (128 // c), 512):
            nbytes = n * n * c
            for shift in (16, 32, 48, 80, 112):
                for kind in (1, 2):
                    raw = np.zeros(nbytes + 512, dtype=np.uint8)
                    base = (-raw.ctypes.data) % 128 + 128 + shift
                    raw[:] = 0x5A
                    g = raw[base:base + nbytes].view(dtype).reshape(n, n)
                    g0 = oracle.fill_hash(n, dtype, 11 + shift, 0)
                    g[...] = g0
                    want = g0.copy()
                    oracle.run_bounding_box(want, g0, 1, kind, 5)
                    gpu.backends.run_block_space(g, g, 64 if n >= 64 else n, (n // min(64, n)).bit_length() - 1,
                                                 S.TUNED, kind=kind, param=5)
                    assert np.array_equal(g, want), (np.dtype(dtype).name, n, shift, kind)
                    assert (raw[:base] == 0x5A).all() and (raw[base + nbytes:] == 0x5A).all(), (n, shift, "guard")
                    del g
    gpu.device.pinned.clear()


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32])
def test_mapped_write_misaligned_host_grids(gpu, oracle, monkeypatch, dtype):
    """The mapped write pass on host grids that do not start on a 128-byte boundary (a
    plain numpy array sits 16 bytes into its pages): the host-aligned kernel
    (host_rows_write16_shift) == the oracle for every 16-byte shift, the bytes around the
    array (another owner's memory) untouched, zero-background mode included."""
    monkeypatch.setenv("GASKET_HOST_TRANSPORT", "mapped")
    S = gpu.geometry.IntraStrategy
    c = np.dtype(dtype).itemsize
    for n in (128 // c, 2 * (128 // c), 1024):
        nbytes = n * n * c
        for shift in range(0, 128, 16):
            for zero in (False, True):
                raw = np.zeros(nbytes + 512, dtype=np.uint8)
                base = (-raw.ctypes.data) % 128 + 128 + shift
                raw[:] = 0xA5
                g = raw[base:base + nbytes].view(dtype).reshape(n, n)
                g0 = np.zeros((n, n), dtype) if zero else oracle.fill_hash(n, dtype, 3 + shift, 0)
                g[...] = g0
                want = g0.copy()
                oracle.run_bounding_box(want, want, 1, 0, -7)
                gpu.backends.run_block_space(g, g, min(32, n), (n // min(32, n)).bit_length() - 1, S.TUNED, kind=0,
                                             param=-7, assume_zero_background=zero)
                assert np.array_equal(g, want), (n, shift, zero)
                assert (raw[:base] == 0xA5).all() and (raw[base + nbytes:] == 0xA5).all(), (n, shift, "guard")
                del g
    gpu.device.pinned.clear()
