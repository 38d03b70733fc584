"""BASELINE.json configs at their own sizes, cell for cell against the CPU oracle.

Config 2 (n = 2^16 write pass, every strategy), config 3 (n = 2^17 int8 8-neighbour
CA step; 4-neighbour too) and the single-GPU leg of config 5 (n = 2^18 int8 CA).
Reference semantics: _cell_value (backends.py:127-141) on the gasket cells only
(backends.py:155-156), each step reading the pre-launch state (engine.py:201).

No checksums: every comparison counts differing words between the device result
and the oracle grid uploaded band by band (tests/gpu_compare.py).  The oracle for
grids the host cannot hold whole is the row-band restatement oracle.steps_band,
itself pinned to the full-grid oracle in tests/test_oracle_golden.py.

This file sorts before the slower GPU files so its cases run first.
"""

import numpy as np
import pytest
import torch

from tests.gpu_compare import band_mismatches, sampled_bands

pytestmark = pytest.mark.gpu

FLAG_DST_FROM_SRC = 2


def _ca_steps(gpu, dst, src, n, kind, steps):
    gpu.native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, dst.element_size(), kind, 1, steps, 0,
                    gpu.device.stream_handle())


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_n16_int8_every_strategy_exact(gpu, oracle, kind):
    """n = 2^16 int8 (BASELINE config 2 and its stencil variants): the tuned kernels at
    every rho, the paper-literal SUBBOX / TABLE / UNROLL and the bounding box ==
    the oracle, every cell (the oracle grid is uploaded once, then compared on the
    device)."""
    n = 1 << 16
    S = gpu.geometry.IntraStrategy
    want = oracle.steps_band(n, np.int8, 3, 0, kind, 1, 0, n, [1])[0]
    want_d = torch.from_numpy(want).cuda()
    del want
    src = gpu.device.fill_hash(n, torch.int8, 3, 0)
    g = torch.empty_like(src)
    cases = [(8, S.TUNED, 0), (16, S.TUNED, 0), (32, S.TUNED, 0), (64, S.TUNED, 0), (16, S.SUBBOX, 0),
             (32, S.TABLE, 0), (16, S.UNROLL, 0)]
    if kind:
        cases.append((64, S.TUNED, FLAG_DST_FROM_SRC))
    for rho, strat, flags in cases:
        g.copy_(src)
        lx, ly = gpu.backends.local_cell_arrays(strat, rho) if strat == S.TABLE else (None, None)
        gpu.backends.run_block_space(g, src, rho, 16 - rho.bit_length() + 1, strat, lx, ly, kind=kind, param=1,
                                     flags=flags)
        assert gpu.device.count_mismatch(g, want_d) == 0, (rho, strat, kind, flags)
    for early in (False, True):
        g.copy_(src)
        gpu.backends.run_bounding_box(g, src, 32, kind, 1, early_exit=early)
        assert gpu.device.count_mismatch(g, want_d) == 0, ("bb", early)


def test_n16_write_zero_background_exact(gpu, oracle):
    """The opt-in zero-background write pass on make_grid zeros (PAPER.md:442-443,
    engine.py:88-90) == the oracle's write pass, every schedule and store width."""
    n = 1 << 16
    S = gpu.geometry.IntraStrategy
    # mode 1 = hashed gasket cells on a zero background; the write pass sets every gasket cell to 1
    want = oracle.steps_band(n, np.int8, 0, 1, 0, 1, 0, n, [1])[0]
    want_d = torch.from_numpy(want).cuda()
    del want
    g = torch.zeros((n, n), dtype=torch.int8, device="cuda")
    nat = gpu.native
    for flags in (0, nat.FLAG_DIGIT_ORDER, nat.FLAG_ROWMAJOR, nat.FLAG_GRID_ROWS, nat.FLAG_GRID_ROWS | nat.FLAG_WRITE_HALVES,
                  nat.FLAG_GRID_ROWS | nat.FLAG_WRITE_LINES,
                  nat.FLAG_GRID_ROWS | nat.FLAG_WRITE_LINES | nat.FLAG_WRITE_HALVES, nat.FLAG_WRITE_SWEEP):
        g.zero_()
        for _ in range(2):  # the reference bench re-runs plan.run(grid, grid) on its own output
            gpu.backends.run_block_space(g, g, 32, 11, S.TUNED, kind=0, param=1, flags=flags,
                                         assume_zero_background=True)
        assert gpu.device.count_mismatch(g, want_d) == 0, flags


def test_n16_int32_nsum4_exact(gpu, oracle):
    """The reference's own dtype (engine.launch accepts int32 only, engine.py:198-199):
    n = 2^16 int32 NEIGHBOR_SUM (16 GiB per grid), tuned (plain and whole-sector
    blend) and SUBBOX, every cell against oracle bands."""
    n = 1 << 16
    S = gpu.geometry.IntraStrategy
    src = gpu.device.fill_hash(n, torch.int32, 21, 0)
    a = src.clone()
    gpu.backends.run_block_space(a, src, 16, 12, S.TUNED, kind=1, param=1)
    bad = band_mismatches(gpu, oracle, {1: a}, n, np.int32, 21, 0, 1, 1, band_rows=8192)
    assert bad == {1: 0}
    b = src.clone()
    for strat, flags in ((S.TUNED, FLAG_DST_FROM_SRC), (S.SUBBOX, 0)):
        b.copy_(src)
        gpu.backends.run_block_space(b, src, 16, 12, strat, kind=1, param=1, flags=flags)
        assert gpu.device.count_mismatch(a, b) == 0, (strat, flags)


@pytest.mark.parametrize("kind", [2, 1])
def test_n17_int8_ca_exact(gpu, oracle, kind):
    """BASELINE config 3: n = 2^17 int8 (16 GiB per grid), NSUM8 (and NSUM4), seed-hashed
    state on every cell.  Every cell of: the tuned single step (default and
    whole-sector blend), the paper-literal SUBBOX step, the fused 2/4/6-step kernels
    (gm_ca_steps) and the CA driver (CARunner, 6 fused steps per launch, CUDA graph)
    after 12 steps -- against the oracle after 1, 2, 4, 6 and 12 steps."""
    from paper_1706_04552_b200 import ca

    n = 1 << 17
    S = gpu.geometry.IntraStrategy
    seed = 9
    src = gpu.device.fill_hash(n, torch.int8, seed, 0)
    results = {}
    runner = ca.CARunner(src.clone(), kind=kind, param=1, temporal=6)
    results[12] = runner.run(12)
    other = runner.bufs[1 - runner.cur]
    del runner
    torch.cuda.synchronize()
    del other
    torch.cuda.empty_cache()
    r1 = src.clone()
    gpu.backends.run_block_space(r1, src, 64, 11, S.TUNED, kind=kind, param=1)
    results[1] = r1
    t = src.clone()
    for rho, strat, flags in ((64, S.TUNED, FLAG_DST_FROM_SRC), (32, S.SUBBOX, 0)):
        t.copy_(src)
        gpu.backends.run_block_space(t, src, rho, 17 - rho.bit_length() + 1, strat, kind=kind, param=1, flags=flags)
        assert gpu.device.count_mismatch(t, r1) == 0, (strat, flags)
    del t
    torch.cuda.empty_cache()
    for steps in (2, 4, 6):
        d = src.clone()
        _ca_steps(gpu, d, src, n, kind, steps)
        results[steps] = d
    # the CA steps with the static left-edge cache (edge.cu) give the same cells
    edge = torch.empty(gpu.native.ca_edge_bytes(n, 1), dtype=torch.uint8, device="cuda")
    gpu.native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, 1, -1, 0, 0, None, 0,
                    gpu.device.stream_handle())
    t = src.clone()
    for steps in (1, 2, 6):
        gpu.native.call("gm_ca_run", t.data_ptr(), src.data_ptr(), n, 1, kind, 1, steps, edge.data_ptr(), 0,
                        gpu.device.stream_handle())
        assert gpu.device.count_mismatch(t, results[steps]) == 0, ("edge cache", steps)
    # the in-place launch (src = grid: engine.launch semantics with a border snapshot only)
    t.copy_(src)
    gpu.backends.run_block_space(t, t, 64, 11, S.TUNED, kind=kind, param=1)
    assert gpu.device.count_mismatch(t, results[1]) == 0, "in-place"
    del t, edge
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    bad = band_mismatches(gpu, oracle, results, n, np.int8, seed, 0, kind, 1, band_rows=4096)
    assert bad == {s: 0 for s in results}, bad


def test_n18_int8_ca_sampled_bands(gpu, oracle):
    """BASELINE config 5 on one GPU: n = 2^18 int8 (64 GiB per grid), NSUM8, the tuned
    single step and the fused 6-step kernel, against the oracle on 24 bands of 1024 rows
    (grid top and bottom, and interior bands straddling tile / sub-gasket rows)."""
    n = 1 << 18
    seed = 5
    S = gpu.geometry.IntraStrategy
    src = gpu.device.fill_hash(n, torch.int8, seed, 0)
    d = src.clone()
    gpu.backends.run_block_space(d, src, 64, 12, S.TUNED, kind=2, param=1)
    bands = sampled_bands(n, 1024, 24)
    assert band_mismatches(gpu, oracle, {1: d}, n, np.int8, seed, 0, 2, 1, bands=bands) == {1: 0}
    d.copy_(src)
    _ca_steps(gpu, d, src, n, 2, 6)
    assert band_mismatches(gpu, oracle, {6: d}, n, np.int8, seed, 0, 2, 1, bands=bands) == {6: 0}


def test_n16_coverage_audit(gpu):
    """The coverage audit (engine.verify_coverage, engine.py:214-258) at BASELINE config 2's
    size: the real kernels count every write into n x n uint32 counters (16 GiB) and the
    comparison runs on the device (gm_coverage_check).  Correct launches are exact; a
    corrupted map (geometry.corrupted_map_fn, the reference's mutation hook) is caught,
    its duplicates and misses row-major like np.argwhere."""
    eng, geo = gpu.engine, gpu.geometry
    S = geo.IntraStrategy
    spec = geo.FractalSpec(n=1 << 16, rho=32)
    for mapping, strat in ((eng.Mapping.BLOCK_SPACE, S.TUNED), (eng.Mapping.BLOCK_SPACE, S.TABLE),
                           (eng.Mapping.BOUNDING_BOX_EXIT, None)):
        rep = eng.verify_coverage(eng.LaunchConfig(spec=spec, mapping=mapping, strategy=strat))
        assert rep.exact and not rep.duplicates and not rep.misses, (mapping, strat)
        del rep
        torch.cuda.empty_cache()
    # one block mapped onto its neighbour's place: that block's cells are missed, the
    # neighbour's written twice -- the audit finds exactly those, row-major
    def one_bad(omega, r_b):
        return geo.map_block((1, 0) if tuple(omega) == (0, 0) else omega, r_b)

    rep = eng.verify_coverage(eng.LaunchConfig(spec=spec, mapping=eng.Mapping.BLOCK_SPACE, strategy=S.SUBBOX), one_bad)
    good, bad = geo.map_block((0, 0), spec.r_b).coord, geo.map_block((1, 0), spec.r_b).coord
    cells = [(x, y) for y in range(32) for x in range(32) if (x & ~y) == 0]  # a block's gasket cells
    want_miss = sorted((good[1] * 32 + y) * spec.n + good[0] * 32 + x for x, y in cells)
    want_dup = sorted((bad[1] * 32 + y) * spec.n + bad[0] * 32 + x for x, y in cells)
    assert [c.y * spec.n + c.x for c in rep.misses] == want_miss
    assert [c.y * spec.n + c.x for c in rep.duplicates] == want_dup
