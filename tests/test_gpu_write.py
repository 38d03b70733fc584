"""The tuned write pass (csrc/write.cu) vs the CPU oracle, bit for bit.

Reference semantics: _block_space_nb with KERNEL_CONST (backends.py:158-222,
_cell_value backends.py:127-141) -- every gasket cell gets `param`, nothing else
changes (backends.py:155-156).  Four schedules (lambda digit order = default, address sweep,
row-major tiles, grid rows) x two store modes (general; opt-in zero background,
valid on the paper's zero-filled matrix).
"""

import numpy as np
import pytest
import torch

from tests.gpu_compare import first_mismatch, mismatches

pytestmark = pytest.mark.gpu

DTYPES = (np.int8, np.int16, np.int32, np.int64)
# schedules: the default (lambda tiles; zero background: grid rows), lambda digit-order tiles, row-major tiles (GM_FLAG_ROWMAJOR), grid rows (GM_FLAG_GRID_ROWS),
# address-ordered sweep of the member lines (GM_FLAG_WRITE_SWEEP)
SCHEDULES = {"default": 0, "lambda": 65536, "rowmajor": 32, "gridrows": 536870912, "sweep": 1073741824}


def _want(oracle, grid0, param):
    """The oracle's write pass (bounding box for small grids, lambda TABLE rho=16 above)."""
    g = grid0.copy()
    n = g.shape[0]
    if n < 256:
        oracle.run_bounding_box(g, g, 1, 0, param)
    else:
        lx, ly = oracle.local_cells(oracle.STRAT_TABLE, 16)
        oracle.run_block_space(g, g, 16, n.bit_length() - 5, oracle.STRAT_TABLE, lx, ly, 0, param)
    return g


def test_write_general_every_schedule_vs_oracle(gpu, oracle):
    """Arbitrary background (splitmix hash): only gasket cells change, every schedule."""
    S = gpu.geometry.IntraStrategy
    for dtype in DTYPES:
        for n in (1, 2, 8, 16, 32, 64, 128, 256, 1024, 4096):
            grid0 = oracle.fill_hash(n, dtype, 31, 0)
            for param in (1, -3, 2**31 - 1):
                want = _want(oracle, grid0, param)
                for name, fl in SCHEDULES.items():
                    for rho in (1, 32):
                        if rho > n:
                            continue
                        g = torch.from_numpy(grid0.copy()).cuda()
                        gpu.backends.run_block_space(g, g, rho, (n // rho).bit_length() - 1, S.TUNED, kind=0,
                                                     param=param, flags=fl)
                        got = g.cpu().numpy()
                        assert np.array_equal(got, want), (np.dtype(dtype).name, n, param, name, rho)


def test_write_zero_background_vs_oracle(gpu, oracle):
    """assume_zero_background on make_grid zeros == the reference result, every schedule and
    cell width; re-running it on its own output (the reference bench's repeated
    plan.run(grid, grid), bench.py:145-150) is idempotent."""
    S = gpu.geometry.IntraStrategy
    for dtype in DTYPES:
        for n in (16, 32, 64, 128, 256, 1024, 4096):
            zeros = np.zeros((n, n), dtype=dtype)
            for param in (1, -7):
                want = _want(oracle, zeros, param)
                for name, fl in SCHEDULES.items():
                    g = torch.zeros((n, n), dtype=getattr(torch, np.dtype(dtype).name), device="cuda")
                    for _ in range(2):
                        gpu.backends.run_block_space(g, g, 1, n.bit_length() - 1, S.TUNED, kind=0, param=param,
                                                     flags=fl, assume_zero_background=True)
                        assert np.array_equal(g.cpu().numpy(), want), (np.dtype(dtype).name, n, param, name)


def test_zero_background_is_opt_in(gpu, oracle):
    """Off by default: a nonzero background survives the default write pass, and the
    opt-in mode is refused for neighbour sums and non-tuned strategies."""
    S = gpu.geometry.IntraStrategy
    n = 1024
    grid0 = oracle.fill_hash(n, np.int8, 5, 0)
    g = torch.from_numpy(grid0.copy()).cuda()
    gpu.backends.run_block_space(g, g, 32, 5, S.TUNED, kind=0, param=1)
    assert np.array_equal(g.cpu().numpy(), _want(oracle, grid0, 1))
    with pytest.raises(ValueError):
        gpu.backends.run_block_space(g, g, 32, 5, S.TUNED, kind=1, param=1, assume_zero_background=True)
    with pytest.raises(ValueError):
        gpu.backends.run_block_space(g, g, 32, 5, S.SUBBOX, kind=0, param=1, assume_zero_background=True)
    # what the assertion buys: on a nonzero background the off-gasket cells of touched
    # sectors are zeroed, nothing else differs (so the flag must never be implied)
    g = torch.from_numpy(grid0.copy()).cuda()
    gpu.backends.run_block_space(g, g, 32, 5, S.TUNED, kind=0, param=1, assume_zero_background=True)
    got = g.cpu().numpy()
    want = _want(oracle, grid0, 1)
    diff = got != want
    assert diff.any() and not got[diff].any()


@pytest.mark.parametrize("mode", ["general", "zero"])
def test_write_n16_int8_exact(gpu, oracle, mode):
    """BASELINE config 2 size (n = 2^16 int8, 4 GiB): every cell vs the oracle, in chunks."""
    n = 1 << 16
    S = gpu.geometry.IntraStrategy
    if mode == "zero":
        grid0 = np.zeros((n, n), dtype=np.int8)
    else:
        grid0 = oracle.fill_hash(n, np.int8, 12, 0)
    want = _want(oracle, grid0, 1)
    del grid0
    for name, fl in SCHEDULES.items():
        g = torch.zeros((n, n), dtype=torch.int8, device="cuda") if mode == "zero" else \
            gpu.device.fill_hash(n, torch.int8, 12, 0)
        gpu.backends.run_block_space(g, g, 32, 11, S.TUNED, kind=0, param=1, flags=fl,
                                     assume_zero_background=mode == "zero")
        bad = mismatches(gpu, g, want)
        assert bad == 0, (mode, name, bad, first_mismatch(g, want))
        del g
        torch.cuda.empty_cache()


def test_write_n17_int8_zero_exact(gpu, oracle):
    """n = 2^17 int8 (16 GiB): the zero-background pass, every cell vs the oracle."""
    n = 1 << 17
    S = gpu.geometry.IntraStrategy
    want = _want(oracle, np.zeros((n, n), dtype=np.int8), 1)
    g = torch.zeros((n, n), dtype=torch.int8, device="cuda")
    gpu.backends.run_block_space(g, g, 32, 12, S.TUNED, kind=0, param=1, assume_zero_background=True)
    assert mismatches(gpu, g, want) == 0
    # the general pass over the same grid leaves it unchanged
    gpu.backends.run_block_space(g, g, 32, 12, S.TUNED, kind=0, param=1)
    assert mismatches(gpu, g, want) == 0


def test_write_partitioned_ranges_cover_once(gpu, oracle):
    """Partitioned write launches (gm_run_part, level-L sub-gasket ranges in lambda digit
    order) over any split of the sub-gaskets == one whole-gasket pass."""
    n = 1 << 12
    for dtype, c in ((np.int8, 1), (np.int32, 4)):
        grid0 = oracle.fill_hash(n, dtype, 3, 0)
        want = _want(oracle, grid0, 9)
        for level, cuts in ((2, (0, 4, 9)), (3, (0, 1, 13, 27)), (5, (0, 100, 243))):
            g = torch.from_numpy(grid0.copy()).cuda()
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                gpu.native.call("gm_run_part", g.data_ptr(), g.data_ptr(), n, c, 0, 9, 0, level, lo, hi,
                                gpu.device.stream_handle())
            assert np.array_equal(g.cpu().numpy(), want), (np.dtype(dtype).name, level, cuts)
