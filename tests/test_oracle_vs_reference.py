"""The CPU oracle against the LIVE reference (container only; skipped where
/root/reference is absent).  Randomised configurations beyond the committed
golden vectors, on identical inputs, compared cell by cell."""

import numpy as np
import pytest


@pytest.mark.parametrize("seed", range(6))
def test_random_configs_match_reference(reference, oracle, seed):
    from gasketmap import backends, blockmap, intra

    rng = np.random.default_rng(seed)
    be = backends.resolve_backend("numba")
    strat_of = {0: intra.IntraStrategy.UNROLL, 1: intra.IntraStrategy.TABLE, 2: intra.IntraStrategy.SUBBOX}
    for _ in range(6):
        dtype = rng.choice([np.int8, np.uint8, np.int16, np.int32])
        r = int(rng.integers(0, 9))
        n = 1 << r
        rho = 1 << int(rng.integers(0, min(r, 5) + 1))
        kind = int(rng.integers(0, 2))
        param = int(rng.integers(-2**31, 2**31))
        src = oracle.fill_hash(n, dtype, int(rng.integers(0, 2**63)), int(rng.integers(0, 2)))
        r_b = (n // rho).bit_length() - 1
        for tag, strat in strat_of.items():
            lx, ly = backends.local_cell_arrays(strat, rho)
            want = src.copy()
            backends.run_block_space(want, src.copy(), rho, r_b, strat, lx, ly, kind, param, be)
            got = src.copy()
            oracle.run_block_space(got, src.copy(), rho, r_b, tag, lx, ly, kind, param)
            assert np.array_equal(got, want), (dtype, n, rho, kind, param, strat)
        want = src.copy()
        backends.run_bounding_box(want, src.copy(), rho, kind, param, be)
        got = src.copy()
        oracle.run_bounding_box(got, src.copy(), rho, kind, param)
        assert np.array_equal(got, want)
        wx = rng.integers(-50, 3**7, size=257)
        wy = rng.integers(-50, 3**7, size=257)
        for rb in (0, 3, 9, 14):
            assert all(np.array_equal(a, b) for a, b in
                       zip(oracle.map_blocks(wx, wy, rb), blockmap.map_blocks_array(wx, wy, rb)))
