#!/usr/bin/env python
"""The CPU reference arm's stand-in (oracle/gasket_oracle.c, OpenMP) against the live
reference (gasketmap's numba backend) on the same host, same workload, same threads:
the lambda TABLE rho=16 pass over an n=2^16 int8 grid, write and 4-neighbour sum.
Container only (needs /root/reference).  python scripts/port_vs_reference.py [reps]"""
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_port")
sys.path.append("/root/reference/pkg/src")

import numpy as np  # noqa: E402

import oracle  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.fmean(ts), min(ts)


def main():
    from gasketmap import backends as ref
    from gasketmap import intra

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    threads = len(os.sched_getaffinity(0))
    ref.set_workers(threads)
    import numba

    r, rho = 16, 16
    n = 1 << r
    r_b = r - 4
    lx, ly = oracle.local_cells(oracle.STRAT_TABLE, rho)
    rlx, rly = ref.local_cell_arrays(intra.IntraStrategy.TABLE, rho)  # the reference's own table
    print(f"host threads {threads}, numba {numba.__version__} threading layer ", end="")
    for kind, name in ((0, "write"), (1, "nsum4")):
        g = np.zeros((n, n), dtype=np.int8)
        src = oracle.fill_hash(n, np.int8, 1, 0, threads=threads) if kind else g
        m_ref, b_ref = timed(lambda: ref.run_block_space(g, src, rho, r_b, intra.IntraStrategy.TABLE, rlx, rly, kind, 1, "numba"), reps)
        if kind == 0:
            print(numba.threading_layer(), flush=True)
        m_port, b_port = timed(lambda: oracle.run_block_space(g, src, rho, r_b, oracle.STRAT_TABLE, lx, ly, kind, 1,
                                                              threads=threads), reps)
        print(f"n=2^{r} int8 {name:5s} TABLE rho={rho}: live reference (numba) {m_ref * 1e3:8.2f} ms "
              f"(best {b_ref * 1e3:.2f}), C port {m_port * 1e3:8.2f} ms (best {b_port * 1e3:.2f}); "
              f"{3**r / m_ref / 1e9:.2f} vs {3**r / m_port / 1e9:.2f} Gcells/s", flush=True)


if __name__ == "__main__":
    main()
