#!/usr/bin/env python
"""Time kernel variants (flags) of the tuned lambda kernels on the GPU.

    python scripts/variants.py [write16] [stencil17] ...
Prints one line per variant: mean event time over K launches, each after an L2 flush.
"""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200 import roofline as R  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def timeit(fn, flush, k=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.fmean(ts), min(ts)


def main():
    which = sys.argv[1:] or ["write16", "stencil17"]
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    if "write16" in which or "write17" in which:
        r = 17 if "write17" in which else 16
        n = 1 << r
        for dt, c in ((torch.int8, 1), (torch.int32, 4)):
            if c == 4 and r == 17:
                continue
            g = torch.zeros((n, n), dtype=dt, device="cuda")
            alg = R.write_bytes(r, c)
            H, E, L = native.FLAG_HOST_ROWS, native.FLAG_EXPLICIT_RMW, native.FLAG_WHOLE_LINES
            for name, fl in (("masked", 0), ("rmw-sectors", E), ("rmw-lines", E | L)):
                m, mn = timeit(lambda: backends.run_block_space(g, g, 32, r - 5, T, kind=0, param=1, flags=fl), flush)
                print(f"write r={r} c={c} {name:10s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                      f"{3**r / (m * 1e-3) / 1e9:7.1f} Gcells/s  alg {alg / (m * 1e-3) / 1e9:6.0f} GB/s", flush=True)
            del g
            torch.cuda.empty_cache()
    if "stencil17" in which or "stencil16" in which:
        r = 17 if "stencil17" in which else 16
        n = 1 << r
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        D, RM, CH = native.FLAG_DST_FROM_SRC, native.FLAG_ROWMAJOR, native.FLAG_CHUNKED
        NT = native.FLAG_NO_TMA
        for name, fl in (("tma", D | native.FLAG_FORCE_TMA), ("cp.async", D | NT), ("masked-tma", 0),
                         ("masked-cp.async", NT)):
            m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=2, param=1, flags=fl), flush, k=10)
            print(f"stencil r={r} nsum8 {name:22s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us", flush=True)
        for kind in (2, 1):
            alg = R.pass_bytes(r, 1, kind)
            for name, fl in (("dst_from_src", native.FLAG_DST_FROM_SRC), ("masked", 0)):
                m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=kind, param=1, flags=fl),
                               flush, k=10)
                print(f"stencil r={r} nsum{4 * kind} {name:12s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                      f"{3**r / (m * 1e-3) / 1e9:7.1f} Gcells/s  alg {alg / (m * 1e-3) / 1e9:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
