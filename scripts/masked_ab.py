#!/usr/bin/env python
"""The drop-in neighbour-sum launch with distinct grid and src (off-gasket cells of grid
kept: the blend reads grid's touched sectors), n=2^17 int8: mean of K flushed launches.
python scripts/masked_ab.py [K]   (A/B two builds with GASKET_B200_LIB)"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = 1 << 17
    flush = device.L2Flusher()
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = device.fill_hash(n, torch.int8, 2, 0)
    for kind in (2, 1):
        for name, fl in (("masked", 0), ("masked+half", native.FLAG_FETCH_HALF)):
            fn = lambda: backends.run_block_space(dst, src, 64, 11, IntraStrategy.TUNED, kind=kind, param=1, flags=fl)  # noqa
            fn()
            ts = []
            for _ in range(k):
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            print(f"nsum{4 * kind} {name:12s} mean {statistics.fmean(ts):7.1f} us", flush=True)


if __name__ == "__main__":
    main()
