#!/usr/bin/env python
"""Single-step tuned stencil at n=2^17 int8: NSUM4 vs NSUM8 (mean of K flushed launches),
with the design-probe flags.  python scripts/time_single.py [K]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    flush = device.L2Flusher()
    n = 1 << 17
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = src.clone()
    D = native.FLAG_DST_FROM_SRC
    for kind in (2, 1):
        for name, fl in (("full", D), ("fetch half", D | native.FLAG_FETCH_HALF),
                         ("fetch mixed", D | native.FLAG_FETCH_HALF | native.FLAG_FETCH_MIXED),
                         ("stages2", D | native.FLAG_STAGES2), ("no compute", D | native.FLAG_PROBE_NOCOMPUTE),
                         ("reads only", D | native.FLAG_PROBE_NOSTORE), ("no memory", D | native.FLAG_PROBE_NOLOAD |
                                                                          native.FLAG_PROBE_NOSTORE)):
            fn = lambda: backends.run_block_space(dst, src, 64, 11, IntraStrategy.TUNED, kind=kind,  # noqa: E731
                                                  param=1, flags=fl)
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
            print(f"nsum{4 * kind} {name:12s} mean {statistics.fmean(ts):7.1f} us  min {min(ts):7.1f} us", flush=True)


if __name__ == "__main__":
    main()
