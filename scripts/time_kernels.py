#!/usr/bin/env python
"""Time the three tuned hot kernels once each (mean of K launches, L2 flushed before each).

    GASKET_TILE_ORDER_LEVEL=L python scripts/time_kernels.py [K]
Used for knob sweeps that are read from the environment at library load (tile order
level); prints one line: write16 / stencil17 NSUM8 / fused CA pair NSUM8 times in us.
"""

import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def timeit(fn, flush, k):
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
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.fmean(ts)


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    out = {}
    g = torch.zeros((1 << 16, 1 << 16), dtype=torch.int8, device="cuda")
    out["write16"] = timeit(lambda: backends.run_block_space(g, g, 32, 11, T, kind=0, param=1), flush, k)
    del g
    torch.cuda.empty_cache()
    n = 1 << 17
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = src.clone()
    D = native.FLAG_DST_FROM_SRC
    out["stencil17"] = timeit(lambda: backends.run_block_space(dst, src, 64, 11, T, kind=2, param=1, flags=D), flush, k)
    out["ca17pair"] = timeit(lambda: native.call("gm_ca_step2", dst.data_ptr(), src.data_ptr(), n, 1, 2, 1, 0,
                                                 device.stream_handle()), flush, k)
    lvl = os.environ.get("GASKET_TILE_ORDER_LEVEL", "0")
    print(f"level {lvl}: " + "  ".join(f"{key} {v:7.1f} us" for key, v in out.items()), flush=True)


if __name__ == "__main__":
    main()
