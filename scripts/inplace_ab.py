#!/usr/bin/env python
"""In-place neighbour-sum launch (gm_run_inplace) vs the same step into a separate buffer,
and the border-snapshot kernel alone: n=2^16 int32 NSUM4 and n=2^17 int8 NSUM8, back to
back.  python scripts/inplace_ab.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def b2b(fn, k=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / k


def main():
    s = device.stream_handle()
    for dt, r, kind in ((torch.int32, 16, 1), (torch.int8, 17, 2)):
        n = 1 << r
        c = torch.empty((), dtype=dt).element_size()
        g = device.fill_hash(n, dt, 1, 0)
        other = g.clone()
        border = torch.empty(native.border_bytes(n, c), dtype=torch.uint8, device="cuda")
        rows = {
            "in place (border + stencil)": lambda: native.call("gm_run_inplace", g.data_ptr(), border.data_ptr(), n, c,
                                                               kind, 1, s),
            "separate dst (DST_FROM_SRC)": lambda: backends.run_block_space(other, g, 64, r - 6, IntraStrategy.TUNED,
                                                                            kind=kind, param=1, flags=2),
        }
        for name, fn in rows.items():
            print(f"{str(dt):12s} n=2^{r} nsum{4 * kind}  {name:30s} {b2b(fn):8.1f} us", flush=True)
        del g, other, border
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
