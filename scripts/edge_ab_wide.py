#!/usr/bin/env python
"""CA step with the static left-edge cache on 2- and 4-byte cells: the default staging ring
(4 deep) vs the 2-deep one (GM_FLAG_STAGES2), and no cache.  python scripts/edge_ab_wide.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import device, native  # noqa: E402


def main():
    flush = device.L2Flusher()
    s = device.stream_handle()
    for dt, r in ((torch.int16, 16), (torch.int32, 16)):
        n = 1 << r
        c = torch.empty((), dtype=dt).element_size()
        src = device.fill_hash(n, dt, 1, 0)
        dst = src.clone()
        edge = torch.empty(native.ca_edge_bytes(n, c), dtype=torch.uint8, device="cuda")
        native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, c, -1, 0, 0, None, 0, s)
        for kind in (1, 2):
            for name, e, fl in (("grid", None, 0), ("edge ring4", edge.data_ptr(), 0),
                                ("edge ring2", edge.data_ptr(), native.FLAG_STAGES2), ("grid ring2", None, native.FLAG_STAGES2)):
                fn = lambda: native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), n, c, kind, 1, 1, e, fl, s)  # noqa
                fn()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    fn()
                b.record()
                b.synchronize()
                print(f"{str(dt):12s} n=2^{r} nsum{4 * kind} {name:11s}: b2b {a.elapsed_time(b) * 1e3 / 20:7.1f} us", flush=True)
        del src, dst, edge
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
