#!/usr/bin/env python
"""The staged host path of a neighbour-sum launch on a numpy grid (engine.launch semantics:
src is the grid), timed part by part with CUDA events: masked snapshot over PCIe, the
device kernel, the whole-line write-back.  python scripts/staged_parts.py [r] [K]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 17
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    n = 1 << r
    grid = np.zeros((n, n), dtype=np.int8)
    grid[:] = device.fill_hash(n, torch.int8, 1, 0).cpu().numpy()
    backends.run_block_space(grid, grid, 64, r - 6, IntraStrategy.TUNED, kind=2, param=1)  # registers the array
    s = device.stream_handle()
    snap = device.scratch.get(f"host_snap:{s}", n * n, torch.int8).view(n, n)
    dst = device.scratch.get(f"host_dst:{s}", n * n, torch.int8).view(n, n)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    parts = {"snapshot": [], "kernel": [], "writeback": []}
    with device.MappedHost(grid) as gptr:
        for _ in range(k):
            ev[0].record()
            native.call("gm_snapshot_stencil", snap.data_ptr(), gptr, n, 1, s)
            ev[1].record()
            backends.run_block_space(dst, snap, 64, r - 6, IntraStrategy.TUNED, kind=2, param=1,
                                     flags=native.FLAG_DST_FROM_SRC)
            ev[2].record()
            native.call("gm_writeback_tiles", gptr, dst.data_ptr(), snap.data_ptr(), n, 1, s)
            ev[3].record()
            ev[3].synchronize()
            parts["snapshot"].append(ev[0].elapsed_time(ev[1]))
            parts["kernel"].append(ev[1].elapsed_time(ev[2]))
            parts["writeback"].append(ev[2].elapsed_time(ev[3]))
    for name, v in parts.items():
        print(f"n=2^{r} int8 NSUM8 staged {name:10s} {min(v):8.2f} ms (min of {k})", flush=True)


if __name__ == "__main__":
    main()
