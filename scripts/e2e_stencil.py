#!/usr/bin/env python
"""Time the mapped (zero-copy) host path of the stencil per kernel flag set.

    python scripts/e2e_stencil.py [r]
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 17
n = 1 << r
src_t = torch.empty((n, n), dtype=torch.int8, pin_memory=True)
src_t.copy_(device.fill_hash(n, torch.int8, 1, 0).cpu())
g_t = torch.empty_like(src_t, pin_memory=True)
g_t.copy_(src_t)
src, g = src_t.numpy(), g_t.numpy()
os.environ[device.HOST_TRANSPORT_ENV] = "mapped"
base = native.FLAG_HOST_ROWS | native.FLAG_EXPLICIT_RMW | native.FLAG_WHOLE_LINES
for name, fl in (("default", base), ("half", base | native.FLAG_FETCH_HALF), ("stages2", base | native.FLAG_STAGES2),
                 ("half+stages2", base | native.FLAG_FETCH_HALF | native.FLAG_STAGES2)):
    os.environ[device.HOST_FLAGS_ENV] = str(fl)
    backends.run_block_space(g, src, 64, r - 6, IntraStrategy.TUNED, kind=2, param=1)
    t0 = time.perf_counter()
    for _ in range(3):
        backends.run_block_space(g, src, 64, r - 6, IntraStrategy.TUNED, kind=2, param=1)
    dt = (time.perf_counter() - t0) / 3
    print(f"e2e nsum8 r={r} {name:14s} {dt * 1e3:8.2f} ms  {3**r / dt / 1e9:6.2f} Gcells/s", flush=True)
