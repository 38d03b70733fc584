#!/usr/bin/env python
"""Why is a registered pageable grid slower than a cudaHostAlloc'd one over PCIe?
Write pass e2e (mapped transport) on: torch pin_memory; np.zeros registered; a 2 MB-aligned
numpy buffer registered."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402

r = 16
n = 1 << r
os.environ[device.HOST_TRANSPORT_ENV] = "mapped"


def aligned(nbytes, align):
    raw = np.zeros(nbytes + align, dtype=np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off:off + nbytes]


cases = []
cases.append(("torch pinned", lambda: torch.zeros((n, n), dtype=torch.int8, pin_memory=True).numpy()))
cases.append(("np.zeros", lambda: np.zeros((n, n), dtype=np.int8)))
cases.append(("np 2MB-aligned", lambda: aligned(n * n, 2 << 20).view(np.int8).reshape(n, n)))
cases.append(("np 64KB-aligned", lambda: aligned(n * n, 64 << 10).view(np.int8).reshape(n, n)))
for label, make in cases:
    g = make()
    print(label, hex(g.ctypes.data % (2 << 20)), flush=True)
    call = lambda: backends.run_block_space(g, g, 32, r - 5, IntraStrategy.TUNED, kind=0, param=1)  # noqa: E731
    call()
    for rep in range(2):
        t0 = time.perf_counter()
        for _ in range(10):
            call()
        dt = (time.perf_counter() - t0) / 10
        print(f"  {label:18s} {dt * 1e3:7.2f} ms  {3**r / dt:.3e} cells/s", flush=True)
    del g
    device.pinned.clear()
