#!/usr/bin/env python
"""e2e of the write pass / staged stencil on a pageable numpy grid, with and without the
huge-page hint before registration (GASKET_HOST_HUGEPAGES), vs a torch pinned grid.
    python scripts/e2e_pageable.py [r] [kind]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << r
os.environ[device.HOST_TRANSPORT_ENV] = "mapped"
for p in ("/sys/kernel/mm/transparent_hugepage/enabled", "/sys/kernel/mm/transparent_hugepage/defrag"):
    try:
        print(p, open(p).read().strip())
    except OSError as e:
        print(p, e)
init = device.fill_hash(n, torch.int8, 1, 0).cpu().numpy() if kind else None
for label, hp, pinned in (("pageable, 4K pages", "0", False), ("pageable, huge-page hint", "1", False),
                          ("torch pinned", "1", True)):
    os.environ["GASKET_HOST_HUGEPAGES"] = hp
    if pinned:
        host = torch.zeros((n, n), dtype=torch.int8, pin_memory=True)
        g = host.numpy()
    else:
        g = np.zeros((n, n), dtype=np.int8)
    if init is not None:
        g[...] = init
    call = lambda: backends.run_block_space(g, g, 32, r - 5, IntraStrategy.TUNED, kind=kind, param=1)  # noqa: E731
    t0 = time.perf_counter()
    call()
    first = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(10):
        call()
    dt = (time.perf_counter() - t0) / 10
    try:
        sm = [l for l in open("/proc/self/smaps_rollup") if "AnonHugePages" in l]
    except OSError:
        sm = []
    print(f"r={r} kind={kind} {label:26s} first {first * 1e3:8.1f} ms  steady {dt * 1e3:7.2f} ms  "
          f"{3**r / dt:.3e} cells/s  {sm[0].strip() if sm else ''}", flush=True)
    del g
    device.pinned.clear()
