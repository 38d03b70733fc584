#!/usr/bin/env python
"""Time the zero-copy host path (backends.run_block_space on a pinned numpy grid) per kernel flag set."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = 1 << r
host = torch.zeros((n, n), dtype=torch.int8, pin_memory=True)
g = host.numpy()
os.environ[device.HOST_TRANSPORT_ENV] = "mapped"
H, E, L = native.FLAG_HOST_ROWS, native.FLAG_EXPLICIT_RMW, native.FLAG_WHOLE_LINES
for name, fl in (("rows-halves", H | E | L), ("rows-sectors", H | E), ("rows-masked", H), ("tiles-lines", E | L)):
    os.environ[device.HOST_FLAGS_ENV] = str(fl)
    backends.run_block_space(g, g, 32, r - 5, IntraStrategy.TUNED, kind=0, param=1)
    t0 = time.perf_counter()
    for _ in range(5):
        backends.run_block_space(g, g, 32, r - 5, IntraStrategy.TUNED, kind=0, param=1)
    dt = (time.perf_counter() - t0) / 5
    print(f"e2e write r={r} {name:12s} {dt * 1e3:8.2f} ms  {3**r / dt / 1e9:6.2f} Gcells/s", flush=True)
