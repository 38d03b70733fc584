#!/usr/bin/env python
"""One in-place neighbour-sum launch (engine.launch semantics, gm_run_inplace) at n=2^r int8,
for ncu captures.  python scripts/inplace_launch.py [r] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 17
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    g = device.fill_hash(1 << r, torch.int8, 1, 0)
    flush = device.L2Flusher()
    for _ in range(reps):
        flush()
        backends.run_block_space(g, g, 64, r - 6, IntraStrategy.TUNED, kind=2, param=1)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
