#!/usr/bin/env python
"""One tuned launch of a workload with given flags (for ncu captures).

    python scripts/one_launch.py stencil17 FLAGS [reps]
    python scripts/one_launch.py write16 FLAGS [reps]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def main():
    wl, flags = sys.argv[1], int(sys.argv[2], 0)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    r = int(wl.replace("x4", "")[-2:])
    n = 1 << r
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    if wl.startswith("ca"):
        from paper_1706_04552_b200 import native
        kind = 1 if "nsum4" in wl else 2
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        steps = 4 if wl.endswith("x4") else 2  # ca17 / ca17x4: 2 or 4 fused steps (gm_ca_steps)
        fn = lambda: native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, steps,  # noqa: E731
                                 flags, device.stream_handle())
    elif wl.startswith("stencil"):
        kind = 1 if "nsum4" in wl else 2
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        fn = lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=kind, param=1, flags=flags)  # noqa: E731
    else:
        g = torch.zeros((n, n), dtype=torch.int8, device="cuda")
        fn = lambda: backends.run_block_space(g, g, 32, r - 5, T, kind=0, param=1, flags=flags)  # noqa: E731
    for _ in range(reps):
        flush()
        fn()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
