#!/usr/bin/env python
"""One tuned launch of a workload with given flags (for ncu captures).

    python scripts/one_launch.py stencil17 FLAGS [reps]
    python scripts/one_launch.py write16 FLAGS [reps]
    python scripts/one_launch.py castep17 FLAGS [reps]   (gm_ca_run, one step, edge cache)
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
    r = int(wl.replace("x4", "").replace("x6", "")[-2:])
    n = 1 << r
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    if wl.startswith("castep"):
        # castep17: one CA step through gm_ca_run with the static left-edge cache (edge.cu)
        from paper_1706_04552_b200 import native
        kind = 1 if "nsum4" in wl else 2
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        edge = torch.empty(native.ca_edge_bytes(n, 1), dtype=torch.uint8, device="cuda")
        native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, 1, -1, 0, 0, None, 0,
                    device.stream_handle())
        fn = lambda: native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, 1,  # noqa: E731
                                 edge.data_ptr(), flags, device.stream_handle())
    elif wl.startswith("ca"):
        from paper_1706_04552_b200 import native
        kind = 1 if "nsum4" in wl else 2
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        steps = 6 if wl.endswith("x6") else 4 if wl.endswith("x4") else 2  # ca17 / ca17x4 / ca17x6 (gm_ca_steps)
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
