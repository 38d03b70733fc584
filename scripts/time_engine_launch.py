#!/usr/bin/env python
"""engine.launch NEIGHBOR_SUM on a device grid, snapshot included (engine.py:201):
the in-place launch with a border-cell snapshot (what engine.launch runs for the tuned
strategy), the masked snapshot (device.stencil_snapshot) and the full grid copy the
reference takes.
    python scripts/time_engine_launch.py [r] [K]      (default n = 2^16 int32, the reference's dtype)"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, engine  # noqa: E402
from paper_1706_04552_b200.geometry import FractalSpec, IntraStrategy  # noqa: E402


def timed(fn, flush, k):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.fmean(ts)


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 16  # (int32: three grids, so r <= 16 on one B200)
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    n, rho = 1 << r, 32
    flush = device.L2Flusher()
    g = device.fill_hash(n, torch.int32, 3, 0)
    spec = FractalSpec(n=n, rho=rho)
    cfg = engine.LaunchConfig(spec=spec, mapping=engine.Mapping.BLOCK_SPACE, strategy=IntraStrategy.TUNED,
                              kernel=engine.CellKernel(engine.KernelKind.NEIGHBOR_SUM, 1))
    snap_full = torch.empty_like(g)

    def full_copy():  # the reference's semantics, literally: copy the whole grid, then launch
        snap_full.copy_(g)
        backends.run_block_space(g, snap_full, rho, spec.r_b, IntraStrategy.TUNED, kind=1, param=1, flags=2)

    def masked():
        engine.launch(cfg, g)

    def kernel_only():
        backends.run_block_space(g, snap_full, rho, spec.r_b, IntraStrategy.TUNED, kind=1, param=1, flags=2)

    def snapshot_only():
        device.stencil_snapshot(g)

    def snapshot_launch():  # the device work of engine.launch, without its host-side bookkeeping
        s = device.stencil_snapshot(g)
        backends.run_block_space(g, s, rho, spec.r_b, IntraStrategy.TUNED, kind=1, param=1, flags=2)

    def inplace():  # src = grid: the tuned kernel in place with the border-cell snapshot (gm_run_inplace)
        backends.run_block_space(g, g, rho, spec.r_b, IntraStrategy.TUNED, kind=1, param=1)

    for name, fn in (("full grid copy + launch", full_copy), ("engine.launch", masked),
                     ("in place (border snapshot)", inplace),
                     ("masked snapshot + launch", snapshot_launch), ("masked snapshot only", snapshot_only),
                     ("launch only", kernel_only)):
        print(f"n=2^{r} int32 NSUM4  {name:34s} {timed(fn, flush, k):8.3f} ms", flush=True)


if __name__ == "__main__":
    main()
