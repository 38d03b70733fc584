#!/usr/bin/env python
"""A/B of the write-pass kernels (write.cu vs the round-1 stream.cu kernel).

    python scripts/write_ab.py [r ...]
Checks every variant against the member mask on small grids, then times each at
n = 2^r (default 16 and 17, int8; 16 int32): L2 flushed before each launch, and
back to back (the touched lines exceed L2, so each launch also pays the previous
one's dirty write-back).
"""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200 import roofline as R  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402

T = IntraStrategy.TUNED
Z = native.FLAG_ZERO_BACKGROUND
VARIANTS = (
    ("lambda", 0),
    ("rowmajor", native.FLAG_ROWMAJOR),
    ("gridrows", native.FLAG_GRID_ROWS),
    ("lambda-zero", Z),
    ("rowmajor-zero", Z | native.FLAG_ROWMAJOR),
    ("gridrows-zero", Z | native.FLAG_GRID_ROWS),
    ("gridrows-zero-halves", Z | native.FLAG_GRID_ROWS | native.FLAG_WRITE_HALVES),
    ("gridrows-zero-lines", Z | native.FLAG_GRID_ROWS | native.FLAG_WRITE_LINES),
    ("gridrows-zero-v8", Z | native.FLAG_GRID_ROWS | native.FLAG_WRITE_LINES | native.FLAG_WRITE_HALVES),
    ("lambda-static", native.FLAG_STATIC_SCHEDULE),
    ("gridrows-zero-static", Z | native.FLAG_GRID_ROWS | native.FLAG_STATIC_SCHEDULE),
    ("lambda-zero-static", Z | native.FLAG_DIGIT_ORDER | native.FLAG_STATIC_SCHEDULE),
    ("lambda-zero-dyn", Z | native.FLAG_DIGIT_ORDER),
    ("sweep", native.FLAG_WRITE_SWEEP),
    ("sweep-zero", Z | native.FLAG_WRITE_SWEEP),
    ("hostrows-zero", Z | native.FLAG_HOST_ROWS | native.FLAG_EXPLICIT_RMW | native.FLAG_WHOLE_LINES),
)
if len(sys.argv) > 1 and sys.argv[1].startswith("only="):
    keep = sys.argv.pop(1)[5:].split(",")
    VARIANTS = tuple(v for v in VARIANTS if v[0] in keep)


def member(n, dt):
    y = torch.arange(n, device="cuda", dtype=torch.int64).view(n, 1)
    x = torch.arange(n, device="cuda", dtype=torch.int64).view(1, n)
    return (x & (n - 1 - y)) == 0


def check():
    bad = 0
    for r in (5, 7, 8, 10, 12):
        n = 1 << r
        for dt in (torch.int8, torch.int16, torch.int32, torch.int64):
            m = member(n, dt)
            for name, fl in VARIANTS:
                if "probe" in name:
                    continue
                for bg in (0, 5):
                    if bg and "zero" in name:
                        continue
                    g = torch.full((n, n), bg, dtype=dt, device="cuda")
                    backends.run_block_space(g, g, 1, r, T, kind=0, param=-3, flags=fl)
                    want = torch.where(m, torch.tensor(-3, dtype=dt, device="cuda"),
                                       torch.tensor(bg, dtype=dt, device="cuda"))
                    ok = bool(torch.equal(g, want))
                    if not ok:
                        bad += 1
                        print(f"MISMATCH r={r} {dt} {name} bg={bg}", flush=True)
    print(f"check: {'ok' if bad == 0 else f'{bad} mismatches'}", flush=True)


def main():
    check()
    rs = [int(a) for a in sys.argv[1:]] or [16, 17]
    flush = device.L2Flusher()
    for r in rs:
        n = 1 << r
        for dt, c in ((torch.int8, 1), (torch.int32, 4)):
            if c == 4 and r != 16:
                continue
            g = torch.zeros((n, n), dtype=dt, device="cuda")
            alg = R.write_bytes(r, c)
            for rep in range(2):
                for name, fl in VARIANTS:
                    fn = lambda: backends.run_block_space(g, g, 32, r - 5, T, kind=0, param=1, flags=fl)  # noqa: E731
                    fn()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(20):
                        flush()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        fn()
                        b.record()
                        b.synchronize()
                        ts.append(a.elapsed_time(b))
                    flush()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    K = 50
                    a.record()
                    for _ in range(K):
                        fn()
                    b.record()
                    b.synchronize()
                    bb = a.elapsed_time(b) / K
                    m = statistics.fmean(ts)
                    print(f"write r={r} c={c} {name:22s} flushed {m * 1e3:7.1f} us (min {min(ts) * 1e3:6.1f})  "
                          f"b2b {bb * 1e3:7.1f} us  frac {alg / (m * 1e-3) / 1e9 / 6548.5:5.3f} / "
                          f"{alg / (bb * 1e-3) / 1e9 / 6548.5:5.3f}", flush=True)
            del g
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
