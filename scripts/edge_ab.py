#!/usr/bin/env python
"""CA steps with and without the static left-edge cache (edge.cu), n=2^17 int8, and
staging-fetch variants of the single step: mean event time of K flushed launches and back
to back, and an exact compare against the default single step.
python scripts/edge_ab.py [r] [K]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import device, native  # noqa: E402


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
        ts.append(a.elapsed_time(b) * 1e3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    b.synchronize()
    return statistics.fmean(ts), min(ts), a.elapsed_time(b) * 1e3 / k


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 17
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    which = sys.argv[3] if len(sys.argv) > 3 else "all"
    n = 1 << r
    flush = device.L2Flusher()
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = src.clone()
    ref = src.clone()
    edge = torch.empty(native.ca_edge_bytes(n, 1), dtype=torch.uint8, device="cuda")
    s = device.stream_handle()
    native.call("gm_ca_edge_build", edge.data_ptr(), src.data_ptr(), n, 1, -1, 0, 0, None, 0, s)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    FH, FM, F256, S2 = native.FLAG_FETCH_HALF, native.FLAG_FETCH_MIXED, native.FLAG_FETCH256, native.FLAG_STAGES2
    E = edge.data_ptr()
    variants = [("grid", None, 0), ("edge", E, 0), ("grid+stages2", None, S2), ("edge+stages2", E, S2),
                ("edge+stages2+256", E, S2 | F256), ("edge+stages2+mixed", E, S2 | FH | FM),
                ("edge (again)", E, 0), ("edge+stages2 (again)", E, S2)]
    for kind in (2, 1):
        for steps in ((1,) if which == "single" else (1, 2, 6)):
            for name, e, fl in (variants if steps == 1 else variants[:2]):
                fn = lambda: native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, steps, e, fl, s)  # noqa
                m, mn, b2b = timed(fn, flush, k)
                if name == "grid":
                    ref.copy_(dst)
                    extra = ""
                else:
                    native.call("gm_count_equal", dst.data_ptr(), ref.data_ptr(), n * n, 1, cnt.data_ptr(), s)
                    extra = f"  differing words vs grid: {int(cnt.item())}"
                print(f"nsum{4 * kind} steps={steps} {name:20s}: flushed mean {m:8.1f} us min {mn:8.1f} us, "
                      f"b2b {b2b:8.1f} us, per step {b2b / steps:7.1f} us{extra}", flush=True)


if __name__ == "__main__":
    main()
