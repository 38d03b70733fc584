#!/usr/bin/env python
"""Time kernel variants (flags) of the tuned lambda kernels on the GPU.

    python scripts/variants.py [write16] [stencil17] ...
Prints one line per variant: mean event time over K launches, each after an L2 flush.
"""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200 import roofline as R  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy  # noqa: E402


def timeit(fn, flush, k=20):
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
    return statistics.fmean(ts), min(ts)


def main():
    which = sys.argv[1:] or ["write16", "stencil17"]
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    if "write16" in which or "write17" in which:
        r = 17 if "write17" in which else 16
        n = 1 << r
        for dt, c in ((torch.int8, 1), (torch.int32, 4)):
            if c == 4 and r == 17:
                continue
            g = torch.zeros((n, n), dtype=dt, device="cuda")
            alg = R.write_bytes(r, c)
            H, E, L = native.FLAG_HOST_ROWS, native.FLAG_EXPLICIT_RMW, native.FLAG_WHOLE_LINES
            F64, FL = native.FLAG_FETCH64, native.FLAG_FETCH_LINE
            RMJ = native.FLAG_ROWMAJOR
            DO, CS = native.FLAG_DIGIT_ORDER, native.FLAG_STORE_CS
            BM = native.FLAG_BAND_MAJOR
            PA = native.FLAG_PREFETCH_AHEAD
            for name, fl in (("masked", 0), ("masked+touchline", F64 | FL), ("masked (again)", 0),
                             ("masked+touchline (again)", F64 | FL), ("masked-prefetch", PA), ("masked-bandmajor", BM),
                             ("masked-digit", DO), ("masked-cs", CS), ("masked+touch64", F64),
                             ("rmw-sectors", E), ("rmw-lines", E | L)):
                m, mn = timeit(lambda: backends.run_block_space(g, g, 32, r - 5, T, kind=0, param=1, flags=fl), flush)
                print(f"write r={r} c={c} {name:10s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                      f"{3**r / (m * 1e-3) / 1e9:7.1f} Gcells/s  alg {alg / (m * 1e-3) / 1e9:6.0f} GB/s", flush=True)
            del g
            torch.cuda.empty_cache()
    if "stencil17" in which or "stencil16" in which:
        r = 17 if "stencil17" in which else 16
        n = 1 << r
        src = device.fill_hash(n, torch.int8, 1, 0)
        dst = src.clone()
        D, RM, CH = native.FLAG_DST_FROM_SRC, native.FLAG_ROWMAJOR, native.FLAG_CHUNKED
        NT = native.FLAG_NO_TMA
        FL = native.FLAG_FETCH_LINE
        V1, S2 = native.FLAG_STENCIL_V1, native.FLAG_STAGES2
        PN, PL = native.FLAG_PROBE_NOSTORE, native.FLAG_PROBE_NOLOAD
        DO, CS = native.FLAG_DIGIT_ORDER, native.FLAG_STORE_CS
        FH = native.FLAG_FETCH_HALF
        F256 = native.FLAG_FETCH256
        for name, fl in (("v2", D), ("v2-256", D | F256), ("v2 (again)", D), ("v2-256 (again)", D | F256),
                         ("v2-half", D | FH), ("v2-half (again)", D | FH),
                         ("v2-mixed", D | FH | native.FLAG_FETCH_MIXED), ("v2-cs", D | CS), ("v2-digit", D | DO), ("v2-stages2", D | S2),
                         ("v2-chunked", D | CH), ("probe v2 no compute", D | native.FLAG_PROBE_NOCOMPUTE),
                         ("probe v2 reads only", D | PN), ("probe v2 reads only, line", D | PN | FL),
                         ("probe v2 stores only", D | PL), ("probe v2 no memory", D | PN | PL),
                         ("probe v2 no compute", D | native.FLAG_PROBE_NOCOMPUTE),
                         ("probe v2 no compute, reads only", D | native.FLAG_PROBE_NOCOMPUTE | PN),
                         ("v2-masked", 0), ("v2-masked-line", FL),
                         ("v1-tma", D | native.FLAG_FORCE_TMA), ("v1-cp.async", D | NT | V1),
                         ("v1-masked-tma", V1), ("v1-masked-cp.async", NT | V1)):
            m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=2, param=1, flags=fl), flush, k=10)
            print(f"stencil r={r} nsum8 {name:22s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us", flush=True)
        for kind in (2, 1):
            alg = R.pass_bytes(r, 1, kind)
            for name, fl in (("dst_from_src", native.FLAG_DST_FROM_SRC), ("masked", 0),
                             ("v1-dst_from_src", native.FLAG_DST_FROM_SRC | native.FLAG_STENCIL_V1)):
                m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=kind, param=1, flags=fl),
                               flush, k=10)
                print(f"stencil r={r} nsum{4 * kind} {name:12s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                      f"{3**r / (m * 1e-3) / 1e9:7.1f} Gcells/s  alg {alg / (m * 1e-3) / 1e9:6.0f} GB/s", flush=True)




def offsets(r=17):
    """Stencil v2 time vs the byte offset between the src and dst allocations (DRAM bank mapping)."""
    n = 1 << r
    flush = device.L2Flusher()
    T = IntraStrategy.TUNED
    src = device.fill_hash(n, torch.int8, 1, 0)
    D = native.FLAG_DST_FROM_SRC
    for off in (0, 128, 2048, 4096, 65536 + 2048, (1 << 20) + 4096, (1 << 21) + 8192 + 128):
        big = torch.empty(n * n + off, dtype=torch.int8, device="cuda")
        dst = big[off:off + n * n].view(n, n)
        dst.copy_(src)
        m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=2, param=1, flags=D), flush, k=10)
        print(f"stencil r={r} nsum8 v2 dst offset {off:8d} (src-dst delta {dst.data_ptr() - src.data_ptr():+d}) "
              f"mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us", flush=True)
        del big, dst
        torch.cuda.empty_cache()


def ca_pairs(r=17):
    """Two fused CA steps (gm_ca_step2) vs one single step, NSUM8/NSUM4 int8."""
    n = 1 << r
    flush = device.L2Flusher()
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = src.clone()
    for kind in (2, 1):
        for name, fl in (("fused pair", 0), ("fused pair line", native.FLAG_FETCH_LINE), ("fused pair (again)", 0),
                         ("fused pair line (again)", native.FLAG_FETCH_LINE),
                         ("probe no compute", native.FLAG_PROBE_NOCOMPUTE),
                         ("probe no memory", native.FLAG_PROBE_NOLOAD | native.FLAG_PROBE_NOSTORE),
                         ("probe no store", native.FLAG_PROBE_NOSTORE), ("probe no load", native.FLAG_PROBE_NOLOAD)):
            fn = lambda: native.call("gm_ca_step2", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, fl,  # noqa: E731
                                     device.stream_handle())
            m, mn = timeit(fn, flush, k=10)
            print(f"ca r={r} nsum{4 * kind} {name:20s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                  f"per step {m * 1e3 / 2:8.1f} us", flush=True)
        for name, fl in (("fused quad", 0), ("fused quad (again)", 0),
                         ("quad probe no compute", native.FLAG_PROBE_NOCOMPUTE),
                         ("quad probe no memory", native.FLAG_PROBE_NOLOAD | native.FLAG_PROBE_NOSTORE)):
            fn = lambda: native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, 4, fl,  # noqa: E731
                                     device.stream_handle())
            m, mn = timeit(fn, flush, k=10)
            print(f"ca r={r} nsum{4 * kind} {name:20s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                  f"per step {m * 1e3 / 4:8.1f} us", flush=True)
        T = IntraStrategy.TUNED
        m, mn = timeit(lambda: backends.run_block_space(dst, src, 64, r - 6, T, kind=kind, param=1,
                                                        flags=native.FLAG_DST_FROM_SRC), flush, k=10)
        print(f"ca r={r} nsum{4 * kind} {'single step':20s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us", flush=True)


def ca_pair_ab(r=17, reps=int(__import__("os").environ.get("CAPAIR_REPS", "4"))):
    """Just the fused pair (gm_ca_step2, present in every build) with the SM clock read
    after each timing: for A/B runs of stencil_tb.cu builds."""
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    n = 1 << r
    flush = device.L2Flusher()
    src = device.fill_hash(n, torch.int8, 1, 0)
    dst = src.clone()
    import os

    probes = (("", 0), (" no compute", native.FLAG_PROBE_NOCOMPUTE), (" no memory", native.FLAG_PROBE_NOLOAD |
              native.FLAG_PROBE_NOSTORE)) if os.environ.get("CAPAIR_PROBES") else (("", 0),)
    for _ in range(reps):
        for kind in (2, 1):
            for label, fl in probes:
                if os.environ.get("CAPAIR_STEPS", "2") == "2":
                    fn = lambda: native.call("gm_ca_step2", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1,  # noqa: E731
                                             fl, device.stream_handle())
                else:
                    fn = lambda: native.call("gm_ca_steps", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1,  # noqa: E731
                                             int(os.environ["CAPAIR_STEPS"]), fl, device.stream_handle())
                m, mn = timeit(fn, flush, k=20)
                mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                print(f"ca r={r} nsum{4 * kind} fused pair{label:12s} mean {m * 1e3:8.1f} us  min {mn * 1e3:8.1f} us  "
                      f"sm {mhz} MHz", flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["offsets"]:
        offsets()
    elif sys.argv[1:] == ["ca"]:
        ca_pairs()
    elif sys.argv[1:] == ["capair"]:
        ca_pair_ab()
    else:
        main()
