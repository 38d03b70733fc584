"""The single CA step without the edge cache (the drop-in launch's staging): fetch-size and
ring-depth variants, n=2^17 int8, back to back.  python scripts/dropin_ab.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1706_04552_b200 import device, native
n = 1 << 17
src = device.fill_hash(n, torch.int8, 1, 0); dst = src.clone()
s = device.stream_handle()
FH, FM, S2 = native.FLAG_FETCH_HALF, native.FLAG_FETCH_MIXED, native.FLAG_STAGES2
for kind in (2, 1):
    for name, fl in (("default", 0), ("mixed", FH | FM), ("stages2", S2), ("mixed+stages2", FH | FM | S2), ("half", FH), ("half+stages2", FH | S2)):
        fn = lambda: native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), n, 1, kind, 1, 1, None, fl, s)
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): fn()
        b.record(); b.synchronize()
        print(f"nsum{4*kind} no-edge {name:14s} b2b {a.elapsed_time(b)*1e3/20:7.1f} us", flush=True)
