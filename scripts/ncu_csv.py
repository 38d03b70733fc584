#!/usr/bin/env python
"""Summarise an `ncu --csv --metrics ...` log: one line per launch (or per kernel with --mean)."""

import collections
import csv
import io
import sys


def load(path: str):
    text = "".join(ln for ln in open(path) if not ln.startswith("==") and ln.strip())
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[iid]), r[ik].split("(")[0].replace("void ", ""))
        try:
            launches.setdefault(key, {})[r[im]] = float(r[iv].replace(",", ""))
        except ValueError:
            launches.setdefault(key, {})[r[im]] = r[iv]
    return launches


def main() -> None:
    path = sys.argv[1]
    skip = sys.argv[2] if len(sys.argv) > 2 else "k_flush|l2_flush"
    import re

    for (i, k), m in load(path).items():
        if re.search(skip, k):
            continue
        short = {name.replace("__", ".").split(".")[0] + "." + name.split("__")[1][:28]: v for name, v in m.items()}
        t = m.get("gpu__time_duration.sum")
        rd = m.get("dram__bytes_read.sum", 0)
        wr = m.get("dram__bytes_write.sum", 0)
        extra = ""
        if t:
            extra = f"  dram {(rd + wr) / t:.0f} GB/s"
        print(f"{i:4d} {k[:60]:60s} t={t and t / 1e3:.1f}us rd={rd / 1e6:.1f}MB wr={wr / 1e6:.1f}MB{extra}")
        others = {n: v for n, v in m.items() if n not in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")}
        if others:
            print("      " + "  ".join(f"{n.split('__', 1)[1]}={v:.4g}" if isinstance(v, float) else f"{n}={v}" for n, v in others.items()))


if __name__ == "__main__":
    main()
