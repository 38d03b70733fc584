#!/usr/bin/env python
"""ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv) -> one line per launch: time, DRAM bytes, DRAM rate.  python scripts/launch_list.py X.csv"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit")
    d = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
                 "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
        d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = v * scale
    for (i, k), m in d.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        name = k.split("(")[0].replace("void ", "")[:60]
        print(f"{i:4d} {name:60s} t={t:.1f}us rd={rd:.1f}MB wr={wr:.1f}MB  dram {(rd + wr) / max(t, 1e-9) * 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
