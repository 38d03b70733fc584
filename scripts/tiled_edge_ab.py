#!/usr/bin/env python
"""One-rank tiled partition CA step (n=2^r int8 NSUM8, level-5 sub-gaskets) with and
without the static left-edge cache, back to back.  python scripts/tiled_edge_ab.py [r] [K]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1706_04552_b200 import partition as P  # noqa: E402


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    plan = P.PartitionPlan(1 << r, 5, 1, eight=True, depth=1)
    for edge in (False, True, False, True):
        ca = P.TiledCA(plan, 0, 2, 1, dtype=torch.int8, seed=1, halo="collective", edge_cache=edge)
        for _ in range(3):
            ca.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            ca.step()
        b.record()
        b.synchronize()
        print(f"n=2^{r} tiled one rank, edge_cache={edge}: {a.elapsed_time(b) / k * 1e3:8.1f} us per step", flush=True)
        del ca
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
