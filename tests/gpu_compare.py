"""Exact device-vs-oracle grid comparison in row chunks (test helper).

The oracle result lives in host memory (numpy); the device result is a CUDA
tensor of the same shape.  Rows are uploaded in chunks and compared cell by cell
on the device (gm_count_equal through device.count_mismatch) -- no checksum, so
nothing can cancel.  Returns the number of differing cells.
"""

from __future__ import annotations

import numpy as np
import torch


def mismatches(gpu, got: torch.Tensor, want: np.ndarray, chunk_bytes: int = 1 << 30) -> int:
    n = want.shape[0]
    assert tuple(got.shape) == tuple(want.shape)
    rows = max(1, min(n, chunk_bytes // max(1, want.strides[0])))
    buf = None
    bad = 0
    for y in range(0, n, rows):
        k = min(rows, n - y)
        host = torch.from_numpy(np.ascontiguousarray(want[y:y + k]))
        if buf is None or buf.shape[0] < k:
            buf = torch.empty((rows, want.shape[1]), dtype=got.dtype, device=got.device)
        buf[:k].copy_(host)
        bad += gpu.device.count_mismatch(got[y:y + k], buf[:k])
    return bad


def first_mismatch(got: torch.Tensor, want: np.ndarray, rows: int = 4096):
    """(y, x, got, want) of the first differing cell, for assertion messages."""
    n = want.shape[0]
    for y in range(0, n, rows):
        g = got[y:y + rows].cpu().numpy()
        d = np.argwhere(g != want[y:y + rows])
        if d.size:
            yy, xx = d[0]
            return int(y + yy), int(xx), g[yy, xx].item(), want[y + yy, xx].item()
    return None


def band_mismatches(gpu, oracle, results: dict, n: int, dtype, seed: int, mode: int, kind: int, param: int,
                    band_rows: int = 4096, bands=None) -> dict:
    """Exact compare of device grids after s steps (``results[s]``) with the oracle's
    row-band restatement (oracle.steps_band) of the same synthetic input
    (fill_hash(seed, mode)), band by band, so no host array larger than a band is
    needed.  ``bands`` = iterable of (y0, y1) (default: every row).  Returns
    {steps: differing 32-bit words}."""
    steps = sorted(results)
    if bands is None:
        bands = [(y, min(n, y + band_rows)) for y in range(0, n, band_rows)]
    bad = {s: 0 for s in steps}
    buf = None
    for y0, y1 in bands:
        outs = oracle.steps_band(n, dtype, seed, mode, kind, param, y0, y1, steps)
        for s, want in zip(steps, outs):
            got = results[s]
            if buf is None or buf.numel() < want.size:
                buf = torch.empty(want.size, dtype=got.dtype, device=got.device)
            b = buf[:want.size].view(y1 - y0, n)
            b.copy_(torch.from_numpy(want))
            bad[s] += gpu.device.count_mismatch(got[y0:y1], b)
    return bad


def sampled_bands(n: int, rows: int, count: int) -> list:
    """`count` bands of `rows` rows: the top and bottom of the grid and evenly spaced
    interior bands offset so they straddle tile and sub-gasket boundaries."""
    out = {(0, rows), (n - rows, n)}
    for i in range(1, count - 1):
        y = (i * n) // (count - 1) - rows // 2 + 1
        y = max(0, min(n - rows, y))
        out.add((y, y + rows))
    return sorted(out)
