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
