"""Reference module name ``gasketmap.blockmap``.

Scalar pieces live in ``geometry``; the array-valued operations
(``map_blocks_array``, ``verify_bijection``) run on the GPU.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch

from . import device, native
from .geometry import (  # noqa: F401
    BijectionReport,
    Coord2,
    MapResult,
    block_region,
    corrupted_map_fn,
    map_block,
    packing_dims,
    reduction_depth,
    region_offset,
    suggested_block_threads,
)

map_blocks_array = device.map_blocks_array  # blockmap.py:91-108 on the device

#: device audits go well beyond the reference's host oracle cap of r_b = 12
MAX_BIJECTION_LEVEL = 16


def verify_bijection(r_b: int, map_fn: Optional[Callable[[tuple[int, int], int], MapResult]] = None) -> BijectionReport:
    """blockmap.py:123-166 on the device: map every omega of the packed rectangle
    and report the first omega (row-major) whose target is off the gasket or
    already taken, plus how many distinct cells were reached before it."""
    if not 0 <= r_b <= MAX_BIJECTION_LEVEL:
        raise ValueError(f"bijection oracle supports levels 0..{MAX_BIJECTION_LEVEL}, got {r_b}")
    device.require_cuda()
    width, height = packing_dims(r_b)
    n_b = 1 << r_b
    if map_fn is None:
        cx, cy = device.map_rectangle(r_b)
    else:
        coords = [map_fn((wx, wy), r_b).coord for wy in range(height) for wx in range(width)]
        cx = torch.tensor([c[0] for c in coords], dtype=torch.int64, device="cuda")
        cy = torch.tensor([c[1] for c in coords], dtype=torch.int64, device="cuda")
    owner = torch.empty(n_b * n_b, dtype=torch.int64, device="cuda")
    result = torch.empty(2, dtype=torch.int64, device="cuda")
    native.call("gm_bijection_check", cx.data_ptr(), cy.data_ptr(), cx.numel(), n_b, owner.data_ptr(),
                result.data_ptr(), device.stream_handle())
    first_bad = int(result[0].item())
    total = width * height
    if first_bad < 0 or first_bad >= total:
        return BijectionReport(True, None, total)
    return BijectionReport(False, Coord2(first_bad % width, first_bad // width), first_bad)


def map_blocks_numpy_compat(wx: np.ndarray, wy: np.ndarray, r_b: int):
    """Alias kept for callers that want numpy in / numpy out explicitly."""
    return device.map_blocks_array(np.asarray(wx), np.asarray(wy), r_b)
