"""Reference module name ``gasketmap.core`` -> implementation in ``geometry``."""
from .geometry import (  # noqa: F401
    MAX_LEVEL,
    ORACLE_MAX_EDGE,
    Coord2,
    FractalSpec,
    OrthotopeDims,
    enumerate_cells,
    hausdorff_exponent,
    is_member,
    member_mask,
    packing_dims,
    scale_level,
    volume,
)
