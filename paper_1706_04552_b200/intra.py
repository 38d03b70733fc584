"""Reference module name ``gasketmap.intra`` -> implementation in ``geometry``."""
from .geometry import (  # noqa: F401
    MAX_TABLE_EDGE,
    PAPER_STRATEGIES,
    IntraStrategy,
    LookupTable,
    build_lookup_table,
    local_cells,
    subbox_thread_map,
    threads_per_block,
    unroll_thread_map,
)
