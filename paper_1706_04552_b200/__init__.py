"""paper_1706_04552_b200 -- B200-native block-space map lambda(omega) and the
embedded Sierpinski-gasket kernels it drives (Navarro et al., arXiv:1706.04552).

Drop-in for the reference ``gasketmap`` hot path: the same module names
(core, blockmap, intra, backends, engine, bench) and launch API, with every
kernel running as hand-written sm_100a CUDA behind the C ABI in
include/gasket_b200.h (libgasket_b200.so, loaded through ``native``).
"""
from . import geometry, native  # noqa: F401
from .geometry import FractalSpec, IntraStrategy  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):  # lazy: torch-dependent modules load on first use
    import importlib

    if name in ("backends", "blockmap", "bench", "ca", "core", "device", "engine", "intra", "partition", "roofline"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
