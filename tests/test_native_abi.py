"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/gasket_b200.h declares (no compute calls here)."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols() -> set[str]:
    text = (ROOT / "include" / "gasket_b200.h").read_text()
    return set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(gm_\w+)\s*\(", text, flags=re.M))


def test_header_declares_expected_surface():
    syms = _declared_symbols()
    assert {"gm_run_bounding_box", "gm_run_block_space", "gm_map_blocks", "gm_launch"} <= syms


def test_library_loads_and_exports_header_symbols():
    from paper_1706_04552_b200 import _build, native

    _build.build()
    lib = native.lib()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert set(native.EXPORTED) == _declared_symbols()
    assert native.version().startswith("gasket_b200")
    assert native.launch_count() == 0  # nothing ran in this CPU process


def test_library_is_sm100a_cubin():
    from paper_1706_04552_b200 import _build

    lib = _build.build()
    out = subprocess.run(["cuobjdump", "-lelf", str(lib)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_errors_without_gpu_are_loud():
    """Product entry points refuse to run (no CPU fallback) when there is no GPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    from paper_1706_04552_b200 import backends, native

    g = np.zeros((8, 8), dtype=np.int32)
    with pytest.raises(native.GasketError):
        backends.run_bounding_box(g, g, 2, 0, 1)


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: only tests/, __graft_entry__.smoke() and bench.py's
    CPU legs may use it; the package itself must not import it (no CPU fallback)."""
    import ast

    pkg = ROOT / "paper_1706_04552_b200"
    for path in pkg.rglob("*.py"):
        tree = ast.parse(path.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert all(not a.name.split(".")[0] == "oracle" for a in node.names), path
            elif isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", path


def test_ca_edge_bytes_host_only():
    """The static left-edge cache size (gm_ca_edge_bytes: no CUDA call): 16 bytes per row
    of every member tile of the launch's tile range."""
    from paper_1706_04552_b200 import native

    assert native.ca_edge_bytes(1 << 17, 1) == 3**10 * 128 * 16
    assert native.ca_edge_bytes(128, 1) == 128 * 16
    assert native.ca_edge_bytes(1 << 12, 4) == 3**7 * 32 * 16
    # a partitioned launch: level-2 sub-gaskets [1, 3) of n=2^12 int8 (27 tiles each)
    assert native.ca_edge_bytes(1 << 12, 1, 2, 1, 3) == 2 * 27 * 128 * 16
    with pytest.raises(ValueError):
        native.ca_edge_bytes(64, 1)  # narrower than a tile
    with pytest.raises(ValueError):
        native.ca_edge_bytes(1 << 12, 8)


def test_border_bytes_host_only():
    """The in-place launch's border buffer: 8 cells per tile of the tile grid."""
    from paper_1706_04552_b200 import native

    assert native.border_bytes(1 << 17, 1) == (1 << 10) ** 2 * 8
    assert native.border_bytes(1 << 16, 4) == (1 << 11) ** 2 * 8 * 4
    with pytest.raises(ValueError):
        native.border_bytes(64, 1)
