"""Build libgasket_b200.so in-tree with nvcc for sm_100a (no torch types in the ABI)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
# A/B builds (GASKET_AB_BUILD=1, scripts/ only): the superseded stencil variants (v1,
# TMA-staged) and the design-probe flags are compiled in, into a separate library that
# scripts load with GASKET_B200_LIB; the product library carries neither.
AB_BUILD = os.environ.get("GASKET_AB_BUILD", "") == "1"
LIB = LIB_DIR / ("libgasket_b200_ab.so" if AB_BUILD else "libgasket_b200.so")
SOURCES = ["literal.cu", "tuned.cu", "stream.cu", "write.cu", "stencil2.cu", "stencil_tb.cu", "hostrows.cu",
           "maps.cu", "capi.cu", "peer.cu", "snapshot.cu", "edge.cu"]
AB_SOURCES = ["stencil.cu", "stencil_tma.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return cand


def sources() -> list[Path]:
    return [CSRC / s for s in SOURCES + (AB_SOURCES if AB_BUILD else [])]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list((PKG.parent / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    obj_dir = LIB_DIR / ("obj_ab" if AB_BUILD else "obj")
    obj_dir.mkdir(parents=True, exist_ok=True)
    extra_inc = ["-I", str(PKG.parent / "include")]
    defines: list[str] = ["-DGM_AB_VARIANTS=1"] if AB_BUILD else []

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra_inc, *defines, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    link = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
