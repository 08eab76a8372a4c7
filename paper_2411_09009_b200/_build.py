"""Build libcce_b200.so in-tree with nvcc for sm_100a (no torch involvement)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libcce_b200.so"
SOURCES = [CSRC / "cce_kernels.cu"]
HEADERS = sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "cce_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(src.stat().st_mtime <= t for src in SOURCES + HEADERS if src.exists())


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Build libcce_b200.so (or, for A/B experiments, a variant with extra -D defines into `out`,
    selected at run time with CCE_LIB=<file name>)."""
    lib = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{x}" for x in (defines or [])], "-I", str(CSRC),
           "-I", str(PKG.parent / "include"), "-o", str(tmp), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2411_09009_b200._build [--force] [--variant NAME DEFINE=VALUE ...]
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], sys.argv[i + 2:]
        print(build(force=True, verbose=True, defines=defs, out=PKG / f"libcce_b200_{name}.so"))
    else:
        build(force="--force" in sys.argv, verbose=True)
        print(LIB)
