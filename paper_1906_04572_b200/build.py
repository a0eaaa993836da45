"""Build libcorutv_b200.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_1906_04572_b200.build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libcorutv_b200.so"
SOURCES = [CSRC / "corutv_b200.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "corutv_b200.h"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def command(out: Path = OUT) -> list[str]:
    return [nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
            "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", str(PKG.parent / "include"),
            "-o", str(out), *map(str, SOURCES)]


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS if p.exists())


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and up_to_date():
        return OUT
    cmd = command(OUT.with_suffix(".so.tmp"))
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT.with_suffix(".so.tmp"), OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
