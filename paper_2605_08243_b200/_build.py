"""Build libsimba.so in-tree with nvcc for sm_100a (no JIT cache)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = [PKG / "csrc" / "simba.cu"]
DEPS = SRC + [PKG / "csrc" / "simba_device.cuh", PKG / "csrc" / "vfb_impl.cuh", ROOT / "include" / "simba.h"]
OUT = PKG / "_lib" / "libsimba.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, out: Path = OUT, defines=()) -> Path:
    if not force and out.exists() and all(out.stat().st_mtime >= p.stat().st_mtime for p in DEPS):
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-Xcompiler", "-fPIC", *ARCH, "-O3", "-lineinfo", "-std=c++17",
           "-I", str(ROOT / "include"), *[f"-D{d}" for d in defines], "-o", str(tmp), *map(str, SRC)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    tmp.replace(out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
