"""In-tree build of the native libraries (no GPU needed; nvcc cross-compiles sm_100a).

* ``paper_2601_17707_b200/libbbc.so``      CUDA path (csrc/bbc_*.cu), sm_100a only
* ``paper_2601_17707_b200/libbbcsynth.so`` host synthetic-graph generator (csrc/synth.c)
* ``oracle/liboracle.so``                  CPU parity oracle (test infrastructure)

Each target is rebuilt only when a source is newer than the output.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

LIBBBC = PKG / "libbbc.so"
LIBSYNTH = PKG / "libbbcsynth.so"
LIBORACLE = ROOT / "oracle" / "liboracle.so"


def _stale(out: Path, srcs: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(s.stat().st_mtime > t for s in srcs)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)


def build_libbbc(force: bool = False) -> Path:
    """Each translation unit compiled in parallel (objects under build/), then one link."""
    srcs = sorted(CSRC.glob("bbc_*.cu"))
    deps = srcs + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "bbc.h"]
    if force or _stale(LIBBBC, deps):
        objdir = ROOT / "build"
        objdir.mkdir(exist_ok=True)
        flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", str(ROOT / "include")]
        flags += os.environ.get("BBC_NVCC_EXTRA", "").split()  # experiments only (e.g. -DBBC_WALK2)
        procs = []
        objs = []
        for src in srcs:
            obj = objdir / (src.stem + ".o")
            objs.append(obj)
            cmd = [NVCC, *flags, "-c", "-o", str(obj), str(src)]
            print("+", " ".join(cmd), file=sys.stderr)
            procs.append((subprocess.Popen(cmd), cmd))
        for p, cmd in procs:
            if p.wait():
                raise subprocess.CalledProcessError(p.returncode, cmd)
        tmp = LIBBBC.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-ldl"])
        os.replace(tmp, LIBBBC)
    return LIBBBC


def build_synth(force: bool = False) -> Path:
    src = CSRC / "synth.c"
    if force or _stale(LIBSYNTH, [src]):
        tmp = LIBSYNTH.with_suffix(".so.tmp")
        _run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", str(tmp), str(src), "-lm"])
        os.replace(tmp, LIBSYNTH)
    return LIBSYNTH


def build_oracle(force: bool = False) -> Path:
    src = ROOT / "oracle" / "bbc_oracle.c"
    if force or _stale(LIBORACLE, [src]):
        tmp = LIBORACLE.with_suffix(".so.tmp")
        _run(["gcc", "-O3", "-march=x86-64-v2", "-shared", "-fPIC", "-o", str(tmp), str(src), "-lpthread"])
        os.replace(tmp, LIBORACLE)
    return LIBORACLE


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_oracle(force)
    build_libbbc(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
