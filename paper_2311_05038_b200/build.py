"""Build libfd.so (the C-ABI library of include/fd.h) for sm_100a with nvcc.

The .so is built IN-TREE (paper_2311_05038_b200/libfd.so) so that it travels
to the GPU box with the repo snapshot.  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libfd.so"
SOURCES = [CSRC / "fd_runtime.cu"] + sorted(CSRC.glob("fd_tab_*.cu"))
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "fd.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I", str(ROOT / "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    """Compile each translation unit to an object in parallel, then link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    tag = f"tmp{os.getpid()}"
    objdir = PKG / "build_obj"
    objdir.mkdir(exist_ok=True)
    # FD_NVCC_EXTRA: extra nvcc flags for A/B experiments (e.g. -DFD_MBAR_SUSPEND_NS=0)
    extra = os.environ.get("FD_NVCC_EXTRA", "").split()
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    if verbose:
        cflags = ["-Xptxas=-v", *cflags]
    objs = [objdir / f"{src.stem}.{tag}.o" for src in SOURCES]

    def compile_one(i: int) -> None:
        subprocess.check_call([nvcc(), *cflags, *extra, "-c", "-o", str(objs[i]), str(SOURCES[i])])

    try:
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            list(ex.map(compile_one, range(len(SOURCES))))
        tmp = LIB.with_suffix(f".so.{tag}")
        subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                               "-o", str(tmp), *map(str, objs), "-ldl"])
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if o.exists():
                o.unlink()
    return LIB


if __name__ == "__main__":
    print(build_lib(force=True, verbose=True))
