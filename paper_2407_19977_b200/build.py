"""Build the native library in-tree: paper_2407_19977_b200/_build/libluxb200.so.

nvcc cross-compiles the CUDA kernels for sm_100a only (no multi-arch, no
PTX fallback); the host BVH builder is plain C++ compiled with
-ffp-contract=off so its float64 arithmetic rounds like the reference.
Run `python -m paper_2407_19977_b200.build` or call build().
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = OUT / "libluxb200.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
             f"-I{INCLUDE}", f"-I{CSRC}"]

CU_SOURCES = ["lt_kernels.cu", "lt_api.cu", "lt_bvh_gpu.cu", "lt_query64.cu", "lt_ingest.cu"]
# per-source extra nvcc flags: the BVH build must round every float64 operation
# like the reference (no FMA contraction)
# (and the float64 query kernels and the glTF flatten reproduce the
# reference's roundings)
CU_EXTRA = {"lt_bvh_gpu.cu": ["-fmad=false"], "lt_query64.cu": ["-fmad=false"],
            "lt_ingest.cu": ["-fmad=false"]}
CPP_SOURCES = ["lt_bvh_build.cpp"]
HEADERS = ["lt_device.cuh", "lt_material.cuh", "lt_traverse.cuh", "lt_kernels.h",
           "lt_internal.h", "lt_staged.h"]


def _run(cmd: list[str], log) -> None:
    print(" ".join(cmd), file=log)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.stdout:
        print(res.stdout, file=log)
    if res.stderr:
        print(res.stderr, file=log)
    if res.returncode != 0:
        raise RuntimeError(f"build step failed ({res.returncode}): {' '.join(cmd)}\n{res.stderr}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Build the library; `variant` builds an experimental copy with extra
    -D `defines` into _build/variant_<name>/ (select it with LUXB200_LIB)."""
    out = OUT if variant is None else OUT / f"variant_{variant}"
    lib = out / "libluxb200.so"
    out.mkdir(parents=True, exist_ok=True)
    headers = [CSRC / h for h in HEADERS] + [INCLUDE / "luxb200.h", Path(__file__)]
    log_path = out / "build.log"
    dflags = [f"-D{d}" for d in defines]
    objs = []
    with open(log_path, "a") as log:
        for src in CU_SOURCES:
            obj = out / (Path(src).stem + ".o")
            objs.append(obj)
            if force or _stale(obj, [CSRC / src] + headers):
                _run([NVCC, *ARCH, *NVCC_FLAGS, *CU_EXTRA.get(src, []), *dflags, "-c", str(CSRC / src),
                      "-o", str(obj)],
                     log)
        for src in CPP_SOURCES:
            obj = out / (Path(src).stem + ".o")
            objs.append(obj)
            if force or _stale(obj, [CSRC / src] + headers):
                _run([CXX, *CXX_FLAGS, "-c", str(CSRC / src), "-o", str(obj)], log)
        if force or _stale(lib, objs):
            _run([NVCC, *ARCH, "-shared", "-o", str(lib), *map(str, objs)], log)
    if verbose:
        print(log_path.read_text()[-4000:])
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
