"""Builds the sm_100a shared library ``lib/libpfe_b200.so`` in-tree.

nvcc compiles every translation unit with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -fmad=false`` (no multiply-add contraction, so elementwise formulas
round exactly like the reference's x86-64 build).  The cuda
runtime is linked statically, so the library does not depend on torch's
CUDA runtime.  Incremental: a TU is recompiled only when it or a header is
newer than its object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OUT_DIR = PKG / "lib"
OBJ_DIR = PKG / "build" / "obj"
LIB = OUT_DIR / "libpfe_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
CXX_FLAGS = ["-std=c++17", "-O3", "-fPIC", "-Wall", "-Wextra", f"-I{INCLUDE}", f"-I{CSRC}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 PFE library must be compiled with nvcc for sm_100a")


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp"))
    return cu, cpp


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))


_INC = re.compile(r'^\s*#\s*include\s*"([^"]+)"', re.M)


def _deps(src: Path, seen: set | None = None) -> set:
    """Project headers `src` includes, transitively (quoted includes found
    under csrc/ or include/)."""
    seen = set() if seen is None else seen
    for name in _INC.findall(src.read_text(errors="ignore")):
        for base in (src.parent, CSRC, INCLUDE):
            h = (base / name).resolve()
            if h.exists() and h not in seen:
                seen.add(h)
                _deps(h, seen)
                break
    return seen


def _stale(obj: Path, src: Path, hdr_mtime: float) -> bool:
    """A TU is rebuilt when it, or a header it includes, is newer than its object."""
    if not obj.exists():
        return True
    m = obj.stat().st_mtime
    if m < src.stat().st_mtime:
        return True
    return any(m < h.stat().st_mtime for h in _deps(src))


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    nvcc = _nvcc()
    cu, cpp = _sources()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    hdr = max((h.stat().st_mtime for h in _headers()), default=0.0)
    cmds = []
    objs = []
    for src in cu:
        obj = OBJ_DIR / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src, hdr):
            cmds.append([nvcc, *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    for src in cpp:
        obj = OBJ_DIR / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src, hdr):
            cmds.append(["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    jobs = jobs or max(1, min(len(cmds), os.cpu_count() or 4))
    if cmds:
        with cf.ThreadPoolExecutor(jobs) as ex:
            list(ex.map(run, cmds))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        run([nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl"])
    return LIB


BINDING = PKG / "binding"
REF_INCLUDE = Path("/root/reference/proj/core/include")
EIGEN_STUB = PKG.parent / "tests" / "cpp" / "eigen_stub"
REF_TEST = BINDING / "build" / "test_ref_binding"


def build_ref_binding(verbose: bool = False) -> Path | None:
    """Compiles the link-level backend (binding/pfe_core_b200.cpp) against the
    reference's own headers into the test program tests/cpp/test_ref_binding.cpp
    (with the test-only Eigen stub; Eigen3 is absent here).  Needs
    /root/reference, so it runs in the build container only; the binary
    travels with the repo snapshot to the GPU box like the library does."""
    if not REF_INCLUDE.exists():
        return None
    src = [PKG.parent / "tests" / "cpp" / "test_ref_binding.cpp", BINDING / "pfe_core_b200.cpp"]
    deps = src + [LIB, INCLUDE / "pfe_b200.h", EIGEN_STUB / "Eigen" / "Dense"]
    if REF_TEST.exists() and REF_TEST.stat().st_mtime >= max(p.stat().st_mtime for p in deps):
        return REF_TEST
    REF_TEST.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{EIGEN_STUB}", f"-I{REF_INCLUDE}", f"-I{INCLUDE}",
           *map(str, src), f"-L{OUT_DIR}", "-lpfe_b200", "-Wl,-rpath,$ORIGIN/../../lib", "-o", str(REF_TEST)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return REF_TEST


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_ref_binding(verbose="-v" in sys.argv))
