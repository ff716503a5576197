"""In-tree build of the CUDA library (sm_100a) behind the C-ABI.

    python -m paper_1103_2635_b200._build        # or __graft_entry__.build()

Each csrc/*.cu is compiled to an object with nvcc in parallel, then linked
into paper_1103_2635_b200/librbc_b200.so (static cudart).  Rebuilds only when
a source or header is newer than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# diagnostic variants: RBC_BUILD_TAG=timing RBC_BUILD_DEFINES=-DRBC_S2_TIMING builds
# librbc_b200_timing.so (load it with RBC_B200_LIB=...); the default build is untouched
_TAG = os.environ.get("RBC_BUILD_TAG", "")
OBJ = os.path.join(PKG, "build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, "librbc_b200" + (f"_{_TAG}" if _TAG else "") + ".so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"), "-Xptxas", "-warn-spills",
] + os.environ.get("RBC_BUILD_DEFINES", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _sources() + _headers() + [os.path.abspath(__file__)])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    cc = nvcc()

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        cmd = [cc, *NVCC_FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, _sources()))
    tmp = LIB + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


TORCH_SRC = os.path.join(PKG, "torch_ext", "rbc_torch_ops.cpp")
TORCH_LIB = os.path.join(PKG, "librbc_torch_ops.so")


def build_torch_ops(force: bool = False) -> str:
    """torch.ops.rbc_b200.* (torch_ext/rbc_torch_ops.cpp): registered operators over the C-ABI,
    linked against librbc_b200.so (found next to it via $ORIGIN)."""
    deps = [TORCH_SRC, os.path.join(ROOT, "include", "rbc_b200.h"), os.path.abspath(__file__)]
    if (not force and os.path.exists(TORCH_LIB)
            and all(os.path.getmtime(p) <= os.path.getmtime(TORCH_LIB) for p in deps)):
        return TORCH_LIB
    import torch
    from torch.utils import cpp_extension

    cxx = shutil.which("g++") or "g++"
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", TORCH_SRC, "-o", TORCH_LIB + ".tmp",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_EXTENSION_NAME=rbc_torch_ops",
           "-I", os.path.join(ROOT, "include")]
    for inc in cpp_extension.include_paths(device_type="cuda"):
        cmd += ["-isystem", inc]
    for lib in cpp_extension.library_paths(device_type="cuda"):
        cmd += ["-L", lib, f"-Wl,-rpath,{lib}"]
    cmd += ["-L", PKG, "-lrbc_b200", "-Wl,-rpath,$ORIGIN", "-lc10", "-ltorch", "-ltorch_cpu", "-ltorch_cuda",
            "-lc10_cuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch ops build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(TORCH_LIB + ".tmp", TORCH_LIB)
    return TORCH_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_torch_ops(force="--force" in sys.argv))
