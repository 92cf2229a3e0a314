"""Build libspidgpu.so (the C ABI + sm_100a kernels) in-tree with nvcc.

    python -m paper_2103_01380_b200.build [--force] [-v]

Every .cu under csrc/ is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo; the host-only .cpp
files (archive metadata JSON, via the nlohmann/json single header that ships
in this image's cudnn_frontend wheel) with g++; everything is linked into
paper_2103_01380_b200/lib/libspidgpu.so (static cudart; the TMA encoder is
resolved through cudaGetDriverEntryPoint, so no -lcuda). The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "lib", "obj")
LIB = os.path.join(HERE, "lib", "libspidgpu.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", f"-I{INCLUDE}"]


CXX = os.environ.get("CXX", shutil.which("g++") or "g++")


def _nlohmann_dir() -> str:
    """Directory holding nlohmann/json's single-header json.hpp (3.11.3)."""
    import sysconfig
    cands = [os.environ.get("SPIDGPU_JSON_DIR", "")]
    for key in ("purelib", "platlib"):
        cands.append(os.path.join(sysconfig.get_paths()[key], "include", "cudnn_frontend",
                                  "thirdparty", "nlohmann"))
    for c in cands:
        if c and os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise RuntimeError("nlohmann json.hpp not found (set SPIDGPU_JSON_DIR)")


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def _stale(target, inputs):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(i) > t for i in inputs)


def _compile(src, verbose):
    base, ext = os.path.splitext(os.path.basename(src))
    obj = os.path.join(OBJ, base + (".o" if ext == ".cu" else ".cpp.o"))
    if not _stale(obj, [src] + _deps()):
        return obj, None
    if ext == ".cpp":
        cmd = [CXX, "-O3", "-std=c++17", "-fPIC", f"-I{INCLUDE}", f"-I{_nlohmann_dir()}", "-c", src,
               "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, (r.stdout + r.stderr).strip() or None


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    if force:
        for f in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(f)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log and verbose:
            print(log, file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
