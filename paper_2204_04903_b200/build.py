"""Build libpicasso.so (sm_100a) in-tree with nvcc.  Sources: csrc/*.cu, csrc/*.cpp."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpicasso.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]



def _nccl_dir():
    """NCCL 2.28 from the nvidia-nccl wheel torch loads (never the system 2.27 copy)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl wheel not found")
    return list(spec.submodule_search_locations)[0]


NCCL = _nccl_dir()
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(NCCL, "include")]
FLAGS += os.environ.get("PICASSO_NVCC_EXTRA", "").split()  # tuning experiments only


def _needs(obj, src, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))
    cmds = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if _needs(o, s, deps):
            lang = ["-x", "cu"] if s.endswith(".cu") else ["-x", "c++"]
            cmds.append([NVCC, *ARCH, *FLAGS, *lang, "-c", s, "-o", o])

    def run(c):
        if verbose:
            print(" ".join(c), flush=True)
        r = subprocess.run(c, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(c)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(jobs) as ex:
        for err in ex.map(run, cmds):
            if verbose and err:
                print(err)
    stale = not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs)
    if cmds or stale:
        nlib = os.path.join(NCCL, "lib")
        link = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-Xcompiler", "-fPIC", "-L", nlib,
                "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nlib, "-Xlinker", "--no-undefined"]
        run(link)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
