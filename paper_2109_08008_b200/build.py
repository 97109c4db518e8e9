"""Build libnmt.so (all CUDA sources, sm_100a) in-tree with nvcc.

The .so lives next to this file so it travels with the repo snapshot to the GPU box
(a JIT cache under ~/.cache would not).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnmt.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas=-v"]
# NMT_EXTRA_NVCC: extra flags for a diagnostic build, e.g. "-DNMT_TRAP_DIAG"
FLAGS += os.environ.get("NMT_EXTRA_NVCC", "").split()
OBJ = os.path.join(HERE, "build")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    # one nvcc per translation unit in parallel, then one link (no relocatable device code:
    # kernels are launched only from host code in their own file)
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()

    def cc(src):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC] + FLAGS + ["-I", INCLUDE, "-c", "-o", obj, src],
                           capture_output=True, text=True)
        return obj, r

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        res = list(ex.map(cc, srcs))
    errs = "".join(r.stdout + r.stderr for _, r in res)
    if verbose or any(r.returncode != 0 for _, r in res):
        sys.stderr.write(errs)
    if any(r.returncode != 0 for _, r in res):
        raise RuntimeError("nvcc failed building libnmt.so")
    tmp = LIB + ".tmp"
    # -z defs: an unresolved symbol fails the link here instead of the dlopen on the GPU box
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-Xlinker", "-z,defs", "-o", tmp] + [o for o, _ in res],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libnmt.so")
    os.replace(tmp, LIB)
    log = os.path.join(HERE, "build_ptxas.log")
    with open(log, "w") as f:
        f.write(errs)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
