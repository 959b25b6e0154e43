"""Build libssa_b200.so in-tree with nvcc for sm_100a (explicit -gencode; no torch arch list).

python -m paper_2505_17412_b200.build  [--force]
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.environ.get("SSA_LIB_OUT", os.path.join(HERE, "libssa_b200.so"))
OBJ = os.path.join(HERE, "_obj" + os.environ.get("SSA_OBJ_SUFFIX", ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", INCLUDE]
FLAGS += [f for f in os.environ.get("SSA_EXTRA_NVCC_FLAGS", "").split() if f]   # e.g. -DSSA_TRACE (debug builds)


def sources():
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    for need in ("tc_fwd.cu", "tc_bwd.cu"):      # the tcgen05 kernels are the product path: no stub build
        if not os.path.exists(os.path.join(CSRC, need)):
            raise RuntimeError(f"missing {need}")
    return srcs


def _digest(path, extra):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        h.update(f.read())
    for e in extra:
        with open(e, "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                     glob.glob(os.path.join(INCLUDE, "*.h")))
    objs = []
    for src in sources():
        dig = _digest(src, headers)
        obj = os.path.join(OBJ, os.path.basename(src) + f".{dig}.o")
        if force or not os.path.exists(obj):
            cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log = os.path.join(OBJ, os.path.basename(src) + ".ptxas.log")
            with open(log, "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                print(r.stderr)
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
