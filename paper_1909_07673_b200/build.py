"""Build libnacs.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnacs.so")
SOURCES = [os.path.join(CSRC, f) for f in ("nacs_kernels.cu", "nacs_warp.cu", "nacs_paths.cu", "nacs_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "nacs_internal.h"), os.path.join(CSRC, "nacs_device.cuh"),
                  os.path.join(ROOT, "include", "nacs.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# NCCL bundled with torch (nvidia-nccl wheel): headers, library, and an rpath so that
# libnacs.so finds the same libnccl.so.2 at run time
try:
    import nvidia.nccl as _nccl
    NCCL = list(_nccl.__path__)[0]
except Exception:  # pragma: no cover
    NCCL = "/usr"
NCCL_FLAGS = ["-I", os.path.join(NCCL, "include"), "-L", os.path.join(NCCL, "lib"), "-lnccl",
              "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    if force or stale():
        cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), *NCCL_FLAGS, "-o", out, *SOURCES]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            sys.stderr.write(p.stdout + p.stderr)
            raise RuntimeError("nvcc failed building libnacs.so")
        if verbose:
            sys.stderr.write(p.stderr)
    return out


if __name__ == "__main__":
    # python build.py [out.so -DFLAG ...]: an experiment build next to the product library
    if len(sys.argv) > 1:
        build(force=True, out=os.path.abspath(sys.argv[1]), extra=sys.argv[2:])
    else:
        build(force=True, verbose=True)
