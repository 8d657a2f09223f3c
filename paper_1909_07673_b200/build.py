"""Build libnacs.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnacs.so")
SOURCES = [os.path.join(CSRC, f) for f in ("nacs_kernels.cu", "nacs_warp.cu", "nacs_paths.cu", "nacs_rank.cu", "nacs_api.cu")]
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
    """Compile the sources in parallel (one nvcc per file, no cross-file device code), then
    link the shared library."""
    if force or stale():
        import tempfile
        from concurrent.futures import ThreadPoolExecutor
        tmp = tempfile.mkdtemp(prefix="nacs_build_")
        compile_flags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
        inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(NCCL, "include")]

        def compile_one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            return obj, subprocess.run([NVCC, *compile_flags, *extra, *inc, "-c", "-o", obj, src],
                                       capture_output=True, text=True)

        with ThreadPoolExecutor(len(SOURCES)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        log = "".join(p.stdout + p.stderr for _, p in results)
        if any(p.returncode != 0 for _, p in results):
            sys.stderr.write(log)
            raise RuntimeError("nvcc failed building libnacs.so")
        link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                "-Xcompiler", "-fPIC", *NCCL_FLAGS, "-o", out, *[o for o, _ in results]]
        p = subprocess.run(link, capture_output=True, text=True)
        if p.returncode != 0:
            sys.stderr.write(log + p.stdout + p.stderr)
            raise RuntimeError("nvcc failed linking libnacs.so")
        if verbose:
            sys.stderr.write(log)
    return out


if __name__ == "__main__":
    # python build.py [out.so -DFLAG ...]: an experiment build next to the product library
    if len(sys.argv) > 1:
        build(force=True, out=os.path.abspath(sys.argv[1]), extra=sys.argv[2:])
    else:
        build(force=True, verbose=True)
