"""Build the C-ABI library ``libmss.so`` in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmss.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_paths():
    try:
        import nvidia.nccl  # noqa: F401  (torch's bundled NCCL wheel)
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    return None, None


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "mss.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include")]
    if os.environ.get("MSS_FAST_BUILD"):
        # development only: --split-compile optimises the kernels of this one translation unit in
        # parallel (5 min -> 1-2 min) but changes code generation (the TMA pair kernel gets 78
        # instead of 84 registers and runs 10 % slower), so the product build does not use it
        cmd += ["--split-compile", "0"]
    inc, lib = _nccl_paths()
    if inc:
        cmd += ["-DMSS_WITH_NCCL=1", "-I", inc, "-L", lib, "-Xlinker", f"-rpath={lib}"]
    cmd += [os.path.join(CSRC, "mss.cu"), "-o", LIB + ".tmp"]
    if inc:
        cmd += ["-l:libnccl.so.2"]
    # cuFFT (NEXT-4 field sampler: a library FFT as a step of the method)
    cudalib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    cmd += ["-L", cudalib, "-lcufft", "-Xlinker", f"-rpath={cudalib}"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
