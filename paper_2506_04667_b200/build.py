"""Builds the two in-tree libraries with nvcc for sm_100a (the only target), in parallel:

  lib/libfdmoe.so      the product: exactly include/fdmoe.h (no ablation bits, no diagnostics,
                       no profiling clocks in the pipeline roles)
  lib/libfdmoe_dev.so  the same sources with -DFDMOE_DEV -DFDMOE_WAIT_ACCOUNTING: FDMOE_DEBUG ablation
                       bits, the MMA-warp chunk log, per-role wait accounting and the
                       include/fdmoe_dev.h diagnostics (tests and tools/ only)

Both statically link the CUDA runtime so they do not depend on which libcudart the hosting process
(e.g. torch) already loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libfdmoe.so")
DEV_LIB = os.path.join(LIB_DIR, "libfdmoe_dev.so")
SOURCES = ["fdmoe_kernel.cu", "fdmoe_abi.cpp", "fdmoe_runtime.cpp"]
HEADERS = ["fdmoe_device.cuh", "fdmoe_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + \
           [os.path.join(ROOT, "include", h) for h in ("fdmoe.h", "fdmoe_dev.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _cmd(out: str, dev: bool, verbose: bool):
    cmd = [
        NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-diag-suppress", "550",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
    ]
    if dev:
        cmd += ["-DFDMOE_DEV", "-DFDMOE_WAIT_ACCOUNTING"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    return cmd + [os.path.join(CSRC, f) for f in SOURCES] + ["-o", out + ".tmp"]


def build(force: bool = False, verbose: bool = False, dev: bool = True) -> str:
    """Builds libfdmoe.so (and libfdmoe_dev.so unless dev=False) when stale; returns the product path."""
    os.makedirs(LIB_DIR, exist_ok=True)
    todo = [(LIB, False)] + ([(DEV_LIB, True)] if dev else [])
    todo = [(lib, d) for lib, d in todo if force or _stale(lib)]
    procs = [(lib, subprocess.Popen(_cmd(lib, d, verbose), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                    text=True)) for lib, d in todo]
    for lib, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc build of {os.path.basename(lib)} failed")
        if verbose:
            sys.stderr.write(err)
        os.replace(lib + ".tmp", lib)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
