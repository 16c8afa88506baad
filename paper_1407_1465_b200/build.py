"""Build librsa_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librsa_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("modexp.cu", "modexp_f64.cu", "modexp_multi.cu", "crt.cu", "rsa_abi.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("mont.cuh", "mont_f64.cuh", "mont_pair.cuh", "mont_sqr.cuh", "mont_multi.cuh", "mont_group.cuh", "plan.h", "host_bn.hpp")] + [
    os.path.join(os.path.dirname(HERE), "include", "rsa_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build the library (to `out` for an A/B variant, loaded with RSA_B200_LIB)."""
    if out:
        extra = os.environ.get("RSA_B200_NVCC_EXTRA", "").split()
        subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                               *extra, "-o", out, *SOURCES])
        return out
    if not force and not stale():
        return LIB
    extra = os.environ.get("RSA_B200_NVCC_EXTRA", "").split()   # A/B experiments, e.g. -DRSA_SMALL_PPT2=8
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *extra,
           "-Xptxas", "-v" if verbose else "-O3", "-o", LIB + ".tmp", *SOURCES]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    # the microbenchmarks (roofline denominator, chain latency), built alongside
    for name in ("imad_peak", "imad_latency", "dfma_latency"):
        mb = os.path.join(CSRC, "microbench", name)
        src = mb + ".cu"
        if os.path.exists(src) and (force or not os.path.exists(mb) or os.path.getmtime(mb) < os.path.getmtime(src)):
            subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-o", mb, src])
    return LIB


if __name__ == "__main__":
    o = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o[0] if o else None))
