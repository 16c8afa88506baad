"""Build librsa_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librsa_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("modexp.cu", "modexp_f64.cu", "modexp_tc.cu", "modexp_multi.cu", "crt.cu", "rsa_abi.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("mont.cuh", "mont_f64.cuh", "mont_pair.cuh", "mont_sqr.cuh", "mont_multi.cuh", "mont_group.cuh", "mont_tc.cuh", "tc_i8.cuh", "tc_digits.cuh", "plan.h", "host_bn.hpp", "devcache.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "rsa_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _compile_link(out: str, extra: list[str], verbose: bool) -> None:
    """One nvcc per translation unit, in parallel, then one link (the units
    are independent; the FP64 and integer kernels dominate the build time)."""
    objdir = os.path.join(HERE, "build", os.path.basename(out).replace(".", "_"))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra,
               "-Xptxas", "-v" if verbose else "-O3", "-c", "-o", obj, src]
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs])


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build the library (to `out` for an A/B variant, loaded with RSA_B200_LIB)."""
    extra = os.environ.get("RSA_B200_NVCC_EXTRA", "").split()   # A/B experiments, e.g. -DRSA_SMALL_PPT2=8
    if out:
        _compile_link(out, extra, verbose)
        return out
    if not force and not stale():
        return LIB
    _compile_link(LIB + ".tmp", extra, verbose)
    os.replace(LIB + ".tmp", LIB)
    # the microbenchmarks (roofline denominator, chain latency), built alongside
    for name in ("imad_peak", "imad_latency", "dfma_latency", "tc_redc"):
        mb = os.path.join(CSRC, "microbench", name)
        src = mb + ".cu"
        # tc_redc includes the product headers (mont_tc.cuh): rebuilt with the library
        if os.path.exists(src) and (force or name == "tc_redc" or not os.path.exists(mb)
                                    or os.path.getmtime(mb) < os.path.getmtime(src)):
            subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-o", mb, src])
    return LIB


if __name__ == "__main__":
    o = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o[0] if o else None))
