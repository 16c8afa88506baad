"""The alternative kernel shapes kept for measurement ('chosen by
measurement') stay bit-exact vs the oracle: the 1024/2048/4096-bit classes on
the integer pipe or the FP64 pipe, 2048-bit as a 2-lane group, 4096-bit as
integer lane pairs or 4-lane groups, and the thread-per-packet kernel for the
small widths (instead of the multi-packet one).  Selected in-process with the
C-ABI knob rsa_set_kernel_path (include/rsa_b200.h); one subprocess checks
that the RSA_B200_* environment switches of the A/B tools are still honoured."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(key, count):
    import torch
    import paper_1407_1465_b200 as R
    k = workload.key(key)
    nb = k["nbits"]
    s = workload.limbs_needed(nb)
    m = workload.packets(count, nb, n=k["n"], config_id=21)
    RR = 1 << (32 * s)                      # inputs at and above n as well (the call is total)
    edge = [v for v in (k["n"], k["n"] + 1, 2 * k["n"] - 1, RR - 1, RR - 2) if v < RR]
    m = np.concatenate([m, workload.ints_to_rows(edge, s)])
    t = torch.from_numpy(m.view(np.int32)).cuda()
    for e in (k["e"], k["d"], 3):
        got = R.rsa_modexp_batch(t, e, k["n"], nb).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, oracle.modexp_batch(m, e, k["n"])[:, :s]), e


def _classes(key):
    s = workload.limbs_needed(workload.key(key)["nbits"])
    return next(c for c in (2, 4, 8, 16, 32, 64, 128) if s <= c)


@pytest.mark.parametrize("path,key,count", [("TC", "rsa4096", 60), ("TC", "rsa3072", 60), ("TC", "rsa2048", 300), ("TC", "rsa1536", 300), ("TC", "rsa1024", 700),
                                            ("TC", "rsa1000", 300), ("TC", "rsa768", 300),
                                            ("INT", "rsa2048", 300), ("INT", "rsa1536", 300),
                                            ("INT", "rsa1024", 300), ("FP64", "rsa1024", 300),
                                            ("FP64", "rsa2048", 300), ("FP64", "rsa1536", 300),
                                            ("INT_GROUP", "rsa2048", 300), ("INT_GROUP", "rsa1536", 300),
                                            ("INT_PAIR", "rsa4096", 60), ("INT_PAIR", "rsa3072", 60),
                                            ("INT_GROUP", "rsa4096", 60), ("INT_GROUP", "rsa3072", 60),
                                            ("FP64", "rsa4096", 60), ("FP64", "rsa3072", 60),
                                            ("INT", "rsa64", 3001), ("INT", "rsa128", 3001),
                                            ("INT", "toy17947", 3001), ("INT_MULTI", "rsa64", 3001)])
def test_alternative_shapes(path, key, count):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    S = _classes(key)
    code = getattr(R, "RSA_PATH_" + path)
    with R.kernel_path(S, code):
        assert R.rsa_get_kernel_path(S) == code
        info = R.rsa_plan_info(workload.key(key)["d"], workload.key(key)["n"], workload.key(key)["nbits"])
        assert (info["fp64_digits"] > 0) == (path in ("FP64", "TC"))
        _check(key, count)


SCRIPT = r'''
import sys
sys.path[:0] = [%r, %r]
import paper_1407_1465_b200 as R
from test_gpu_shapes import _check
assert R.rsa_get_kernel_path(64) == R.RSA_PATH_INT, R.rsa_get_kernel_path(64)
assert R.rsa_get_kernel_path(128) == R.RSA_PATH_INT_PAIR
_check("rsa2048", 200)
print("shape ok")
''' % (ROOT, os.path.join(ROOT, "tests"))


def test_environment_switch_still_honoured():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, RSA_B200_F64="0"))
    assert r.returncode == 0 and "shape ok" in r.stdout, (r.stdout + r.stderr)[-2000:]
