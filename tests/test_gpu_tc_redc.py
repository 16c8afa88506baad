"""The tensor-core Montgomery reduction on its own (csrc/mont_tc.cuh through
csrc/microbench/tc_redc.cu, built with the library): for T = A B with A, B < n
(random, the extremes A = B = n - 1, A = 0, A = B = 1, and T constructed so that
(T + m n) / R lands at n - d, n, n + d: the conditional subtraction's rare path
where the top words tie and the full borrow chain decides), the quotient
m = (T mod R) n' mod R read back from the staging buffer and the result
U = T R^-1 mod n (canonical) are compared with Python integers, R = 2^2048,
over a full persistent wave (148 x 256 packets, two tiles per CTA)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1407_1465_b200", "csrc", "microbench", "tc_redc")


def test_tc_reduction_bit_exact(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(EXE):
        from paper_1407_1465_b200 import build
        build.build(force=True)
    assert os.path.exists(EXE)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tc_redc_check.py"), EXE, str(148 * 256)],
                       cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bad_m 0, bad_u 0" in r.stdout
