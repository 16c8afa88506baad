"""Structured edge moduli for the FP64-pipe kernels (paper_1407_1465_b200/csrc/
mont_f64.cuh; the default for the 1024-, 2048- and 4096-bit classes): moduli
whose 52-bit digits are all ones or nearly all zeros (every column at its
carry extreme), the smallest and largest modulus of each class (R / n from
2^4 to 2^1056), bases at 0, 1, n - 1, n, 2^(32 s) - 1 (the call is total), and
exponents with long zero runs (window edges).  Bit-exact vs the oracle."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workload  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def moduli(nb):
    """Odd moduli of exactly nb bits at the carry extremes."""
    top = 1 << (nb - 1)
    return [
        (1 << nb) - 1,                       # all ones: every digit 2^52 - 1
        top + 1,                             # smallest nb-bit odd modulus (largest R / n)
        top | 0xFFFFF,                       # nearly all-zero digits
        (1 << nb) - (1 << 52) - 1,           # one zero digit
        sum(1 << (52 * k) for k in range(nb // 52)) | top | 1,   # a one at each digit boundary
        (1 << nb) - 3,
    ]


@pytest.mark.parametrize("nb", [513, 1000, 1024, 1025, 1536, 2047, 2048, 2049, 3072, 4095, 4096])
def test_f64_edge_moduli(R, nb):
    rnd = random.Random(52 * nb)
    s = workload.limbs_needed(nb)
    full = (1 << (32 * s)) - 1
    for n in moduli(nb):
        assert n.bit_length() == nb and n & 1
        vals = [v for v in (0, 1, 2, n - 1, n, n + 1, full, full - 1) if v <= full]
        vals += [rnd.getrandbits(32 * s) for _ in range(9)]
        base = workload.ints_to_rows(vals, s)
        t = torch.from_numpy(base.view(np.int32)).cuda()
        for e in (3, 65537, (1 << 300) + 1, rnd.getrandbits(nb) | 1 | (1 << (nb - 1))):
            got = R.rsa_modexp_batch(t, e, n, nb).cpu().numpy().view(np.uint32)
            want = oracle.modexp_batch(base, e, n)[:, :s]
            assert np.array_equal(got, want), (nb, hex(n)[:20], e.bit_length())
