"""Structured edge moduli for the FP64-pipe arithmetic (paper_1407_1465_b200/csrc/
mont_f64.cuh: the whole multiply at 4096 bits; the product half of the
tensor-core kernels, the default at 513-2048 bits, whose n' = -n^-1 mod R
then takes its extreme byte patterns too): moduli
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


@pytest.mark.parametrize("nb,path", [(513, None), (1000, None), (1024, None), (1025, None), (1536, None),
                                     (2047, None), (2048, None), (2049, None), (3072, None), (4095, None),
                                     (4096, None), (1024, "FP64"), (2048, "FP64"), (1025, "FP64"),
                                     (4096, "FP64"), (3072, "FP64")])
def test_f64_edge_moduli(R, nb, path):
    if path is None:
        _edges(R, nb)
    else:                                   # the FP64 kernel, selectable where the TC path is the default
        with R.kernel_path(next(c for c in (32, 64, 128) if workload.limbs_needed(nb) <= c),
                           getattr(R, "RSA_PATH_" + path)):
            _edges(R, nb)


def _edges(R, nb):
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
