"""Fuzz across width-class boundaries: random odd moduli of every awkward bit
length (class edges 32k-1 / 32k / 32k+1 up to 4096 bits, where the kernel
width S pads the packet's limbs), random exponents of mixed lengths, random
bases below 2^(32 s), multi-key batches of mixed moduli -- all bit-exact vs
the oracle."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workload  # noqa: E402

EDGE_BITS = [2, 3, 5, 17, 31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 128, 129, 255, 256, 257, 511, 512, 513,
             1023, 1024, 1025, 2047, 2048, 2049, 3000, 4095, 4096]


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def run(R, vals, e, n, nb):
    s = workload.limbs_needed(nb)
    base = workload.ints_to_rows(vals, s)
    t = torch.from_numpy(base.view(np.int32)).cuda()
    got = R.rsa_modexp_batch(t, e, n, nb)
    torch.cuda.synchronize()
    return workload.rows_to_ints(got.cpu().numpy().view(np.uint32)), base


@pytest.mark.parametrize("nb", EDGE_BITS)
def test_fuzz_width_edges(R, nb):
    rnd = random.Random(7000 + nb)
    s = workload.limbs_needed(nb)
    for trial in range(3 if nb <= 1100 else 2):
        n = rnd.getrandbits(nb) | 1 | (1 << (nb - 1))
        if n < 3:
            n = 3
        count = rnd.choice([1, 7, 33, 300]) if nb > 1100 else rnd.choice([1, 31, 1000, 5000])
        vals = [rnd.getrandbits(32 * s) for _ in range(count)]
        ebits = rnd.choice([1, 2, 17, 64, nb]) if nb > 1100 else rnd.choice([1, 5, 17, 64, 200, nb + 7])
        e = rnd.getrandbits(min(ebits, 32 * s)) | 1
        got, base = run(R, vals, e, n, nb)
        want = workload.rows_to_ints(oracle.modexp_batch(base, e, n)[:, :s])
        assert got == want, (nb, trial, e.bit_length())


def test_fuzz_multikey_mixed_moduli(R):
    rnd = random.Random(99)
    for nb in (64, 100, 700, 1500, 2048):
        s = workload.limbs_needed(nb)
        count = 700 if nb <= 700 else 150
        mods = [rnd.getrandbits(rnd.randrange(max(2, nb - 70), nb + 1)) | 1 for _ in range(count)]
        mods = [max(m, 3) for m in mods]
        base = [rnd.getrandbits(32 * s) for _ in range(count)]
        eb = rnd.choice([5, 17, 100, 32 * s])
        exps = [rnd.getrandbits(eb) for _ in range(count)]
        B, E, M = (workload.ints_to_rows(v, s) for v in (base, exps, mods))
        tb, te, tm = (torch.from_numpy(x.view(np.int32)).cuda() for x in (B, E, M))
        got = R.rsa_modexp_batch_multi(tb, te, tm, nb, exp_bits=eb)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().view(np.uint32), oracle.modexp_multi(B, E, M)), nb
