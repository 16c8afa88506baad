"""The paper's single-word exponentiation schedules as GPU kernels (SURVEY.md
sec. 8(f) row f2): Fig 4 naive, Fig 5a right-to-left and
Fig 5b left-to-right binary, Fig 12 halving
(PAPER.md:374-406), bit-exact against the oracle's implementations of the
same figures (oracle.naive, oracle.modexp_variant, oracle.halving) and the
oracle's Fig 5 batch path."""
import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def _run(R, vals, e, m, sched):
    import torch
    t = torch.from_numpy(np.asarray(vals, dtype=np.uint32).view(np.int32)).cuda()
    return [int(v) for v in R.rsa_modexp_batch_schedule(t, e, m, sched).cpu().numpy().view(np.uint32)]


SCHEDS = ["NAIVE", "R2L", "L2R", "HALVING"]


def _oracle(sched, g, e, m):
    if sched == "NAIVE":
        return oracle.naive(g, e, m)
    if sched == "R2L":
        return oracle.modexp_variant("r2l", g, e, m)
    if sched == "L2R":
        return oracle.modexp_variant("l2r", g, e, m)
    return oracle.halving(g, e, m, faithful=False)


@pytest.mark.parametrize("sched", SCHEDS)
def test_fig4_worked_example(R, sched):
    """4^13 mod 497 = 445 by every schedule."""
    assert _run(R, [4], 13, 497, getattr(R, "RSA_SCHED_" + sched)) == [445]


@pytest.mark.parametrize("sched", SCHEDS)
def test_toy_key_exhaustive(R, sched):
    """Every residue of the sec. 2 toy key n = 17947: encrypt with e = 131,
    decrypt with d = 14171 (reading Z1), vs the oracle's Fig 5 batch path;
    the full round trip returns every packet."""
    k = workload.key("toy17947")
    n, e, d = k["n"], k["e"], k["d"]
    g = np.arange(n, dtype=np.uint32)
    code = getattr(R, "RSA_SCHED_" + sched)
    c = _run(R, g, e, n, code)
    assert c == [int(v) for v in oracle.modexp_batch(g.reshape(-1, 1), e, n).ravel()]
    assert _run(R, c, d, n, code) == list(range(n))


@pytest.mark.parametrize("sched", SCHEDS)
def test_random_single_word(R, sched):
    """Random moduli below 2^31 (Fig 12's envelope) or 2^32, random bases
    (also >= m), exponents 0 .. 2^12 (the O(e) schedules) or full 32/64-bit
    (the binary ones), against the oracle's implementation of the same figure."""
    rng = np.random.default_rng(1465)
    code = getattr(R, "RSA_SCHED_" + sched)
    for trial in range(12):
        top = 2**31 if sched == "HALVING" else 2**32
        m = int(rng.integers(1, top)) if trial else 1
        big_e = sched in ("R2L", "L2R")
        e = int(rng.integers(0, 2**63 if big_e else 2**12)) if trial > 1 else trial
        g = rng.integers(0, 2**32, 64, dtype=np.uint64).astype(np.uint32)
        g[:4] = [0, 1, m - 1 if m > 1 else 0, min(m, 2**32 - 1)]
        got = _run(R, g, e, m, code)
        want = [_oracle(sched, int(x), e, m) for x in g]
        assert got == want, (sched, m, e)
        assert got == [pow(int(x), e, m) for x in g]


def test_faithful_fig12_exponent_zero(R):
    """Reading Z5: Fig 12 as printed returns g mod m for e = 0."""
    got = _run(R, [5, 12, 0], 0, 7, R.RSA_SCHED_HALVING_FAITHFUL)
    assert got == [oracle.halving(g, 0, 7, faithful=True) for g in (5, 12, 0)] == [5, 5, 0]


def test_schedule_errors(R):
    import torch
    t = torch.zeros(4, dtype=torch.int32, device="cuda")
    for args, code in [((3, 0, R.RSA_SCHED_R2L), R.RSA_ERANGE), ((2**32, 7, R.RSA_SCHED_NAIVE), R.RSA_ERANGE),
                       ((3, 2**31, R.RSA_SCHED_HALVING), R.RSA_ERANGE), ((3, 7, 9), R.RSA_EINVAL)]:
        with pytest.raises(R.RsaError) as ei:
            R.rsa_modexp_batch_schedule(t, *args)
        assert ei.value.code == code
