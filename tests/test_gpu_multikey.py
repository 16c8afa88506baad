"""SURVEY.md sec. 8(f) row f1 on the GPU: multi-key batches (per-packet
modulus and exponent) and the Miller-Rabin prime search behind key
generation, parity against the oracle (expected values from oracle/ only;
candidates from workload/'s independent copy of the generator)."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def random_odd_moduli(count, nbits, rnd, full=True):
    vals = []
    for _ in range(count):
        b = nbits if full else rnd.randrange(max(2, nbits - 40), nbits + 1)
        v = rnd.getrandbits(b) | 1 | (1 << (b - 1))
        vals.append(max(v, 3))
    return vals


@pytest.mark.parametrize("nbits", [64, 100, 256, 512, 1000, 1024, 2048])
def test_multikey_parity(R, nbits):
    rnd = random.Random(nbits)
    s = workload.limbs_needed(nbits)
    count = {64: 50000, 100: 30000, 256: 20000, 512: 6000}.get(nbits, 1500)
    mods = random_odd_moduli(count, nbits, rnd, full=(nbits % 2 == 0))
    base = [rnd.getrandbits(32 * s) for _ in range(count)]
    exps = [rnd.getrandbits(32 * s) for _ in range(count)]
    exps[:4] = [0, 1, 2, 65537]
    B, E, M = (workload.ints_to_rows(v, s) for v in (base, exps, mods))
    got = host(R.rsa_modexp_batch_multi(dev(B), dev(E), dev(M), nbits))
    assert np.array_equal(got, oracle.modexp_multi(B, E, M))


def test_multikey_many_rsa_keys_public_exponent(R):
    """Encrypt to many recipients: 1024-bit keys (fixture keys reused) with
    e = 65537 scanned over 17 bits."""
    keys = [workload.key(k) for k in ("rsa1024", "rsa1000")]
    rnd = random.Random(3)
    count = 4096
    s = 32
    mods = [keys[i % 2]["n"] for i in range(count)]
    base = [rnd.randrange(m) for m in mods]
    E = workload.ints_to_rows([65537] * count, s)
    B, M = workload.ints_to_rows(base, s), workload.ints_to_rows(mods, s)
    got = host(R.rsa_modexp_batch_multi(dev(B), dev(E), dev(M), 1024, exp_bits=17))
    assert np.array_equal(got, oracle.modexp_multi(B, E, M))


def test_multikey_bad_moduli_status(R):
    s = 8
    mods = [2 ** 255 + 1, 2 ** 255 + 2, 1, 0, 7]
    M = workload.ints_to_rows(mods, s)
    B = workload.ints_to_rows([5] * 5, s)
    E = workload.ints_to_rows([3] * 5, s)
    st = torch.zeros(5, dtype=torch.int32, device="cuda")
    got = host(R.rsa_modexp_batch_multi(dev(B), dev(E), dev(M), 256, status=st))
    status = st.cpu().numpy()
    assert list(status) == [0, -3, -3, -3, 0]
    assert workload.rows_to_ints(got)[0] == pow(5, 3, mods[0]) and workload.rows_to_ints(got)[4] == 125 % 7
    assert all(v == 0 for v in workload.rows_to_ints(got)[1:4])


@pytest.mark.parametrize("nbits", [64, 512, 1024])
def test_candidate_generator_matches_independent_copy(R, nbits):
    got = host(R.rsa_prime_candidates(nbits, 1407, 100, 500))
    assert np.array_equal(got, workload.prime_candidates(nbits, 1407, 100, 500))


@pytest.mark.parametrize("nbits,count", [(64, 20000), (256, 6000), (512, 3000), (1024, 1200)])
def test_sieve_and_mr_rounds_match_oracle(R, nbits, count):
    cand = workload.prime_candidates(nbits, 77, 0, count)
    vals = workload.rows_to_ints(cand)
    sv = host(R.rsa_prime_sieve(dev(cand), nbits)).view(np.int32)
    small = [p for p in range(3, 4096, 2) if all(p % f for f in range(3, int(p ** 0.5) + 1, 2))]
    want_sv = [int(all(v % p for p in small)) for v in vals]
    assert list(sv) == want_sv
    idx = [i for i, f in enumerate(want_sv) if f][:600]
    sub = cand[idx]
    for a in (2, 3, 5):
        mr = host(R.rsa_miller_rabin_batch(dev(sub), nbits, a)).view(np.int32)
        assert [bool(x) for x in mr] == [oracle.mr_round(vals[i], a) for i in idx]


def test_mr_strong_pseudoprimes(R):
    """Strong pseudoprimes to base 2 (2047 = 23*89, 3277, 4033, 4681, 8321)
    pass one base-2 round, fail base 3 -- exactly one MR round's semantics."""
    sp = [2047, 3277, 4033, 4681, 8321, 15841, 29341, 42799, 49141, 52633]
    C = workload.ints_to_rows(sp, 1)
    for a in (2, 3):
        got = host(R.rsa_miller_rabin_batch(dev(C), 16, a)).view(np.int32)
        assert [bool(x) for x in got] == [oracle.mr_round(v, a) for v in sp]
    assert all(oracle.mr_round(v, 2) for v in sp)


@pytest.mark.parametrize("nbits", [64, 512, 1024])
def test_prime_search(R, nbits):
    primes, tried = R.rsa_prime_search(nbits, 5, 6, rounds=8)
    assert len(primes) == 6 and tried > 0
    for p in primes:
        assert p.bit_length() == nbits and (p >> (nbits - 2)) == 3 and oracle.is_prime(p)
    # deterministic, and the first primes of the candidate stream in index order
    again, _ = R.rsa_prime_search(nbits, 5, 6, rounds=8)
    assert again == primes
    if nbits <= 512:
        cand = workload.rows_to_ints(workload.prime_candidates(nbits, 5, 0, 4000))
        want = [c for c in cand if oracle.is_prime(c)][:6]
        assert primes == want


@pytest.mark.parametrize("nbits", [512, 2048])
def test_keygen_end_to_end(R, nbits):
    k = R.rsa_keygen(nbits, 65537, seed=11)
    assert k["n"].bit_length() == nbits and k["n"] == k["p"] * k["q"]
    assert oracle.is_prime(k["p"]) and oracle.is_prime(k["q"]) and k["p"] != k["q"]
    assert oracle.keygen_check(k["p"], k["q"], 65537) == (k["n"], k["phi"], k["d"])
    m = workload.packets(257, nbits, n=k["n"], config_id=9)
    t = dev(m)
    c = R.rsa_modexp_batch(t, 65537, k["n"], nbits)
    y = R.rsa_modexp_batch(c, k["d"], k["n"], nbits)
    assert np.array_equal(host(y), m)


@pytest.mark.parametrize("nbits", [64, 96, 1000])
def test_keygen_odd_sizes(R, nbits):
    k = R.rsa_keygen(nbits, 65537, seed=3)
    assert k["n"].bit_length() == nbits and k["n"] == k["p"] * k["q"] and k["p"] != k["q"]
    assert oracle.is_prime(k["p"]) and oracle.is_prime(k["q"])
    assert oracle.keygen_check(k["p"], k["q"], 65537) == (k["n"], k["phi"], k["d"])
