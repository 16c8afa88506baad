"""SURVEY.md sec. 8(f) row f3 on the GPU: CRT decryption == the plain
definition M = C^d mod n (oracle), for the paper's keys and seeded keys up to
4096 bits, including ciphertexts sharing a factor with n."""
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


@pytest.mark.parametrize("key", ["toy17947", "table2_513581", "fig2_187", "rsa64", "rsa96", "rsa512", "rsa1000",
                                 "rsa1024", "rsa2048", "rsa3072", "rsa4096"])
def test_crt_matches_oracle(R, key):
    k = workload.key(key)
    n, nb = k["n"], k["n"].bit_length()
    s = workload.limbs_needed(nb)
    count = 3000 if nb <= 1024 else 400
    m = workload.packets(count, nb, n=n, config_id=12) if nb > 20 else \
        np.arange(min(n, 3000), dtype=np.uint32).reshape(-1, 1)
    vals = workload.rows_to_ints(m)
    extra = [0, 1, n - 1, k["p"], k["q"], 2 * k["p"] % n, (k["p"] * 5) % n]
    C = oracle.modexp_batch(workload.ints_to_rows(vals + extra, s), k["e"], n)[:, :s]
    got = host(R.rsa_decrypt_crt_batch(dev(C), k["p"], k["q"], k["d"], nb))
    want = oracle.modexp_batch(C[:200], k["d"], n)[:, :s]
    assert np.array_equal(got[:200], want)
    # decryption inverts encryption on every packet (exact: x -> x^e is a bijection)
    assert workload.rows_to_ints(got) == vals + [x % n for x in extra]


def test_crt_equals_full_exponent_path(R):
    k = workload.key("rsa2048")
    c = workload.packets(70000, 2048, n=k["n"], config_id=13)
    t = dev(c)
    a = host(R.rsa_decrypt_crt_batch(t, k["p"], k["q"], k["d"], 2048))
    b = host(R.rsa_modexp_batch(t, k["d"], k["n"], 2048))
    assert np.array_equal(a, b)


def test_crt_prime_order_and_errors(R):
    k = workload.key("rsa1024")
    c = dev(workload.packets(100, 1024, n=k["n"], config_id=14))
    a = host(R.rsa_decrypt_crt_batch(c, k["p"], k["q"], k["d"], 1024))
    b = host(R.rsa_decrypt_crt_batch(c, k["q"], k["p"], k["d"], 1024))      # swapped primes
    assert np.array_equal(a, b)
    with pytest.raises(R.RsaError) as ei:
        R.rsa_decrypt_crt_batch(c, k["p"], k["p"], k["d"], 1024)
    assert ei.value.code == R.RSA_EEQUAL
    with pytest.raises(R.RsaError) as ei:
        R.rsa_decrypt_crt_batch(c, k["p"] + 1, k["q"], k["d"], 1024)
    assert ei.value.code == R.RSA_EEVEN
