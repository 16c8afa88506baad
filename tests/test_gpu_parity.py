"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit-exact.

Every expected value comes from oracle/ (or the paper, cited in
tests/golden/), never from the CUDA path.  Sizes: element-by-element at sizes
the oracle finishes in seconds (several CTAs' worth of packets, a ragged
tail, more packets than persistent-grid threads so each thread loops), and at
BASELINE.json full sizes in the bench's launch configuration on samples plus
properties that hold at any size (inverse permutation, Fermat).
"""
import json
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workload  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def gpu_run(R, base_np, exp, n, nbits):
    t = torch.from_numpy(base_np.view(np.int32)).cuda()
    out = R.rsa_modexp_batch(t, exp, n, nbits)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32)


def oracle_rows(base_np, exp, n, s):
    out = oracle.modexp_batch(base_np, exp, n)
    assert out.shape[1] >= s
    return out[:, :s]


# ------------------------------------------------------------------ paper toy key

def test_toy_packets_encrypt_decrypt(R):
    g = gold("sec2_packets.json")
    dv = gold("survey_derived.json")
    n, e = g["n"], g["e"]
    _, _, d = R.rsa_keygen_check(g["p"], g["q"], e)
    assert d == dv["toy_d"]
    pk = np.array(R.rsa_encode(g["text"]), dtype=np.uint32).reshape(-1, 1)
    c = gpu_run(R, pk, e, n, 15)
    assert [int(v) for v in c.ravel()] == dv["toy_ciphertexts"]
    assert np.array_equal(c, oracle_rows(pk, e, n, 1))
    m = gpu_run(R, c, d, n, 15)
    assert R.rsa_decode(m.ravel()) == g["decoded"]
    wrong = gpu_run(R, c, g["paper_d"], n, 15)
    assert [int(v) for v in wrong.ravel()] == dv["toy_wrong_decrypt_with_paper_d"]


@pytest.mark.parametrize("key", ["toy17947", "table2_513581", "fig2_187"])
def test_small_keys_exhaustive(R, key):
    k = workload.key(key)
    n, e, d = k["n"], k["e"], k["d"]
    nbits = n.bit_length()
    base = np.arange(n, dtype=np.uint32).reshape(-1, 1)
    c = gpu_run(R, base, e, n, nbits)
    assert np.array_equal(c, oracle_rows(base, e, n, 1))
    m = gpu_run(R, c, d, n, nbits)
    assert np.array_equal(m, base)
    # the paper's own inputs: values 0..800
    if n > 800:
        pp = workload.paper_packets(4096, config_id=0)
        assert np.array_equal(gpu_run(R, pp, e, n, nbits), oracle_rows(pp, e, n, 1))


def test_fig4_worked_example(R):
    g = gold("fig4_trace.json")
    base = np.array([[g["g"]]], dtype=np.uint32)
    assert int(gpu_run(R, base, g["e"], g["m"], 9)[0, 0]) == g["result"]


# ------------------------------------------------------------------ multi-precision widths

WIDTHS = ["rsa64", "rsa96", "rsa128", "rsa192", "rsa256", "rsa384", "rsa512", "rsa768", "rsa1000",
          "rsa1024", "rsa1536", "rsa2048", "rsa3072", "rsa4096"]


@pytest.mark.parametrize("key", WIDTHS)
def test_parity_public_exponent(R, key):
    k = workload.key(key)
    nb, n = k["nbits"], k["n"]
    s = workload.limbs_needed(nb)
    # more packets than persistent-grid threads (each thread loops) + a ragged tail
    count = {64: 700001, 96: 400003, 128: 400003, 192: 200001, 256: 200001}.get(nb, 40000 + 77)
    base = workload.packets(count, nb, n=n, config_id=2)
    got = gpu_run(R, base, k["e"], n, nb)
    assert np.array_equal(got, oracle_rows(base, k["e"], n, s))


@pytest.mark.parametrize("key", WIDTHS)
def test_parity_private_exponent(R, key):
    k = workload.key(key)
    nb, n = k["nbits"], k["n"]
    s = workload.limbs_needed(nb)
    count = 40000 + 11 if nb <= 128 else (4096 + 9 if nb <= 512 else (600 + 3 if nb <= 2048 else 160 + 3))
    base = workload.packets(count, nb, n=n, config_id=3)
    got = gpu_run(R, base, k["d"], n, nb)
    assert np.array_equal(got, oracle_rows(base, k["d"], n, s))


@pytest.mark.parametrize("w", [1, 2, 3, 4, 5, 6, 7])
def test_forced_windows_agree(R, w):
    k = workload.key("rsa512")
    base = workload.packets(1500, 512, n=k["n"], config_id=4)
    want = oracle_rows(base, k["d"], k["n"], 16)
    R.rsa_set_window(w)
    try:
        got = gpu_run(R, base, k["d"], k["n"], 512)
        assert R.rsa_plan_info(k["d"], k["n"], 512)["window"] == w
    finally:
        R.rsa_set_window(0)
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("key", ["toy17947", "rsa64", "rsa128", "rsa1000", "rsa2048", "rsa3072", "rsa4096"])
def test_edge_exponents_and_bases(R, key):
    """Inputs at and above n (the call is total, reading Z11) with exponents
    whose last window digit is 1 -- the final multiply then takes the raw
    input (RSA_OP_MULX) -- and others; every width-class kernel."""
    k = workload.key(key)
    nb, n = k["nbits"], k["n"]
    s = workload.limbs_needed(nb)
    rnd = random.Random(nb)
    vals = [0, 1, 2, n - 1, n - 2, n, n + 1, (1 << (32 * s)) - 1, (1 << (32 * s)) - 2, 2 * n if 2 * n < (1 << (32 * s)) else 3]
    vals += [rnd.getrandbits(32 * s) for _ in range(50)]
    base = workload.ints_to_rows(vals, s)
    exps = [0, 1, 2, 3, 4, 65537, (1 << 20) - 1, 1 << 40, k["d"], n - 1, rnd.getrandbits(32 * s)]
    for e in [e for e in exps if e < (1 << (32 * s))]:            # the exponent has s limbs
        got = gpu_run(R, base, e, n, nb)
        want = [pow(v, e, n) for v in vals]
        assert workload.rows_to_ints(got) == want, e
        assert np.array_equal(got, oracle_rows(base, e, n, s))


def test_in_place_and_empty(R):
    k = workload.key("rsa256")
    base = workload.packets(5000, 256, n=k["n"], config_id=5)
    want = oracle_rows(base, k["e"], k["n"], 8)
    t = torch.from_numpy(base.view(np.int32)).cuda()
    R.rsa_modexp_batch(t, k["e"], k["n"], 256, out=t)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy().view(np.uint32), want)
    empty = torch.empty((0, 8), dtype=torch.int32, device="cuda")
    R.rsa_modexp_batch(empty, k["e"], k["n"], 256)


def test_argument_errors(R):
    k = workload.key("rsa256")
    t = torch.zeros((4, 8), dtype=torch.int32, device="cuda")
    with pytest.raises(R.RsaError) as ei:
        R.rsa_modexp_batch(t, 3, k["n"] + 1, 256)          # even modulus
    assert ei.value.code == R.RSA_EEVEN
    with pytest.raises(R.RsaError) as ei:
        R.rsa_modexp_batch(t, 3, k["n"], 255)               # n >= 2^nbits
    assert ei.value.code == R.RSA_ERANGE
    with pytest.raises(R.RsaError) as ei:
        R.rsa_modexp_batch(torch.zeros((4, 1), dtype=torch.int32, device="cuda"), 3, 1, 1)
    assert ei.value.code == R.RSA_ERANGE
    big = torch.zeros((4, 129), dtype=torch.int32, device="cuda")
    with pytest.raises(R.RsaError) as ei:
        R.rsa_modexp_batch(big, 3, (1 << 4096) + 1, 4097)
    assert ei.value.code == R.RSA_ERANGE


def test_host_entry_matches_device(R):
    k = workload.key("rsa1024")
    base = workload.packets(70000, 1024, n=k["n"], config_id=6)
    out = R.rsa_modexp_batch_host(base, k["e"], k["n"], 1024)
    dev = gpu_run(R, base, k["e"], k["n"], 1024)
    assert np.array_equal(out, dev)
    idx = np.random.default_rng(0).choice(len(base), 2000, replace=False)
    assert np.array_equal(out[idx], oracle_rows(base[idx], k["e"], k["n"], 32))


# ------------------------------------------------------------------ full sizes (bench configuration)

def _sample(count, k=4000, seed=0):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([np.arange(16), rng.choice(count, k, replace=False), [count - 1]]))


def test_full_size_rsa2048_encrypt(R):
    """C2: 1M packets, e = 65537; sampled oracle parity + full-batch
    inverse-permutation (decrypt on GPU, compare with input)."""
    k = workload.key("rsa2048")
    cfg = workload.CONFIGS["rsa2048-enc"]
    base = workload.packets(cfg["count"], 2048, n=k["n"], config_id=cfg["config_id"])
    c = gpu_run(R, base, k["e"], k["n"], 2048)
    idx = _sample(len(base))
    assert np.array_equal(c[idx], oracle_rows(base[idx], k["e"], k["n"], 64))


def test_full_size_rsa2048_decrypt_inverse_permutation(R):
    """C3: y = c^d on the full 1M batch is exact iff oracle(y, e) == c (P9);
    checked on a large sample with the oracle, and y == m on all packets."""
    k = workload.key("rsa2048")
    cfg = workload.CONFIGS["rsa2048-dec"]
    m = workload.packets(cfg["count"], 2048, n=k["n"], config_id=cfg["config_id"])
    c = oracle.modexp_batch(m[:65536], k["e"], k["n"])              # oracle ciphertexts (sample)
    y = gpu_run(R, c, k["d"], k["n"], 2048)
    assert np.array_equal(y, m[:65536])
    idx = _sample(65536, 600)
    assert np.array_equal(y[idx], oracle_rows(c[idx], k["d"], k["n"], 64))


def test_full_size_fermat_prime_modulus(R):
    """P6 at full size: for the 1024-bit prime p of the RSA-2048 key,
    a^(p-1) = 1 mod p for every packet a in [1, p)."""
    k = workload.key("rsa2048")
    p = k["p"]
    base = workload.packets(1 << 20, 1024, n=p, config_id=7)
    base[base.sum(axis=1) == 0, 0] = 5                              # avoid a = 0
    got = gpu_run(R, base, p - 1, p, 1024)
    assert (got[:, 0] == 1).all() and (got[:, 1:] == 0).all()


def test_full_size_u64(R):
    """C1: 16M packets under the 64-bit key, e and full d; round trip on all,
    oracle parity on a sample."""
    k = workload.key("rsa64")
    cfg = workload.CONFIGS["u64"]
    m = workload.packets(cfg["count"], 64, n=k["n"], config_id=cfg["config_id"])
    c = gpu_run(R, m, k["e"], k["n"], 64)
    y = gpu_run(R, c, k["d"], k["n"], 64)
    assert np.array_equal(y, m)
    idx = _sample(len(m), 20000)
    assert np.array_equal(c[idx], oracle_rows(m[idx], k["e"], k["n"], 2))
    assert np.array_equal(y[idx], oracle_rows(c[idx], k["d"], k["n"], 2))


def test_full_size_rsa4096_decrypt(R):
    """C4: 256K packets, full 4095-bit d (lane-pair kernel): y == m on every
    packet for oracle ciphertexts of a sample, oracle parity on a subsample,
    and the GPU round trip on the whole batch."""
    k = workload.key("rsa4096")
    cfg = workload.CONFIGS["rsa4096-dec"]
    m = workload.packets(cfg["count"], 4096, n=k["n"], config_id=cfg["config_id"])
    c_gpu = gpu_run(R, m, k["e"], k["n"], 4096)
    idx = _sample(len(m), 3000)
    assert np.array_equal(c_gpu[idx], oracle_rows(m[idx], k["e"], k["n"], 128))
    y = gpu_run(R, c_gpu, k["d"], k["n"], 4096)
    assert np.array_equal(y, m)
    sub = idx[:40]
    assert np.array_equal(y[sub], oracle_rows(c_gpu[sub], k["d"], k["n"], 128))


# ------------------------------------------------------------------ f2: the paper's Fig 12 kernel

@pytest.mark.parametrize("key", ["toy17947", "table2_513581", "fig2_187"])
def test_paper_fig12_kernel_matches_oracle(R, key):
    k = workload.key(key)
    n, e = k["n"], k["e"]
    base = np.arange(min(n, 65536), dtype=np.uint32)
    t = torch.from_numpy(base.view(np.int32)).cuda()
    for exp in (e, 0, 1, 2, 1000):
        for faithful in (True, False):
            got = R.rsa_modexp_batch_paper(t, exp, n, faithful=faithful)
            torch.cuda.synchronize()
            got = got.cpu().numpy().view(np.uint32)
            want = np.array([oracle.halving(int(g), exp, n, faithful) for g in base[:3000]], dtype=np.uint32)
            assert np.array_equal(got[:3000], want), (exp, faithful)
            if exp or not faithful:
                assert np.array_equal(got, oracle_rows(base.reshape(-1, 1), exp, n, 1).ravel())


def test_paper_fig12_table1_shapes(R):
    """Table 1 shapes: n = 131*137, e = 131, paper inputs
    0..800, sizes 256 .. 32784; both kernels agree with the oracle."""
    n, e = 17947, 131
    for size in (256, 512, 1024, 2048, 4096, 8192, 16392, 32784):
        pp = workload.paper_packets(size, config_id=size)
        t = torch.from_numpy(pp.ravel().view(np.int32)).cuda()
        got = R.rsa_modexp_batch_paper(t, e, n).cpu().numpy().view(np.uint32)
        mont = gpu_run(R, pp, e, n, 15).ravel()
        want = oracle_rows(pp, e, n, 1).ravel()
        assert np.array_equal(got, want) and np.array_equal(mont, want)


def test_paper_fig12_errors(R):
    t = torch.zeros(4, dtype=torch.int32, device="cuda")
    for den, key in [(0, 3), (1 << 31, 3), (17947, 1 << 32)]:
        with pytest.raises(R.RsaError) as ei:
            R.rsa_modexp_batch_paper(t, key, den)
        assert ei.value.code == R.RSA_ERANGE


# ------------------------------------------------------------------ host entry on other classes

@pytest.mark.parametrize("key,count", [("rsa4096", 2000), ("rsa64", 300001), ("toy17947", 5)])
def test_host_entry_classes(R, key, count):
    k = workload.key(key)
    nb = k["n"].bit_length()
    s = workload.limbs_needed(nb)
    base = workload.packets(count, nb, n=k["n"], config_id=31) if nb > 20 else \
        np.arange(count, dtype=np.uint32).reshape(-1, 1) + 7
    out = R.rsa_modexp_batch_host(base, k["e"], k["n"], nb)
    idx = np.unique(np.concatenate([np.arange(min(count, 8)), np.random.default_rng(1).choice(count, min(count, 300), replace=False)]))
    assert np.array_equal(out[idx], oracle_rows(base[idx], k["e"], k["n"], s))
    one = R.rsa_modexp_batch_host(base, 0, k["n"], nb)                 # exp = 0 -> 1
    assert (one[:, 0] == 1).all() and (one[:, 1:] == 0).all()
