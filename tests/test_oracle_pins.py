"""Pins for the CPU oracle (oracle/): it is checked against what the paper and
the mathematics fix -- never against itself or the CUDA path.

P1  Fig 4 worked trace          -> tests/golden/fig4_trace.json
P2  Fig 2 key + exhaustive round trip -> tests/golden/fig2_key.json
P3  sec. 2 packetisation          -> tests/golden/sec2_packets.json
P4  sec. 2 key validity: d=137 fails, residue 267  (closed form)
P5  gcd(e, phi) = 1 and d*e = 1 mod phi for every fixture key (math.gcd, Python ints)
P6  Fermat / Euler closed forms
P7  exponent splitting identity (sec. 6)
P8  brute force on tiny inputs (pure-Python repeated multiplication)
P10 special values ((n-1)^d, 1^x, 0^x, x^1, x^0, multiplicativity)
P11 CPython pow() / pow(e, -1, phi) as an independent library routine
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
import workload

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ P1

def test_p1_fig4_naive_trace():
    g = gold("fig4_trace.json")
    res, tr = oracle.naive(g["g"], g["e"], g["m"], trace=True)
    assert tr == g["trace"]
    assert res == g["result"]


@pytest.mark.parametrize("variant,k", [("l2r", 1), ("r2l", 1), ("kary", 1), ("kary", 2), ("kary", 3),
                                       ("sliding", 1), ("sliding", 3), ("sliding", 5)])
def test_p1_fig4_all_schedules(variant, k):
    g = gold("fig4_trace.json")
    assert oracle.modexp_variant(variant, g["g"], g["e"], g["m"], k) == g["result"]


def test_p1_fig12_halving_loop():
    g = gold("fig4_trace.json")
    assert oracle.halving(g["g"], g["e"], g["m"], faithful=True) == g["result"]
    # reading Z5: Fig 12 returns base % den for e = 0
    assert oracle.halving(5, 0, 7, faithful=True) == 5
    assert oracle.halving(5, 0, 7, faithful=False) == 1
    assert oracle.modexp(5, 0, 7) == 1


@pytest.mark.parametrize("m", [1, 2, 3, 7, 497, 17947, 513581, 65537, 2**31 - 1, 2**30 + 3, 1000000006])
def test_p11_fig12_halving_every_exponent(m):
    """Fig 12 computes (g^2)^floor(e/2) * g^(e mod 2) mod m:
    pinned to CPython pow (an independent library routine) for every exponent
    0..300, both parities, bases below and above m (g % den first),
    so a wrong even-e or odd-e branch fails here, not only on the GPU."""
    rng = random.Random(m)
    bases = [0, 1, 2, m - 1, m, m + 1, rng.randrange(m), rng.randrange(2**32), 2**40 + 17]
    for g in bases:
        g = max(g, 0)
        for e in range(0, 301):
            want = pow(g, e, m)
            assert oracle.halving(g, e, m, faithful=False) == want, (g, e, m)
            # faithful mode differs only at e = 0 (reading Z5: returns g % den)
            assert oracle.halving(g, e, m, faithful=True) == (g % m if e == 0 else want), (g, e, m)


def test_p11_fig12_halving_large_exponents():
    rng = random.Random(1212)
    for _ in range(200):
        m = rng.randrange(2, 2**31)
        g = rng.randrange(2**40)
        e = rng.randrange(1, 2**20)
        assert oracle.halving(g, e, m, faithful=True) == pow(g, e, m)


# ------------------------------------------------------------------ P2

def test_p2_fig2_key():
    k = gold("fig2_key.json")
    n, phi, d = oracle.keygen_check(k["p"], k["q"], k["e"])
    assert (n, phi, d) == (k["n"], k["phi"], k["d"])


def test_p2_fig2_roundtrip_exhaustive():
    k = gold("fig2_key.json")
    for m in range(k["n"]):
        c = oracle.modexp(m, k["e"], k["n"])
        assert oracle.modexp(c, k["d"], k["n"]) == m


# ------------------------------------------------------------------ P3

def test_p3_sec2_packets():
    g = gold("sec2_packets.json")
    assert oracle.encode(g["text"]) == g["packets"]
    assert oracle.decode(g["packets"]) == g["decoded"]


@pytest.mark.parametrize("text,code", [("a", oracle.EODD), ("abc", oracle.EODD), ("aB", oracle.ECHAR),
                                       ("a1", oracle.ECHAR)])
def test_p3_codec_errors(text, code):
    with pytest.raises(oracle.OracleError) as ei:
        oracle.encode(text)
    assert ei.value.code == code


def test_p3_codec_edges():
    assert oracle.encode("ab") == [1]
    assert oracle.encode("") == []
    assert oracle.decode([0]) == "aa"
    assert oracle.decode([2525]) == "zz"
    for bad in ([2600], [26], [99]):
        with pytest.raises(oracle.OracleError) as ei:
            oracle.decode(bad)
        assert ei.value.code == oracle.EPACKET


def test_p3_codec_roundtrip_random():
    rnd = random.Random(5)
    for _ in range(200):
        s = "".join(rnd.choice("abcdefghijklmnopqrstuvwxyz") for _ in range(2 * rnd.randint(0, 20)))
        assert oracle.decode(oracle.encode(s)) == s


# ------------------------------------------------------------------ P4

def test_p4_paper_key_is_invalid():
    g = gold("sec2_packets.json")
    dv = gold("survey_derived.json")
    ok, residue = oracle.validate_key(g["e"], g["paper_d"], g["p"], g["q"])
    assert not ok and residue == dv["toy_de_mod_phi_paper_d"] == (131 * 137) % 17680
    n, phi, d = oracle.keygen_check(g["p"], g["q"], g["e"])
    assert (n, phi, d) == (g["n"], dv["toy_phi"], dv["toy_d"])
    assert (d * g["e"]) % phi == 1


def test_p4_paper_packets_encrypt_decrypt():
    g = gold("sec2_packets.json")
    dv = gold("survey_derived.json")
    c = [oracle.modexp(m, g["e"], g["n"]) for m in g["packets"]]
    assert c == dv["toy_ciphertexts"] == [pow(m, g["e"], g["n"]) for m in g["packets"]]
    back = [oracle.modexp(x, dv["toy_d"], g["n"]) for x in c]
    assert back == g["packets"]
    wrong = [oracle.modexp(x, g["paper_d"], g["n"]) for x in c]
    assert wrong == dv["toy_wrong_decrypt_with_paper_d"]
    assert wrong != g["packets"]


def test_p4_paper_d_fixed_points():
    dv = gold("survey_derived.json")
    n = 17947
    fixed = [m for m in range(n) if pow(pow(m, 131, n), 137, n) == m]
    assert fixed == dv["toy_roundtrip_fixed_points"]
    for m in fixed[:4] + fixed[-2:]:
        assert oracle.modexp(oracle.modexp(m, 131, n), 137, n) == m


def test_keygen_errors():
    assert oracle.keygen_check(131, 137, 3)[2] == gold("survey_derived.json")["keygen_131_137_e3_d"]
    cases = [((13, 13, 3), oracle.EEQUAL), ((15, 17, 3), oracle.ENOTPRIME), ((17, 11, 2), oracle.ENOTCOPRIME),
             ((17, 11, 1), oracle.ERANGE), ((17, 11, 160), oracle.ERANGE), ((17, 11, 161), oracle.ERANGE),
             ((1005, 509, 131), oracle.ENOTPRIME)]
    for (p, q, e), code in cases:
        with pytest.raises(oracle.OracleError) as ei:
            oracle.keygen_check(p, q, e)
        assert ei.value.code == code, (p, q, e)


def test_table2_key_reading_z7():
    dv = gold("survey_derived.json")
    assert not oracle.is_prime(1005) and oracle.is_prime(1009) and oracle.is_prime(509)
    n, phi, d = oracle.keygen_check(1009, 509, 131)
    assert n == dv["table2_n"] and d == dv["table2_d_e131"]


# ------------------------------------------------------------------ P5

def test_p5_fixture_keys():
    for name, k in workload.load_keys().items():
        assert k["n"] == k["p"] * k["q"], name
        assert k["phi"] == (k["p"] - 1) * (k["q"] - 1), name
        assert math.gcd(k["e"], k["phi"]) == 1, name
        assert (k["d"] * k["e"]) % k["phi"] == 1 and 0 < k["d"] < k["phi"], name
        assert k["d"] == pow(k["e"], -1, k["phi"]), name
        if name.startswith("rsa"):
            assert k["n"].bit_length() == k["nbits"]


def test_p5_primality_against_trial_division():
    for x in range(0, 5000):
        truth = x >= 2 and all(x % p for p in range(2, int(x ** 0.5) + 1))
        assert oracle.is_prime(x) == truth, x
    # Carmichael numbers and strong pseudoprimes to small bases
    for c in [561, 1105, 1729, 2465, 2821, 6601, 8911, 3215031751, 2152302898747, 3474749660383,
              341550071728321, 3825123056546413051]:
        assert not oracle.is_prime(c), c
    for p in [2**31 - 1, 2**61 - 1, 2**89 - 1, 2**107 - 1, 2**127 - 1, 2**521 - 1]:
        assert oracle.is_prime(p)
        assert not oracle.is_prime(p * (2**31 - 1))


# ------------------------------------------------------------------ P6

def test_p6_fermat_on_fixture_primes():
    rnd = random.Random(6)
    for name in ["rsa64", "rsa512", "rsa2048", "rsa4096"]:
        k = workload.key(name)
        for p in (k["p"], k["q"]):
            for _ in range(3):
                a = rnd.randrange(1, p)
                assert oracle.modexp(a, p - 1, p) == 1
                assert oracle.modexp(a, p, p) == a


def test_p6_euler_on_rsa_moduli():
    rnd = random.Random(7)
    for name in ["rsa64", "rsa256", "rsa1024"]:
        k = workload.key(name)
        n, phi = k["n"], k["phi"]
        for _ in range(4):
            a = rnd.randrange(2, n)
            if math.gcd(a, n) == 1:
                assert oracle.modexp(a, phi, n) == 1
            kk = rnd.randrange(1, 5)
            assert oracle.modexp(a, kk * phi + 1, n) == a


def test_p6_mersenne_closed_form():
    # 2^63 = 2 * 2^62 and 2^62 = 0 mod (p-1) = 2*3^2*7*11*31*151*331? use order: 7^(2^63) = 7^(2^63 mod (p-1))
    p = 2**31 - 1
    assert oracle.modexp(7, 2**63, p) == 7 ** 8 == 5764801


# ------------------------------------------------------------------ P7

def test_p7_exponent_splitting():
    rnd = random.Random(8)
    k = workload.key("rsa512")
    n = k["n"]
    for _ in range(10):
        g = rnd.randrange(n)
        e = rnd.getrandbits(300)
        x = rnd.randrange(e)
        lhs = (oracle.modexp(g, e - x, n) * oracle.modexp(g, x, n)) % n
        assert lhs == oracle.modexp(g, e, n)


# ------------------------------------------------------------------ P8

def test_p8_brute_force_tiny():
    for m in range(1, 64):
        for g in range(0, m + 3):
            c = 1 % m
            for e in range(0, 24):
                assert oracle.modexp(g, e, m) == c, (g, e, m)
                c = (c * g) % m


def test_p8_naive_vs_l2r_small_odd_moduli():
    rnd = random.Random(9)
    for _ in range(3000):
        m = rnd.randrange(1, 4096) | 1
        g = rnd.randrange(0, m)
        e = rnd.randrange(1, 256)
        assert oracle.naive(g, e, m) == oracle.modexp(g, e, m)


# ------------------------------------------------------------------ P10

def test_p10_special_values():
    rnd = random.Random(10)
    for name in ["rsa64", "rsa1024", "rsa2048"]:
        k = workload.key(name)
        n, e, d = k["n"], k["e"], k["d"]
        if d % 2:
            assert oracle.modexp(n - 1, d, n) == n - 1
        x = rnd.randrange(2, n)
        assert oracle.modexp(1, d, n) == 1
        assert oracle.modexp(0, e, n) == 0
        assert oracle.modexp(0, 0, n) == 1
        assert oracle.modexp(x, 1, n) == x
        assert oracle.modexp(x, 0, n) == 1
        a, b = rnd.randrange(n), rnd.randrange(n)
        assert (oracle.modexp(a, e, n) * oracle.modexp(b, e, n)) % n == oracle.modexp(a * b % n, e, n)


# ------------------------------------------------------------------ P11

@pytest.mark.parametrize("bits", [2, 15, 31, 32, 33, 63, 64, 65, 96, 127, 128, 255, 512, 1000, 1024, 2048, 4096])
def test_p11_cpython_pow_random(bits):
    rnd = random.Random(bits)
    n_cases = 300 if bits <= 1024 else 40
    for _ in range(n_cases):
        m = rnd.getrandbits(bits) | (1 << (bits - 1)) | rnd.getrandbits(1)
        g = rnd.getrandbits(min(bits + rnd.randrange(0, 33), 4096))
        e = rnd.getrandbits(rnd.choice([1, 2, 17, 64, min(bits, 300)]))
        assert oracle.modexp(g, e, m) == pow(g, e, m), (g, e, m)


def test_p11_structured_limbs_division():
    """Limb patterns that drive Algorithm D's q-hat correction / add-back."""
    rnd = random.Random(11)
    pats = [0, 1, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFF, 0xFFFFFFFE, 0x00010000]
    for _ in range(6000):
        nl = rnd.randrange(2, 8)
        ml = rnd.randrange(1, 6)
        g = sum(rnd.choice(pats + [rnd.getrandbits(32)]) << (32 * i) for i in range(nl))
        m = sum(rnd.choice(pats + [rnd.getrandbits(32)]) << (32 * i) for i in range(ml))
        m |= 1 << (32 * ml - rnd.randrange(1, 32))
        assert oracle.modexp(g, 1, m) == g % m
        assert oracle.modexp(g, 2, m) == (g * g) % m


def test_p11_schedules_agree():
    rnd = random.Random(12)
    for bits in (64, 300, 1024):
        for _ in range(4):
            m = rnd.getrandbits(bits) | 1 | (1 << (bits - 1))
            g, e = rnd.getrandbits(bits), rnd.getrandbits(bits)
            ref = pow(g, e, m)
            assert oracle.modexp_variant("r2l", g, e, m) == ref
            for k in (1, 2, 4, 5, 8):
                assert oracle.modexp_variant("kary", g, e, m, k) == ref
                assert oracle.modexp_variant("sliding", g, e, m, k) == ref


def test_p11_batch_matches_pow():
    k = workload.key("rsa2048")
    base = workload.packets(512, 2048, n=k["n"], config_id=2)
    out = oracle.modexp_batch(base, k["e"], k["n"], nthreads=4)
    vals = workload.rows_to_ints(base)
    got = workload.rows_to_ints(out)
    assert got == [pow(v, k["e"], k["n"]) for v in vals]
    assert out.shape == base.shape


def test_p11_batch_full_d_sample():
    k = workload.key("rsa1024")
    base = workload.packets(16, 1024, n=k["n"], config_id=3)
    out = oracle.modexp_batch(base, k["d"], k["n"], nthreads=4)
    assert workload.rows_to_ints(out) == [pow(v, k["d"], k["n"]) for v in workload.rows_to_ints(base)]


def test_workload_packets_below_n():
    for name in ["rsa64", "rsa96", "rsa1000", "rsa2048"]:
        k = workload.key(name)
        pk = workload.packets(4096, k["nbits"], n=k["n"], config_id=1)
        vals = workload.rows_to_ints(pk)
        assert all(0 <= v < k["n"] for v in vals)
        assert vals[:4] == [0, 1, 2, 3] and vals[4] == k["n"] - 1
        assert max(vals[16:]) < 2 ** (k["nbits"] - 1)
        # deterministic
        assert np.array_equal(pk, workload.packets(4096, k["nbits"], n=k["n"], config_id=1))


# ------------------------------------------------------------------ f1 oracle helpers

def test_mr_round_known_strong_pseudoprimes():
    """Strong pseudoprimes from the literature: 2047 (base 2), 1373653 (2, 3),
    25326001 (2, 3, 5), 3215031751 (2, 3, 5, 7) -- each passes exactly those
    bases and fails the next prime base."""
    table = {2047: [2], 1373653: [2, 3], 25326001: [2, 3, 5], 3215031751: [2, 3, 5, 7]}
    for n, ok in table.items():
        for a in ok:
            assert oracle.mr_round(n, a)
        nxt = {1: 3, 2: 5, 3: 7, 4: 11}[len(ok)]
        assert not oracle.mr_round(n, nxt)
    for p in [1000003, 2 ** 61 - 1, 2 ** 127 - 1]:
        assert all(oracle.mr_round(p, a) for a in (2, 3, 5, 7, 11))


def test_modexp_multi_matches_pow():
    rnd = random.Random(21)
    s = 8
    mods = [rnd.getrandbits(256) | 1 | (1 << 255) for _ in range(200)]
    base = [rnd.getrandbits(256) for _ in range(200)]
    exps = [rnd.getrandbits(rnd.choice([1, 17, 256])) for _ in range(200)]
    B, E, M = (workload.ints_to_rows(v, s) for v in (base, exps, mods))
    got = workload.rows_to_ints(oracle.modexp_multi(B, E, M))
    assert got == [pow(b, e, m) for b, e, m in zip(base, exps, mods)]


def test_candidate_generator_spec():
    """workload.prime_candidates: exactly nbits bits, top two bits and bit 0
    set, deterministic, index-addressable."""
    for nb in (64, 100, 1024):
        c = workload.rows_to_ints(workload.prime_candidates(nb, 3, 10, 20))
        assert all(v.bit_length() == nb and (v >> (nb - 2)) == 3 and v & 1 for v in c)
        assert c[5:] == workload.rows_to_ints(workload.prime_candidates(nb, 3, 15, 15))
