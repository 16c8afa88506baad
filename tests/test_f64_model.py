"""Design check of the FP64-pipe Montgomery multiply (paper_1407_1465_b200/csrc/
mont_f64.cuh) on CPU: the header's own template code, compiled for the host
(tests/tools/f64_model.cu) with the rounding mode toward zero, against the
plain definition a*b*R^-1 mod n with R = 2^(52 ND) (Python ints).  Pins the
exact hi/lo digit split, the exponent-field bias bookkeeping and the
in-place column shift before any GPU run; the GPU parity tests then pin the
kernel (tests/test_gpu_parity.py runs every class through it)."""
import os
import random
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tools", "f64_model.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nd_of(S):
    return ((32 * S + 2 + 51) // 52 + 1) // 2 * 2


@pytest.fixture(scope="module")
def model(tmp_path_factory):
    if not os.path.exists(NVCC) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("f64") / "f64_model")
    subprocess.check_call([NVCC, "-O2", "-std=c++17", *os.environ.get("F64_MODEL_FLAGS", "").split(), "-o", exe, SRC])
    p = subprocess.Popen([exe], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)

    def call(line):
        p.stdin.write(line + "\n")
        p.stdin.flush()
        return p.stdout.readline().strip()
    yield call
    p.stdin.close()
    p.wait()


def rand_modulus(rng, S, nbits=None):
    nbits = nbits or 32 * S
    n = rng.getrandbits(nbits) | (1 << (nbits - 1)) | 1
    return n


@pytest.mark.parametrize("S", [8, 16, 32, 64, 128])
def test_montmul_f64_matches_definition(model, S):
    rng = random.Random(1407 + S)
    ND = nd_of(S)
    R = 1 << (52 * ND)
    for trial in range(60):
        nbits = 32 * S if trial % 3 else rng.randint(32 * S // 2 + 1, 32 * S)
        n = rand_modulus(rng, S, nbits)
        rinv = pow(R, -1, n)
        if trial % 5 == 0:
            a, b = 2 * n - 1, 2 * n - 1             # the extreme almost-Montgomery inputs
        elif trial % 5 == 1:
            a, b = 0, rng.randrange(2 * n)
        else:
            a, b = rng.randrange(2 * n), rng.randrange(2 * n)
        for op in "MAIF":                          # registers / A parked / A living in the slot (+ fused rows)
            out = model(f"{op} {S} {n:x} {a:x} {b:x}")
            assert out != "MISMATCH", "double digits disagree with integer digits"
            r = int(out, 16)
            assert r < 2 * n, "almost-Montgomery bound r < 2n"
            assert r % n == a * b * rinv % n


@pytest.mark.parametrize("S", [16, 64])
def test_montmul_f64_raw_input_below_R(model, S):
    # RSA_OP_MULX: b is the raw packet (any value < 2^(32 S)), a < 2n
    rng = random.Random(99 + S)
    ND = nd_of(S)
    R = 1 << (52 * ND)
    for _ in range(30):
        n = rand_modulus(rng, S)
        a, b = rng.randrange(2 * n), rng.getrandbits(32 * S)
        r = int(model(f"M {S} {n:x} {a:x} {b:x}"), 16)
        assert r < 2 * n and r % n == a * b * pow(R, -1, n) % n


@pytest.mark.parametrize("S", [16, 64])
def test_canonicalise(model, S):
    rng = random.Random(5 + S)
    for k in range(40):
        n = rand_modulus(rng, S)
        r = [0, n - 1, n, n + 1, 2 * n - 1][k % 5] if k < 10 else rng.randrange(2 * n)
        assert int(model(f"C {S} {n:x} {r:x}"), 16) == r % n


@pytest.mark.parametrize("S", [8, 64])
def test_limb_digit_round_trip(model, S):
    rng = random.Random(3 * S)
    for k in range(40):
        x = [0, (1 << (32 * S)) - 1, 1 << (32 * S - 1)][k] if k < 3 else rng.getrandbits(32 * S)
        assert int(model(f"L {S} {x:x}"), 16) == x


@pytest.mark.parametrize("S,op", [(8, "S"), (16, "S"), (32, "S"), (64, "S"), (8, "Q"), (32, "Q"), (64, "Q"),
                                  (128, "Q")])
def test_montsqr_f64_matches_definition(model, S, op):
    """montsqr (A in registers, T in a 2 ND slot) and montsqr_slot (A living in
    one ND-digit slot, T_high parked in A's dead registers: the 4096-bit
    kernel's squaring) against a^2 R^-1 mod n."""
    rng = random.Random(2024 + S)
    ND = nd_of(S)
    R = 1 << (52 * ND)
    for trial in range(60):
        nbits = 32 * S if trial % 3 else rng.randint(32 * S // 2 + 1, 32 * S)
        n = rand_modulus(rng, S, nbits)
        a = [2 * n - 1, 0, 1, n - 1, n][trial] if trial < 5 else rng.randrange(2 * n)
        out = model(f"{op} {S} {n:x} {a:x} {a:x}")
        assert out != "MISMATCH"
        r = int(out, 16)
        assert r < 2 * n, "almost-Montgomery bound r < 2n"
        assert r % n == a * a * pow(R, -1, n) % n


@pytest.mark.parametrize("nd", [20, 40, 80])
def test_normalize_carry_lookahead(model, nd):
    """normalize(): columns < 2^62 -> 52-bit digits of the same number (mod 2^(52 nd)),
    incl. carries rippling through runs of all-ones digits and across the 64-column
    mask word boundary (nd = 80)."""
    rng = random.Random(nd)
    M = (1 << 52) - 1
    cases = [[0] * nd, [M] * nd, [M + 1] + [M] * (nd - 1), [(1 << 62) - 1] * nd]
    for start in (0, 5, 62, 63, 64):
        if start < nd:
            c = [M] * nd
            c[start] = M + 1                      # generate at `start`, then propagate to the top
            cases.append(c)
    for _ in range(40):
        cases.append([rng.choice([rng.getrandbits(62), M, M + 1, rng.getrandbits(52), 0]) for _ in range(nd)])
    for cols in cases:
        want = sum(v << (52 * k) for k, v in enumerate(cols)) % (1 << (52 * nd))
        got = int(model("Z %d %s" % (nd, " ".join("%x" % v for v in cols))), 16)
        assert got == want
