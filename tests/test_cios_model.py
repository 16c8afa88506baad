"""Design check of the kernel's carry scheme (paper_1407_1465_b200/csrc/mont.cuh)
on CPU: a bit-exact Python model of cios_step/montmul -- register arrays X, Y,
`hi`, the PTX carry flag -- compared with the plain definition
a*b*R^-1 mod n (Python ints).  This pins the even/odd + pre-shift fold
bookkeeping before any GPU run; the GPU parity tests then pin the kernel."""
import random

import pytest

M32 = 0xFFFFFFFF


class CC:
    """PTX carry flag semantics for add.cc/addc/mad*.cc."""
    def __init__(self):
        self.c = 0

    def add_cc(self, a, b, cin=0):
        s = a + b + cin
        self.c = s >> 32
        return s & M32

    def mad_lo_cc(self, a, b, c, cin=0):
        return self.add_cc((a * b) & M32, c, cin)

    def mad_hi_cc(self, a, b, c, cin=0):
        return self.add_cc((a * b) >> 32, c, cin)


def cios_step(X, Y, hi, a, b, n, n0inv):
    S = len(a)
    cc = CC()
    X[0] = cc.add_cc(X[0], Y[1])
    for j in range(1, S - 2, 2):
        c = cc.c; Y[j - 1] = cc.mad_lo_cc(a[j], b, Y[j + 1], c)
        c = cc.c; Y[j] = cc.mad_hi_cc(a[j], b, Y[j + 2], c)
    c = cc.c; Y[S - 2] = cc.mad_lo_cc(a[S - 1], b, 0, c)
    c = cc.c; Y[S - 1] = cc.mad_hi_cc(a[S - 1], b, hi, c)
    hi = cc.c
    X[0] = cc.mad_lo_cc(a[0], b, X[0])
    c = cc.c; X[1] = cc.mad_hi_cc(a[0], b, X[1], c)
    for j in range(2, S, 2):
        c = cc.c; X[j] = cc.mad_lo_cc(a[j], b, X[j], c)
        c = cc.c; X[j + 1] = cc.mad_hi_cc(a[j], b, X[j + 1], c)
    c = cc.c; Y[S - 1] = cc.add_cc(Y[S - 1], 0, c)
    hi = hi + cc.c
    m = (X[0] * n0inv) & M32
    Y[0] = cc.mad_lo_cc(n[1], m, Y[0])
    c = cc.c; Y[1] = cc.mad_hi_cc(n[1], m, Y[1], c)
    for j in range(3, S, 2):
        c = cc.c; Y[j - 1] = cc.mad_lo_cc(n[j], m, Y[j - 1], c)
        c = cc.c; Y[j] = cc.mad_hi_cc(n[j], m, Y[j], c)
    hi = hi + cc.c
    X[0] = cc.mad_lo_cc(n[0], m, X[0])
    assert X[0] == 0
    c = cc.c; X[1] = cc.mad_hi_cc(n[0], m, X[1], c)
    for j in range(2, S, 2):
        c = cc.c; X[j] = cc.mad_lo_cc(n[j], m, X[j], c)
        c = cc.c; X[j + 1] = cc.mad_hi_cc(n[j], m, X[j + 1], c)
    c = cc.c; Y[S - 1] = cc.add_cc(Y[S - 1], 0, c)
    hi = hi + cc.c
    assert hi < 2**32
    return hi


def montmul_model(a, b, n, S):
    n0inv = (-pow(n[0], -1, 2**32)) % 2**32
    X, Y, hi = [0] * S, [0] * S, 0
    for i in range(S):
        if i % 2 == 0:
            hi = cios_step(X, Y, hi, a, b[i], n, n0inv)
        else:
            hi = cios_step(Y, X, hi, a, b[i], n, n0inv)
    cc = CC()
    X[0] = cc.add_cc(X[0], Y[1])
    for k in range(1, S - 1):
        c = cc.c; X[k] = cc.add_cc(X[k], Y[k + 1], c)
    c = cc.c; X[S - 1] = cc.add_cc(X[S - 1], 0, c)
    hi = hi + cc.c
    r = sum(v << (32 * k) for k, v in enumerate(X)) + (hi << (32 * S))
    N = sum(v << (32 * k) for k, v in enumerate(n))
    return r - N if r >= N else r


def L(x, S):
    return [(x >> (32 * k)) & M32 for k in range(S)]


@pytest.mark.parametrize("S", [2, 4, 8, 16])
def test_cios_model_random(S):
    rnd = random.Random(S)
    R = 1 << (32 * S)
    for _ in range(300):
        N = rnd.getrandbits(32 * S) | 1 | (rnd.choice([1, 0]) << (32 * S - 1))
        if N < 3:
            continue
        A = rnd.randrange(R)                  # a < R (to-Montgomery case)
        B = rnd.randrange(N)
        got = montmul_model(L(A, S), L(B, S), L(N, S), S)
        assert got == (A * B * pow(R, -1, N)) % N


@pytest.mark.parametrize("S", [2, 4, 8])
def test_cios_model_extremes(S):
    R = 1 << (32 * S)
    for N in [R - 1, R - 3, (R >> 1) + 1, 3, 0xFFFFFFFF, (R >> 1) | 1]:
        for A in [0, 1, N - 1, R - 1, N // 2]:
            for B in [0, 1, N - 1, N // 2]:
                got = montmul_model(L(A, S), L(B, S), L(N, S), S)
                assert got == (A * B * pow(R, -1, N)) % N, (N, A, B)


# ---------------------------------------------------------------- lane-pair (S = 2L) scheme

def cios_step_pair(st, a, b, n, n0inv, L):
    """Both lanes run cios_step on their halves; lane 0's m is broadcast; lane
    1's dropped low word moves to lane 0's top (mont_pair.cuh)."""
    # products on each lane; m from lane 0
    X0, Y0, h0 = st[0]
    X1, Y1, h1 = st[1]
    out = []
    ms = []
    for lane in (0, 1):
        X, Y, hi = st[lane]
        cc = CC()
        X[0] = cc.add_cc(X[0], Y[1])
        for j in range(1, L - 2, 2):
            c = cc.c; Y[j - 1] = cc.mad_lo_cc(a[lane][j], b, Y[j + 1], c)
            c = cc.c; Y[j] = cc.mad_hi_cc(a[lane][j], b, Y[j + 2], c)
        c = cc.c; Y[L - 2] = cc.mad_lo_cc(a[lane][L - 1], b, 0, c)
        c = cc.c; Y[L - 1] = cc.mad_hi_cc(a[lane][L - 1], b, hi, c)
        hi = cc.c
        X[0] = cc.mad_lo_cc(a[lane][0], b, X[0])
        c = cc.c; X[1] = cc.mad_hi_cc(a[lane][0], b, X[1], c)
        for j in range(2, L, 2):
            c = cc.c; X[j] = cc.mad_lo_cc(a[lane][j], b, X[j], c)
            c = cc.c; X[j + 1] = cc.mad_hi_cc(a[lane][j], b, X[j + 1], c)
        c = cc.c; Y[L - 1] = cc.add_cc(Y[L - 1], 0, c)
        hi = hi + cc.c
        st[lane] = (X, Y, hi)
        ms.append((X[0] * n0inv) & M32)
    m = ms[0]
    for lane in (0, 1):
        X, Y, hi = st[lane]
        nn = n[lane]
        cc = CC()
        Y[0] = cc.mad_lo_cc(nn[1], m, Y[0])
        c = cc.c; Y[1] = cc.mad_hi_cc(nn[1], m, Y[1], c)
        for j in range(3, L, 2):
            c = cc.c; Y[j - 1] = cc.mad_lo_cc(nn[j], m, Y[j - 1], c)
            c = cc.c; Y[j] = cc.mad_hi_cc(nn[j], m, Y[j], c)
        hi = hi + cc.c
        X[0] = cc.mad_lo_cc(nn[0], m, X[0])
        c = cc.c; X[1] = cc.mad_hi_cc(nn[0], m, X[1], c)
        for j in range(2, L, 2):
            c = cc.c; X[j] = cc.mad_lo_cc(nn[j], m, X[j], c)
            c = cc.c; X[j + 1] = cc.mad_hi_cc(nn[j], m, X[j + 1], c)
        c = cc.c; Y[L - 1] = cc.add_cc(Y[L - 1], 0, c)
        hi = hi + cc.c
        st[lane] = (X, Y, hi)
    assert st[0][0][0] == 0
    w = [st[1][0][0], st[0][0][0]]          # shfl_xor(X[0], 1)
    for lane in (0, 1):
        X, Y, hi = st[lane]
        cc = CC()
        Y[L - 1] = cc.add_cc(Y[L - 1], w[lane])  # new even array's top, carry -> hi
        hi = hi + cc.c
        assert hi < 2**32
        st[lane] = (Y, X, hi)                  # role swap


def montmul_pair_model(A, B, N, L):
    S = 2 * L
    n0inv = (-pow(N & M32, -1, 2**32)) % 2**32
    a = [L_(A, 0, L), L_(A, L, L)]
    n = [L_(N, 0, L), L_(N, L, L)]
    st = [([0] * L, [0] * L, 0), ([0] * L, [0] * L, 0)]
    for i in range(S):
        cios_step_pair(st, a, (B >> (32 * i)) & M32, n, n0inv, L)
    vals = []
    for lane in (0, 1):
        X, Y, hi = st[lane]
        r = X[0] + Y[1] + sum((X[k] + Y[k + 1]) << (32 * k) for k in range(1, L - 1)) \
            + (X[L - 1] << (32 * (L - 1))) + (hi << (32 * L))
        vals.append(r)
    T = vals[0] + (vals[1] << (32 * L))
    return T - N if T >= N else T


def L_(x, off, L):
    return [(x >> (32 * (off + k))) & M32 for k in range(L)]


@pytest.mark.parametrize("L", [2, 4, 8])
def test_cios_pair_model(L):
    rnd = random.Random(100 + L)
    S = 2 * L
    R = 1 << (32 * S)
    cases = [(R - 1, R - 1, R - 2), (R - 3, R - 4, 1)]
    for _ in range(200):
        N = rnd.getrandbits(32 * S) | 1 | (rnd.choice([1, 0]) << (32 * S - 1))
        cases.append((N, rnd.randrange(R), rnd.randrange(N)))
    for N, A, B in cases:
        if N < 3:
            continue
        B %= N
        got = montmul_pair_model(A, B, N, L)
        assert got == (A * B * pow(R, -1, N)) % N


# ---------------------------------------------------------------- squaring (mont_sqr.cuh)

def red_step(X, Y, hi, n, n0inv):
    S = len(X)
    cc = CC()
    X[0] = cc.add_cc(X[0], Y[1])
    m = (X[0] * n0inv) & M32
    for j in range(1, S - 2, 2):
        c = cc.c; Y[j - 1] = cc.mad_lo_cc(n[j], m, Y[j + 1], c)
        c = cc.c; Y[j] = cc.mad_hi_cc(n[j], m, Y[j + 2], c)
    c = cc.c; Y[S - 2] = cc.mad_lo_cc(n[S - 1], m, 0, c)
    c = cc.c; Y[S - 1] = cc.mad_hi_cc(n[S - 1], m, hi, c)
    hi = cc.c
    X[0] = cc.mad_lo_cc(n[0], m, X[0])
    assert X[0] == 0
    c = cc.c; X[1] = cc.mad_hi_cc(n[0], m, X[1], c)
    for j in range(2, S, 2):
        c = cc.c; X[j] = cc.mad_lo_cc(n[j], m, X[j], c)
        c = cc.c; X[j + 1] = cc.mad_hi_cc(n[j], m, X[j + 1], c)
    c = cc.c; Y[S - 1] = cc.add_cc(Y[S - 1], 0, c)
    hi = hi + cc.c
    return hi


def montsqr_model(a, n, S):
    n0inv = (-pow(n[0], -1, 2**32)) % 2**32
    # phase 1: triangle by product scanning, two accumulators per column
    T = [0] * (2 * S)
    c0 = c1 = c2 = 0
    for k in range(1, 2 * S - 2):
        lo, hi_ = max(0, k - S + 1), (k - 1) // 2
        d0 = d1 = d2 = 0
        for i in range(lo, hi_ + 1):
            p = a[i] * a[k - i]
            if (i - lo) % 2 == 0:
                s = c0 + (c1 << 32) + p
                c0, c1 = s & M32, (s >> 32) & M32
                c2 += s >> 64
            else:
                s = d0 + (d1 << 32) + p
                d0, d1 = s & M32, (s >> 32) & M32
                d2 += s >> 64
        cc = CC()
        c0 = cc.add_cc(c0, d0)
        c = cc.c; c1 = cc.add_cc(c1, d1, c)
        c2 = (c2 + d2 + cc.c) & M32
        T[k] = c0
        c0, c1, c2 = c1, c2, 0
    T[2 * S - 2] = c0
    T[2 * S - 1] = c1
    # phase 2: double;  phase 3: + diagonal
    cc = CC()
    T[0] = cc.add_cc(T[0], T[0])
    for k in range(1, 2 * S):
        c = cc.c; T[k] = cc.add_cc(T[k], T[k], c)
    assert cc.c == 0
    cc = CC()
    for i in range(S):
        c = cc.c if i else 0
        T[2 * i] = cc.mad_lo_cc(a[i], a[i], T[2 * i], c)
        c = cc.c; T[2 * i + 1] = cc.mad_hi_cc(a[i], a[i], T[2 * i + 1], c)
    assert cc.c == 0
    A = sum(v << (32 * k) for k, v in enumerate(a))
    assert sum(v << (32 * k) for k, v in enumerate(T)) == A * A
    # phase 4: reduce T_low
    X, Y, hi = T[:S], [0] * S, 0
    for i in range(S):
        hi = red_step(X, Y, hi, n, n0inv) if i % 2 == 0 else red_step(Y, X, hi, n, n0inv)
    cc = CC()
    X[0] = cc.add_cc(X[0], Y[1])
    for k in range(1, S - 1):
        c = cc.c; X[k] = cc.add_cc(X[k], Y[k + 1], c)
    c = cc.c; X[S - 1] = cc.add_cc(X[S - 1], 0, c)
    hi = hi + cc.c
    # + T_high
    cc = CC()
    for k in range(S):
        c = cc.c if k else 0
        X[k] = cc.add_cc(X[k], T[S + k], c)
    hi = hi + cc.c
    r = sum(v << (32 * k) for k, v in enumerate(X)) + (hi << (32 * S))
    N = sum(v << (32 * k) for k, v in enumerate(n))
    assert r < 2 * N
    return r - N if r >= N else r


@pytest.mark.parametrize("S", [2, 4, 8, 16])
def test_montsqr_model(S):
    rnd = random.Random(200 + S)
    R = 1 << (32 * S)
    cases = []
    for N in [R - 1, R - 3, (R >> 1) | 1]:
        cases += [(N, N - 1), (N, 0), (N, 1), (N, N // 2)]
    for _ in range(200):
        N = rnd.getrandbits(32 * S) | 1 | (rnd.choice([1, 0]) << (32 * S - 1))
        if N >= 3:
            cases.append((N, rnd.randrange(N)))
    for N, A in cases:
        got = montsqr_model(L(A, S), L(N, S), S)
        assert got == (A * A * pow(R, -1, N)) % N


# ---------------------------------------------------------------- v2 squaring: fused doubling + diagonal

def square_fused_columns(a, S):
    """Column loop of mont_v2.cuh: per column, fresh off-diagonal accumulators
    (two interleaved), doubled, + diagonal, + the running 2-word carry."""
    T = [0] * (2 * S)
    r0 = r1 = 0
    for k in range(2 * S):
        lo, top = max(0, k - S + 1), (k - 1) // 2
        c = [0, 0, 0]
        d = [0, 0, 0]
        for i in range(lo, top + 1):
            acc = c if (i - lo) % 2 == 0 else d
            v = acc[0] + (acc[1] << 32) + (acc[2] << 64) + a[i] * a[k - i]
            acc[0], acc[1], acc[2] = v & M32, (v >> 32) & M32, v >> 64
        v = c[0] + (c[1] << 32) + (c[2] << 64) + d[0] + (d[1] << 32) + (d[2] << 64)
        v = 2 * v
        if k % 2 == 0 and k // 2 < S:
            v += a[k // 2] * a[k // 2]
        v += r0 + (r1 << 32)
        assert v < 1 << 96
        T[k] = v & M32
        r0, r1 = (v >> 32) & M32, v >> 64
        assert r1 < 2**32
    assert r0 == 0 and r1 == 0
    return T


@pytest.mark.parametrize("S", [2, 4, 8, 64])
def test_square_fused_columns(S):
    rnd = random.Random(300 + S)
    for A in [0, 1, (1 << (32 * S)) - 1] + [rnd.getrandbits(32 * S) for _ in range(50)]:
        T = square_fused_columns(L(A, S), S)
        assert sum(v << (32 * k) for k, v in enumerate(T)) == A * A


# ---------------------------------------------------------------------------
# montmul2_ps (mont.cuh): the S = 2 product-scanning Montgomery multiply used by
# the small-width kernel, modelled instruction by instruction (mad.lo.cc takes
# no carry in, madc.* / addc do).

def montmul2_ps_model(a, b, n):
    a0, a1 = a & M32, a >> 32
    b0, b1 = b & M32, b >> 32
    n0, n1 = n & M32, n >> 32
    n0inv = (-pow(n0, -1, 2**32)) % 2**32
    cc = CC()
    p = a0 * b0
    c0, c1 = p & M32, p >> 32
    m0 = (c0 * n0inv) & M32
    c0 = cc.mad_lo_cc(m0, n0, c0)
    assert c0 == 0
    c = cc.c; c1 = cc.mad_hi_cc(m0, n0, c1, c)
    c2 = cc.c
    # column 1
    c1 = cc.mad_lo_cc(a0, b1, c1)
    c = cc.c; c2 = cc.mad_hi_cc(a0, b1, c2, c)
    c3 = cc.c
    c1 = cc.mad_lo_cc(a1, b0, c1)
    c = cc.c; c2 = cc.mad_hi_cc(a1, b0, c2, c)
    c3 = c3 + cc.c
    c1 = cc.mad_lo_cc(m0, n1, c1)
    c = cc.c; c2 = cc.mad_hi_cc(m0, n1, c2, c)
    c3 = c3 + cc.c
    m1 = (c1 * n0inv) & M32
    c1 = cc.mad_lo_cc(m1, n0, c1)
    assert c1 == 0
    c = cc.c; c2 = cc.mad_hi_cc(m1, n0, c2, c)
    c3 = c3 + cc.c
    assert c3 < 2**32
    # column 2
    c2 = cc.mad_lo_cc(a1, b1, c2)
    c = cc.c; c3 = cc.mad_hi_cc(a1, b1, c3, c)
    c4 = cc.c
    c2 = cc.mad_lo_cc(m1, n1, c2)
    c = cc.c; c3 = cc.mad_hi_cc(m1, n1, c3, c)
    c4 = c4 + cc.c
    assert c4 <= 1
    # conditional subtraction: borrow chain, keep = c4 - borrow
    d = (c3 << 32 | c2) - n
    borrow = 1 if d < 0 else 0
    keep = (c4 - borrow) & M32
    return (c3 << 32 | c2) if keep else d & (2**64 - 1)


def test_montmul2_ps_model():
    rng = random.Random(14071465)
    R = 2**64
    mods = [3, 17947, 513581, 2**32 - 5, 2**32 + 15, 2**63 + 29, 2**64 - 59, 2**64 - 1]
    mods += [rng.randrange(3, 2**64) | 1 for _ in range(200)]
    for n in mods:
        rinv = pow(R, -1, n)
        cases = [(R - 1, n - 1), (0, n - 1), (R - 1, 0), (1, 1), (n - 1, n - 1)]
        cases += [(rng.randrange(R), rng.randrange(n)) for _ in range(50)]
        for a, b in cases:
            assert montmul2_ps_model(a, b, n) == a * b * rinv % n, (a, b, n)
