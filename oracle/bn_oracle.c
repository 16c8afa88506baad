/*
 * oracle/bn_oracle.c -- CPU ORACLE for batched RSA modular exponentiation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1407_1465_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the product.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arXiv 1407.1465):
 *   out = g^e mod m, the unique value in [0, m)   (sec. 2;
 *   PAPER.md:65, sec. 3.3).  The method reaches exactly this value, so the
 *   oracle is that definition written out with textbook steps:
 *     - multi-precision numbers: little-endian arrays of 32-bit limbs;
 *     - multiply: schoolbook, O(s^2) with 64-bit partial products;
 *     - reduce: Knuth TAOCP vol.2 sec. 4.3.1 Algorithm D (long division),
 *       i.e. the "(u * v) mod m" of Fig 3;
 *     - exponentiate: left-to-right binary square-and-multiply exactly as
 *       Fig 5.
 *   Alternates, used only to cross-check the oracle against itself and the
 *   paper's worked example: naive repeated multiplication with trace
 *   (Fig 4), right-to-left binary (Fig 5),
 *   left-to-right k-ary (Fig 6), sliding window (Fig 7,
 *   PAPER.md:169-180), and the paper's own halving loop (Fig 12,
 *   PAPER.md:374-406) for single-word moduli.
 *   Key generation check (Fig 1): n = p*q, phi = (p-1)(q-1),
 *   1 < e < phi, gcd(e, phi) = 1, d = e^-1 mod phi with 0 < d < phi.
 *   Packet codec (sec. 2): a=00 .. z=25, two letters per
 *   packet, packet = hi*100 + lo.
 *
 * Parallelism: a plain pthread pool over packets (the harness splits the
 * batch; the per-packet algorithm is unchanged).
 *
 * Parity pins (tests/test_oracle_pins.py): Fig 4 trace, Fig 2 key, sec. 2
 * packets, closed forms (Fermat/Euler), brute force on tiny inputs, CPython
 * pow() as an independent library routine.  Nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Max limbs of any intermediate: 4096-bit modulus (128 limbs) squared is 256
 * limbs; keygen of two 64-limb primes gives a 128-limb n.  Headroom added. */
#define BN_MAX 264

typedef struct {
    int len;                 /* number of significant limbs (0 for zero) */
    uint32_t d[BN_MAX];      /* little-endian limbs */
} bn_t;

/* status codes -- the values are fixed by the C-ABI contract in DESIGN.md
 * (SURVEY.md sec. 8(b)); the oracle defines its own copy. */
enum {
    OR_OK = 0,
    OR_EINVAL = -1,
    OR_ERANGE = -2,
    OR_EEVEN = -3,
    OR_ENOTPRIME = -4,
    OR_EEQUAL = -5,
    OR_ENOTCOPRIME = -6,
    OR_ECHAR = -7,
    OR_EODD = -8,
    OR_ENOSPC = -9,
    OR_EPACKET = -10,
    OR_EBADKEY = -11,
};

/* ------------------------------------------------------------------ */
/* basic representation                                                 */
/* ------------------------------------------------------------------ */

static void bn_norm(bn_t *a)
{
    while (a->len > 0 && a->d[a->len - 1] == 0)
        a->len--;
}

static void bn_zero(bn_t *a) { a->len = 0; }

static void bn_set_u32(bn_t *a, uint32_t v)
{
    a->d[0] = v;
    a->len = 1;
    bn_norm(a);
}

static void bn_set_u64(bn_t *a, uint64_t v)
{
    a->d[0] = (uint32_t)v;
    a->d[1] = (uint32_t)(v >> 32);
    a->len = 2;
    bn_norm(a);
}

static void bn_from_limbs(bn_t *a, const uint32_t *limbs, int n)
{
    int i;
    for (i = 0; i < n; i++)
        a->d[i] = limbs[i];
    a->len = n;
    bn_norm(a);
}

static void bn_to_limbs(uint32_t *limbs, int n, const bn_t *a)
{
    int i;
    for (i = 0; i < n; i++)
        limbs[i] = (i < a->len) ? a->d[i] : 0u;
}

static void bn_copy(bn_t *r, const bn_t *a)
{
    int i;
    for (i = 0; i < a->len; i++)
        r->d[i] = a->d[i];
    r->len = a->len;
}

static int bn_is_zero(const bn_t *a) { return a->len == 0; }

static uint64_t bn_to_u64(const bn_t *a)
{
    uint64_t v = 0;
    if (a->len > 0)
        v = a->d[0];
    if (a->len > 1)
        v |= (uint64_t)a->d[1] << 32;
    return v;
}

static int bn_is_one(const bn_t *a) { return a->len == 1 && a->d[0] == 1; }

static int bn_cmp(const bn_t *a, const bn_t *b)
{
    int i;
    if (a->len != b->len)
        return a->len < b->len ? -1 : 1;
    for (i = a->len - 1; i >= 0; i--)
        if (a->d[i] != b->d[i])
            return a->d[i] < b->d[i] ? -1 : 1;
    return 0;
}

static int bn_bitlen(const bn_t *a)
{
    uint32_t top;
    int bits;
    if (a->len == 0)
        return 0;
    top = a->d[a->len - 1];
    bits = 0;
    while (top) {
        bits++;
        top >>= 1;
    }
    return 32 * (a->len - 1) + bits;
}

static int bn_bit(const bn_t *a, int i)
{
    int w = i / 32;
    if (w >= a->len)
        return 0;
    return (a->d[w] >> (i % 32)) & 1u;
}

/* ------------------------------------------------------------------ */
/* add / sub / mul                                                       */
/* ------------------------------------------------------------------ */

/* r = a + b (r may alias a or b) */
static void bn_add(bn_t *r, const bn_t *a, const bn_t *b)
{
    int n = a->len > b->len ? a->len : b->len;
    uint64_t carry = 0;
    int i;
    for (i = 0; i < n; i++) {
        uint64_t s = carry;
        if (i < a->len)
            s += a->d[i];
        if (i < b->len)
            s += b->d[i];
        r->d[i] = (uint32_t)s;
        carry = s >> 32;
    }
    r->d[n] = (uint32_t)carry;
    r->len = n + 1;
    bn_norm(r);
}

/* r = a - b, requires a >= b (r may alias a or b) */
static void bn_sub(bn_t *r, const bn_t *a, const bn_t *b)
{
    int64_t borrow = 0;
    int i;
    for (i = 0; i < a->len; i++) {
        int64_t s = (int64_t)a->d[i] - borrow - (i < b->len ? (int64_t)b->d[i] : 0);
        if (s < 0) {
            s += ((int64_t)1 << 32);
            borrow = 1;
        } else {
            borrow = 0;
        }
        r->d[i] = (uint32_t)s;
    }
    r->len = a->len;
    bn_norm(r);
}

/* r = a * b, schoolbook.  r must not alias a or b. */
static void bn_mul(bn_t *r, const bn_t *a, const bn_t *b)
{
    int i, j;
    if (a->len == 0 || b->len == 0) {
        bn_zero(r);
        return;
    }
    for (i = 0; i < a->len + b->len; i++)
        r->d[i] = 0;
    for (i = 0; i < a->len; i++) {
        uint64_t carry = 0;
        for (j = 0; j < b->len; j++) {
            uint64_t t = (uint64_t)a->d[i] * b->d[j] + r->d[i + j] + carry;
            r->d[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        r->d[i + b->len] = (uint32_t)carry;
    }
    r->len = a->len + b->len;
    bn_norm(r);
}

/* ------------------------------------------------------------------ */
/* long division: Knuth TAOCP 4.3.1 Algorithm D                          */
/* ------------------------------------------------------------------ */

static int nlz32(uint32_t x)
{
    int n = 0;
    if (x == 0)
        return 32;
    while (!(x & 0x80000000u)) {
        n++;
        x <<= 1;
    }
    return n;
}

/* q = u / v, r = u mod v.  v != 0.  q or r may be NULL.  q, r must not
 * alias u or v. */
static void bn_divmod(bn_t *q, bn_t *r, const bn_t *u, const bn_t *v)
{
    const uint64_t b = (uint64_t)1 << 32;
    int m, n, j, i, sh;
    uint32_t un[BN_MAX + 1], vn[BN_MAX];
    bn_t qq;

    n = v->len;
    m = u->len - n;
    if (bn_cmp(u, v) < 0) {
        /* quotient 0, remainder u */
        if (q)
            bn_zero(q);
        if (r)
            bn_copy(r, u);
        return;
    }
    if (n == 1) {
        /* short division by a single limb */
        uint64_t rem = 0;
        for (j = u->len - 1; j >= 0; j--) {
            uint64_t cur = (rem << 32) | u->d[j];
            qq.d[j] = (uint32_t)(cur / v->d[0]);
            rem = cur % v->d[0];
        }
        qq.len = u->len;
        bn_norm(&qq);
        if (q)
            bn_copy(q, &qq);
        if (r)
            bn_set_u32(r, (uint32_t)rem);
        return;
    }

    /* D1. normalise: shift so the divisor's top bit is set */
    sh = nlz32(v->d[n - 1]);
    for (i = n - 1; i > 0; i--)
        vn[i] = (v->d[i] << sh) | (sh ? (uint32_t)((uint64_t)v->d[i - 1] >> (32 - sh)) : 0u);
    vn[0] = v->d[0] << sh;
    un[m + n] = sh ? (uint32_t)((uint64_t)u->d[m + n - 1] >> (32 - sh)) : 0u;
    for (i = m + n - 1; i > 0; i--)
        un[i] = (u->d[i] << sh) | (sh ? (uint32_t)((uint64_t)u->d[i - 1] >> (32 - sh)) : 0u);
    un[0] = u->d[0] << sh;

    /* D2..D7. main loop over quotient digits, most significant first */
    for (j = m; j >= 0; j--) {
        uint64_t num = ((uint64_t)un[j + n] << 32) | un[j + n - 1];
        uint64_t qhat = num / vn[n - 1];
        uint64_t rhat = num % vn[n - 1];
        int64_t t, borrow;

        /* D3. test qhat: correct an estimate that is at most 2 too big */
        while (qhat >= b || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
            qhat--;
            rhat += vn[n - 1];
            if (rhat >= b)
                break;
        }

        /* D4. multiply and subtract qhat * vn from un[j .. j+n] */
        borrow = 0;
        for (i = 0; i < n; i++) {
            uint64_t p = qhat * vn[i];
            t = (int64_t)un[i + j] - borrow - (int64_t)(p & 0xFFFFFFFFu);
            un[i + j] = (uint32_t)t;
            borrow = (int64_t)(p >> 32) - (t >> 32);
        }
        t = (int64_t)un[j + n] - borrow;
        un[j + n] = (uint32_t)t;

        /* D5/D6. if the result went negative, add back once */
        qq.d[j] = (uint32_t)qhat;
        if (t < 0) {
            uint64_t carry = 0;
            qq.d[j]--;
            for (i = 0; i < n; i++) {
                uint64_t s = (uint64_t)un[i + j] + vn[i] + carry;
                un[i + j] = (uint32_t)s;
                carry = s >> 32;
            }
            un[j + n] = (uint32_t)((uint64_t)un[j + n] + carry);
        }
    }
    qq.len = m + 1;
    bn_norm(&qq);
    if (q)
        bn_copy(q, &qq);

    /* D8. unnormalise the remainder */
    if (r) {
        for (i = 0; i < n - 1; i++)
            r->d[i] = (un[i] >> sh) | (sh ? (uint32_t)((uint64_t)un[i + 1] << (32 - sh)) : 0u);
        r->d[n - 1] = un[n - 1] >> sh;
        r->len = n;
        bn_norm(r);
    }
}

/* r = a mod m (r may alias a) */
static void bn_mod(bn_t *r, const bn_t *a, const bn_t *m)
{
    bn_t t;
    bn_divmod(NULL, &t, a, m);
    bn_copy(r, &t);
}

/* r = (a * b) mod m  -- Fig 3, third identity */
static void bn_mulmod(bn_t *r, const bn_t *a, const bn_t *b, const bn_t *m)
{
    bn_t p;
    bn_mul(&p, a, b);
    bn_mod(r, &p, m);
}

/* ------------------------------------------------------------------ */
/* modular exponentiation                                                */
/* ------------------------------------------------------------------ */

/* THE ORACLE.  Left-to-right binary modular exponentiation, Fig 5
 * (PAPER.md:139-152):
 *   1. A = 1.
 *   2. For i from t down to 0: 2.1 A = (A*A) mod m; 2.2 if e_i = 1, A = (A*g) mod m.
 *   3. Return A.
 * The final "mod m" covers e = 0 and m = 1 (A = 1 is returned as 1 mod m). */
static void bn_modexp_l2r(bn_t *A, const bn_t *g, const bn_t *e, const bn_t *m)
{
    bn_t T;
    int i, t = bn_bitlen(e) - 1;
    bn_set_u32(A, 1);
    for (i = t; i >= 0; i--) {
        bn_mulmod(&T, A, A, m);              /* 2.1 */
        if (bn_bit(e, i))
            bn_mulmod(A, &T, g, m);          /* 2.2 */
        else
            bn_copy(A, &T);
    }
    bn_mod(A, A, m);
}

/* Right-to-left binary, Fig 5:
 *   1. A = 1; S = g; E = e.
 *   2. while E != 0: 2.1 if E odd: A = A*S mod m, E = E-1; 2.2 E = E/2;
 *      2.3 if E != 0: S = S*S mod m.
 *   3. return A. */
static void bn_modexp_r2l(bn_t *A, const bn_t *g, const bn_t *e, const bn_t *m)
{
    bn_t S, T;
    int i, nb = bn_bitlen(e);
    bn_set_u32(A, 1);
    bn_copy(&S, g);
    /* walking the bits of e from bit 0 upwards is exactly steps 2.1-2.3:
     * "E odd" is bit i, "E = (E - e_i)/2" moves to bit i+1, and "E != 0"
     * holds while a higher set bit remains (i < nb - 1). */
    for (i = 0; i < nb; i++) {
        if (bn_bit(e, i)) {
            bn_mulmod(&T, A, &S, m);
            bn_copy(A, &T);
        }
        if (i < nb - 1) {
            bn_mulmod(&T, &S, &S, m);
            bn_copy(&S, &T);
        }
    }
    bn_mod(A, A, m);
}

/* Left-to-right k-ary, Fig 6.  Reading Z6: the table
 * entries are reduced mod m (the paper prints g_i = g_{i-1} * g without it).
 *   1. g_0 = 1; g_i = g_{i-1} * g mod m for i = 1 .. 2^k - 1.
 *   2. A = 1.
 *   3. for each base-2^k digit e_i from the top: A = A^(2^k) mod m;
 *      A = A * g_{e_i} mod m.
 *   4. return A. */
static int bn_modexp_kary(bn_t *A, const bn_t *g, const bn_t *e, const bn_t *m, int k)
{
    bn_t *tab, T;
    int i, j, ndig, nent;
    if (k < 1 || k > 8)
        return OR_EINVAL;
    nent = 1 << k;
    tab = (bn_t *)malloc(sizeof(bn_t) * (size_t)nent);
    if (!tab)
        return OR_EINVAL;
    bn_set_u32(&tab[0], 1);
    bn_mod(&tab[0], &tab[0], m);
    for (i = 1; i < nent; i++)
        bn_mulmod(&tab[i], &tab[i - 1], g, m);
    bn_set_u32(A, 1);
    ndig = (bn_bitlen(e) + k - 1) / k;
    for (i = ndig - 1; i >= 0; i--) {
        int digit = 0;
        for (j = 0; j < k; j++) {
            bn_mulmod(&T, A, A, m);
            bn_copy(A, &T);
        }
        for (j = k - 1; j >= 0; j--)
            digit = (digit << 1) | bn_bit(e, i * k + j);
        bn_mulmod(&T, A, &tab[digit], m);
        bn_copy(A, &T);
    }
    bn_mod(A, A, m);
    free(tab);
    return OR_OK;
}

/* Sliding window, Fig 7.  Reading Z6: "find the longest
 * bitstring e_i e_{i-1} .. e_l such that i - l + 1 <= k and e_l = 1" (the
 * printed e_1 is read as e_l).
 *   1. g_1 = g, g_2 = g^2, g_{2i+1} = g_{2i-1} * g_2 mod m, i = 1 .. 2^(k-1)-1.
 *   2. A = 1, i = t.
 *   3. while i >= 0: if e_i = 0: A = A^2 mod m, i = i - 1;
 *      else find l; A = A^(2^(i-l+1)) * g_{(e_i..e_l)_2} mod m; i = l - 1.
 *   4. return A. */
static int bn_modexp_sliding(bn_t *A, const bn_t *g, const bn_t *e, const bn_t *m, int k)
{
    bn_t *tab, g2, T;
    int i, l, j, nodd;
    if (k < 1 || k > 8)
        return OR_EINVAL;
    nodd = 1 << (k - 1);
    tab = (bn_t *)malloc(sizeof(bn_t) * (size_t)nodd); /* tab[j] = g^(2j+1) */
    if (!tab)
        return OR_EINVAL;
    bn_mod(&tab[0], g, m);
    bn_mulmod(&g2, g, g, m);
    for (j = 1; j < nodd; j++)
        bn_mulmod(&tab[j], &tab[j - 1], &g2, m);
    bn_set_u32(A, 1);
    i = bn_bitlen(e) - 1;
    while (i >= 0) {
        if (!bn_bit(e, i)) {
            bn_mulmod(&T, A, A, m);
            bn_copy(A, &T);
            i = i - 1;
        } else {
            int val = 0;
            l = i - k + 1;
            if (l < 0)
                l = 0;
            while (!bn_bit(e, l))
                l++;
            for (j = i; j >= l; j--)
                val = (val << 1) | bn_bit(e, j);
            for (j = 0; j < i - l + 1; j++) {
                bn_mulmod(&T, A, A, m);
                bn_copy(A, &T);
            }
            bn_mulmod(&T, A, &tab[val >> 1], m);
            bn_copy(A, &T);
            i = l - 1;
        }
    }
    bn_mod(A, A, m);
    free(tab);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* number theory for the key-generation check (Fig 1)   */
/* ------------------------------------------------------------------ */

/* Euclid: r = gcd(a, b) */
static void bn_gcd(bn_t *r, const bn_t *a, const bn_t *b)
{
    bn_t x, y, t;
    bn_copy(&x, a);
    bn_copy(&y, b);
    while (!bn_is_zero(&y)) {
        bn_mod(&t, &x, &y);
        bn_copy(&x, &y);
        bn_copy(&y, &t);
    }
    bn_copy(r, &x);
}

/* Extended Euclid with the Bezout coefficient of e kept reduced mod phi:
 * invariant t_i * e == r_i (mod phi).  Returns 1 and d in (0, phi) when
 * gcd(e, phi) = 1, else 0. */
static int bn_inverse(bn_t *d, const bn_t *e, const bn_t *phi)
{
    bn_t r0, r1, t0, t1, qt, q, rr, tmp, tn;
    bn_copy(&r0, phi);
    bn_mod(&r1, e, phi);
    bn_zero(&t0);
    bn_set_u32(&t1, 1);
    while (!bn_is_zero(&r1)) {
        bn_divmod(&q, &rr, &r0, &r1);
        /* t_new = t0 - q * t1 (mod phi) */
        bn_mul(&tmp, &q, &t1);
        bn_mod(&qt, &tmp, phi);
        if (bn_cmp(&t0, &qt) >= 0) {
            bn_sub(&tn, &t0, &qt);
        } else {
            bn_add(&tmp, &t0, phi);
            bn_sub(&tn, &tmp, &qt);
        }
        bn_copy(&r0, &r1);
        bn_copy(&r1, &rr);
        bn_copy(&t0, &t1);
        bn_copy(&t1, &tn);
    }
    if (!bn_is_one(&r0))
        return 0;
    bn_copy(d, &t0);
    return 1;
}

/* splitmix64: counter-based generator for Miller-Rabin bases */
static uint64_t splitmix64(uint64_t *state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static const uint32_t small_primes[] = {
    2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71,
    73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151,
    157, 163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223, 227, 229, 233,
    239, 241, 251};

/* one Miller-Rabin round to base a: n - 1 = 2^r * q, q odd */
static int mr_round(const bn_t *n, const bn_t *nm1, const bn_t *q, int r, const bn_t *a)
{
    bn_t x, t;
    int i;
    bn_modexp_l2r(&x, a, q, n);
    if (bn_is_one(&x) || bn_cmp(&x, nm1) == 0)
        return 1;
    for (i = 1; i < r; i++) {
        bn_mulmod(&t, &x, &x, n);
        bn_copy(&x, &t);
        if (bn_cmp(&x, nm1) == 0)
            return 1;
        if (bn_is_one(&x))
            return 0;
    }
    return 0;
}

/* Primality: trial division by the primes < 256, then Miller-Rabin.  For
 * n < 2^64 the 12 prime bases 2..37 are a deterministic test; above that,
 * 64 rounds with bases drawn from splitmix64(seed = 1407146500). */
static int bn_is_prime(const bn_t *n)
{
    bn_t one, nm1, q, a, t;
    int i, r, np = (int)(sizeof(small_primes) / sizeof(small_primes[0]));
    if (n->len == 0 || bn_is_one(n))
        return 0;
    for (i = 0; i < np; i++) {
        bn_t p, rem;
        bn_set_u32(&p, small_primes[i]);
        if (bn_cmp(n, &p) == 0)
            return 1;
        bn_mod(&rem, n, &p);
        if (bn_is_zero(&rem))
            return 0;
    }
    bn_set_u32(&one, 1);
    bn_sub(&nm1, n, &one);
    bn_copy(&q, &nm1);
    r = 0;
    while (!bn_bit(&q, 0)) {
        /* q = q / 2 */
        int k;
        for (k = 0; k < q.len; k++)
            q.d[k] = (q.d[k] >> 1) | (k + 1 < q.len ? (q.d[k + 1] << 31) : 0u);
        bn_norm(&q);
        r++;
    }
    if (bn_bitlen(n) <= 64) {
        for (i = 0; i < 12; i++) {
            bn_set_u32(&a, small_primes[i]);
            if (!mr_round(n, &nm1, &q, r, &a))
                return 0;
        }
        return 1;
    } else {
        uint64_t st = 1407146500ull;
        bn_t three, span;
        bn_set_u32(&three, 3);
        bn_sub(&span, n, &three);           /* bases in [2, n-2] */
        for (i = 0; i < 64; i++) {
            bn_t raw;
            int k;
            raw.len = n->len;
            for (k = 0; k < n->len; k++)
                raw.d[k] = (uint32_t)splitmix64(&st);
            bn_norm(&raw);
            bn_mod(&t, &raw, &span);
            bn_set_u32(&a, 2);
            bn_add(&a, &a, &t);
            if (!mr_round(n, &nm1, &q, r, &a))
                return 0;
        }
        return 1;
    }
}

/* ------------------------------------------------------------------ */
/* exported C API (ctypes, see oracle/__init__.py)                        */
/* ------------------------------------------------------------------ */

#define CHECK_LEN(x) do { if ((x) < 0 || (x) > 128) return OR_EINVAL; } while (0)

/* out[0 .. ml) = g^e mod m.  Returns 0, or OR_EINVAL (m == 0). */
int oracle_modexp(const uint32_t *g, int gl, const uint32_t *e, int el,
                  const uint32_t *m, int ml, uint32_t *out)
{
    bn_t G, E, M, A;
    CHECK_LEN(gl); CHECK_LEN(el); CHECK_LEN(ml);
    bn_from_limbs(&G, g, gl);
    bn_from_limbs(&E, e, el);
    bn_from_limbs(&M, m, ml);
    if (bn_is_zero(&M))
        return OR_EINVAL;
    bn_modexp_l2r(&A, &G, &E, &M);
    bn_to_limbs(out, ml, &A);
    return OR_OK;
}

/* variant: 0 = L2R (Fig 5b), 1 = R2L (Fig 5a), 2 = k-ary (Fig 6),
 * 3 = sliding (Fig 7) */
int oracle_modexp_variant(int variant, int k, const uint32_t *g, int gl,
                          const uint32_t *e, int el, const uint32_t *m, int ml,
                          uint32_t *out)
{
    bn_t G, E, M, A;
    int st = OR_OK;
    CHECK_LEN(gl); CHECK_LEN(el); CHECK_LEN(ml);
    bn_from_limbs(&G, g, gl);
    bn_from_limbs(&E, e, el);
    bn_from_limbs(&M, m, ml);
    if (bn_is_zero(&M))
        return OR_EINVAL;
    switch (variant) {
    case 0: bn_modexp_l2r(&A, &G, &E, &M); break;
    case 1: bn_modexp_r2l(&A, &G, &E, &M); break;
    case 2: st = bn_modexp_kary(&A, &G, &E, &M, k); break;
    case 3: st = bn_modexp_sliding(&A, &G, &E, &M, k); break;
    default: return OR_EINVAL;
    }
    if (st != OR_OK)
        return st;
    bn_to_limbs(out, ml, &A);
    return OR_OK;
}

/* Naive repeated multiplication, Fig 4, single-word:
 * c_1 = g mod m; c_j = (c_{j-1} * g) mod m for j = 2 .. e (e - 1 modular
 * multiplications).  trace[j-1] = c_j if trace != NULL.  e = 0 returns
 * 1 mod m (empty product). */
int oracle_naive_u64(uint64_t g, uint64_t e, uint64_t m, uint64_t *out, uint64_t *trace)
{
    bn_t G, M, C, T;
    uint64_t j;
    if (m == 0)
        return OR_EINVAL;
    bn_set_u64(&G, g);
    bn_set_u64(&M, m);
    if (e == 0) {
        bn_set_u32(&C, 1);
        bn_mod(&C, &C, &M);
    } else {
        bn_mod(&C, &G, &M);
        if (trace)
            trace[0] = bn_to_u64(&C);
        for (j = 2; j <= e; j++) {
            bn_mulmod(&T, &C, &G, &M);
            bn_copy(&C, &T);
            if (trace)
                trace[j - 1] = bn_to_u64(&C);
        }
    }
    *out = bn_to_u64(&C);
    return OR_OK;
}

/* The paper's own device function, Fig 12, as printed,
 * in exact integer arithmetic for m < 2^31 (its overflow envelope, SURVEY
 * fact 0.3): a = (g%m)^2; ret = 1; floor(e/2) times ret = ret*a % m; if e
 * odd, ret = ret*(g%m) % m.  faithful = 1 keeps "if (exponent == 0) return
 * base % den" (reading Z5); faithful = 0 returns 1 % m for e = 0.  The
 * float counter of Fig 12 is replaced by its exact integer meaning
 * (reading Z15: identical for e < 2^24). */
int oracle_halving_u64(uint64_t g, uint64_t e, uint64_t m, int faithful, uint64_t *out)
{
    bn_t G, M, A, R, T;
    uint64_t j, half;
    if (m == 0 || m >= (1ull << 31))
        return OR_ERANGE;
    bn_set_u64(&G, g);
    bn_set_u64(&M, m);
    bn_mod(&G, &G, &M);                       /* g % den */
    if (e == 0) {
        if (faithful) {
            *out = bn_to_u64(&G);
        } else {
            *out = 1 % m;
        }
        return OR_OK;
    }
    bn_mul(&A, &G, &G);                       /* a = (g%den)*(g%den), unreduced */
    bn_set_u32(&R, 1);
    half = e / 2;
    for (j = 0; j < half; j++) {              /* size > 0.5 branch */
        bn_mulmod(&T, &R, &A, &M);
        bn_copy(&R, &T);
    }
    if (e & 1) {                              /* size == 0.5 branch */
        bn_mulmod(&T, &R, &G, &M);
        bn_copy(&R, &T);
    }
    bn_mod(&R, &R, &M);                       /* ret = 1 when e/2 loop never ran and m = 1 */
    *out = bn_to_u64(&R);
    return OR_OK;
}

int oracle_is_prime(const uint32_t *x, int xl)
{
    bn_t X;
    if (xl < 0 || xl > 128)
        return OR_EINVAL;
    bn_from_limbs(&X, x, xl);
    return bn_is_prime(&X);
}

/* Fig 1: n = p*q; phi = (p-1)(q-1); require p, q prime,
 * p != q, 1 < e < phi, gcd(e, phi) = 1; d = e^-1 mod phi, 0 < d < phi.
 * Outputs hold 2*pl limbs each. */
int oracle_keygen_check(const uint32_t *p, const uint32_t *q, int pl,
                        const uint32_t *e, int el,
                        uint32_t *n_out, uint32_t *phi_out, uint32_t *d_out)
{
    bn_t P, Q, E, N, PHI, P1, Q1, one, G, D;
    if (!p || !q || !e || !n_out || !phi_out || !d_out || pl < 1 || pl > 64 || el < 1 || el > 128)
        return OR_EINVAL;
    bn_from_limbs(&P, p, pl);
    bn_from_limbs(&Q, q, pl);
    bn_from_limbs(&E, e, el);
    if (!bn_is_prime(&P) || !bn_is_prime(&Q))
        return OR_ENOTPRIME;
    if (bn_cmp(&P, &Q) == 0)
        return OR_EEQUAL;
    bn_set_u32(&one, 1);
    bn_mul(&N, &P, &Q);
    bn_sub(&P1, &P, &one);
    bn_sub(&Q1, &Q, &one);
    bn_mul(&PHI, &P1, &Q1);
    bn_to_limbs(n_out, 2 * pl, &N);
    bn_to_limbs(phi_out, 2 * pl, &PHI);
    if (bn_cmp(&E, &one) <= 0 || bn_cmp(&E, &PHI) >= 0)
        return OR_ERANGE;
    bn_gcd(&G, &E, &PHI);
    if (!bn_is_one(&G))
        return OR_ENOTCOPRIME;
    if (!bn_inverse(&D, &E, &PHI))
        return OR_ENOTCOPRIME;
    bn_to_limbs(d_out, 2 * pl, &D);
    return OR_OK;
}

/* residue_out = (d * e) mod phi, phi = (p-1)(q-1).  Returns OR_OK when the
 * residue is 1 (valid pair), OR_EBADKEY otherwise. */
int oracle_validate_key(const uint32_t *e, const uint32_t *d, const uint32_t *p,
                        const uint32_t *q, int limbs, uint32_t *residue_out)
{
    bn_t E, D, P, Q, one, P1, Q1, PHI, R;
    if (!e || !d || !p || !q || !residue_out || limbs < 1 || limbs > 64)
        return OR_EINVAL;
    bn_from_limbs(&E, e, limbs);
    bn_from_limbs(&D, d, limbs);
    bn_from_limbs(&P, p, limbs);
    bn_from_limbs(&Q, q, limbs);
    bn_set_u32(&one, 1);
    bn_sub(&P1, &P, &one);
    bn_sub(&Q1, &Q, &one);
    bn_mul(&PHI, &P1, &Q1);
    bn_mulmod(&R, &D, &E, &PHI);
    bn_to_limbs(residue_out, 2 * limbs, &R);
    return bn_is_one(&R) ? OR_OK : OR_EBADKEY;
}

/* ---------------- batch driver (pthread pool over packets) ---------------- */

typedef struct {
    const uint32_t *base;
    int s;                    /* limbs per input packet */
    const bn_t *E, *M;
    int ml;                   /* limbs per output packet */
    uint32_t *out;
    size_t lo, hi;
} batch_job_t;

static void *batch_worker(void *arg)
{
    batch_job_t *jb = (batch_job_t *)arg;
    size_t i;
    for (i = jb->lo; i < jb->hi; i++) {
        bn_t G, A;
        bn_from_limbs(&G, jb->base + i * (size_t)jb->s, jb->s);
        bn_modexp_l2r(&A, &G, jb->E, jb->M);
        bn_to_limbs(jb->out + i * (size_t)jb->ml, jb->ml, &A);
    }
    return NULL;
}

/* out[i] = base[i]^e mod m for i < count; base is [count][s], out is
 * [count][ml], little-endian limbs.  nthreads >= 1. */
int oracle_modexp_batch(const uint32_t *base, size_t count, int s,
                        const uint32_t *e, int el, const uint32_t *m, int ml,
                        uint32_t *out, int nthreads)
{
    bn_t E, M;
    pthread_t *th;
    batch_job_t *jobs;
    int t;
    size_t per;
    CHECK_LEN(s); CHECK_LEN(el); CHECK_LEN(ml);
    if (nthreads < 1)
        nthreads = 1;
    bn_from_limbs(&E, e, el);
    bn_from_limbs(&M, m, ml);
    if (bn_is_zero(&M))
        return OR_EINVAL;
    if ((size_t)nthreads > count)
        nthreads = count ? (int)count : 1;
    th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    jobs = (batch_job_t *)malloc(sizeof(batch_job_t) * (size_t)nthreads);
    per = (count + (size_t)nthreads - 1) / (size_t)nthreads;
    for (t = 0; t < nthreads; t++) {
        jobs[t].base = base;
        jobs[t].s = s;
        jobs[t].E = &E;
        jobs[t].M = &M;
        jobs[t].ml = ml;
        jobs[t].out = out;
        jobs[t].lo = (size_t)t * per < count ? (size_t)t * per : count;
        jobs[t].hi = (size_t)(t + 1) * per < count ? (size_t)(t + 1) * per : count;
        pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    }
    for (t = 0; t < nthreads; t++)
        pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return OR_OK;
}

/* ---------------- packet codec, sec. 2 ---------------- */

/* Strip ASCII spaces (reading Z16); each remaining char must be a..z
 * (a = 00 .. z = 25); consecutive pairs become hi*100 + lo
 * (PAPER.md:40).  On OR_ECHAR, *count_out = index of the bad char in text. */
int oracle_encode(const char *text, uint32_t *packets, size_t cap, size_t *count_out)
{
    size_t i, nl = 0, np = 0;
    int have_hi = 0;
    uint32_t hi = 0;
    if (!text || !count_out)
        return OR_EINVAL;
    for (i = 0; text[i]; i++) {
        if (text[i] == ' ')
            continue;
        if (text[i] < 'a' || text[i] > 'z') {
            *count_out = i;
            return OR_ECHAR;
        }
        nl++;
    }
    if (nl % 2)
        return OR_EODD;
    if (nl / 2 > cap) {
        *count_out = nl / 2;
        return OR_ENOSPC;
    }
    for (i = 0; text[i]; i++) {
        uint32_t v;
        if (text[i] == ' ')
            continue;
        v = (uint32_t)(text[i] - 'a');
        if (!have_hi) {
            hi = v;
            have_hi = 1;
        } else {
            packets[np++] = hi * 100u + v;
            have_hi = 0;
        }
    }
    *count_out = np;
    return OR_OK;
}

/* Inverse of oracle_encode (spaces are not recovered).  text receives
 * 2*count letters and a NUL; cap counts bytes including the NUL. */
int oracle_decode(const uint32_t *packets, size_t count, char *text, size_t cap)
{
    size_t i;
    if ((!packets && count) || !text)
        return OR_EINVAL;
    if (2 * count + 1 > cap)
        return OR_ENOSPC;
    for (i = 0; i < count; i++) {
        uint32_t hi = packets[i] / 100u, lo = packets[i] % 100u;
        if (hi > 25 || lo > 25)
            return OR_EPACKET;
        text[2 * i] = (char)('a' + hi);
        text[2 * i + 1] = (char)('a' + lo);
    }
    text[2 * count] = 0;
    return OR_OK;
}

/* ---------------- multi-key batch: per-packet exponent and modulus ------------- */

typedef struct {
    const uint32_t *base, *exps, *mods;
    int s;
    uint32_t *out;
    size_t lo, hi;
} multi_job_t;

static void *multi_worker(void *arg)
{
    multi_job_t *jb = (multi_job_t *)arg;
    size_t i;
    for (i = jb->lo; i < jb->hi; i++) {
        bn_t G, E, M, A;
        bn_from_limbs(&G, jb->base + i * (size_t)jb->s, jb->s);
        bn_from_limbs(&E, jb->exps + i * (size_t)jb->s, jb->s);
        bn_from_limbs(&M, jb->mods + i * (size_t)jb->s, jb->s);
        if (bn_is_zero(&M)) {
            bn_zero(&A);
        } else {
            bn_modexp_l2r(&A, &G, &E, &M);       /* Fig 5 */
        }
        bn_to_limbs(jb->out + i * (size_t)jb->s, jb->s, &A);
    }
    return NULL;
}

/* out[i] = base[i]^exps[i] mod mods[i]; all [count][s] limbs. */
int oracle_modexp_multi(const uint32_t *base, const uint32_t *exps, const uint32_t *mods, size_t count,
                        int s, uint32_t *out, int nthreads)
{
    pthread_t *th;
    multi_job_t *jobs;
    int t;
    size_t per;
    CHECK_LEN(s);
    if (nthreads < 1)
        nthreads = 1;
    if ((size_t)nthreads > count)
        nthreads = count ? (int)count : 1;
    th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    jobs = (multi_job_t *)malloc(sizeof(multi_job_t) * (size_t)nthreads);
    per = (count + (size_t)nthreads - 1) / (size_t)nthreads;
    for (t = 0; t < nthreads; t++) {
        jobs[t].base = base;
        jobs[t].exps = exps;
        jobs[t].mods = mods;
        jobs[t].s = s;
        jobs[t].out = out;
        jobs[t].lo = (size_t)t * per < count ? (size_t)t * per : count;
        jobs[t].hi = (size_t)(t + 1) * per < count ? (size_t)(t + 1) * per : count;
        pthread_create(&th[t], NULL, multi_worker, &jobs[t]);
    }
    for (t = 0; t < nthreads; t++)
        pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return OR_OK;
}

/* One Miller-Rabin round to base a on odd n >= 5: returns 1 if n is a strong
 * probable prime to base a (n - 1 = 2^r q, a^q = 1 or a^(2^j q) = n - 1 for
 * some j < r), else 0. */
int oracle_mr_round(const uint32_t *n, int nl, uint32_t a)
{
    bn_t N, one, nm1, q, A;
    int r;
    if (nl < 1 || nl > 128)
        return OR_EINVAL;
    bn_from_limbs(&N, n, nl);
    bn_set_u32(&one, 1);
    bn_sub(&nm1, &N, &one);
    bn_copy(&q, &nm1);
    r = 0;
    while (!bn_bit(&q, 0)) {
        int k;
        for (k = 0; k < q.len; k++)
            q.d[k] = (q.d[k] >> 1) | (k + 1 < q.len ? (q.d[k + 1] << 31) : 0u);
        bn_norm(&q);
        r++;
    }
    bn_set_u32(&A, a);
    return mr_round(&N, &nm1, &q, r, &A);
}
