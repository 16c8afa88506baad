// host_bn.hpp -- small host-side multi-precision helpers for the product's
// key precompute (n', R^2 mod n) and rsa_keygen_check.  Product code: it shares
// nothing with oracle/ (different algorithms on purpose: shift-subtract
// division, signed extended Euclid, Montgomery-based Miller-Rabin).
#pragma once
#include <stdint.h>

#include <vector>

namespace rsa_host {

typedef std::vector<uint32_t> BN;   // little-endian limbs, normalised (no top zeros)

inline void trim(BN& a) {
    while (!a.empty() && a.back() == 0) a.pop_back();
}
inline BN from_limbs(const uint32_t* p, int n) {
    BN a(p, p + n);
    trim(a);
    return a;
}
inline BN from_u64(uint64_t v) {
    BN a{(uint32_t)v, (uint32_t)(v >> 32)};
    trim(a);
    return a;
}
inline void to_limbs(const BN& a, uint32_t* p, int n) {
    for (int i = 0; i < n; i++) p[i] = i < (int)a.size() ? a[i] : 0u;
}
inline bool is_zero(const BN& a) { return a.empty(); }
inline bool is_one(const BN& a) { return a.size() == 1 && a[0] == 1; }
inline int bits(const BN& a) {
    if (a.empty()) return 0;
    return 32 * (int)(a.size() - 1) + (32 - __builtin_clz(a.back()));
}
inline int bit(const BN& a, int i) {
    size_t w = (size_t)i / 32;
    return w < a.size() ? (int)((a[w] >> (i % 32)) & 1u) : 0;
}
inline int cmp(const BN& a, const BN& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
inline BN add(const BN& a, const BN& b) {
    BN r(std::max(a.size(), b.size()) + 1, 0);
    uint64_t c = 0;
    for (size_t i = 0; i + 1 < r.size(); i++) {
        c += (uint64_t)(i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
        r[i] = (uint32_t)c;
        c >>= 32;
    }
    r.back() = (uint32_t)c;
    trim(r);
    return r;
}
// a - b, requires a >= b
inline BN sub(const BN& a, const BN& b) {
    BN r(a.size(), 0);
    uint32_t borrow = 0;
    for (size_t i = 0; i < a.size(); i++) {
        uint64_t bi = (uint64_t)(i < b.size() ? b[i] : 0) + borrow;
        uint64_t ai = a[i];
        r[i] = (uint32_t)(ai - bi);
        borrow = ai < bi ? 1u : 0u;
    }
    trim(r);
    return r;
}
inline BN mul(const BN& a, const BN& b) {
    if (a.empty() || b.empty()) return BN();
    BN r(a.size() + b.size(), 0);
    for (size_t j = 0; j < b.size(); j++) {
        uint64_t c = 0;
        for (size_t i = 0; i < a.size(); i++) {
            c += (uint64_t)a[i] * b[j] + r[i + j];
            r[i + j] = (uint32_t)c;
            c >>= 32;
        }
        r[j + a.size()] = (uint32_t)c;
    }
    trim(r);
    return r;
}
inline BN shl(const BN& a, int s) {
    if (a.empty()) return a;
    int w = s / 32, b = s % 32;
    BN r(a.size() + w + 1, 0);
    for (size_t i = 0; i < a.size(); i++) {
        r[i + w] |= a[i] << b;
        if (b) r[i + w + 1] |= a[i] >> (32 - b);
    }
    trim(r);
    return r;
}
inline BN shr1(const BN& a) {
    BN r(a.size(), 0);
    for (size_t i = 0; i < a.size(); i++)
        r[i] = (a[i] >> 1) | (i + 1 < a.size() ? (a[i + 1] << 31) : 0u);
    trim(r);
    return r;
}
// binary shift-subtract long division: q = a / m, r = a mod m (m != 0)
inline void divmod(const BN& a, const BN& m, BN* q, BN* r) {
    BN rem = a, quo;
    int sh = bits(a) - bits(m);
    if (sh < 0) {
        if (q) *q = BN();
        if (r) *r = rem;
        return;
    }
    quo.assign((size_t)sh / 32 + 1, 0);
    BN d = shl(m, sh);
    for (int i = sh; i >= 0; i--) {
        if (cmp(rem, d) >= 0) {
            rem = sub(rem, d);
            quo[(size_t)i / 32] |= 1u << (i % 32);
        }
        d = shr1(d);
    }
    trim(quo);
    if (q) *q = quo;
    if (r) *r = rem;
}
inline BN mod(const BN& a, const BN& m) {
    BN r;
    divmod(a, m, nullptr, &r);
    return r;
}

// -n^-1 mod 2^32 for odd n0 (Newton: x <- x (2 - n0 x) doubles the bits)
inline uint32_t neg_inv32(uint32_t n0) {
    uint32_t x = n0;            // correct to 3 bits for odd n0
    for (int i = 0; i < 5; i++) x *= 2u - n0 * x;
    return 0u - x;
}

// 2^k mod n by repeated doubling (n odd >= 3)
inline BN pow2_mod(int k, const BN& n) {
    BN v{1u};
    for (int i = 0; i < k; i++) {
        v = shl(v, 1);
        if (cmp(v, n) >= 0) v = sub(v, n);
    }
    return v;
}

// ---- Montgomery arithmetic over a fixed odd modulus (host, for Miller-Rabin)
struct HostMont {
    BN n;
    int s;
    uint32_t ninv;
    BN r2;      // R^2 mod n, R = 2^(32 s)
    explicit HostMont(const BN& n_) : n(n_), s((int)n_.size()), ninv(neg_inv32(n_[0])) {
        r2 = pow2_mod(64 * s, n);
    }
    // a, b: s limbs each (< n); returns a b R^-1 mod n (s limbs, padded)
    std::vector<uint32_t> mulm(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) const {
        std::vector<uint32_t> t(s + 2, 0);
        for (int i = 0; i < s; i++) {
            uint64_t c = 0;
            for (int j = 0; j < s; j++) {
                c += (uint64_t)a[j] * b[i] + t[j];
                t[j] = (uint32_t)c;
                c >>= 32;
            }
            uint64_t u = (uint64_t)t[s] + c;
            t[s] = (uint32_t)u;
            t[s + 1] = (uint32_t)(u >> 32);
            uint32_t m = t[0] * ninv;
            c = ((uint64_t)m * n[0] + t[0]) >> 32;
            for (int j = 1; j < s; j++) {
                c += (uint64_t)m * n[j] + t[j];
                t[j - 1] = (uint32_t)c;
                c >>= 32;
            }
            u = (uint64_t)t[s] + c;
            t[s - 1] = (uint32_t)u;
            t[s] = t[s + 1] + (uint32_t)(u >> 32);
            t[s + 1] = 0;
        }
        // conditional subtract
        std::vector<uint32_t> d(s, 0);
        int64_t br = 0;
        for (int j = 0; j < s; j++) {
            int64_t v = (int64_t)t[j] - n[j] - br;
            br = v < 0;
            d[j] = (uint32_t)v;
        }
        bool ge = t[s] != 0 || br == 0;
        if (ge) return d;
        t.resize(s);
        return t;
    }
    std::vector<uint32_t> pad(const BN& a) const {
        std::vector<uint32_t> v(s, 0);
        for (size_t i = 0; i < a.size() && (int)i < s; i++) v[i] = a[i];
        return v;
    }
    // g^e mod n, g < n
    BN powm(const BN& g, const BN& e) const {
        std::vector<uint32_t> one(s, 0);
        one[0] = 1;
        std::vector<uint32_t> x = mulm(pad(g), pad(r2));      // to Montgomery
        std::vector<uint32_t> acc = mulm(one, pad(r2));       // R mod n
        for (int i = bits(e) - 1; i >= 0; i--) {
            acc = mulm(acc, acc);
            if (bit(e, i)) acc = mulm(acc, x);
        }
        acc = mulm(acc, one);
        BN r(acc.begin(), acc.end());
        trim(r);
        return r;
    }
};

// xorshift64* -- Miller-Rabin base generator (fixed seed, deterministic)
inline uint64_t xs64(uint64_t& s) {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    return s * 2685821657736338717ull;
}

// Miller-Rabin: trial division by primes < 1000, then deterministic bases
// for n < 2^64 and 48 pseudo-random bases above.
inline bool is_probable_prime(const BN& n) {
    if (n.empty()) return false;
    if (n.size() == 1 && n[0] < 4) return n[0] >= 2;
    if ((n[0] & 1u) == 0) return false;
    for (uint32_t p = 3; p < 1000; p += 2) {
        bool prime = true;
        for (uint32_t f = 3; f * f <= p; f += 2)
            if (p % f == 0) { prime = false; break; }
        if (!prime) continue;
        // n mod p by Horner on limbs
        uint64_t r = 0;
        for (size_t i = n.size(); i-- > 0;) r = ((r << 32) | n[i]) % p;
        if (r == 0) return n.size() == 1 && n[0] == p;
    }
    BN one{1u};
    BN nm1 = sub(n, one);
    BN d = nm1;
    int r = 0;
    while (!bit(d, 0)) { d = shr1(d); r++; }
    HostMont mt(n);
    auto witness = [&](const BN& a) -> bool {   // true if a proves n composite
        BN x = mt.powm(a, d);
        if (is_one(x) || cmp(x, nm1) == 0) return false;
        for (int i = 1; i < r; i++) {
            x = mod(mul(x, x), n);
            if (cmp(x, nm1) == 0) return false;
            if (is_one(x)) return true;
        }
        return true;
    };
    if (bits(n) <= 64) {
        static const uint32_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
        for (uint32_t b : bases)
            if (witness(BN{b})) return false;
        return true;
    }
    uint64_t st = 0x1407146500000001ull;
    BN span = sub(n, BN{3u});
    for (int i = 0; i < 48; i++) {
        BN raw(n.size(), 0);
        for (auto& w : raw) w = (uint32_t)(xs64(st) >> 16);
        trim(raw);
        BN a = add(mod(raw, span), BN{2u});
        if (witness(a)) return false;
    }
    return true;
}

// gcd by Euclid (shift-subtract division)
inline BN gcd(BN a, BN b) {
    while (!b.empty()) {
        BN r = mod(a, b);
        a = b;
        b = r;
    }
    return a;
}

// e^-1 mod phi by the extended Euclidean algorithm with signed coefficient
// bookkeeping (sign, magnitude).  Returns false if gcd(e, phi) != 1.
inline bool inverse(const BN& e, const BN& phi, BN* d) {
    BN r0 = phi, r1 = mod(e, phi);
    BN s0, s1{1u};          // coefficients of e: s_i * e == r_i (mod phi)
    bool n0 = false, n1 = false;   // signs (true = negative)
    while (!r1.empty()) {
        BN q, r2;
        divmod(r0, r1, &q, &r2);
        // s2 = s0 - q s1 (signed)
        BN qs = mul(q, s1);
        BN s2;
        bool n2;
        if (n0 != n1) {             // s0 and q*s1 have opposite signs -> magnitudes add
            s2 = add(s0, qs);
            n2 = n0;
        } else if (cmp(s0, qs) >= 0) {
            s2 = sub(s0, qs);
            n2 = n0;
        } else {
            s2 = sub(qs, s0);
            n2 = !n0;
        }
        if (s2.empty()) n2 = false;
        r0 = r1; r1 = r2;
        s0 = s1; n0 = n1;
        s1 = s2; n1 = n2;
    }
    if (!is_one(r0)) return false;
    BN v = mod(s0, phi);
    if (n0 && !v.empty()) v = sub(phi, v);
    *d = v;
    return true;
}

}  // namespace rsa_host
