// mont_f64.cuh -- Montgomery multiplication on the FP64 pipe (52-bit digits).
//
// Same operation as mont.cuh (Fig 3 "(u*v) mod
// m", realised by Montgomery reduction), different number
// representation: numbers are ND digits of D = 52 bits held as doubles, and
// every 52x52 -> 104-bit digit product is split exactly into its high and low
// halves by two fused multiply-adds:
//
//   h = fma_rz(x, y, 2^104)          = 2^104 + floor(x y / 2^52) 2^52
//   l = fma_rz(x, y, 2^104 + 2^52 - h) = 2^52 + (x y mod 2^52)        (exact)
//
// (the first rounds toward zero inside the binade [2^104, 2^105) whose ulp is
// 2^52; the second is an integer in [2^52, 2^53) and so exact).  Both results
// carry their integer in the low 52 bits of their IEEE bit pattern, on top of
// a constant exponent field (Bh = 0x467 << 52, Bl = 0x433 << 52).  Column sums
// therefore accumulate the raw bit patterns with 64-bit integer adds (IADD3 +
// IADD3.X on the ALU pipe); the exponent fields add a known multiple of 2^52
// per term (mod 2^64), which is subtracted only where a carry is taken.  No
// carry chains: a column of the CIOS accumulator receives 4 terms < 2^52 per
// iteration and lives <= ND iterations, so its true value stays < 2^60.
//
// Why: on B200 the DFMA pipe issues ~53-64 results/clk/SM (profiles/
// r01_imad_peak.jsonl, r01_dfma_latency.jsonl) and one 52x52 product costs 3
// FP64 ops (DFMA, DADD, DFMA) + one 64-bit add: the measured mix sustains ~41
// FP64 ops/clk/SM = ~13.7 products x 2704 bit^2 per clk, against ~28
// IMAD.WIDE.X products x 1024 bit^2 on the integer pipe: ~1.3x the multiply
// throughput (the RSA kernels: +13% at 2048 bits, +24% at 4096).
//
// CIOS (operand scanning) with R = 2^(52 ND), for i = 0 .. ND-1:
//   T += A b_i ;  q = T_0 n' mod 2^52 ;  T += q n ;  T /= 2^52
// The division is a register rename folded into the adds: column j of the
// new T is written from column j+1 of the old one (t[j-1] = t[j] + ...), in
// place, so a loop iteration needs no moves and no unrolling.  montsqr is the
// squaring (product scan + reduction loop), normalize the carry-lookahead
// end-of-op normalisation (used at ND >= 64).
//
// Bounds: A, B < 2n and 4n < R give T < 2n (almost-Montgomery: no
// subtraction inside the exponentiation; the caller canonicalises once at the
// end).  Pinned on CPU by tests/test_f64_model.py (this header compiled for
// the host with the rounding mode set to toward-zero).
#pragma once
#include <stdint.h>

#ifndef __CUDA_ARCH__
#include <cmath>
#include <cstring>
#endif

#ifndef RSA_F64_LOOKAHEAD
#define RSA_F64_LOOKAHEAD 0   // carry-lookahead normalisation at ND < 64 (A/B: 565K vs 591K at 2048)
#endif
#ifndef RSA_F64_LOOKAHEAD_SMALL
#define RSA_F64_LOOKAHEAD_SMALL 0   // ... at ND <= 20 (A/B: CRT-2048 2.04M vs 2.19M)
#endif
#ifndef RSA_F64_LOOKAHEAD_BIG
#define RSA_F64_LOOKAHEAD_BIG 1   // ... at ND >= 64 (A/B: 60.2K vs 56.5K at 4096)
#endif
#ifndef RSA_F64_NREG
#define RSA_F64_NREG 0   // A/B: n in registers in the reduction loop, 552K vs 591K at 2048 (CRT-2048 even)
#endif
#ifndef RSA_F64_NCONST
#define RSA_F64_NCONST 0  // n's digits as constant-bank DFMA operands (kernel parameters) instead of smem pairs
#endif
#ifndef RSA_F64_SQBATCH
#define RSA_F64_SQBATCH 4  // recursive product scan: digit products issued per batch (even; A/B at
#endif                     // 4096: 2/4/8/12 -> 62.5K/63.5K/63.4K/63.0K)
#ifndef RSA_F64_SQACC2
#define RSA_F64_SQACC2 0   // recursive product scan: two partial sums per column sum (A/B)
#endif
#ifndef RSA_F64_SQLOOP
#define RSA_F64_SQLOOP 40  // product scan as plain unrolled loops up to this ND (ptxas stops unrolling
#endif                     // the loop form at ND = 80: the recursive form expands at compile time)
#ifndef RSA_F64_MU
#define RSA_F64_MU 1      // CIOS loop trips unrolled (A/B: 2 -> 561K vs 565K at 2048, 37.4K vs 60.2K at 4096)
#endif
#ifndef RSA_F64_RU
#define RSA_F64_RU 4      // squaring's reduction loop trips unrolled at ND >= 40 (A/B knob:
#endif                    // 1/2/4/5 -> 565K/581K/590K/585K RSA-2048 decrypts/s)
#ifndef RSA_F64_RU_SMALL
#define RSA_F64_RU_SMALL 1   // ... at ND < 40 (A/B, CRT-2048: 1/2/4 -> 2.19M/2.14M/1.87M)
#endif

namespace rsa_b200 {
namespace f64 {

constexpr int kMU = RSA_F64_MU, kRU = RSA_F64_RU, kRUs = RSA_F64_RU_SMALL;
constexpr int D = 52;
constexpr uint64_t M52 = (1ull << 52) - 1;
constexpr uint64_t BL = 0x433ull << 52;            // bit pattern of 2^52
constexpr uint64_t BH = 0x467ull << 52;            // bit pattern of 2^104
constexpr uint64_t BETA = 2 * BL + 2 * BH;         // exponent fields added to an interior column per iteration
constexpr double C104 = 20282409603651670423947251286016.0;   // 2^104
constexpr double C2 = 20282409603651674927546878656512.0;     // 2^104 + 2^52
constexpr double C52 = 4503599627370496.0;                      // 2^52

// digits needed for a Montgomery radix R = 2^(52 ND) > 4n with n < 2^(32 S)
// (rounded up to even: the kernels move digit pairs; plan.h rsa_f64_digits is the same)
template <int S> struct Digits { static constexpr int ND = ((32 * S + 2 + D - 1) / D + 1) / 2 * 2; };

__host__ __device__ __forceinline__ uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}
__host__ __device__ __forceinline__ double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x; memcpy(&x, &u, 8); return x;
#endif
}
// host: the caller runs with fesetround(FE_TOWARDZERO) (the only inexact op)
__host__ __device__ __forceinline__ double fma_rz(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rz(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}
__host__ __device__ __forceinline__ double sub_rn(double a, double b) {   // exact where used
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
// digits 2g, 2g+1 of n.  On the device nd points to a per-block shared copy
// and the load is volatile: ptxas may neither hoist the ND digits into
// registers ahead of the loop (which starves the product schedule) nor fold
// them into uniform registers (too few: they spill).
// RSA_F64_NCONST: nd points to the kernel-parameter copy instead; the loads
// are plain, so ptxas can take each digit as a constant-bank operand of the
// DFMAs (no load instruction, no register read).
__host__ __device__ __forceinline__ void nd_pair(const double* nd, int g, double& x, double& y) {
#ifdef __CUDA_ARCH__
    if constexpr (RSA_F64_NCONST != 0) {
        x = nd[2 * g];
        y = nd[2 * g + 1];
        return;
    }
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(x), "=d"(y) : "r"((unsigned)__cvta_generic_to_shared(nd + 2 * g)));
#else
    x = nd[2 * g];
    y = nd[2 * g + 1];
#endif
}

// integer d < 2^52 -> double (exact)
__host__ __device__ __forceinline__ double digit_to_double(uint64_t d) { return sub_rn(from_bits(BL | d), C52); }

// x (S little-endian 32-bit limbs) -> ND digits of 52 bits as doubles
template <int S, int ND>
__host__ __device__ __forceinline__ void limbs_to_digits(const uint32_t (&x)[S], double (&a)[ND]) {
#pragma unroll
    for (int k = 0; k < ND; k++) {
        const int o = D * k, L = o / 32, sh = o % 32;
        uint64_t v = 0;
        if (L < S) v = (uint64_t)x[L] >> sh;
        if (L + 1 < S) v |= (uint64_t)x[L + 1] << (32 - sh);
        if (L + 2 < S && 64 - sh < 52) v |= (uint64_t)x[L + 2] << (64 - sh);
        a[k] = digit_to_double(v & M52);
    }
}

// canonical digits (uint64, < 2^52 each, value < 2^(32 S)) -> S limbs
template <int S, int ND>
__host__ __device__ __forceinline__ void digits_to_limbs(const uint64_t (&d)[ND], uint32_t (&x)[S]) {
#pragma unroll
    for (int m = 0; m < S; m++) {
        const int o = 32 * m, k = o / D, sh = o % D;
        uint64_t v = d[k] >> sh;
        if (k + 1 < ND && D - sh < 32) v |= d[k + 1] << (D - sh);
        x[m] = (uint32_t)v;
    }
}

// A <- A B R^-1 (mod n), R = 2^(52 ND), result < 2n for A, B < 2n.
// b(i) returns digit i of B as a double; nd: n's digits as doubles (constant
// bank on the device); np = -n^-1 mod 2^52; c104 = 2^104, passed in from the
// kernel parameters: as a register operand it leaves the DFMA's constant-bank
// slot to n's digits (with the immediate 2^104 ptxas hoists all ND digits of
// n into registers instead, and the product schedule starves).  The result digits are returned
// normalised both as doubles (a) and as integers (ai, for the final store).
// t[p] (true column values < 2^62) -> digits < 2^52 of the same number (the
// carry out of the top column is 0 by the callers' bounds).  Carry-lookahead
// instead of a 2 ND-deep serial chain: one local pass (low 52 bits + the
// previous column's high bits leaves a 0/1 carry per column), then the single-bit
// carries resolve with one 64-bit addition on bitmasks (generate G, propagate
// P: carry-in = (G + (G | P)) ^ P), then one more local pass.
template <int ND>
__host__ __device__ __forceinline__ void normalize(uint64_t (&t)[ND]) {
    constexpr int NW = (ND + 63) / 64;
    uint64_t G[NW], P[NW];
#pragma unroll
    for (int w = 0; w < NW; w++) { G[w] = 0; P[w] = 0; }
    uint64_t hprev = 0;
#pragma unroll
    for (int p = 0; p < ND; p++) {
        const uint64_t v = t[p];
        const uint64_t w = (v & M52) + hprev;
        hprev = v >> D;
        const uint64_t r = w & M52;
        t[p] = r;
        G[p >> 6] |= (w >> D) << (p & 63);
        P[p >> 6] |= (uint64_t)(r == M52) << (p & 63);
    }
    uint64_t C[NW], cin = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
        const uint64_t b = G[w] | P[w];
        const uint64_t s1 = G[w] + b;
        const uint64_t s2 = s1 + cin;
        cin = (s1 < G[w]) | (s2 < s1);
        C[w] = s2 ^ P[w];
    }
#pragma unroll
    for (int p = 0; p < ND; p++) t[p] = (t[p] + ((C[p >> 6] >> (p & 63)) & 1)) & M52;
}

// volatile load of a thread-private shared-memory digit (not hoisted)
__host__ __device__ __forceinline__ double ld_digit(const double* p) {
#ifdef __CUDA_ARCH__
    double x;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(x) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return x;
#else
    return *p;
#endif
}

// ASMEM: A is parked in this thread's shared-memory slot (aslot[k * stride])
// for the loop and re-read digit by digit, so its ND registers are free for
// the product schedule; the result comes back in registers.
// AIN: A lives in the slot (no copy in, the result digits go back to the slot
// and a[] is not touched).
// FUSEJ: one j-loop for both product rows (A b_i and q n), each column written
// once per iteration (fewer live partial results; for the 4096-bit kernel).
template <int ND, bool ASMEM = false, typename BF, bool AIN = false, bool FUSEJ = false>
__host__ __device__ __forceinline__ void montmul(double (&a)[ND], BF b, const double* __restrict__ nd, uint64_t np,
                                                 double c104, uint64_t (&t)[ND], double* aslot = nullptr,
                                                 int stride = 0) {
    static_assert(!AIN || ASMEM, "AIN needs the slot");
    if constexpr (ASMEM && !AIN) {
#pragma unroll
        for (int k = 0; k < ND; k++) aslot[k * stride] = a[k];
    }
    auto A = [&](int k) -> double {
        if constexpr (ASMEM) return ld_digit(aslot + k * stride);
        else return a[k];
    };
#pragma unroll
    for (int k = 0; k < ND; k++) t[k] = 0;
    uint64_t bias0 = 2 * BL;
    // Software-pipelined like montsqr's reduction: the quotient digit of
    // iteration i+1 needs only the new column 0 (complete after the j = 1
    // products) and a_0 b_{i+1}, so it is computed mid-iteration.
    double bi = b(0);
    uint64_t hp0, c0;
    {
        const double a0 = A(0);
        const double h0 = fma_rz(a0, bi, C104);
        const double l0 = fma_rz(a0, bi, sub_rn(C2, h0));
        hp0 = bits(h0);
        c0 = bits(l0);                                   // t[0] = 0
    }
    double qd = digit_to_double(((c0 & M52) * np) & M52);
#ifdef __CUDA_ARCH__
#pragma unroll kMU
#endif
    for (int i = 0; i < ND; i++) {
        const double bn = b(i + 1 < ND ? i + 1 : i);
        double n0, n1;
        nd_pair(nd, 0, n0, n1);
        const double hq0 = fma_rz(qd, n0, c104);
        const double lq0 = fma_rz(qd, n0, sub_rn(C2, hq0));
        const uint64_t carry = (c0 + bits(lq0) - bias0) >> D;     // column 0 is 0 mod 2^52
        const double a1 = A(1);
        const double h1 = fma_rz(a1, bi, C104);
        const double l1 = fma_rz(a1, bi, sub_rn(C2, h1));
        const double hq1 = fma_rz(qd, n1, c104);
        const double lq1 = fma_rz(qd, n1, sub_rn(C2, hq1));
        t[0] = t[1] + bits(l1) + hp0 + bits(lq1) + bits(hq0) + carry;
        // next iteration's column 0: + a_0 b_{i+1}
        const double a0 = A(0);
        const double hn = fma_rz(a0, bn, C104);
        const double ln = fma_rz(a0, bn, sub_rn(C2, hn));
        const uint64_t c0n = t[0] + bits(ln);
        const double qnext = digit_to_double(((c0n & M52) * np) & M52);
        uint64_t hp = bits(h1), hqp = bits(hq1);
        if constexpr (FUSEJ) {
#pragma unroll
            for (int j = 2; j < ND; j++) {
                const double aj = A(j);
                const double h = fma_rz(aj, bi, C104);
                const double l = fma_rz(aj, bi, sub_rn(C2, h));
                double nj = n1;
                if ((j & 1) == 0) nd_pair(nd, j / 2, nj, n1);
                const double hq = fma_rz(qd, nj, c104);
                const double lq = fma_rz(qd, nj, sub_rn(C2, hq));
                t[j - 1] = t[j] + bits(l) + hp + bits(lq) + hqp;
                hp = bits(h);
                hqp = bits(hq);
            }
        } else {
#pragma unroll
        for (int j = 2; j < ND; j++) {
            const double aj = A(j);
            const double h = fma_rz(aj, bi, C104);
            const double l = fma_rz(aj, bi, sub_rn(C2, h));
            t[j - 1] = t[j] + bits(l) + hp;
            hp = bits(h);
        }
#pragma unroll
        for (int j = 2; j < ND; j++) {
            double nj = n1;
            if ((j & 1) == 0) nd_pair(nd, j / 2, nj, n1);
            const double h = fma_rz(qd, nj, c104);
            const double l = fma_rz(qd, nj, sub_rn(C2, h));
            t[j - 1] += bits(l) + hqp;
            hqp = bits(h);
        }
        }
        t[ND - 1] = hp + hqp;
        c0 = c0n;
        hp0 = bits(hn);
        qd = qnext;
        bi = bn;
        bias0 += BETA;
    }
    // remove the exponent fields and propagate carries: column p now carries
    // 2 BH + (ND-1-p) BETA (mod 2^64) on top of its true value
    if constexpr ((ND >= 64) ? RSA_F64_LOOKAHEAD_BIG : (ND <= 20 ? RSA_F64_LOOKAHEAD_SMALL : RSA_F64_LOOKAHEAD)) {
#pragma unroll
        for (int p = 0; p < ND; p++) t[p] -= 2 * BH + (uint64_t)(ND - 1 - p) * BETA;
        normalize<ND>(t);
#pragma unroll
        for (int p = 0; p < ND; p++) {
            if constexpr (AIN) aslot[p * stride] = digit_to_double(t[p]);
            else a[p] = digit_to_double(t[p]);
        }
    } else {
        uint64_t carry = 0;
#pragma unroll
        for (int p = 0; p < ND; p++) {
            const uint64_t v = t[p] - (2 * BH + (uint64_t)(ND - 1 - p) * BETA) + carry;
            t[p] = v & M52;
            carry = v >> D;
            if constexpr (AIN) aslot[p * stride] = digit_to_double(t[p]);
            else a[p] = digit_to_double(t[p]);
        }
    }
}

// Squaring, separated operand scanning (SOS), in three pieces shared by
// montsqr (registers + a 2 ND-digit slot) and montsqr_slot (one ND-digit slot):
//
// number of cross products a_i a_j (i < j, i + j = k, j < ND) in column k
template <int ND>
__host__ __device__ constexpr int sqr_ncross(int k) {
    const int lo = k - ND + 1 > 0 ? k - ND + 1 : 0, hi = (k - 1) / 2;
    return (k >= 1 && hi >= lo) ? hi - lo + 1 : 0;
}

// One column K of the product scan, then (recursively, fully expanded at
// compile time) the columns after it.  xh = the previous column's cross
// products' high halves, already summed (raw patterns): each product's high
// half goes straight into the next column's running sum instead of being held
// until then (at ND = 80 the ~40 pending highs would take 80 registers next to
// A's 160 and starve the product schedule); lows and highs are added two
// products at a time (3-input 64-bit adds).
template <int ND, int K, int SQB_ = RSA_F64_SQBATCH, int ACC2 = RSA_F64_SQACC2, typename Put>
__host__ __device__ __forceinline__ void sqr_col(const double (&a)[ND], uint64_t xh, uint64_t hd, uint64_t carry,
                                                 Put& put) {
    if constexpr (K < 2 * ND) {
        constexpr int ILO = K - ND + 1 > 0 ? K - ND + 1 : 0;
        constexpr int NH = sqr_ncross<ND>(K), NHP = (K >= 1) ? sqr_ncross<ND>(K - 1) : 0;
        uint64_t x = xh, xn = 0, x2 = 0, xn2 = 0;
        // products in batches of SQB (every h, then every s = C2 - h, then every
        // l): the batch is the number of exact splits in flight per warp
        constexpr int SQB = SQB_;
#pragma unroll
        for (int m0 = 0; m0 < NH; m0 += SQB) {
            double hb[SQB], lb[SQB];
#pragma unroll
            for (int u = 0; u < SQB; u++)
                if (m0 + u < NH) hb[u] = fma_rz(a[ILO + m0 + u], a[K - ILO - m0 - u], C104);
#pragma unroll
            for (int u = 0; u < SQB; u++)
                if (m0 + u < NH) lb[u] = sub_rn(C2, hb[u]);
#pragma unroll
            for (int u = 0; u < SQB; u++)
                if (m0 + u < NH) lb[u] = fma_rz(a[ILO + m0 + u], a[K - ILO - m0 - u], lb[u]);
#pragma unroll
            for (int u = 0; u < SQB; u += 2) {
                // RSA_F64_SQACC2: alternate pairs go to second partial sums
                uint64_t& xs = (ACC2 && ((m0 + u) / 2) % 2) ? x2 : x;
                uint64_t& xns = (ACC2 && ((m0 + u) / 2) % 2) ? xn2 : xn;
                if (m0 + u + 1 < NH) {
                    xs += bits(lb[u]) + bits(lb[u + 1]);
                    xns += bits(hb[u]) + bits(hb[u + 1]);
                } else if (m0 + u < NH) {
                    xs += bits(lb[u]);
                    xns += bits(hb[u]);
                }
            }
        }
        x += x2;
        xn += xn2;
        // exponent fields: BL per low half, BH per high half carried in
        constexpr uint64_t XB = (uint64_t)NH * BL + (uint64_t)NHP * BH;
        uint64_t y = hd;
        constexpr uint64_t YB0 = ((K - 1) >= 0 && ((K - 1) & 1) == 0 && (K - 1) / 2 < ND) ? BH : 0;
        uint64_t yb = YB0, hdn = 0;
        if constexpr ((K & 1) == 0 && K / 2 < ND) {
            const double ai = a[K / 2];
            const double h = fma_rz(ai, ai, C104);
            const double l = fma_rz(ai, ai, sub_rn(C2, h));
            y += bits(l);
            yb += BL;
            hdn = bits(h);
        }
        const uint64_t v = 2 * (x - XB) + (y - yb) + carry;
        put(K, v & M52);
        sqr_col<ND, K + 1, SQB_, ACC2>(a, xn, hdn, v >> D, put);
    }
}

// sqr_scan: T = A^2 by product scanning, fully unrolled: column k sums the
// low halves of its cross products a_i a_j (i < j, i + j = k) and the high
// halves of column k-1's, once; the column is then doubled and the diagonal
// a_{k/2}^2 added (one 64-bit shift-add per column, not per product).  Column
// k's digit (< 2^52) is handed to put(k, v) as soon as it completes.
template <int ND, typename Put>
__host__ __device__ __forceinline__ void sqr_scan(const double (&a)[ND], Put put) {
    if constexpr (ND <= RSA_F64_SQLOOP) {
        uint64_t carry = 0;
        uint64_t hx[ND], hd = 0;          // high halves pending for the next column (cross, diagonal)
        int nhx = 0;
#pragma unroll
        for (int k = 0; k < 2 * ND; k++) {
            uint64_t x = 0, xb = 0;       // cross sum (raw patterns) and its exponent fields
#pragma unroll
            for (int m = 0; m < ND; m++)
                if (m < nhx) { x += hx[m]; xb += BH; }
            int nh = 0;
#pragma unroll
            for (int i = 0; i < ND; i++) {
                const int j = k - i;
                if (i < j && j < ND) {
                    const double h = fma_rz(a[i], a[j], C104);
                    const double l = fma_rz(a[i], a[j], sub_rn(C2, h));
                    x += bits(l);
                    xb += BL;
                    hx[nh++] = bits(h);
                }
            }
            nhx = nh;
            uint64_t y = hd, yb = (k > 0 && ((k - 1) & 1) == 0 && (k - 1) / 2 < ND) ? BH : 0;
            hd = 0;
            if ((k & 1) == 0 && k / 2 < ND) {
                const double ai = a[k / 2];
                const double h = fma_rz(ai, ai, C104);
                const double l = fma_rz(ai, ai, sub_rn(C2, h));
                y += bits(l);
                yb += BL;
                hd = bits(h);
            }
            const uint64_t v = 2 * (x - xb) + (y - yb) + carry;
            carry = v >> D;
            put(k, v & M52);
        }
    } else {
        sqr_col<ND, 0>(a, 0, 0, 0, put);
    }
}

// sqr_reduce: Montgomery reduction of T_low (in t): ND reduction-only CIOS
// iterations q = t_0 n' mod 2^52; t = (t + q n) / 2^52.  Software-pipelined:
// the new column 0 is complete once the j = 1 product is in, so the next
// quotient digit (an IMAD/LOP/DADD chain) is computed there and overlaps the
// remaining ND-2 products.  Leaves column p carrying BH + (ND-1-p)(BL+BH).
template <int ND, int RU>
__host__ __device__ __forceinline__ void sqr_reduce(uint64_t (&t)[ND], const double* __restrict__ nd, uint64_t np,
                                                    double c104) {
    uint64_t bias0 = BL;
    double qd = digit_to_double(((t[0] & M52) * np) & M52);
    // RSA_F64_NREG: n's digits held in registers for the loop (A's registers are
    // free here) instead of ND/2 shared-memory pair loads per iteration (A/B)
    [[maybe_unused]] double nr[RSA_F64_NREG ? ND : 2];
    if constexpr (RSA_F64_NREG != 0) {
#pragma unroll
        for (int g = 0; g < ND / 2; g++) nd_pair(nd, g, nr[2 * g], nr[2 * g + 1]);
    }
    auto npair = [&](int g, double& x, double& y) {
        if constexpr (RSA_F64_NREG != 0) { x = nr[2 * g]; y = nr[2 * g + 1]; }
        else nd_pair(nd, g, x, y);
    };
#ifdef __CUDA_ARCH__
#pragma unroll RU
#endif
    for (int i = 0; i < ND; i++) {
        double n0, n1;
        npair(0, n0, n1);
        const double hq0 = fma_rz(qd, n0, c104);
        const double lq0 = fma_rz(qd, n0, sub_rn(C2, hq0));
        const uint64_t cr = (t[0] + bits(lq0) - bias0) >> D;   // column 0 is 0 mod 2^52
        const double hq1 = fma_rz(qd, n1, c104);
        const double lq1 = fma_rz(qd, n1, sub_rn(C2, hq1));
        t[0] = t[1] + bits(lq1) + bits(hq0) + cr;
        const double qnext = digit_to_double(((t[0] & M52) * np) & M52);
        uint64_t hqp = bits(hq1);
#pragma unroll
        for (int j = 2; j < ND; j++) {
            double nj = n1;
            if ((j & 1) == 0) npair(j / 2, nj, n1);
            const double h = fma_rz(qd, nj, c104);
            const double l = fma_rz(qd, nj, sub_rn(C2, h));
            t[j - 1] = t[j] + bits(l) + hqp;
            hqp = bits(h);
        }
        t[ND - 1] = hqp;
        qd = qnext;
        bias0 += BL + BH;
    }
}

// sqr_finish: t + T_high (high(p) = digit p of T_high), bias removed and
// carries normalised; out(p, digit) receives the result digits (< 2n in all:
// T / R + Q n / R < 4n^2/R + n < 2n).
template <int ND, typename High, typename Out>
__host__ __device__ __forceinline__ void sqr_finish(uint64_t (&t)[ND], High high, Out out) {
    if constexpr ((ND >= 64) ? RSA_F64_LOOKAHEAD_BIG : (ND <= 20 ? RSA_F64_LOOKAHEAD_SMALL : RSA_F64_LOOKAHEAD)) {
#pragma unroll
        for (int p = 0; p < ND; p++) t[p] = t[p] - (BH + (uint64_t)(ND - 1 - p) * (BL + BH)) + high(p);
        normalize<ND>(t);
#pragma unroll
        for (int p = 0; p < ND; p++) out(p, t[p]);
    } else {
        uint64_t carry = 0;
#pragma unroll
        for (int p = 0; p < ND; p++) {
            const uint64_t v = t[p] - (BH + (uint64_t)(ND - 1 - p) * (BL + BH)) + high(p) + carry;
            t[p] = v & M52;
            carry = v >> D;
            out(p, t[p]);
        }
    }
}

// (montsqr keeps its own inline copy of the scan / reduction / finish rather
// than calling sqr_scan / sqr_reduce / sqr_finish below: with the shared
// pieces ptxas schedules the 2048-bit squaring ~7% slower, 552K vs 591K
// decrypts/s, measured.)
// A <- A^2 R^-1 (mod n), result < 2n for A < 2n (squarings are ~85% of a
// full-d exponentiation).  A square has ND (ND+1)/2 distinct digit products
// instead of ND^2, so this is separated operand scanning (SOS):
//   1. T = A^2 by product scanning, fully unrolled: column k sums the low
//      halves of its cross products a_i a_j (i < j, i + j = k) and the high
//      halves of column k-1's, once; the column is then doubled and the
//      diagonal a_{k/2}^2 added (one 64-bit shift-add per column, not per
//      product).  The 2 ND digits of T go to this thread's shared-memory
//      slot th[k * stride] as they complete (registers hold A and the
//      in-flight products only), and the low half is reloaded into t.
//   2. Reduction-only CIOS on t: q = t_0 n' mod 2^52; t = (t + q n) / 2^52,
//      ND times (loop, not unrolled).
//   3. t + T_high, normalised: T / R + Q n / R < 4n^2/R + n < 2n.
template <int ND, int RU = (ND >= 40 ? kRU : kRUs)>
__host__ __device__ __forceinline__ void montsqr(double (&a)[ND], const double* __restrict__ nd, uint64_t np,
                                                 double c104, uint64_t (&t)[ND], uint64_t* th, int stride) {
    // 1. T = A^2
    if constexpr (ND > RSA_F64_SQLOOP) {
        sqr_scan<ND>(a, [&](int kk, uint64_t v) { th[kk * stride] = v; });
    } else {
        uint64_t carry = 0;
        uint64_t hx[ND], hd = 0;          // high halves pending for the next column (cross, diagonal)
        int nhx = 0;
#pragma unroll
        for (int k = 0; k < 2 * ND; k++) {
            uint64_t x = 0, xb = 0;       // cross sum (raw patterns) and its exponent fields
#pragma unroll
            for (int m = 0; m < ND; m++)
                if (m < nhx) { x += hx[m]; xb += BH; }
            int nh = 0;
#pragma unroll
            for (int i = 0; i < ND; i++) {
                const int j = k - i;
                if (i < j && j < ND) {
                    const double h = fma_rz(a[i], a[j], C104);
                    const double l = fma_rz(a[i], a[j], sub_rn(C2, h));
                    x += bits(l);
                    xb += BL;
                    hx[nh++] = bits(h);
                }
            }
            nhx = nh;
            uint64_t y = hd, yb = (k > 0 && ((k - 1) & 1) == 0 && (k - 1) / 2 < ND) ? BH : 0;
            hd = 0;
            if ((k & 1) == 0 && k / 2 < ND) {
                const double ai = a[k / 2];
                const double h = fma_rz(ai, ai, C104);
                const double l = fma_rz(ai, ai, sub_rn(C2, h));
                y += bits(l);
                yb += BL;
                hd = bits(h);
            }
            const uint64_t v = 2 * (x - xb) + (y - yb) + carry;
            carry = v >> D;
            th[k * stride] = v & M52;
        }
    }
#pragma unroll
    for (int p = 0; p < ND; p++) t[p] = th[p * stride];
    // 2. reduce T_low.  Software-pipelined: the new column 0 is complete once
    // the j = 1 product is in, so the next quotient digit (an IMAD/LOP/DADD
    // chain) is computed there and overlaps the remaining ND-2 products.
    uint64_t bias0 = BL;
    double qd = digit_to_double(((t[0] & M52) * np) & M52);
    // RSA_F64_NREG: n's digits held in registers for the loop (A's registers are
    // free here) instead of ND/2 shared-memory pair loads per iteration (A/B)
    [[maybe_unused]] double nr[RSA_F64_NREG ? ND : 2];
    if constexpr (RSA_F64_NREG != 0) {
#pragma unroll
        for (int g = 0; g < ND / 2; g++) nd_pair(nd, g, nr[2 * g], nr[2 * g + 1]);
    }
    auto npair = [&](int g, double& x, double& y) {
        if constexpr (RSA_F64_NREG != 0) { x = nr[2 * g]; y = nr[2 * g + 1]; }
        else nd_pair(nd, g, x, y);
    };
#ifdef __CUDA_ARCH__
#pragma unroll RU
#endif
    for (int i = 0; i < ND; i++) {
        double n0, n1;
        npair(0, n0, n1);
        const double hq0 = fma_rz(qd, n0, c104);
        const double lq0 = fma_rz(qd, n0, sub_rn(C2, hq0));
        const uint64_t cr = (t[0] + bits(lq0) - bias0) >> D;   // column 0 is 0 mod 2^52
        const double hq1 = fma_rz(qd, n1, c104);
        const double lq1 = fma_rz(qd, n1, sub_rn(C2, hq1));
        t[0] = t[1] + bits(lq1) + bits(hq0) + cr;
        const double qnext = digit_to_double(((t[0] & M52) * np) & M52);
        uint64_t hqp = bits(hq1);
#pragma unroll
        for (int j = 2; j < ND; j++) {
            double nj = n1;
            if ((j & 1) == 0) npair(j / 2, nj, n1);
            const double h = fma_rz(qd, nj, c104);
            const double l = fma_rz(qd, nj, sub_rn(C2, h));
            t[j - 1] = t[j] + bits(l) + hqp;
            hqp = bits(h);
        }
        t[ND - 1] = hqp;
        qd = qnext;
        bias0 += BL + BH;
    }
    // 3. + T_high, normalise (column p carries BH + (ND-1-p)(BL+BH))
    if constexpr ((ND >= 64) ? RSA_F64_LOOKAHEAD_BIG : (ND <= 20 ? RSA_F64_LOOKAHEAD_SMALL : RSA_F64_LOOKAHEAD)) {
#pragma unroll
        for (int p = 0; p < ND; p++) t[p] = t[p] - (BH + (uint64_t)(ND - 1 - p) * (BL + BH)) + th[(ND + p) * stride];
        normalize<ND>(t);
#pragma unroll
        for (int p = 0; p < ND; p++) a[p] = digit_to_double(t[p]);
    } else {
        uint64_t carry = 0;
#pragma unroll
        for (int p = 0; p < ND; p++) {
            const uint64_t v = t[p] - (BH + (uint64_t)(ND - 1 - p) * (BL + BH)) + th[(ND + p) * stride] + carry;
            t[p] = v & M52;
            carry = v >> D;
            a[p] = digit_to_double(t[p]);
        }
    }
}

// The same squaring with A living in this thread's ND-digit shared-memory
// slot aslot[k * stride] (the 4096-bit kernel, where a second slot does not
// fit): A is read into registers, T_low goes to the slot as its columns
// complete, T_high stays in registers: column k uses a_i only for
// i >= k - ND + 1, so once column k >= ND is done a_0 .. a_{k-ND+1} are dead
// and T_high digit k - ND takes one of their registers (the live count stays
// ~2 ND registers).  T_low and T_high then swap places
// (t <- slot, slot <- T_high), the reduction runs on t, and the result goes
// back to the slot.  ND (ND+1)/2 + ND^2 digit products instead of the
// multiply's 2 ND^2.  The slot is accessed through one type (64-bit patterns)
// only, so no load or store in here can be reordered across another.
template <int ND, int RU = (ND >= 40 ? kRU : kRUs)>
__host__ __device__ __forceinline__ void montsqr_slot(const double* __restrict__ nd, uint64_t np, double c104,
                                                      uint64_t (&t)[ND], double* aslot, int stride) {
    uint64_t* const s64 = reinterpret_cast<uint64_t*>(aslot);
    double a[ND];
#pragma unroll
    for (int k = 0; k < ND; k++) a[k] = from_bits(s64[k * stride]);
    uint64_t th[ND];
    sqr_scan<ND>(a, [&](int k, uint64_t v) {
        if (k < ND) s64[k * stride] = v;
        else th[k - ND] = v;
    });
#pragma unroll
    for (int p = 0; p < ND; p++) {
        t[p] = s64[p * stride];
        s64[p * stride] = th[p];
    }
    sqr_reduce<ND, RU>(t, nd, np, c104);
    sqr_finish<ND>(t, [&](int p) { return s64[p * stride]; },
                   [&](int p, uint64_t d) { s64[p * stride] = bits(digit_to_double(d)); });
}

// r <- r - n if r >= n (digits, r < 2n); nu: n's digits as integers
template <int ND>
__host__ __device__ __forceinline__ void canonicalise(uint64_t (&r)[ND], const uint64_t* __restrict__ nu) {
    uint64_t d[ND];
    int64_t br = 0;
#pragma unroll
    for (int p = 0; p < ND; p++) {
        const int64_t v = (int64_t)r[p] - (int64_t)nu[p] + br;
        d[p] = (uint64_t)v & M52;
        br = v >> D;                 // 0 or -1
    }
    const bool keep = br < 0;        // r < n
#pragma unroll
    for (int p = 0; p < ND; p++) r[p] = keep ? r[p] : d[p];
}

}  // namespace f64
}  // namespace rsa_b200
