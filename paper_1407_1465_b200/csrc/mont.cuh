// mont.cuh -- multi-precision Montgomery multiplication for sm_100a.
//
// Operation (Fig 3 "(u*v) mod m", PAPER.md:89,
// realised by Montgomery reduction): given A, B < 2^(32 S) with B < n and
// n odd, compute A * B * R^-1 mod n, R = 2^(32 S), canonical in [0, n).
//
// Shape: one thread owns one packet.  A lives in S registers; B streams in G
// limbs at a time from this thread's shared-memory slot (limb-major across the
// block, so LDS.128 is conflict free); n and n' are constant-bank operands
// (kernel parameter).  The accumulator is split across two register arrays so
// that every 32x32->64 product is ONE IMAD.WIDE.U32(.X) with predicate carry
// chains and every 64-bit accumulator pair is register-aligned:
//
//   X[k]   holds position k            (even-aligned pairs (2k, 2k+1))
//   Y[k]   holds position k + 1        (odd-aligned pairs)
//   hi     holds position S + 1
//
// One CIOS iteration (operand scanning, b_i, i = 0 .. S-1):
//   T += A * b_i ;  m = T_0 * n' mod 2^32 ;  T += m * n ;  T /= 2^32
// The division by 2^32 costs no instruction: the even array's content now sits
// at odd alignment shifted by two words, and the NEXT iteration's odd product
// chain reads Y[j+1], Y[j+2] and writes Y[j-1], Y[j] ("rshift"), so the two
// arrays swap roles every iteration and a loop unrolled by 2 closes the cycle.
// The one word left over at position 0 (old position 1) is folded in with a
// single add whose carry feeds the next odd chain.
//
// Bounds: with A < R and B < n every intermediate T < R + n < 2R, so T fits
// S limbs + 1 bit after each shift; every chain carry is captured (into the
// odd array's top word or `hi`), none is dropped.  The final T < 2n is brought
// into [0, n) by one branch-free conditional subtraction.
#pragma once
#include <stdint.h>

namespace rsa_b200 {

__device__ __forceinline__ void add_cc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void addc_cc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void addc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("addc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void sub_cc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void subc_cc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void subc(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("subc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
}
__device__ __forceinline__ void mad_lo_cc(uint32_t& d, uint32_t a, uint32_t b, uint32_t c) {
    asm volatile("mad.lo.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
}
__device__ __forceinline__ void madc_lo_cc(uint32_t& d, uint32_t a, uint32_t b, uint32_t c) {
    asm volatile("madc.lo.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
}
__device__ __forceinline__ void madc_hi_cc(uint32_t& d, uint32_t a, uint32_t b, uint32_t c) {
    asm volatile("madc.hi.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
}

// One CIOS iteration.  X: even-aligned array, Y: odd-aligned array in
// "pre-shift" form (Y[j] at position j-1, Y[1] = leftover word at position 0,
// position S-1 empty, `hi` at position S).  On return the roles are swapped:
// Y is even-aligned and X is the pre-shift odd array.
template <int S>
__device__ __forceinline__ void cios_step(uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t& hi,
                                          const uint32_t (&a)[S], uint32_t b,
                                          const uint32_t* __restrict__ n, uint32_t n0inv) {
    // fold the leftover word (position 0); its carry enters the odd chain
    add_cc(X[0], X[0], Y[1]);
    // odd products a_j * b, j odd, positions (j, j+1), with the shift by two
#pragma unroll
    for (int j = 1; j + 2 < S; j += 2) {
        madc_lo_cc(Y[j - 1], a[j], b, Y[j + 1]);
        madc_hi_cc(Y[j], a[j], b, Y[j + 2]);
    }
    madc_lo_cc(Y[S - 2], a[S - 1], b, 0u);
    madc_hi_cc(Y[S - 1], a[S - 1], b, hi);
    addc(hi, 0u, 0u);
    // even products a_j * b, j even, positions (j, j+1)
    mad_lo_cc(X[0], a[0], b, X[0]);
    madc_hi_cc(X[1], a[0], b, X[1]);
#pragma unroll
    for (int j = 2; j < S; j += 2) {
        madc_lo_cc(X[j], a[j], b, X[j]);
        madc_hi_cc(X[j + 1], a[j], b, X[j + 1]);
    }
    addc_cc(Y[S - 1], Y[S - 1], 0u);
    addc(hi, hi, 0u);
    // Montgomery quotient digit
    const uint32_t m = X[0] * n0inv;
    // odd products m * n_j
    mad_lo_cc(Y[0], n[1], m, Y[0]);
    madc_hi_cc(Y[1], n[1], m, Y[1]);
#pragma unroll
    for (int j = 3; j < S; j += 2) {
        madc_lo_cc(Y[j - 1], n[j], m, Y[j - 1]);
        madc_hi_cc(Y[j], n[j], m, Y[j]);
    }
    addc(hi, hi, 0u);
    // even products m * n_j; X[0] becomes 0
    mad_lo_cc(X[0], n[0], m, X[0]);
    madc_hi_cc(X[1], n[0], m, X[1]);
#pragma unroll
    for (int j = 2; j < S; j += 2) {
        madc_lo_cc(X[j], n[j], m, X[j]);
        madc_hi_cc(X[j + 1], n[j], m, X[j + 1]);
    }
    addc_cc(Y[S - 1], Y[S - 1], 0u);
    addc(hi, hi, 0u);
}

// After S CIOS iterations (S even, so X is even-aligned again):
// merge r = X + (Y pre-shift) + hi * 2^(32 S), then the conditional
// subtraction r - n (keep r if it borrowed) -> a, canonical in [0, n).
template <int S>
__device__ __forceinline__ void mont_finish(uint32_t (&a)[S], uint32_t (&X)[S], const uint32_t (&Y)[S], uint32_t hi,
                                            const uint32_t* __restrict__ n) {
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int k = 1; k + 1 < S; k++) addc_cc(X[k], X[k], Y[k + 1]);
    addc_cc(X[S - 1], X[S - 1], 0u);
    addc(hi, hi, 0u);
    sub_cc(a[0], X[0], n[0]);
#pragma unroll
    for (int k = 1; k < S; k++) subc_cc(a[k], X[k], n[k]);
    uint32_t keep;
    subc(keep, hi, 0u);               // 0 if r >= n, 0xFFFFFFFF if r < n
#pragma unroll
    for (int k = 0; k < S; k++) a[k] = (X[k] & keep) | (a[k] & ~keep);
}

// 2-limb Montgomery multiply by product scanning (S = 2, R = 2^64): columns 0..2
// of T = A B + m N accumulate in a 3-word window (c_k, c_k+1, c_k+2); m_0 and
// m_1 are taken when their column is complete.  Same result as montmul_regb<2>
// (A B R^-1 mod n, canonical for A < R, B < n) in fewer instructions than the
// two-step CIOS, whose odd/even split is pointless at S = 2.
__device__ __forceinline__ void montmul2_ps(uint32_t (&a)[2], const uint32_t (&b)[2], const uint32_t* __restrict__ n,
                                            uint32_t n0inv) {
    const uint32_t a0 = a[0], a1 = a[1], b0 = b[0], b1 = b[1], n0 = n[0], n1 = n[1];
    uint32_t c0, c1, c2, c3, c4, m0, m1;
    // column 0: a0 b0 + m0 n0 (low word becomes 0)
    asm("mul.lo.u32 %0, %2, %3;\n\t"
        "mul.hi.u32 %1, %2, %3;" : "=r"(c0), "=r"(c1) : "r"(a0), "r"(b0));
    m0 = c0 * n0inv;
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, 0, 0;" : "+r"(c0), "+r"(c1), "=r"(c2) : "r"(m0), "r"(n0));
    // column 1: a0 b1 + a1 b0 + m0 n1, then m1 n0
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "mad.lo.cc.u32 %0, %7, %8, %0;\n\t"
        "madc.hi.cc.u32 %1, %7, %8, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(c1), "+r"(c2), "=r"(c3) : "r"(a0), "r"(b1), "r"(a1), "r"(b0), "r"(m0), "r"(n1));
    m1 = c1 * n0inv;
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;" : "+r"(c1), "+r"(c2), "+r"(c3) : "r"(m1), "r"(n0));
    // column 2: a1 b1 + m1 n1 -> result (c4 : c3 : c2) < 2n
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(c2), "+r"(c3), "=r"(c4) : "r"(a1), "r"(b1), "r"(m1), "r"(n1));
    // conditional subtraction
    uint32_t d0, d1, keep;
    asm("sub.cc.u32 %0, %3, %5;\n\t"
        "subc.cc.u32 %1, %4, %6;\n\t"
        "subc.u32 %2, %7, 0;" : "=r"(d0), "=r"(d1), "=r"(keep) : "r"(c2), "r"(c3), "r"(n0), "r"(n1), "r"(c4));
    a[0] = keep ? c2 : d0;
    a[1] = keep ? c3 : d1;
}

template <int S> struct BVec;
template <> struct BVec<2> { typedef uint2 T; static constexpr int G = 2; };
template <int S> struct BVec { typedef uint4 T; static constexpr int G = 4; };

// A <- A * B * R^-1 mod n, canonical.  bslot points at this thread's first
// B group; group g is at bslot[g * stride].
template <int S>
__device__ __forceinline__ void montmul(uint32_t (&a)[S], const typename BVec<S>::T* __restrict__ bslot,
                                        int stride, const uint32_t* __restrict__ n, uint32_t n0inv) {
    constexpr int G = BVec<S>::G;
    uint32_t X[S], Y[S], hi = 0;
#pragma unroll
    for (int k = 0; k < S; k++) { X[k] = 0; Y[k] = 0; }

    if constexpr (S <= 8) {
#pragma unroll
        for (int g = 0; g < S / G; g++) {
            const typename BVec<S>::T bv = bslot[g * stride];
            cios_step<S>(X, Y, hi, a, bv.x, n, n0inv);
            cios_step<S>(Y, X, hi, a, bv.y, n, n0inv);
            if constexpr (G == 4) {
                cios_step<S>(X, Y, hi, a, bv.z, n, n0inv);
                cios_step<S>(Y, X, hi, a, bv.w, n, n0inv);
            }
        }
    } else {
        // 8 CIOS iterations per loop trip: with 4 per trip ptxas permutes the
        // rotated X/Y registers at the back edge with IMAD.MOV / XOR swaps
        // (fmaheavy slots); with 8 it allocates them in place.
#pragma unroll 1
        for (int g0 = 0; g0 < S / G; g0 += 2) {
#pragma unroll
            for (int g = g0; g < g0 + 2; g++) {
                const typename BVec<S>::T bv = bslot[g * stride];
                cios_step<S>(X, Y, hi, a, bv.x, n, n0inv);
                cios_step<S>(Y, X, hi, a, bv.y, n, n0inv);
                cios_step<S>(X, Y, hi, a, bv.z, n, n0inv);
                cios_step<S>(Y, X, hi, a, bv.w, n, n0inv);
            }
        }
    }

    mont_finish<S>(a, X, Y, hi, n);
}

// A <- A * B * R^-1 mod n with B in registers (small widths: no shared-memory
// staging; B may alias A -- every B word is read before A is written).
template <int S>
__device__ __forceinline__ void montmul_regb(uint32_t (&a)[S], const uint32_t (&b)[S],
                                             const uint32_t* __restrict__ n, uint32_t n0inv) {
    static_assert(S % 2 == 0, "S must be even");
    uint32_t X[S], Y[S], hi = 0;
#pragma unroll
    for (int k = 0; k < S; k++) { X[k] = 0; Y[k] = 0; }
#pragma unroll
    for (int i = 0; i < S; i += 2) {
        cios_step<S>(X, Y, hi, a, b[i], n, n0inv);
        cios_step<S>(Y, X, hi, a, b[i + 1], n, n0inv);
    }
    mont_finish<S>(a, X, Y, hi, n);
}

}  // namespace rsa_b200
