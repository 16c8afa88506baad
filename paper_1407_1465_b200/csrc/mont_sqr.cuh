// mont_sqr.cuh -- Montgomery squaring A <- A^2 R^-1 mod n (thread per packet).
//
// The squarings are ~87% of a full-d exponentiation,
// and a square has only S(S+1)/2 distinct limb products.  Instead of CIOS
// (2S^2 + S products) this computes, in 1.5 S^2 + 1.5 S products:
//   1. T' = sum_{i<j} a_i a_j 2^(32(i+j))  by product scanning (column by
//      column, two interleaved 3-word accumulators per column; every product
//      is one IMAD.WIDE.U32 with carry-out plus an IADD3.X on the ALU pipe);
//   2. T = 2 T' + sum_i a_i^2 2^(64 i)  (one add chain, one IMAD.WIDE.X chain
//      on register-aligned even pairs);
//   3. Montgomery reduction of T_low = T mod R with S reduction-only CIOS
//      steps (the odd m*n chain does the free shift, as in mont.cuh);
//   4. + T_high, one conditional subtraction (acc <= n, T_high < n - 1).
// Pinned on CPU by tests/test_cios_model.py::test_montsqr_model.
#pragma once
#include <stdint.h>

#include "mont.cuh"

namespace rsa_b200 {

// One reduction-only CIOS step: T += m n, T /= 2^32 (X even-aligned, Y pre-shift).
template <int S>
__device__ __forceinline__ void red_step(uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t& hi,
                                         const uint32_t* __restrict__ n, uint32_t n0inv) {
    add_cc(X[0], X[0], Y[1]);
    const uint32_t m = X[0] * n0inv;
#pragma unroll
    for (int j = 1; j + 2 < S; j += 2) {
        madc_lo_cc(Y[j - 1], n[j], m, Y[j + 1]);
        madc_hi_cc(Y[j], n[j], m, Y[j + 2]);
    }
    madc_lo_cc(Y[S - 2], n[S - 1], m, 0u);
    madc_hi_cc(Y[S - 1], n[S - 1], m, hi);
    addc(hi, 0u, 0u);
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

// (c1:c0) += x * y, c2 += carry
__device__ __forceinline__ void mac3(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t x, uint32_t y) {
    mad_lo_cc(c0, x, y, c0);
    madc_hi_cc(c1, x, y, c1);
    addc(c2, c2, 0u);
}

// T = a^2 (2S limbs): steps 1-3 above (independent of the modulus)
template <int S>
__device__ __forceinline__ void square_full(const uint32_t (&a)[S], uint32_t (&T)[2 * S]) {
    // 1. off-diagonal triangle, product scanning
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    T[0] = 0;
#pragma unroll
    for (int k = 1; k <= 2 * S - 3; k++) {
        const int lo = (k - S + 1) > 0 ? (k - S + 1) : 0;
        const int top = (k - 1) / 2;
        uint32_t d0 = 0, d1 = 0, d2 = 0;
#pragma unroll
        for (int i = lo; i <= top; i++) {
            if (((i - lo) & 1) == 0) mac3(c0, c1, c2, a[i], a[k - i]);
            else mac3(d0, d1, d2, a[i], a[k - i]);
        }
        add_cc(c0, c0, d0);
        addc_cc(c1, c1, d1);
        addc(c2, c2, d2);
        T[k] = c0;
        c0 = c1;
        c1 = c2;
        c2 = 0;
    }
    T[2 * S - 2] = c0;
    T[2 * S - 1] = c1;
    // 2. double
    add_cc(T[1], T[1], T[1]);
#pragma unroll
    for (int k = 2; k < 2 * S; k++) addc_cc(T[k], T[k], T[k]);      // no carry out: 2T' < 2^(64 S)
    // 3. + diagonal a_i^2 at (2i, 2i+1)
    mad_lo_cc(T[0], a[0], a[0], T[0]);
    madc_hi_cc(T[1], a[0], a[0], T[1]);
#pragma unroll
    for (int i = 1; i < S; i++) {
        madc_lo_cc(T[2 * i], a[i], a[i], T[2 * i]);
        madc_hi_cc(T[2 * i + 1], a[i], a[i], T[2 * i + 1]);
    }
}

// a <- T R^-1 mod n for a 2S-limb T with T_high = T >> 32S < n (steps 3-4):
// reduction-only CIOS steps on T_low, then + T_high, one conditional subtract.
template <int S>
__device__ __forceinline__ void reduce_wide(uint32_t (&a)[S], const uint32_t (&T)[2 * S],
                                            const uint32_t* __restrict__ n, uint32_t n0inv) {
    // 4. reduce T_low
    uint32_t X[S], Y[S], hi = 0;
#pragma unroll
    for (int k = 0; k < S; k++) { X[k] = T[k]; Y[k] = 0; }
    if constexpr (S <= 8) {
#pragma unroll
        for (int i = 0; i < S; i += 2) {
            red_step<S>(X, Y, hi, n, n0inv);
            red_step<S>(Y, X, hi, n, n0inv);
        }
    } else {
#pragma unroll 1
        for (int i = 0; i < S; i += 8) {
            red_step<S>(X, Y, hi, n, n0inv);
            red_step<S>(Y, X, hi, n, n0inv);
            red_step<S>(X, Y, hi, n, n0inv);
            red_step<S>(Y, X, hi, n, n0inv);
            red_step<S>(X, Y, hi, n, n0inv);
            red_step<S>(Y, X, hi, n, n0inv);
            red_step<S>(X, Y, hi, n, n0inv);
            red_step<S>(Y, X, hi, n, n0inv);
        }
    }
    // merge the redundant accumulator, add T_high
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int k = 1; k + 1 < S; k++) addc_cc(X[k], X[k], Y[k + 1]);
    addc_cc(X[S - 1], X[S - 1], 0u);
    addc(hi, hi, 0u);
    add_cc(X[0], X[0], T[S]);
#pragma unroll
    for (int k = 1; k < S; k++) addc_cc(X[k], X[k], T[S + k]);
    addc(hi, hi, 0u);
    // conditional subtraction (r < 2n)
    sub_cc(a[0], X[0], n[0]);
#pragma unroll
    for (int k = 1; k < S; k++) subc_cc(a[k], X[k], n[k]);
    uint32_t keep;
    subc(keep, hi, 0u);
#pragma unroll
    for (int k = 0; k < S; k++) a[k] = (X[k] & keep) | (a[k] & ~keep);
}

template <int S>
__device__ __forceinline__ void montsqr(uint32_t (&a)[S], const uint32_t* __restrict__ n, uint32_t n0inv) {
    uint32_t T[2 * S];
    square_full<S>(a, T);
    reduce_wide<S>(a, T, n, n0inv);
}

}  // namespace rsa_b200
