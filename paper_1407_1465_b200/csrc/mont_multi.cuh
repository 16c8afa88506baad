// mont_multi.cuh -- Montgomery arithmetic with a per-thread modulus (multi-key
// batches).
//
// Same CIOS / squaring schemes as mont.cuh and mont_sqr.cuh (even/odd
// IMAD.WIDE.U32.X chains, free shift), but n differs per packet, so it cannot
// be a constant-bank operand: each thread keeps its n in its shared-memory
// slot, split into odd- and even-indexed limbs (limb-major across the block,
// conflict free), read with one LDS.128 per four products of a reduction
// chain.  The loads are volatile so ptxas keeps them next to their chains
// instead of hoisting S registers' worth of n out of the loop.
#pragma once
#include <stdint.h>

#include "mont.cuh"
#include "mont_sqr.cuh"

namespace rsa_b200 {

// Per-thread n in shared memory: group q of the odd limbs
// (n[8q+1], n[8q+3], n[8q+5], n[8q+7]) is at nodd[q * stride]; even limbs
// (n[8q], n[8q+2], n[8q+4], n[8q+6]) at neven[q * stride].  S % 8 == 0.
// STRIDE (uint4 elements between a thread's groups) is the block size, a
// compile-time constant, so every address folds into an LDS immediate.
template <int STRIDE>
struct NSharedT {
    const uint4* nodd;
    const uint4* neven;
    static constexpr int stride = STRIDE;
    __device__ __forceinline__ uint4 odd(int q) const { return ldsv(nodd + q * STRIDE); }
    __device__ __forceinline__ uint4 even(int q) const { return ldsv(neven + q * STRIDE); }
    __device__ __forceinline__ uint32_t limb(int j) const {
        const uint32_t* p = reinterpret_cast<const uint32_t*>((j & 1) ? nodd : neven);
        const int k = j >> 1;                  // index among odd (even) limbs
        return p[(k >> 2) * STRIDE * 4 + (k & 3)];
    }
    static __device__ __forceinline__ uint4 ldsv(const uint4* p) {
        uint4 v;
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
        asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
        return v;
    }
};

// Per-thread n held in registers (classes small enough to afford S more
// registers): same interface as NSharedT, no shared-memory traffic for n.
// STRIDE is still the b slot stride of montmul_sm.
template <int S, int STRIDE>
struct NRegsT {
    const uint32_t (&n)[S];
    static constexpr int stride = STRIDE;
    __device__ __forceinline__ uint4 odd(int q) const {
        return make_uint4(n[8 * q + 1], n[8 * q + 3], n[8 * q + 5], n[8 * q + 7]);
    }
    __device__ __forceinline__ uint4 even(int q) const {
        return make_uint4(n[8 * q], n[8 * q + 2], n[8 * q + 4], n[8 * q + 6]);
    }
    __device__ __forceinline__ uint32_t limb(int j) const { return n[j]; }
};

// T += m * n (odd limbs into Y, shifted as in the CIOS step when `rshift`;
// in place otherwise) -- helpers for the chains below.
template <int S, class NShared>
__device__ __forceinline__ void red_odd_inplace(uint32_t (&Y)[S], uint32_t& hi, uint32_t m, const NShared& n) {
    uint4 nxt = n.odd(0);
#pragma unroll
    for (int q = 0; q < S / 8; q++) {
        const uint4 v = nxt;                   // prefetched one group ahead (LDS latency)
        if (q + 1 < S / 8) nxt = n.odd(q + 1);
        const int j = 8 * q + 1;
        if (q == 0) mad_lo_cc(Y[0], v.x, m, Y[0]);
        else madc_lo_cc(Y[j - 1], v.x, m, Y[j - 1]);
        madc_hi_cc(Y[j], v.x, m, Y[j]);
        madc_lo_cc(Y[j + 1], v.y, m, Y[j + 1]);
        madc_hi_cc(Y[j + 2], v.y, m, Y[j + 2]);
        madc_lo_cc(Y[j + 3], v.z, m, Y[j + 3]);
        madc_hi_cc(Y[j + 4], v.z, m, Y[j + 4]);
        madc_lo_cc(Y[j + 5], v.w, m, Y[j + 5]);
        madc_hi_cc(Y[j + 6], v.w, m, Y[j + 6]);
    }
    addc(hi, hi, 0u);
}

template <int S, class NShared>
__device__ __forceinline__ void red_even_inplace(uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t& hi, uint32_t m,
                                                 const NShared& n) {
    uint4 nxt = n.even(0);
#pragma unroll
    for (int q = 0; q < S / 8; q++) {
        const uint4 v = nxt;
        if (q + 1 < S / 8) nxt = n.even(q + 1);
        const int j = 8 * q;
        if (q == 0) mad_lo_cc(X[0], v.x, m, X[0]);
        else madc_lo_cc(X[j], v.x, m, X[j]);
        madc_hi_cc(X[j + 1], v.x, m, X[j + 1]);
        madc_lo_cc(X[j + 2], v.y, m, X[j + 2]);
        madc_hi_cc(X[j + 3], v.y, m, X[j + 3]);
        madc_lo_cc(X[j + 4], v.z, m, X[j + 4]);
        madc_hi_cc(X[j + 5], v.z, m, X[j + 5]);
        madc_lo_cc(X[j + 6], v.w, m, X[j + 6]);
        madc_hi_cc(X[j + 7], v.w, m, X[j + 7]);
    }
    addc_cc(Y[S - 1], Y[S - 1], 0u);
    addc(hi, hi, 0u);
}

// CIOS step with a per-thread n (cf. cios_step in mont.cuh)
template <int S, class NShared>
__device__ __forceinline__ void cios_step_sm(uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t& hi,
                                             const uint32_t (&a)[S], uint32_t b, const NShared& n, uint32_t n0inv) {
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int j = 1; j + 2 < S; j += 2) {
        madc_lo_cc(Y[j - 1], a[j], b, Y[j + 1]);
        madc_hi_cc(Y[j], a[j], b, Y[j + 2]);
    }
    madc_lo_cc(Y[S - 2], a[S - 1], b, 0u);
    madc_hi_cc(Y[S - 1], a[S - 1], b, hi);
    addc(hi, 0u, 0u);
    mad_lo_cc(X[0], a[0], b, X[0]);
    madc_hi_cc(X[1], a[0], b, X[1]);
#pragma unroll
    for (int j = 2; j < S; j += 2) {
        madc_lo_cc(X[j], a[j], b, X[j]);
        madc_hi_cc(X[j + 1], a[j], b, X[j + 1]);
    }
    addc_cc(Y[S - 1], Y[S - 1], 0u);
    addc(hi, hi, 0u);
    const uint32_t m = X[0] * n0inv;
    red_odd_inplace<S, NShared>(Y, hi, m, n);
    red_even_inplace<S, NShared>(X, Y, hi, m, n);
}

// reduction-only step with the shift done by the odd chain (cf. red_step)
template <int S, class NShared>
__device__ __forceinline__ void red_step_sm(uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t& hi, const NShared& n,
                                            uint32_t n0inv) {
    uint4 nxt = n.odd(0);
    add_cc(X[0], X[0], Y[1]);
    const uint32_t m = X[0] * n0inv;
#pragma unroll
    for (int q = 0; q < S / 8; q++) {
        const uint4 v = nxt;
        if (q + 1 < S / 8) nxt = n.odd(q + 1);
        const int j = 8 * q + 1;
        madc_lo_cc(Y[j - 1], v.x, m, Y[j + 1]);
        madc_hi_cc(Y[j], v.x, m, Y[j + 2]);
        madc_lo_cc(Y[j + 1], v.y, m, Y[j + 3]);
        madc_hi_cc(Y[j + 2], v.y, m, Y[j + 4]);
        madc_lo_cc(Y[j + 3], v.z, m, Y[j + 5]);
        madc_hi_cc(Y[j + 4], v.z, m, Y[j + 6]);
        if (q + 1 < S / 8) {
            madc_lo_cc(Y[j + 5], v.w, m, Y[j + 7]);
            madc_hi_cc(Y[j + 6], v.w, m, Y[j + 8]);
        } else {                                   // last pair: positions S-1, S
            madc_lo_cc(Y[S - 2], v.w, m, 0u);
            madc_hi_cc(Y[S - 1], v.w, m, hi);
        }
    }
    addc(hi, 0u, 0u);
    red_even_inplace<S, NShared>(X, Y, hi, m, n);
}

// merge (X, Y pre-shift, hi) + optional addend, conditional subtract -> a
template <int S, class NShared>
__device__ __forceinline__ void finish_sm(uint32_t (&a)[S], uint32_t (&X)[S], uint32_t (&Y)[S], uint32_t hi,
                                          const uint32_t* addend, const NShared& n) {
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int k = 1; k + 1 < S; k++) addc_cc(X[k], X[k], Y[k + 1]);
    addc_cc(X[S - 1], X[S - 1], 0u);
    addc(hi, hi, 0u);
    if (addend) {
        add_cc(X[0], X[0], addend[0]);
#pragma unroll
        for (int k = 1; k < S; k++) addc_cc(X[k], X[k], addend[k]);
        addc(hi, hi, 0u);
    }
#pragma unroll
    for (int q = 0; q < S / 8; q++) {
        const uint4 e = n.even(q), o = n.odd(q);
        const uint32_t nv[8] = {e.x, o.x, e.y, o.y, e.z, o.z, e.w, o.w};
#pragma unroll
        for (int t = 0; t < 8; t++) {
            if (q == 0 && t == 0) sub_cc(a[0], X[0], nv[0]);
            else subc_cc(a[8 * q + t], X[8 * q + t], nv[t]);
        }
    }
    uint32_t keep;
    subc(keep, hi, 0u);
#pragma unroll
    for (int k = 0; k < S; k++) a[k] = (X[k] & keep) | (a[k] & ~keep);
}

#ifndef RSA_MULTI_RED
#define RSA_MULTI_RED 16   // montsqr_sm reduction steps per loop trip (A/B, multi-key RSA-2048 encrypt: 4/8/16 -> 22.0M/22.8M/23.2M; with 16 ptxas keeps the rotated registers off the IMAD pipe)
#endif
#ifndef RSA_MULTI_MUL
#define RSA_MULTI_MUL 8    // montmul_sm CIOS steps per loop trip (multiple of 4)
#endif

// A <- A * B R^-1 mod n (B in this thread's smem slot, group g at bslot[g*stride])
template <int S, class NShared>
__device__ __forceinline__ void montmul_sm(uint32_t (&a)[S], const uint4* __restrict__ bslot, int /*stride*/,
                                           const NShared& n, uint32_t n0inv) {
    constexpr int stride = NShared::stride;
    uint32_t X[S], Y[S], hi = 0;
#pragma unroll
    for (int k = 0; k < S; k++) { X[k] = 0; Y[k] = 0; }
    constexpr int MG = (RSA_MULTI_MUL < S ? RSA_MULTI_MUL : S) / 4;   // limb groups per loop trip
#pragma unroll 1
    for (int g0 = 0; g0 < S / 4; g0 += MG) {
#pragma unroll
        for (int g = g0; g < g0 + MG; g++) {
            const uint4 bv = bslot[g * stride];
            cios_step_sm<S, NShared>(X, Y, hi, a, bv.x, n, n0inv);
            cios_step_sm<S, NShared>(Y, X, hi, a, bv.y, n, n0inv);
            cios_step_sm<S, NShared>(X, Y, hi, a, bv.z, n, n0inv);
            cios_step_sm<S, NShared>(Y, X, hi, a, bv.w, n, n0inv);
        }
    }
    finish_sm<S, NShared>(a, X, Y, hi, nullptr, n);
}

// A <- A^2 R^-1 mod n (triangle of mont_sqr.cuh, reduction with smem n)
template <int S, class NShared>
__device__ __forceinline__ void montsqr_sm(uint32_t (&a)[S], const NShared& n, uint32_t n0inv) {
    uint32_t T[2 * S];
    square_full<S>(a, T);
    uint32_t X[S], Y[S], hi = 0;
#pragma unroll
    for (int k = 0; k < S; k++) { X[k] = T[k]; Y[k] = 0; }
    // RSA_MULTI_RED: reduction steps per loop trip (at most S)
    constexpr int RED = RSA_MULTI_RED < S ? RSA_MULTI_RED : S;
#pragma unroll 1
    for (int i = 0; i < S; i += RED) {
#pragma unroll
        for (int u = 0; u < RED; u += 2) {
            red_step_sm<S, NShared>(X, Y, hi, n, n0inv);
            red_step_sm<S, NShared>(Y, X, hi, n, n0inv);
        }
    }
    finish_sm<S, NShared>(a, X, Y, hi, T + S, n);
}

}  // namespace rsa_b200
