// mont_group.cuh -- Montgomery multiplication with TPI lanes per packet
// (generalises mont_pair.cuh from 2 to TPI in {2, 4} lanes; S = TPI * L limbs).
//
// Lane k of a group owns positions [kL, (k+1)L) of the CIOS accumulator and
// the matching limbs of A and n:
//   T = sum_k 2^(32 kL) T_k          (T_k in lane k's X/Y/hi, redundant)
//   per CIOS iteration:  T_k += A_k b_i ;  m = (T_0 mod 2^32) n'  (lane 0,
//   broadcast) ;  T_k += m n_k ;  T /= 2^32: lane k+1's lowest word moves to
//   lane k's top position L-1 (shfl_down within the group; the top lane gets 0).
//   Lane k's overflow (< 4 * 2^(32L)) stays in its hi word until the end,
//   where it is rippled into lane k+1 (TPI-1 rounds), then T - n is formed with
//   the borrow rippled upwards (TPI rounds) and the group's top lane decides.
// n_k differs per lane: read from shared memory (odd/even limbs).  Pinned on
// CPU by tests/test_cios_model.py (the pair case; the group case is the same
// recurrence with more boundaries).
#pragma once
#include <stdint.h>

#include "mont.cuh"
#include "mont_pair.cuh"

namespace rsa_b200 {

template <int L, int TPI>
__device__ __forceinline__ void cios_step_group(uint32_t (&X)[L], uint32_t (&Y)[L], uint32_t& hi,
                                                const uint32_t (&a)[L], uint32_t b,
                                                const uint4* __restrict__ nodd4, const uint4* __restrict__ neven4,
                                                uint32_t n0inv, int src, bool top_lane) {
    static_assert(L % 8 == 0, "L must be a multiple of 8");
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int j = 1; j + 2 < L; j += 2) {
        madc_lo_cc(Y[j - 1], a[j], b, Y[j + 1]);
        madc_hi_cc(Y[j], a[j], b, Y[j + 2]);
    }
    madc_lo_cc(Y[L - 2], a[L - 1], b, 0u);
    madc_hi_cc(Y[L - 1], a[L - 1], b, hi);
    addc(hi, 0u, 0u);
    mad_lo_cc(X[0], a[0], b, X[0]);
    madc_hi_cc(X[1], a[0], b, X[1]);
#pragma unroll
    for (int j = 2; j < L; j += 2) {
        madc_lo_cc(X[j], a[j], b, X[j]);
        madc_hi_cc(X[j + 1], a[j], b, X[j + 1]);
    }
    addc_cc(Y[L - 1], Y[L - 1], 0u);
    addc(hi, hi, 0u);
    const uint32_t m = __shfl_sync(0xffffffffu, X[0] * n0inv, src);
#pragma unroll
    for (int q = 0; q < L / 8; q++) {
        const uint4 v = lds128(nodd4 + q);
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
#pragma unroll
    for (int q = 0; q < L / 8; q++) {
        const uint4 v = lds128(neven4 + q);
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
    addc_cc(Y[L - 1], Y[L - 1], 0u);
    addc(hi, hi, 0u);
    // lane k+1's dropped word -> lane k's new top (Y is even-aligned after the swap)
    uint32_t w = __shfl_down_sync(0xffffffffu, X[0], 1, TPI);
    w = top_lane ? 0u : w;
    add_cc(Y[L - 1], Y[L - 1], w);
    addc(hi, hi, 0u);
}

template <int L, int TPI>
__device__ __forceinline__ void montmul_group(uint32_t (&a)[L], const uint4* __restrict__ bslot, int pstride,
                                              const uint4* __restrict__ nodd4, const uint4* __restrict__ neven4,
                                              uint32_t n0inv, int lig) {
    constexpr int NG = (TPI * L) / 4;
    const int src = (threadIdx.x & 31) & ~(TPI - 1);
    const bool top_lane = (lig == TPI - 1);
    uint32_t X[L], Y[L], hi = 0;
#pragma unroll
    for (int k = 0; k < L; k++) { X[k] = 0; Y[k] = 0; }
#pragma unroll 1
    for (int g0 = 0; g0 < NG; g0 += 2) {
#pragma unroll
        for (int g = g0; g < g0 + 2; g++) {
            const uint4 bv = bslot[g * pstride];
            cios_step_group<L, TPI>(X, Y, hi, a, bv.x, nodd4, neven4, n0inv, src, top_lane);
            cios_step_group<L, TPI>(Y, X, hi, a, bv.y, nodd4, neven4, n0inv, src, top_lane);
            cios_step_group<L, TPI>(X, Y, hi, a, bv.z, nodd4, neven4, n0inv, src, top_lane);
            cios_step_group<L, TPI>(Y, X, hi, a, bv.w, nodd4, neven4, n0inv, src, top_lane);
        }
    }
    // local merge: r_k = X + (Y pre-shift) + hi * 2^(32 L)
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int k = 1; k + 1 < L; k++) addc_cc(X[k], X[k], Y[k + 1]);
    addc_cc(X[L - 1], X[L - 1], 0u);
    addc(hi, hi, 0u);
    // ripple the overflow words upwards: round r moves lane r's hi into lane r+1
#pragma unroll
    for (int r = 0; r < TPI - 1; r++) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, hi, 1, TPI);
        const uint32_t inc = (lig == r + 1) ? up : 0u;
        if (lig == r) hi = 0u;                   // moved to lane r+1
        add_cc(X[0], X[0], inc);
#pragma unroll
        for (int k = 1; k < L; k++) addc_cc(X[k], X[k], 0u);
        addc(hi, hi, 0u);
    }
    // T = sum_k 2^(32kL) r_k + 2^(32 S) hi_top < 2n.  d = T - n with the borrow
    // rippled upwards: round r finalises lane r.
    const uint32_t* nodd = reinterpret_cast<const uint32_t*>(nodd4);
    const uint32_t* neven = reinterpret_cast<const uint32_t*>(neven4);
    uint32_t bin = 0, br = 0;
#pragma unroll
    for (int r = 0; r < TPI; r++) {
        uint32_t dummy;
        sub_cc(dummy, 0u, bin);                  // borrow flag = bin
#pragma unroll
        for (int k = 0; k < L; k++) subc_cc(a[k], X[k], (k & 1) ? nodd[k >> 1] : neven[k >> 1]);
        subc(br, 0u, 0u);                        // 0xFFFFFFFF if this lane borrowed out
        const uint32_t below = __shfl_up_sync(0xffffffffu, br, 1, TPI);
        if (r + 1 < TPI && lig == r + 1) bin = below & 1u;
        (void)dummy;
    }
    // top lane: keep = hi - borrow = hi + br  (0 if T >= n, 0xFFFFFFFF if T < n)
    const uint32_t bfin = hi + br;
    const uint32_t keep = __shfl_sync(0xffffffffu, bfin, src + TPI - 1);
#pragma unroll
    for (int k = 0; k < L; k++) a[k] = (X[k] & keep) | (a[k] & ~keep);
}

}  // namespace rsa_b200
