// mont_pair.cuh -- Montgomery multiplication with two lanes per packet, for
// moduli too wide for one thread's registers (S = 2L limbs, L = 64: 4096-bit).
//
// Same operation as mont.cuh (A * B * R^-1 mod n, R = 2^(32 S), canonical),
// same even/odd IMAD.WIDE.U32.X chains; the packet's accumulator is split by
// position between the lanes of a pair (lane 0: positions [0, L), lane 1:
// [L, 2L)), each lane owning the matching half of A:
//
//   T = T_0 + 2^(32 L) T_1          (T_l in lane l's X/Y/hi, redundant)
//   per CIOS iteration i:
//     T_l += A_l * b_i ;  m = (T_0 mod 2^32) n'  (lane 0, broadcast by shfl)
//     T_l += m * n_l   ;  T /= 2^32
//   The division: T_0 / 2^32 is exact; lane 1's lowest word (T_1 mod 2^32)
//   moves to lane 0's top position L-1 (one shfl_xor), the rest of T_1 shifts
//   locally.  Lane 0 never hands its overflow (< 4 * 2^(32 L)) to lane 1 during
//   the loop; it is added to lane 1 once, at the end, before the conditional
//   subtraction.  Both lanes execute the same instruction stream (no
//   divergence): the shuffles deliver lane 0's m to both lanes, and give lane 1
//   lane 0's X[0] (= 0 exactly after the reduction), so it adds nothing.
// n_l differs per lane, so it is read from shared memory (odd- and
// even-indexed limbs in separate arrays, one LDS.128 per 4 products) instead
// of the constant bank.  Pinned on CPU by tests/test_cios_model.py.
#pragma once
#include <stdint.h>

#include "mont.cuh"

namespace rsa_b200 {

// Shared-memory 128-bit load kept in program order among the carry-chain asm
// (so the compiler does not hoist all n limbs into registers at once).
__device__ __forceinline__ uint4 lds128(const uint4* p) {
    uint4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Lane-local n half in shared memory: nodd4[2q] = n_l[8q+1, 8q+3, 8q+5, 8q+7],
// neven4[2q] = n_l[8q, 8q+2, 8q+4, 8q+6]; the two lanes' groups are
// interleaved (16 B apart, different banks) so each LDS.128 of a warp -- two
// distinct addresses -- is a single wavefront.
template <int L>
__device__ __forceinline__ void cios_step_pair(uint32_t (&X)[L], uint32_t (&Y)[L], uint32_t& hi,
                                               const uint32_t (&a)[L], uint32_t b,
                                               const uint4* __restrict__ nodd4, const uint4* __restrict__ neven4,
                                               uint32_t n0inv, int src) {
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
    // quotient digit of the pair: lane 0's position-0 word
    const uint32_t m = __shfl_sync(0xffffffffu, X[0] * n0inv, src);
    // odd products m * n_j (j = 8q + 1, 3, 5, 7)
#pragma unroll
    for (int q = 0; q < L / 8; q++) {
        const uint4 v = lds128(nodd4 + 2 * q);
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
    // even products m * n_j (j = 8q, 8q + 2, 4, 6); lane 0's X[0] becomes 0
#pragma unroll
    for (int q = 0; q < L / 8; q++) {
        const uint4 v = lds128(neven4 + 2 * q);
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
    // the shift across the lane boundary: lane 1's dropped word -> lane 0's
    // new top position L-1 (Y is the even-aligned array after the swap)
    const uint32_t w = __shfl_xor_sync(0xffffffffu, X[0], 1);
    add_cc(Y[L - 1], Y[L - 1], w);
    addc(hi, hi, 0u);
}

// A <- A * B * R^-1 mod n for the lane's half of A (a[L]).  bslot: the
// packet's B slot, group g (4 limbs) at bslot[g * pstride], g < 2L/4.
// nodd4/neven4: this lane's n half (see above); nodd/neven: the same as
// uint32 arrays.  half: 0 or 1 (lane within the pair).
template <int L>
__device__ __forceinline__ void montmul_pair(uint32_t (&a)[L], const uint4* __restrict__ bslot, int pstride,
                                             const uint4* __restrict__ nodd4, const uint4* __restrict__ neven4,
                                             uint32_t n0inv, int half) {
    constexpr int NG = (2 * L) / 4;
    const int src = (threadIdx.x & 31) & ~1;
    uint32_t X[L], Y[L], hi = 0;
#pragma unroll
    for (int k = 0; k < L; k++) { X[k] = 0; Y[k] = 0; }
#pragma unroll 1
    for (int g0 = 0; g0 < NG; g0 += 2) {
#pragma unroll
        for (int g = g0; g < g0 + 2; g++) {
            const uint4 bv = bslot[g * pstride];
            cios_step_pair<L>(X, Y, hi, a, bv.x, nodd4, neven4, n0inv, src);
            cios_step_pair<L>(Y, X, hi, a, bv.y, nodd4, neven4, n0inv, src);
            cios_step_pair<L>(X, Y, hi, a, bv.z, nodd4, neven4, n0inv, src);
            cios_step_pair<L>(Y, X, hi, a, bv.w, nodd4, neven4, n0inv, src);
        }
    }
    // local merge: r_l = X + (Y pre-shift) + hi * 2^(32 L)
    add_cc(X[0], X[0], Y[1]);
#pragma unroll
    for (int k = 1; k + 1 < L; k++) addc_cc(X[k], X[k], Y[k + 1]);
    addc_cc(X[L - 1], X[L - 1], 0u);
    addc(hi, hi, 0u);
    // lane 0's overflow (its hi) enters lane 1 at position 0
    const uint32_t t0 = __shfl_xor_sync(0xffffffffu, hi, 1);
    const uint32_t inc = half ? t0 : 0u;
    add_cc(X[0], X[0], inc);
#pragma unroll
    for (int k = 1; k < L; k++) addc_cc(X[k], X[k], 0u);
    addc(hi, hi, 0u);
    // T = r_0 + 2^(32L) r_1 + 2^(64L) hi_1 < 2n.  d = T - n across the pair:
    // phase 1 gives lane 0's borrow, phase 2 redoes lane 1 with it.
    const uint32_t* nodd = reinterpret_cast<const uint32_t*>(nodd4);
    const uint32_t* neven = reinterpret_cast<const uint32_t*>(neven4);
    // limb k of this lane's n: odd/even array, group (k>>1)>>2 (stride 2 groups), component (k>>1)&3
#define NLIMB(k) (((k) & 1) ? nodd[(((k) >> 1) >> 2) * 8 + (((k) >> 1) & 3)] \
                            : neven[(((k) >> 1) >> 2) * 8 + (((k) >> 1) & 3)])
    sub_cc(a[0], X[0], neven[0]);
#pragma unroll
    for (int k = 1; k < L; k++) subc_cc(a[k], X[k], NLIMB(k));
    uint32_t br;
    subc(br, 0u, 0u);                          // 0xFFFFFFFF if borrow
    const uint32_t b0 = __shfl_xor_sync(0xffffffffu, br, 1);
    const uint32_t bin = half ? (b0 & 1u) : 0u;
    uint32_t dummy;
    sub_cc(dummy, 0u, bin);                     // sets the borrow flag iff bin
#pragma unroll
    for (int k = 0; k < L; k++) subc_cc(a[k], X[k], NLIMB(k));
#undef NLIMB
    uint32_t keep1;
    subc(keep1, hi, 0u);                        // lane 1: 0 if T >= n, 0xFFFFFFFF if T < n
    const uint32_t keep = __shfl_sync(0xffffffffu, keep1, src | 1);
#pragma unroll
    for (int k = 0; k < L; k++) a[k] = (X[k] & keep) | (a[k] & ~keep);
    (void)dummy;
}

}  // namespace rsa_b200
