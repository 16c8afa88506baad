// tc_digits.cuh -- the CUDA-core half of the tensor-core Montgomery multiply
// (modexp_tc.cu): the product T = A B on the FP64 pipe (52-bit digits, the
// exact DFMA.RZ split of mont_f64.cuh) streamed out as 32-bit words for the
// tensor-core reduction (mont_tc.cuh), and the reduced words back to digits.
//
//   mul_scan:  T = A B by product scanning (column k = sum_{i+j=k} a_i b_j),
//              each column's digit handed to put(k, d) as soon as it is final
//              (f64::sqr_scan is the squaring counterpart: ND (ND+1)/2
//              products instead of ND^2)
//   Packer:    digit stream (52-bit digits in order) -> 32-bit words, each
//              word handed to word(w, v) as soon as its 32 bits are in
//   words_to_digits: 32-bit words -> 52-bit digits as doubles (A of the next op)
//
// Host-compilable: tests/test_tc_model.py runs them against Python integers.
#pragma once
#include <stdint.h>

#include "mont_f64.cuh"

namespace rsa_b200 {
namespace tcd {

using f64::BH;
using f64::BL;
using f64::C104;
using f64::C2;
using f64::D;
using f64::M52;
using f64::bits;
using f64::fma_rz;
using f64::sub_rn;

// T = A B (2 ND digits), column by column.  b(j) returns digit j of B (a
// double < 2^52).  Column k's sum: the low halves of its products, the high
// halves of column k-1's (summed as they are produced), and the carry; every
// term < 2^52 and at most 2 ND of them, so the 64-bit sums never overflow.
template <int ND, typename BF, typename Put>
__host__ __device__ __forceinline__ void mul_scan(const double (&a)[ND], BF b, Put put) {
    uint64_t carry = 0, hprev = 0, hprevb = 0;
#pragma unroll
    for (int k = 0; k < 2 * ND; k++) {
        uint64_t x = hprev, xb = hprevb, hs = 0, hsb = 0;
#pragma unroll
        for (int i = 0; i < ND; i++) {
            const int j = k - i;
            if (j >= 0 && j < ND) {
                const double bj = b(j);
                const double h = fma_rz(a[i], bj, C104);
                const double l = fma_rz(a[i], bj, sub_rn(C2, h));
                x += bits(l);
                xb += BL;
                hs += bits(h);
                hsb += BH;
            }
        }
        const uint64_t v = x - xb + carry;
        carry = v >> D;
        put(k, v & M52);
        hprev = hs;
        hprevb = hsb;
    }
}

// digit stream -> 32-bit words (words 0 .. NWORDS-1; bits beyond are dropped).
// put(k, d) must be called for k = 0, 1, 2, ... in order.
template <int NWORDS, typename Word>
struct Packer {
    Word word;
    uint64_t prev;
    __host__ __device__ __forceinline__ void put(int k, uint64_t d) {
        const int lo = D * k, hi = D * k + D;
#pragma unroll
        for (int w = lo / 32; w < NWORDS && 32 * w + 32 <= hi; w++) {
            const int sb = 32 * w;
            uint32_t v;
            if (sb >= lo) v = (uint32_t)(d >> (sb - lo));
            else v = (uint32_t)((prev >> (sb - lo + D)) | (d << (lo - sb)));
            word(w, v);
        }
        prev = d;
    }
};

// words (w(i) = word i, 0 beyond the number) -> ND digits of 52 bits as doubles
template <int ND, typename WF>
__host__ __device__ __forceinline__ void words_to_digits(WF wd, double (&a)[ND]) {
#pragma unroll
    for (int k = 0; k < ND; k++) {
        const int o = D * k, w0 = o / 32, sh = o % 32;
        uint64_t v = ((uint64_t)wd(w0) >> sh) | ((uint64_t)wd(w0 + 1) << (32 - sh));
        if (sh > 12) v |= (uint64_t)wd(w0 + 2) << (64 - sh);
        a[k] = f64::digit_to_double(v & M52);
    }
}

}  // namespace tcd
}  // namespace rsa_b200
