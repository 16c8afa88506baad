// tc_digits.cuh -- the CUDA-core half of the tensor-core Montgomery multiply
// (modexp_tc.cu): the product T = A B on the FP64 pipe (52-bit digits, the
// exact DFMA.RZ split of mont_f64.cuh) streamed out as 32-bit words for the
// tensor-core reduction (mont_tc.cuh), and the reduced words back to digits.
//
//   mul_rows:  T = A B by rows, the loop rolled (the fully unrolled column
//              scan of the first version was ~160 KB of SASS), the digits
//              handed to put(k, d) in order (f64::sqr_col / sqr_scan are the
//              squaring's column scans: ND (ND+1)/2 products instead of ND^2)
//   Packer:    digit stream (52-bit digits in order) -> 32-bit words, each
//              word handed to word(w, v) as soon as its 32 bits are in
//   words_to_digits: 32-bit words -> 52-bit digits as doubles (A of the next op)
//
// Host-compilable: tests/test_tc_model.py runs them against Python integers.
#pragma once
#include <stdint.h>

#include <type_traits>

#include "mont_f64.cuh"

#ifndef TCD_SQ_PAIR_UNROLL
#define TCD_SQ_PAIR_UNROLL 1   // sqr_blocks' pair loop unroll: A/B at 4096 bits, 2 -> 97.3-98.4K vs 105.8-106.0K
#endif

namespace rsa_b200 {
namespace tcd {

constexpr int kSqPairUnroll = TCD_SQ_PAIR_UNROLL;

using f64::BH;
using f64::BL;
using f64::C104;
using f64::C2;
using f64::D;
using f64::M52;
using f64::bits;
using f64::fma_rz;
using f64::sub_rn;

// T = A B by rows (operand scanning), the loop NOT unrolled (~40 products of
// code instead of an unrolled ND^2 column scan): iteration j adds a_i b_j to ND running
// 64-bit columns (low half to column j+i, high half to j+i+1), emits the
// completed column j through lowout(j, digit), and shifts the columns down
// by one in place (t[i-1] = t[i] + ...: CIOS's rename without the q n row).
// lowout may overwrite b's digit j (b(j) is read one iteration ahead).  After
// the loop the low digits are replayed into put in order (lowin(k) returns
// what lowout(k) stored), then the high columns are normalised into put.
// Column bounds: <= 2 terms < 2^52 per column per iteration, <= ND iterations.
// mul_rows_f: the same with A read through a(i) (registers, or the thread's
// shared-memory slot at 4096 bits) and, for REPLAY = false, no replay of the
// low digits (lowout then consumes them, e.g. as words written at run time).
//
// NR < ND rows (b(0 .. NR-1)) give the partial product A (b_0 .. b_{NR-1}):
// lowout receives its columns 0 .. NR-1, put its columns NR .. NR+ND-1
// (model-tested; a split of one product's rows over two threads was measured
// slower at 4096 bits, profiles/r02_ab_summary.md).
template <int ND, bool REPLAY, typename AF, typename BF, typename LO, typename LI, typename Put, int NR = ND>
__host__ __device__ __forceinline__ void mul_rows_f(AF a, BF b, LO lowout, LI lowin, Put put) {
    static_assert(NR >= 1 && NR <= ND, "rows");
    uint64_t t[ND];
#pragma unroll
    for (int i = 0; i < ND; i++) t[i] = 0;
    uint64_t bias = BL, carry = 0;
    double bj = b(0);
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int j = 0; j < NR; j++) {
        const double bn = b(j + 1 < NR ? j + 1 : j);
        const double a0 = a(0);
        const double h0 = fma_rz(a0, bj, C104);
        const double l0 = fma_rz(a0, bj, sub_rn(C2, h0));
        const uint64_t v = t[0] + bits(l0) - bias + carry;   // column j: (j+1) lows, j highs
        carry = v >> D;
        lowout(j, v & M52);
        uint64_t hp = bits(h0);
#pragma unroll
        for (int i = 1; i < ND; i++) {
            const double ai = a(i);
            const double h = fma_rz(ai, bj, C104);
            const double l = fma_rz(ai, bj, sub_rn(C2, h));
            t[i - 1] = t[i] + bits(l) + hp;
            hp = bits(h);
        }
        t[ND - 1] = hp;
        bias += BL + BH;
        bj = bn;
    }
    if constexpr (REPLAY) {
#pragma unroll
        for (int k = 0; k < NR; k++) put(k, lowin(k));
    }
    // t[p] = column NR + p: min(NR, ND-1-p) lows, min(NR, ND-p) highs
#pragma unroll
    for (int p = 0; p < ND; p++) {
        const uint64_t nl = (NR < ND - 1 - p) ? NR : ND - 1 - p, nh = (NR < ND - p) ? NR : ND - p;
        const uint64_t v = t[p] - (nl * BL + nh * BH) + carry;
        carry = v >> D;
        put(NR + p, v & M52);
    }
}

template <int ND, typename BF, typename LO, typename LI, typename Put>
__host__ __device__ __forceinline__ void mul_rows(const double (&a)[ND], BF b, LO lowout, LI lowin, Put put) {
    mul_rows_f<ND, true>([&](int i) -> double { return a[i]; }, b, lowout, lowin, put);
}

// sqr_blocks: T = A^2 with the triangle's ND (ND+1) / 2 digit products in a
// ROLLED loop (mul_rows_f's A A costs ND^2; the unrolled column scan sqr_col
// is too much code at ND = 80).  A's digits are cut into NB = ND / BS blocks;
// step s (0 .. 2 NB - 1) adds every block pair (p, s - p), p < s - p, as a
// static BS x BS product, and for even s the diagonal block's strict upper
// triangle, into a 2 BS-column window w (column BS s + d), then finishes
// columns BS s .. BS s + BS - 1:
//   T_c = 2 (W_c - bias_c) + [a_{c/2}^2's low (c even) / high (c odd) half] + carry,
// bias_c = nl(c) BL + nl(c - 1) BH with nl(c) = #{i < j < ND : i + j = c} (the
// exponent fields of the summed bit patterns), and slides the window by BS.
// Columns 0 .. ND-1 leave through lowout(c, digit); columns ND + k through
// hiout(k, digit) -- the caller may store them over A's block s - NB, which no
// later step reads -- and are replayed from hiin(k) into put(ND + k) at the end.
template <int ND, int BS, typename AF, typename LO, typename HO, typename HI, typename Put>
__host__ __device__ __forceinline__ void sqr_blocks(AF a, LO lowout, HO hiout, HI hiin, Put put) {
    static_assert(ND % BS == 0 && BS % 2 == 0, "blocks");
    constexpr int NB = ND / BS;
    uint64_t w[2 * BS];
#pragma unroll
    for (int d = 0; d < 2 * BS; d++) w[d] = 0;
    uint64_t carry = 0;
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int s = 0; s < 2 * NB; s++) {
        const int pmin = s - (NB - 1) > 0 ? s - (NB - 1) : 0, pend = (s + 1) / 2;   // p < s - p
#ifdef __CUDA_ARCH__
#pragma unroll kSqPairUnroll
#endif
        for (int p = pmin; p < pend; p++) {
            double x[BS], y[BS];
#pragma unroll
            for (int k = 0; k < BS; k++) {
                x[k] = a(BS * p + k);
                y[k] = a(BS * (s - p) + k);
            }
#pragma unroll
            for (int i = 0; i < BS; i++) {
                uint64_t hp = 0;
#pragma unroll
                for (int k = 0; k < BS; k++) {
                    const double h = fma_rz(x[k], y[i], C104);
                    const double l = fma_rz(x[k], y[i], sub_rn(C2, h));
                    w[i + k] += bits(l) + hp;
                    hp = bits(h);
                }
                w[i + BS] += hp;
            }
        }
        if ((s & 1) == 0 && s / 2 < NB) {      // diagonal block s / 2: pairs k1 < k2
            double x[BS];
#pragma unroll
            for (int k = 0; k < BS; k++) x[k] = a(BS * (s / 2) + k);
#pragma unroll
            for (int k1 = 0; k1 < BS - 1; k1++) {
                uint64_t hp = 0;
#pragma unroll
                for (int k2 = k1 + 1; k2 < BS; k2++) {
                    const double h = fma_rz(x[k1], x[k2], C104);
                    const double l = fma_rz(x[k1], x[k2], sub_rn(C2, h));
                    w[k1 + k2] += bits(l) + hp;
                    hp = bits(h);
                }
                w[k1 + BS] += hp;
            }
        }
        // finish columns c = BS s + d with the digit squares a_i^2, i = BS s / 2 + m.  Every
        // column of a step lies on one side of ND (ND % BS == 0), where nl is linear:
        //   c <  ND: nl(BS s + e) = (BS/2) s + (e+1)/2
        //   c >= ND: nl(BS s + e) = ND - 1 - (BS/2) s + (e+1)/2 - e      (e = -1 .. BS-1)
        // (the two agree at c = ND - 1), so bias_c = base_s (BL + BH) + a static constant.
        auto finish = [&](auto hiside) {
            constexpr bool HIGH = decltype(hiside)::value;
            const uint64_t base = HIGH ? (uint64_t)(ND - 1 - (BS / 2) * s) : (uint64_t)((BS / 2) * s);
            const uint64_t q2 = 2 * base * (BL + BH);
#pragma unroll
            for (int m = 0; m < BS / 2; m++) {
                const double ai = a(BS * s / 2 + m);
                const double h = fma_rz(ai, ai, C104);
                const double l = fma_rz(ai, ai, sub_rn(C2, h));
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int d = 2 * m + e;
                    constexpr auto g = [](int x) -> int64_t { return HIGH ? (x + 1) / 2 - x : (x + 1) / 2; };
                    // 2 bias_c - 2 base (BL + BH) + the square half's exponent field
                    const uint64_t k = 2 * ((uint64_t)g(d) * BL + (uint64_t)g(d - 1) * BH) + (e ? BH : BL);
                    const uint64_t v = 2 * w[d] + (e ? bits(h) : bits(l)) + carry - q2 - k;
                    carry = v >> D;
                    if constexpr (HIGH) hiout(BS * s + d - ND, v & M52);
                    else lowout(BS * s + d, v & M52);
                }
            }
        };
        if (s < NB) finish(std::false_type{});
        else finish(std::true_type{});
#pragma unroll
        for (int d = 0; d < BS; d++) {
            w[d] = w[d + BS];
            w[d + BS] = 0;
        }
    }
#pragma unroll
    for (int k = 0; k < ND; k++) put(ND + k, hiin(k));
}

// mul_blocks: T = A B in the same rolled block structure (every block pair
// (p, s - p) at step s, no doubling, no digit squares): column c finishes as
// W_c - bias_c + carry with bias_c = nm(c) BL + nm(c - 1) BH, nm(c) =
// #{i, j < ND : i + j = c} (a per-step base plus static constants).  A's block s - NB is dead at step s (hiout may
// overwrite it); b is only read.
template <int ND, int BS, typename AF, typename BF, typename LO, typename HO, typename HI, typename Put>
__host__ __device__ __forceinline__ void mul_blocks(AF a, BF b, LO lowout, HO hiout, HI hiin, Put put) {
    static_assert(ND % BS == 0, "blocks");
    constexpr int NB = ND / BS;
    uint64_t w[2 * BS];
#pragma unroll
    for (int d = 0; d < 2 * BS; d++) w[d] = 0;
    uint64_t carry = 0;
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int s = 0; s < 2 * NB; s++) {
        const int pmin = s - (NB - 1) > 0 ? s - (NB - 1) : 0, pend = s < NB - 1 ? s + 1 : NB;
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
        for (int p = pmin; p < pend; p++) {
            double x[BS], y[BS];
#pragma unroll
            for (int k = 0; k < BS; k++) {
                x[k] = a(BS * p + k);
                y[k] = b(BS * (s - p) + k);
            }
#pragma unroll
            for (int i = 0; i < BS; i++) {
                uint64_t hp = 0;
#pragma unroll
                for (int k = 0; k < BS; k++) {
                    const double h = fma_rz(x[k], y[i], C104);
                    const double l = fma_rz(x[k], y[i], sub_rn(C2, h));
                    w[i + k] += bits(l) + hp;
                    hp = bits(h);
                }
                w[i + BS] += hp;
            }
        }
        // nm is linear on each side of ND (as in sqr_blocks): c = BS s + e,
        //   c < ND: nm = BS s + e + 1;   c >= ND: nm = 2 ND - 1 - BS s - e
        auto finish = [&](auto hiside) {
            constexpr bool HIGH = decltype(hiside)::value;
            const uint64_t base = HIGH ? (uint64_t)(2 * ND - 1 - BS * s) : (uint64_t)(BS * s);
            const uint64_t q = base * (BL + BH);
#pragma unroll
            for (int d = 0; d < BS; d++) {
                constexpr auto g = [](int x) -> int64_t { return HIGH ? -x : x + 1; };
                const uint64_t k = (uint64_t)g(d) * BL + (uint64_t)g(d - 1) * BH;
                const uint64_t v = w[d] + carry - q - k;
                carry = v >> D;
                if constexpr (HIGH) hiout(BS * s + d - ND, v & M52);
                else lowout(BS * s + d, v & M52);
                w[d] = w[d + BS];
                w[d + BS] = 0;
            }
        };
        if (s < NB) finish(std::false_type{});
        else finish(std::true_type{});
    }
#pragma unroll
    for (int k = 0; k < ND; k++) put(ND + k, hiin(k));
}

// digit stream -> 32-bit words at RUN TIME (digits arrive inside a rolled loop):
// each 52-bit digit joins the < 32 pending bits in a 64-bit buffer and whole
// words leave through emit(v), in order (one or two per digit).
// SEL: no branches; emit(v, valid) is called twice per digit, the second time
// with valid = whether the digit completed a second word (the emitter stores
// an invalid word to a scratch slot and does not advance).
template <typename Emit, bool SEL = false>
struct WordEmitter {
    Emit emit;
    uint64_t acc;
    int nb;
    __host__ __device__ __forceinline__ void digit(uint64_t d) {
        const uint64_t lo64 = acc | (d << nb);
        const uint64_t hi = nb > 12 ? (d >> (64 - nb)) : 0;   // bits 64 .. nb + 51
        uint64_t rest = (lo64 >> 32) | (hi << 32);
        int n = nb + 20;
        if constexpr (SEL) {
            emit((uint32_t)lo64, true);
            const bool two = n >= 32;
            emit((uint32_t)rest, two);
            rest = two ? rest >> 32 : rest;
            n = two ? n - 32 : n;
        } else {
            emit((uint32_t)lo64);
            if (n >= 32) {
                emit((uint32_t)rest);
                rest >>= 32;
                n -= 32;
            }
        }
        acc = rest;
        nb = n;
    }
};

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

// words (w(i) = word i, 0 beyond the number) -> ND digits of 52 bits as
// doubles, handed to out(k, digit) (words_to_digits: into an array)
template <int ND, typename WF, typename OF>
__host__ __device__ __forceinline__ void words_to_digits_f(WF wd, OF out) {
#pragma unroll
    for (int k = 0; k < ND; k++) {
        const int o = D * k, w0 = o / 32, sh = o % 32;
        uint64_t v = ((uint64_t)wd(w0) >> sh) | ((uint64_t)wd(w0 + 1) << (32 - sh));
        if (sh > 12) v |= (uint64_t)wd(w0 + 2) << (64 - sh);
        out(k, f64::digit_to_double(v & M52));
    }
}

template <int ND, typename WF>
__host__ __device__ __forceinline__ void words_to_digits(WF wd, double (&a)[ND]) {
    words_to_digits_f<ND>(wd, [&](int k, double v) { a[k] = v; });
}

}  // namespace tcd
}  // namespace rsa_b200
