// mont_tc.cuh -- Montgomery reduction of a 128-packet tile on the tensor core
// (operands of KB bytes, R = 2^(8 KB), n < R odd, byte digits for the MMAs;
// KB = 128 / 256 / 512 for the 1024- / 2048- / 4096-bit classes.  The numbers
// below are for KB = 256; every column index scales with KB).
//
// The operation is the reduction half of Fig 3's "(u*v) mod m" (PAPER.md:89,
// sec. 3.6.1) realised by Montgomery's method, in
// separated form with a FULL-WIDTH quotient:
//
//   T = A B  (< n R, computed on the CUDA cores by the caller)
//   m = (T mod R) n' mod R,            n' = -n^-1 mod R
//   U = (T + m n) / R  (< 2n),   U -= n if U >= n   ->   U = A B R^-1 mod n
//
// Both products have a constant operand (n', n: one key per batch), so for a
// tile of 128 packets they are [128 x 256] x [256 x N] u8 matrix products on
// the tensor core (tc_i8.cuh) against Toeplitz matrices, read out of TMEM as
// exact column sums c_j = sum_k x_k y_{j-k} (<= KB 255^2: < 2^24 at KB <= 256,
// < 2^25 at 512; s32 accumulators) whose carries the thread of each packet
// resolves:
//   GEMM1: columns 0..255 of T_low x n'   (two N = 128 blocks; the upper
//          block-triangle is zero and skipped: 12 MMAs of K = 32)
//   GEMM2: columns 252..507 of m x n       (8 MMAs, N = 256); columns
//          508..510 (6 byte products) on the CUDA cores.
// The carry out of the low half of T + m n: its value V = (T_low + sum_{j<256}
// c_j 2^(8j)) / R is an integer (T + m n = 0 mod R), and columns below 252
// move V 2^32 by less than 2^18 (c_j < 2^25), so V = ceil(X / 2^32) with
// X = T_low's top word + c_252 + c_253 2^8 + c_254 2^16 + c_255 2^24.
//
// Shared memory (per CTA of two tiles): the n' and n "strips" (every
// Toeplitz block is a row window of one strip, see tc_i8.cuh), and per tile a
// 128 x 256-byte staging buffer holding T_low, then m (A operand of both
// GEMMs).  TMEM: 256 columns per tile (GEMM1 and GEMM2 reuse them).
#pragma once
#include <stdint.h>

#include "tc_i8.cuh"

namespace rsa_b200 {
namespace tc {

constexpr int TILE = 128;                     // packets per tile (MMA M, TMEM lanes)
constexpr int STAGE_LBO = TILE * 16;          // bytes between 16-byte K chunks of a staging buffer

// Geometry for operands of KB bytes (R = 2^(8 KB); KB = 256 at 2048 bits, 128 at 1024)
template <int KB_>
struct Geom {
    static constexpr int KB = KB_;
    static constexpr int NW = KB / 4;                         // 32-bit words per operand
    static constexpr int STAGE_BYTES = KB / 16 * STAGE_LBO;   // 128 rows x KB bytes
    // n' strip: GEMM1 blocks c0 = 128 b, K blocks I <= 4 b + 3: rows rho = c0 + nn - 32 I in [-96, KB)
    static constexpr int NP_RHO0 = -96, NP_ROWS = KB + 96, NP_LBO = NP_ROWS * 16;
    // n strip: GEMM2 columns G2_C0 .. G2_C0 + KB - 1, K blocks 0 .. KB/32 - 1: rows [28, 2 KB - 5]
    static constexpr int G2_C0 = KB - 4;
    static constexpr int N_RHO0 = G2_C0 - (KB - 32), N_ROWS = 2 * KB - 32, N_LBO = N_ROWS * 16;
    static constexpr int NP_STRIP_BYTES = 2 * NP_LBO, N_STRIP_BYTES = 2 * N_LBO;
    static constexpr int G2_N = KB < 256 ? KB : 256;          // MMA N of GEMM2
    static constexpr int G2_NB = KB / G2_N;                   // GEMM2 N blocks per K block (2 at KB = 512)
    static_assert(KB == 128 || KB == 256 || KB == 512, "operand widths of the TC kernels");
};

template <int KB, int TILES>
struct __align__(16) TcShared {
    using G = Geom<KB>;
    uint8_t stage[TILES][G::STAGE_BYTES];     // per tile: T_low, then m
    uint8_t np_strip[G::NP_STRIP_BYTES];
    uint8_t n_strip[G::N_STRIP_BYTES];
    uint32_t nw[G::NW];                       // n as words (conditional subtraction)
    // per tile; at KB = 512 a second one per tile (index TILES + tile, the address
    // mbar + 8 TILES): GEMM2's first N half (RSA_TC_SPLIT512)
    unsigned long long mbar[KB == 512 ? 2 * TILES : TILES];
    uint32_t tmem_base;
};

// strip byte (chunk q, row rho, byte b) = y_{rho - 16 q - b} (0 outside [0, KB))
template <int KB, int TILES>
__device__ __forceinline__ void build_strips(TcShared<KB, TILES>& sh, const uint8_t* __restrict__ npb,
                                             const uint8_t* __restrict__ nb) {
    using G = Geom<KB>;
    for (int i = threadIdx.x; i < G::NP_STRIP_BYTES; i += blockDim.x) {
        const int q = i / G::NP_LBO, rem = i % G::NP_LBO, rho = rem / 16 + G::NP_RHO0, b = rem % 16;
        const int idx = rho - 16 * q - b;
        sh.np_strip[i] = (idx >= 0 && idx < KB) ? npb[idx] : 0;
    }
    for (int i = threadIdx.x; i < G::N_STRIP_BYTES; i += blockDim.x) {
        const int q = i / G::N_LBO, rem = i % G::N_LBO, rho = rem / 16 + G::N_RHO0, b = rem % 16;
        const int idx = rho - 16 * q - b;
        sh.n_strip[i] = (idx >= 0 && idx < KB) ? nb[idx] : 0;
    }
}

// staging address of 16-byte chunk c (bytes 16c .. 16c+15) of tile row r
template <int KB, int TILES>
__device__ __forceinline__ uint4* stage_chunk(TcShared<KB, TILES>& sh, int tile, int r, int c) {
    return reinterpret_cast<uint4*>(sh.stage[tile] + c * STAGE_LBO + r * 16);
}

// GEMM1 (m's columns 0 .. KB-1): N = 128 blocks c0 = 128 b with K blocks
// 0 .. 4b+3 (the rest of the block-triangle is zero)
template <int KB, int TILES>
__device__ __forceinline__ void issue_gemm1(TcShared<KB, TILES>& sh, int tile, uint32_t tmem) {
    using G = Geom<KB>;
    const uint32_t st = smem_u32(sh.stage[tile]), sp = smem_u32(sh.np_strip);
    constexpr uint32_t id = idesc_u8(128, 128);
#pragma unroll
    for (int blk = 0; blk < KB / 128; blk++) {
        const int c0 = 128 * blk;
#pragma unroll
        for (int I = 0; I < 4 + 4 * blk; I++) {
            const uint64_t a = sdesc(st + 2 * I * STAGE_LBO, STAGE_LBO, 128);
            const uint64_t b = sdesc(sp + (c0 - 32 * I - G::NP_RHO0) * 16, G::NP_LBO, 128);
            mma_u8(tmem + c0, a, b, id, I > 0);
        }
    }
}

#ifndef RSA_TC_SPLIT512
#define RSA_TC_SPLIT512 1   // KB = 512: GEMM2's two N halves completed separately (the first half's
#endif                      // carries resolve while the second computes; its readout writes registers only)

// one N block (h) of GEMM2
template <int KB, int TILES>
__device__ __forceinline__ void issue_gemm2_half(TcShared<KB, TILES>& sh, int tile, uint32_t tmem, int h) {
    using G = Geom<KB>;
    const uint32_t st = smem_u32(sh.stage[tile]), sn = smem_u32(sh.n_strip);
    constexpr uint32_t id = idesc_u8(128, G::G2_N);
#pragma unroll
    for (int I = 0; I < KB / 32; I++) {
        const uint64_t a = sdesc(st + 2 * I * STAGE_LBO, STAGE_LBO, 128);
        const uint64_t b = sdesc(sn + (G::G2_C0 + G::G2_N * h - 32 * I - G::N_RHO0) * 16, G::N_LBO, 128);
        mma_u8(tmem + G::G2_N * h, a, b, id, I > 0);
    }
}

// GEMM2 (columns G2_C0 .. G2_C0 + KB - 1 of m n): KB / G2_N blocks of N = G2_N per K block
template <int KB, int TILES>
__device__ __forceinline__ void issue_gemm2(TcShared<KB, TILES>& sh, int tile, uint32_t tmem) {
    using G = Geom<KB>;
    const uint32_t st = smem_u32(sh.stage[tile]), sn = smem_u32(sh.n_strip);
    constexpr uint32_t id = idesc_u8(128, G::G2_N);
#pragma unroll
    for (int h = 0; h < G::G2_NB; h++) {
#pragma unroll
        for (int I = 0; I < KB / 32; I++) {
            const uint64_t a = sdesc(st + 2 * I * STAGE_LBO, STAGE_LBO, 128);
            const uint64_t b = sdesc(sn + (G::G2_C0 + G::G2_N * h - 32 * I - G::N_RHO0) * 16, G::N_LBO, 128);
            mma_u8(tmem + G::G2_N * h, a, b, id, I > 0);
        }
    }
}

// 4 column sums at byte offsets 0, 8, 16, 24 of a word (independent per
// word: three IMAD.WIDE; the carries between words are resolved afterwards by
// one add-with-carry per word)
__device__ __forceinline__ uint64_t col4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    return (uint64_t)c0 + ((uint64_t)c1 << 8) + ((uint64_t)c2 << 16) + ((uint64_t)c3 << 24);
}

// carry-chain steps (PTX condition code; consecutive volatile asm statements,
// nothing between them writes CC)
__device__ __forceinline__ uint32_t add_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t addc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t addc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t sub_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t subc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Per-thread state of the reduction: the tile's TMEM columns and mbarrier phase.
struct TcTile {
    int tile;          // 0 or 1
    int r;             // row in the tile (0..127) = TMEM lane
    uint32_t tmem;     // this tile's first TMEM column (lane 0)
    uint32_t tlane;    // this warp's lane offset (32 (warp % 4)) << 16
    uint32_t mbar;
    uint32_t phase;    // bit 0: mbar's parity; bit 1 (KB = 512 split): the second barrier's
};

// U = (T + m n) / R reduced below n.  On entry T_low (words 0..63) is in the
// tile's staging buffer (written by this thread, generic proxy), t63 = its top
// word, th[] = T_high (words 64..127).  On exit th[] holds U < n.
// Carries: word w of a GEMM's output is P_w = sum_i c_{4w+i} 2^(8i) < 2^50,
// computed for 8 words at a time independently; the words then follow from
// one add-with-carry chain lo(P_w) + hi(P_{w-1}) + carry.
template <int KB, int TILES>
__device__ __forceinline__ void redc(TcShared<KB, TILES>& sh, TcTile& tt, uint32_t t63,
                                     uint32_t (&th)[Geom<KB>::NW]) {
    constexpr int NW = Geom<KB>::NW, NCH = KB / 32;   // words, 32-column TMEM chunks
    const int tile = tt.tile, r = tt.r;
    // ---- GEMM1: m's column sums
    fence_async_smem();
    fence_before();
    bar_sync(1 + tile, TILE);
    if (r == 0) {
        fence_after();
        issue_gemm1(sh, tile, tt.tmem);
        commit(tt.mbar);
    }
    mbar_wait(tt.mbar, tt.phase & 1);
    tt.phase ^= 1;
    fence_after();
    uint32_t hprev = 0;
    uint32_t m253 = 0, m254 = 0, m255 = 0;
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) {
        uint32_t v[32];
        tmem_ld32(tt.tmem + tt.tlane + 32 * ch, v);
        tmem_ld_wait();
        uint32_t lo[8], hi[8], w[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint64_t p = col4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            lo[q] = (uint32_t)p;
            hi[q] = (uint32_t)(p >> 32);
        }
        w[0] = add_cc(lo[0], hprev);
#pragma unroll
        for (int q = 1; q < 8; q++) w[q] = addc_cc(lo[q], hi[q - 1]);
        hprev = addc(hi[7], 0u);
        *stage_chunk(sh, tile, r, 2 * ch) = make_uint4(w[0], w[1], w[2], w[3]);
        *stage_chunk(sh, tile, r, 2 * ch + 1) = make_uint4(w[4], w[5], w[6], w[7]);
        if (ch == NCH - 1) {               // m's top bytes KB-3 .. KB-1
            m253 = (w[7] >> 8) & 0xFF;
            m254 = (w[7] >> 16) & 0xFF;
            m255 = w[7] >> 24;
        }
    }
    // ---- GEMM2: columns 252..507 of m n
    fence_async_smem();
    fence_before();
    bar_sync(1 + tile, TILE);
    constexpr bool SPLIT2 = (Geom<KB>::G2_NB == 2) && RSA_TC_SPLIT512;
    if (r == 0) {
        fence_after();
        if constexpr (SPLIT2) {
            issue_gemm2_half(sh, tile, tt.tmem, 0);
            commit(tt.mbar + 8 * TILES);
            issue_gemm2_half(sh, tile, tt.tmem, 1);
        } else {
            issue_gemm2(sh, tile, tt.tmem);
        }
        commit(tt.mbar);
    }
    // columns 2KB-4 .. 2KB-2 (the top byte products) meanwhile
    const uint32_t n63 = sh.nw[NW - 1];
    const uint32_t n253 = n63 >> 8 & 0xFF, n254 = n63 >> 16 & 0xFF, n255 = n63 >> 24;
    const uint32_t c508 = m253 * n255 + m254 * n254 + m255 * n253;
    const uint32_t c509 = m254 * n255 + m255 * n254;
    const uint32_t c510 = m255 * n255;
    if constexpr (SPLIT2) {
        mbar_wait(tt.mbar + 8 * TILES, (tt.phase >> 1) & 1);
        tt.phase ^= 2;
    } else {
        mbar_wait(tt.mbar, tt.phase & 1);
        tt.phase ^= 1;
    }
    fence_after();
    // TMEM column idx = global column KB-4 + idx.  Word w of U (bits 8 KB + 32 w)
    // is P_w over global columns KB + 4w .. KB + 3 + 4w = idx 4 + 4w .. 7 + 4w.
    // The carry V out of the low half enters as the "previous high" of word 0.
    uint32_t carry = 0;
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) {
        if (SPLIT2 && ch == NCH / 2) {     // second N half complete
            mbar_wait(tt.mbar, tt.phase & 1);
            tt.phase ^= 1;
            fence_after();
        }
        uint32_t v[32];
        tmem_ld32(tt.tmem + tt.tlane + 32 * ch, v);
        tmem_ld_wait();
        // words w0 + q, q = 0..7 (chunk 0: q = 0 is the low half's top columns)
        const int w0 = 8 * ch - 1;
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint64_t p = col4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            lo[q] = (uint32_t)p;
            hi[q] = (uint32_t)(p >> 32);
        }
        if (ch == 0) {
            // V = ceil((T_low's top word + c252 + c253 2^8 + c254 2^16 + c255 2^24) / 2^32)
            const uint64_t x = (uint64_t)t63 + lo[0] + ((uint64_t)hi[0] << 32);
            hprev = (uint32_t)((x + 0xFFFFFFFFull) >> 32);
        }
        // x_w = lo(P_w) + hi(P_{w-1}) (chain A; the previous chunk's carries
        // enter with the first word), U_w = th_w + x_w (chain B)
        const int q0 = (ch == 0) ? 1 : 0;
        uint32_t x[8];
        x[q0] = add_cc(lo[q0], hprev + carry);
#pragma unroll
        for (int q = q0 + 1; q < 8; q++) x[q] = addc_cc(lo[q], hi[q - 1]);
        hprev = addc(hi[7], 0u);
        th[w0 + q0] = add_cc(th[w0 + q0], x[q0]);
#pragma unroll
        for (int q = q0 + 1; q < 8; q++) th[w0 + q] = addc_cc(th[w0 + q], x[q]);
        carry = addc(0u, 0u);
    }
    // word NW-1 = columns 2KB-4 .. 2KB-1 (past the last chunk), then bit 8 KB
    {
        const uint64_t p = col4(c508, c509, c510, 0) + hprev + carry;
        th[NW - 1] = add_cc(th[NW - 1], (uint32_t)p);
        carry = addc(0u, (uint32_t)(p >> 32));
    }
    // U < 2n: subtract n once if U >= n (U's bit 2048 is `carry`).  The top
    // words decide unless they are equal (probability ~2^-32): then the full
    // borrow chain of U - n does.
    bool ge = carry != 0 || th[NW - 1] > n63;
    if (carry == 0 && th[NW - 1] == n63) {
        uint32_t borrow = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) borrow = (uint32_t)(((uint64_t)th[w] - sh.nw[w] - borrow) >> 32) & 1;
        ge = borrow == 0;
    }
    const uint32_t mask = ge ? 0xFFFFFFFFu : 0u;
    th[0] = sub_cc(th[0], sh.nw[0] & mask);
#pragma unroll
    for (int w = 1; w < NW; w++) th[w] = subc_cc(th[w], sh.nw[w] & mask);
}

}  // namespace tc
}  // namespace rsa_b200
