// modexp_tc.cu -- batched modular exponentiation with the Montgomery
// reduction on the tensor core (sm_100a), width classes S = 64 (1025..2048-bit
// moduli) and S = 32 (513..1024 bits; also the CRT halves of RSA-2048).
//
// Same contract and op list as modexp_kernel / modexp_f64_kernel: out[i] =
// base[i]^exp mod n for every packet (sec. 2, sec.
// 3.3), one thread per packet, the shared exponent's op list executed
// warp-uniformly.  Each Montgomery multiply A <- A B R^-1 mod n (R = 2^(32 S))
// is split between the two engines of the SM:
//   CUDA cores (FP64 pipe): T = A B by product scanning (tc_digits.cuh;
//     squarings by the compile-time-expanded f64::sqr_col, ND (ND+1)/2 = 820
//     digit products at S = 64 instead of the 2420 of a full FP64 Montgomery
//     squaring; multiplies by the rolled row form tcd::mul_rows), streamed out
//     as words: T_low into the tile's staging buffer, T_high into registers;
//   tensor core: m = T_low n' mod R and the columns of m n (mont_tc.cuh),
//     the carries resolved by each packet's thread; U < n after one
//     conditional subtraction (so every intermediate is canonical).
// CTA = TILES tiles of 128 packets (2 at S = 64: 255 registers; 4 at S = 32:
// 128 registers), one CTA per SM; each tile owns KB TMEM columns and an
// mbarrier and synchronises its MMAs with named barriers of its own 128
// threads; all tiles start every Montgomery op together (RSA_TC_LOCK: the
// unrolled squaring is ~85 KB of SASS, and tiles on different code lines
// stall on instruction fetch).
//
// Shared memory: TcShared (n' and n Toeplitz strips, TILES x 128 x KB-byte
// staging) and a per-thread B slot (ND doubles, digit-major across the
// block) for the multiplies' second operand.  The window table is the FP64
// kernel's format (entries as digit pairs, entry-major then pair-major
// across the grid).
#include <cuda_runtime.h>
#include <stdint.h>

#include "devcache.h"
#include "mont_tc.cuh"
#include "plan.h"
#include "tc_digits.cuh"

namespace rsa_b200 {

#ifndef RSA_TC_TILES32
#define RSA_TC_TILES32 4    // 1024-bit class: tiles of 128 packets per CTA (TMEM 128 columns each)
#endif
#ifndef RSA_TC_SQREC32
#define RSA_TC_SQREC32 1    // squarings by the compile-time-expanded scan (sqr_col) instead of the loop
#endif                      // form (sqr_scan): A/B CRT-2048 3.24M vs 0.45M (loop not unrolled at ND = 20)
#ifndef RSA_TC_SQREC64
#define RSA_TC_SQREC64 1    // ... at 2048 bits: 949K vs 901K decrypts/s
#endif
#ifndef RSA_TC_SQB64
#define RSA_TC_SQB64 2      // products per batch of the scan, A/B at 2048 bits: 2/4/6/8 -> 949-953K/942K/955K/947K
#endif
#ifndef RSA_TC_SQB32
#define RSA_TC_SQB32 4      // ... CRT-2048 (1024-bit halves): 2/4/6 -> 3.20M/3.24M/3.24M
#endif
#ifndef RSA_TC_SQACC2
#define RSA_TC_SQACC2 0     // two partial sums per column (A/B: 927K vs 953K at 2048 bits)
#endif
#ifndef RSA_TC_JOBS
#define RSA_TC_JOBS 1       // 2048-bit: tile jobs (A/B at the 8-GPU slice: 897K vs 829K; 1M: 953K vs 947K)
#endif
#ifndef RSA_TC_JOBS32
#define RSA_TC_JOBS32 0     // 1024-bit (4 tiles): thread mapping (A/B CRT-2048: 3.42M vs 3.35M with jobs)
#endif
#ifndef RSA_TC_SQB128
#define RSA_TC_SQB128 4     // 4096-bit squaring scan batch (the FP64 kernel's measured best at ND = 80)
#endif
#ifndef RSA_TC_SQROWS128
#define RSA_TC_SQROWS128 1  // 4096-bit squarings by the rolled row form: ND^2 = 6400 digit products instead
#endif                      // of 3240, but a few KB of code: A/B 70.4K vs 57.8K decrypts/s (the ~300 KB
                            // expanded scan starves on instruction fetch at 4 warps/SM: no_instruction 2.2)
#ifndef RSA_TC_BSPEC128
#define RSA_TC_BSPEC128 1   // 4096-bit row loop instantiated per B source: A/B 75.2K vs 71.3K (the per-row
                            // run-time dispatch on the op kind sat in the loop)
#endif
#ifndef RSA_TC_EMITSEL
#define RSA_TC_EMITSEL 2    // 4096-bit run-time word stores: 0 branches, 1 branch-free stores, 2 + branch-free second word
#endif
#ifndef RSA_TC_SQBLK128
#define RSA_TC_SQBLK128 10  // 4096-bit squarings by the rolled block triangle (tcd::sqr_blocks, blocks of this
#endif                      // many digits; 3240 digit products instead of the row form's 6400; 0 = rows)
// 4096-bit window multiplies by the rolled block product (tcd::mul_blocks, blocks of this many digits):
// A/B 96.3K (10) / 95.5K (8) vs 98.9K decrypts/s for the row form (102.5K vs 105.8K once both squaring
// and multiply finish columns from per-step constants); the row form loads one table digit per row
// a row ahead; the blocks load B from global memory in bursts.  0 = rows (default).
#ifndef RSA_TC_MULBLK128
#define RSA_TC_MULBLK128 0
#endif
#ifndef RSA_TC_APAIR
#define RSA_TC_APAIR 0      // 4096-bit A slot as digit pairs (A/B)
#endif
#ifndef RSA_TC_LOCK32
#define RSA_TC_LOCK32 0     // 1024-bit class: no CTA barrier per op (A/B: CRT-2048 3.44M vs 3.24M; its code is small)
#endif
#ifndef RSA_TC_LOCK
#define RSA_TC_LOCK 1   // both tiles start every op together (A/B: 900.5K vs 809K: the unrolled squaring is
                        // ~85 KB of SASS and two tiles on different code lines stall on instruction fetch)
#endif

// Class S (32-bit limbs): KB = 4 S bytes per operand, ND digits of 52 bits
// (A < n < 2^(32 S)), TILES tiles of 128 packets per CTA (TMEM: KB columns each).
template <int S>
struct TcCfg {
    static constexpr int KB = 4 * S;
    static constexpr int ND = rsa_f64_digits(S);      // 40 at S = 64, 20 at S = 32, 80 at S = 128
    static constexpr int TILES = (S == 64) ? 2 : (S == 128 ? 1 : RSA_TC_TILES32);
    // S = 128: one tile (512 TMEM columns); A lives in the thread's shared-memory
    // slot between ops (registers: the square's 160 for A, or the row-form
    // multiply's 80 columns), the multiply's B is read in place
    static constexpr bool SLOTA = (S == 128);
    static constexpr bool LOCK = (S == 64) ? RSA_TC_LOCK : (S == 32 ? RSA_TC_LOCK32 : 0);
    static constexpr int BLOCK = TILES * tc::TILE;
    static constexpr int TMEM_COLS = (KB * TILES <= 256) ? 256 : 512;
    static_assert(KB * TILES <= 512, "TMEM: KB columns per tile");
};

template <int S>
__global__ void __launch_bounds__(TcCfg<S>::BLOCK, 1) modexp_tc_kernel(const __grid_constant__ ModexpTcParams<S> p) {
    using C = TcCfg<S>;
    constexpr int TC_S = S, TC_BLOCK = C::BLOCK;
    constexpr int ND = C::ND, NP = ND / 2, NW = tc::Geom<C::KB>::NW;
    using Shared = tc::TcShared<C::KB, C::TILES>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    double* const bslot = reinterpret_cast<double*>(smem_raw + sizeof(Shared)) + threadIdx.x;
    __shared__ __align__(16) double r2d[ND];
    __shared__ uint32_t tc_ovf[C::SLOTA && RSA_TC_EMITSEL ? 3 * TC_BLOCK : 1];   // S = 128: T words NW, NW+1, scratch
    const ModexpParams<TC_S>& ip = p.f.ip;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tc::tmem_alloc(tc::smem_u32(&sh.tmem_base), C::TMEM_COLS);
    if (threadIdx.x == 0) {
        for (int i = 0; i < (int)(sizeof(sh.mbar) / sizeof(sh.mbar[0])); i++) tc::mbar_init(tc::smem_u32(&sh.mbar[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::build_strips(sh, p.npb, reinterpret_cast<const uint8_t*>(ip.n));
    for (int i = threadIdx.x; i < NW; i += blockDim.x) sh.nw[i] = ip.n[i];
    if (threadIdx.x < 32) {
        double d[ND];
        tcd::words_to_digits<ND>([&](int w) -> uint32_t { return w < TC_S ? ip.r2[w] : 0u; }, d);
        for (int k = threadIdx.x; k < ND; k += 32) r2d[k] = d[k];
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tc::TcTile tt;
    tt.tile = threadIdx.x / tc::TILE;
    tt.r = threadIdx.x % tc::TILE;
    tt.tmem = sh.tmem_base + C::KB * tt.tile;
    tt.tlane = (uint32_t)(32 * (warp % 4)) << 16;
    tt.mbar = tc::smem_u32(&sh.mbar[tt.tile]);
    tt.phase = 0;

    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned nthr = gridDim.x * blockDim.x;
    double2* const table = reinterpret_cast<double2*>(ip.table);
    // Work comes in jobs of 128 packets (one tile), dealt round-robin to the
    // grid's tile slots, tile 0 of every CTA first: in a partial last trip the
    // busy CTAs run one tile where they can, which is faster than two (e.g. the
    // 131 072-packet slice of an 8-GPU run: 3.46 trips of two tiles, the last
    // one with one).  Every CTA runs the same trips; an idle tile still joins
    // the CTA barriers (lockstep), and a ragged job recomputes the batch's last
    // packet and skips the store.
    // JOBS (RSA_TC_JOBS / RSA_TC_JOBS32): tile jobs as above; else packet =
    // thread + trip x grid threads (every tile busy in every trip)
    constexpr bool JOBS = (S == 64) ? RSA_TC_JOBS : (S == 32 ? RSA_TC_JOBS32 : 0);
    const unsigned long long slots = (unsigned long long)gridDim.x * C::TILES;
    const unsigned long long slot = (unsigned long long)tt.tile * gridDim.x + blockIdx.x;
    const unsigned long long jobs = (ip.count + tc::TILE - 1) / tc::TILE;
    const unsigned long long trips = JOBS ? (jobs + slots - 1) / slots : (ip.count + nthr - 1) / nthr;
    for (unsigned long long tr = 0; tr < trips; tr++) {
        const unsigned long long job = slot + tr * slots;
        const bool active = !JOBS || job < jobs;          // uniform over the tile
        if (JOBS && __syncthreads_count(active) == 0) break;   // the whole CTA idle: done
        const unsigned long long pkt0 = JOBS ? job * tc::TILE + tt.r : gtid + tr * nthr;
        const bool valid = active && pkt0 < ip.count;
        const unsigned long long pkt = valid ? pkt0 : ip.count - 1;
        const uint32_t* src = ip.base + pkt * (unsigned long long)ip.s_io;
        auto load_input = [&](double (&x)[ND]) {
            uint32_t l[TC_S];
            if (ip.s_io == TC_S) {
#pragma unroll
                for (int k = 0; k < TC_S; k += 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + k));
                    l[k] = v.x; l[k + 1] = v.y; l[k + 2] = v.z; l[k + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < TC_S; k++) l[k] = (k < ip.s_io) ? __ldg(src + k) : 0u;
            }
            tcd::words_to_digits<ND>([&](int w) -> uint32_t { return w < TC_S ? l[w] : 0u; }, x);
        };
        double a[ND];
        uint32_t th[NW];
        // SLOTA: A's digits in the thread's slot, digit-major (stride TC_BLOCK) or, with
        // RSA_TC_APAIR, as digit pairs (digit k at pair k/2, 16 bytes per thread per pair)
        double* const aslot = RSA_TC_APAIR ? reinterpret_cast<double*>(smem_raw + sizeof(Shared)) + 2 * threadIdx.x
                                           : bslot;
        auto slot_at = [&](int k) -> double* {
            if constexpr (RSA_TC_APAIR != 0) return aslot + (k >> 1) * 2 * TC_BLOCK + (k & 1);
            else return aslot + k * TC_BLOCK;
        };
        auto set_digit = [&](int k, double v) {
            if constexpr (C::SLOTA) *slot_at(k) = v;
            else a[k] = v;
        };
        auto get_digit = [&](int k) -> double {
            if constexpr (C::SLOTA) return f64::ld_digit(slot_at(k));
            else return a[k];
        };
        // the row loop's A: two digits per 128-bit load when paired
        double apair_hi = 0.0;
        auto get_digit_rows = [&](int k) -> double {
            if constexpr (C::SLOTA && RSA_TC_APAIR != 0) {
                if ((k & 1) == 0) {
                    double x;
                    f64::nd_pair(slot_at(k), 0, x, apair_hi);
                    return x;
                }
                return apair_hi;
            } else {
                return get_digit(k);
            }
        };
        if (!active) {
            // an idle tile in a partial trip: only the CTA barriers of the busy one
            if constexpr (C::LOCK)
                for (int i = 0; i < ip.nops; i++)
                    for (int r = 0; r < ip.ops[i].rep; r++) __syncthreads();
            continue;
        }
        if constexpr (C::SLOTA) {
            double x[ND];
            load_input(x);
#pragma unroll
            for (int k = 0; k < ND; k++) set_digit(k, x[k]);
        } else {
            load_input(a);
        }

        for (int i = 0; i < ip.nops; i++) {
            const RsaOp op = ip.ops[i];
            if (op.flags & RSA_F_LOADA) {
#pragma unroll
                for (int g = 0; g < NP; g++) {
                    const double2 v = table[((size_t)op.lidx * NP + g) * nthr + gtid];
                    set_digit(2 * g, v.x);
                    set_digit(2 * g + 1, v.y);
                }
            }
            // the second operand of a multiply goes to this thread's slot (once per op: only
            // squarings repeat, rep > 1; the plan builder guarantees rep == 1 for the others,
            // whose row-form product overwrites the slot with T's low digits)
            if (C::SLOTA) {
                // (S = 128: B is read in place by the row-form multiply)
            } else if (op.kind == RSA_OP_MUL) {
#pragma unroll
                for (int g = 0; g < NP; g++) {
                    const double2 v = table[((size_t)op.bidx * NP + g) * nthr + gtid];
                    bslot[(2 * g) * TC_BLOCK] = v.x;
                    bslot[(2 * g + 1) * TC_BLOCK] = v.y;
                }
            } else if (op.kind == RSA_OP_R2) {
#pragma unroll
                for (int k = 0; k < ND; k++) bslot[k * TC_BLOCK] = r2d[k];
            } else if (op.kind == RSA_OP_MULX) {
                double x[ND];
                load_input(x);
#pragma unroll
                for (int k = 0; k < ND; k++) bslot[k * TC_BLOCK] = x[k];
            } else if (op.kind == RSA_OP_ONE) {
#pragma unroll
                for (int k = 0; k < ND; k++) bslot[k * TC_BLOCK] = (k == 0) ? 1.0 : 0.0;
            }
            for (int r = 0; r < op.rep; r++) {
                if constexpr (C::LOCK) __syncthreads();   // all tiles on the same code lines
                // T = A B: words 0..63 to the staging buffer (16-byte chunks), 64..127 to th
                uint32_t t63 = 0, wb0 = 0, wb1 = 0, wb2 = 0;
                auto word = [&](int w, uint32_t v) {
                    if (w < NW) {
                        if ((w & 3) == 0) wb0 = v;
                        else if ((w & 3) == 1) wb1 = v;
                        else if ((w & 3) == 2) wb2 = v;
                        else *tc::stage_chunk(sh, tt.tile, tt.r, w >> 2) = make_uint4(wb0, wb1, wb2, v);
                        if (w == NW - 1) t63 = v;
                    } else {
                        th[w - NW] = v;
                    }
                };
                tcd::Packer<2 * NW, decltype(word)> pk{word, 0};
                auto put = [&](int k, uint64_t d) { pk.put(k, d); };
                if (op.kind == RSA_OP_SQR && !(C::SLOTA && RSA_TC_SQROWS128)) {
                    if constexpr (C::SLOTA) {
#pragma unroll
                        for (int k = 0; k < ND; k++) a[k] = get_digit(k);
                        f64::sqr_col<ND, 0, RSA_TC_SQB128, 0>(a, 0, 0, 0, put);
                    } else if constexpr ((S == 32 && RSA_TC_SQREC32) || (S == 64 && RSA_TC_SQREC64))
                        // the compile-time-expanded scan (the loop form is not unrolled at ND = 20
                        // here; at ND = 40, A/B: 949K vs 901K decrypts/s)
                        f64::sqr_col<ND, 0, (S == 64 ? RSA_TC_SQB64 : RSA_TC_SQB32), RSA_TC_SQACC2>(a, 0, 0, 0, put);
                    else
                        f64::sqr_scan<ND>(a, put);
                } else if constexpr (C::SLOTA) {
                    // rows with A read from its slot and B in place (table / R^2 / 1);
                    // T's low digits leave as words at run time: words 0 .. NW-1 to the
                    // staging buffer, NW and NW+1 (digit ND-1's top bits) to th
                    auto bget = [&](int j) -> double {
                        if (op.kind == RSA_OP_SQR) return get_digit(j);   // RSA_TC_SQROWS128: A A by rows
                        if (op.kind == RSA_OP_MUL) {
                            const double2 v = table[((size_t)op.bidx * NP + (j >> 1)) * nthr + gtid];
                            return (j & 1) ? v.y : v.x;
                        }
                        if (op.kind == RSA_OP_R2) return r2d[j];
                        return j == 0 ? 1.0 : 0.0;                   // RSA_OP_ONE (no MULX at S = 128)
                    };
                    int ew = 0;
                    // branch-free (RSA_TC_EMITSEL): words >= NW (digit ND-1's top bits) go to a small
                    // overflow area, and a digit's second word, when it has none, to a scratch slot
                    auto emit_sel = [&](uint32_t v, bool valid) {
                        uint32_t* const sp = reinterpret_cast<uint32_t*>(sh.stage[tt.tile] + (ew >> 2) * tc::STAGE_LBO +
                                                                         tt.r * 16) + (ew & 3);
                        uint32_t* const op_ = tc_ovf + (ew - NW) * TC_BLOCK + threadIdx.x;
                        uint32_t* const dst = ew < NW ? sp : op_;
                        *(valid ? dst : tc_ovf + 2 * TC_BLOCK + threadIdx.x) = v;
                        ew += valid ? 1 : 0;
                    };
                    auto emit = [&](uint32_t v) {
                        if constexpr (RSA_TC_EMITSEL == 1) {
                            emit_sel(v, true);
                        } else if (ew < NW) {
                            reinterpret_cast<uint32_t*>(sh.stage[tt.tile] + (ew >> 2) * tc::STAGE_LBO +
                                                        tt.r * 16)[ew & 3] = v;
                            if (ew == NW - 1) t63 = v;
                        } else if (ew == NW) {
                            th[0] = v;
                        } else {
                            th[1] = v;
                        }
                        ew++;
                    };
                    tcd::WordEmitter<decltype(emit)> we{emit, 0, 0};
                    tcd::WordEmitter<decltype(emit_sel), true> wes{emit_sel, 0, 0};
                    auto lout = [&](int, uint64_t d) {
                        if constexpr (RSA_TC_EMITSEL == 2) wes.digit(d);
                        else we.digit(d);
                    };
                    auto lin = [&](int) -> uint64_t { return 0; };
                    if constexpr (RSA_TC_BSPEC128 != 0) {
                        // one row-loop instance per B source: the per-row fetch is a single load
                        if (op.kind == RSA_OP_SQR) {
                            if constexpr (RSA_TC_SQBLK128 != 0) {
                                // T's high digits go over A's dead blocks, then to th through put
                                auto hiout = [&](int k, uint64_t d) { *slot_at(k) = f64::from_bits(d); };
                                auto hiin = [&](int k) -> uint64_t { return f64::bits(get_digit(k)); };
                                tcd::sqr_blocks<ND, RSA_TC_SQBLK128>(get_digit, lout, hiout, hiin, put);
                            } else {
                                tcd::mul_rows_f<ND, false>(get_digit_rows, get_digit, lout, lin, put);
                            }
                        } else if (op.kind == RSA_OP_MUL) {
                            auto btab = [&](int j) -> double {
                                const double2 v = table[((size_t)op.bidx * NP + (j >> 1)) * nthr + gtid];
                                return (j & 1) ? v.y : v.x;
                            };
                            if constexpr (RSA_TC_MULBLK128 != 0) {
                                auto hiout = [&](int k, uint64_t d) { *slot_at(k) = f64::from_bits(d); };
                                auto hiin = [&](int k) -> uint64_t { return f64::bits(get_digit(k)); };
                                tcd::mul_blocks<ND, RSA_TC_MULBLK128>(get_digit, btab, lout, hiout, hiin, put);
                            } else {
                                tcd::mul_rows_f<ND, false>(get_digit_rows, btab, lout, lin, put);
                            }
                        } else {
                            tcd::mul_rows_f<ND, false>(get_digit_rows, bget, lout, lin, put);
                        }
                    } else {
                        tcd::mul_rows_f<ND, false>(get_digit_rows, bget, lout, lin, put);
                    }
                    if constexpr (RSA_TC_EMITSEL != 0) {
                        t63 = reinterpret_cast<const uint32_t*>(sh.stage[tt.tile] + ((NW - 1) >> 2) * tc::STAGE_LBO +
                                                                tt.r * 16)[(NW - 1) & 3];
                        th[0] = tc_ovf[threadIdx.x];
                        th[1] = tc_ovf[TC_BLOCK + threadIdx.x];
                    }
                } else {
                    // rows, rolled (the unrolled column scan is ~160 KB of code);
                    // T's low digits go back into b's slot as b's digits are used up
                    auto bget = [&](int j) -> double { return f64::ld_digit(bslot + j * TC_BLOCK); };
                    auto lout = [&](int j, uint64_t d) { reinterpret_cast<uint64_t*>(bslot)[j * TC_BLOCK] = d; };
                    auto lin = [&](int j) -> uint64_t { return reinterpret_cast<const uint64_t*>(bslot)[j * TC_BLOCK]; };
                    tcd::mul_rows<ND>(a, bget, lout, lin, put);
                }
                tc::redc(sh, tt, t63, th);
                tcd::words_to_digits_f<ND>([&](int w) -> uint32_t { return w < NW ? th[w] : 0u; }, set_digit);
            }
            if (op.flags & RSA_F_STORE) {
#pragma unroll
                for (int g = 0; g < NP; g++)
                    table[((size_t)op.sidx * NP + g) * nthr + gtid] = make_double2(get_digit(2 * g), get_digit(2 * g + 1));
            }
        }
        // the last op (RSA_OP_ONE or RSA_OP_MULX) left the canonical result in th
        uint32_t* dst = ip.out + pkt * (unsigned long long)ip.s_io;
        if (!valid) {
        } else if (ip.s_io == TC_S) {
#pragma unroll
            for (int k = 0; k < TC_S; k += 4)
                *reinterpret_cast<uint4*>(dst + k) = make_uint4(th[k], th[k + 1], th[k + 2], th[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < TC_S; k++)
                if (k < ip.s_io) dst[k] = th[k];
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(sh.tmem_base, C::TMEM_COLS);
    }
}

template <int S>
static size_t tc_smem_bytes() {
    return sizeof(tc::TcShared<TcCfg<S>::KB, TcCfg<S>::TILES>) + sizeof(double) * TcCfg<S>::ND * TcCfg<S>::BLOCK;
}

template <int S>
static cudaError_t launch_tc(const void* params, int sms, cudaStream_t stream, int* grid_out, int* block_out,
                             size_t* slots_out, bool query_only) {
    const int block = TcCfg<S>::BLOCK;
    const size_t smem = tc_smem_bytes<S>();
    static OccCache cache;
    int occ = 0;
    cudaError_t ce = cached_occupancy(
        cache, [&](int* o) { return occupancy_with_smem(modexp_tc_kernel<S>, block, smem, o); }, &occ);
    if (ce != cudaSuccess) return ce;
    // resident CTAs per SM: TMEM holds 512 columns
    const int tmem_cap = 512 / TcCfg<S>::TMEM_COLS;
    if (occ > tmem_cap) occ = tmem_cap;
    int grid = sms * occ;
    if (grid_out) *grid_out = grid;
    if (block_out) *block_out = block;
    if (slots_out) *slots_out = (size_t)grid * block;
    if (query_only) return cudaSuccess;
    const ModexpTcParams<S>& prm = *static_cast<const ModexpTcParams<S>*>(params);
    const unsigned long long need = (prm.f.ip.count + block - 1) / block;
    if (need < (unsigned long long)grid) grid = (int)need;
    modexp_tc_kernel<S><<<grid, block, smem, stream>>>(prm);
    return cudaGetLastError();
}

}  // namespace rsa_b200

// 1 if class S's squarings run a dedicated squaring (ND (ND+1)/2 digit products on
// the CUDA cores), 0 if the row-form product (ND^2)
int rsa_b200_tc_sqr(int S) { return (S == 128 && RSA_TC_SQROWS128 && !(RSA_TC_BSPEC128 && RSA_TC_SQBLK128)) ? 0 : 1; }

cudaError_t rsa_b200_launch_tc(int S, const void* params, int sms, cudaStream_t stream, int* grid, int* block,
                               size_t* slots, bool query_only) {
    switch (S) {
    case 32: return rsa_b200::launch_tc<32>(params, sms, stream, grid, block, slots, query_only);
    case 64: return rsa_b200::launch_tc<64>(params, sms, stream, grid, block, slots, query_only);
    case 128: return rsa_b200::launch_tc<128>(params, sms, stream, grid, block, slots, query_only);
    default: return cudaErrorInvalidValue;
    }
}
