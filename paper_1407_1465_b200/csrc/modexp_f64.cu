// modexp_f64.cu -- batched modular exponentiation on the FP64 pipe (sm_100a).
//
// Same contract and operation list as modexp_kernel (modexp.cu): out[i] =
// base[i]^exp mod n for every packet (sec. 2; PAPER.md:65,
// sec. 3.3), one thread per packet, the shared exponent's op list executed
// warp-uniformly.  The Montgomery multiply is mont_f64.cuh: 52-bit digits in
// doubles, products split exactly by DFMA.RZ, column sums in 64-bit integers.
//
// Per thread (S = 32, 64): A (ND doubles) and the accumulator (ND 64-bit
// columns) in registers; a 2 ND-digit shared-memory slot (digit-major across
// the block: conflict-free LDS.64) holds the b operand and A while a multiply
// runs (A re-read per digit), or the square's 2 ND digits.  S = 128: A lives
// in an ND-digit slot and b is read in place (see F64Cfg::ONESLOT).  n's digits
// come from one per-block shared copy (volatile pair loads).  The window table
// holds entries as digit pairs (double2), entry-major then digit-pair-major
// across the grid's threads (coalesced).  Intermediates stay < 2n
// (R = 2^(52 ND) > 4n), and one subtraction canonicalises the result.
#include <cuda_runtime.h>
#include <stdint.h>

#include "devcache.h"
#include "mont_f64.cuh"
#include "plan.h"

namespace rsa_b200 {

#ifndef RSA_F64_SQR
#define RSA_F64_SQR 1
#endif
#ifndef RSA_F64_BLOCK
#define RSA_F64_BLOCK 256
#endif
#ifndef RSA_F64_ASMEM
#define RSA_F64_ASMEM 1
#endif
#ifndef RSA_F64_FUSEJ
#define RSA_F64_FUSEJ 0     // 4096-bit kernel: one fused j-loop (A/B: 54.4K vs 56.4K, no spills but less overlap)
#endif
#ifndef RSA_F64_SQRSMEM
#define RSA_F64_SQRSMEM 0   // 4096-bit kernel: separate squaring instance with LDS b reads (A/B: 56.6K vs 60.2K)
#endif
#ifndef RSA_F64_FUSEJ64
#define RSA_F64_FUSEJ64 0   // 1024/2048-bit multiply: fused j-loop (A/B)
#endif
#ifndef RSA_F64_MINB128
#define RSA_F64_MINB128 2
#endif
#ifndef RSA_F64_MINB32
#define RSA_F64_MINB32 4
#endif
#ifndef RSA_F64_EARLYEXIT
#define RSA_F64_EARLYEXIT 0   // non-lockstep classes: threads stop when the batch runs out (A/B: CRT-2048 2.14M vs 2.19M, off)
#endif
#ifndef RSA_F64_SQR128
#define RSA_F64_SQR128 1    // 4096-bit kernel: dedicated squaring with A in its one slot (montsqr_slot)
#endif
#ifndef RSA_F64_BLOCK128
#define RSA_F64_BLOCK128 256   // 4096-bit kernel CTA: 256 threads in lockstep (the unrolled squaring is long)
#endif
template <int S>
struct F64Cfg {
    static constexpr int ND = rsa_f64_digits(S);
    // S = 64: one 256-thread CTA per SM and a barrier per Montgomery op keep
    // the SM's 8 warps on the same code lines: the unrolled squaring is ~80 KB
    // of SASS, and drifting warps stall on instruction fetch (ncu:
    // no_instruction).  S = 32 (ND = 20): ~80 registers of state, small code,
    // several independent CTAs per SM.
    static constexpr int BLOCK = (S == 64) ? RSA_F64_BLOCK : (S == 128 ? RSA_F64_BLOCK128 : 128);
    static constexpr int MINB = (S == 64)    ? (RSA_F64_BLOCK >= 256 ? 1 : 256 / RSA_F64_BLOCK)
                                : (S == 128) ? (RSA_F64_BLOCK128 >= 256 ? 1 : RSA_F64_MINB128)
                                             : RSA_F64_MINB32;
#ifndef RSA_F64_LOCK
#define RSA_F64_LOCK 0      // A/B: lockstep barriers with 2 x 128-thread CTAs (557K vs 589K)
#endif
    static constexpr bool LOCKSTEP = ((S == 64) && (RSA_F64_BLOCK >= 256 || RSA_F64_LOCK)) ||
                                     ((S == 128) && RSA_F64_BLOCK128 >= 256);
    // S = 128 (ND = 80): the square's 2 ND digits and A + B slots do not fit shared memory at
    // 8 warps/SM, so every op is the CIOS multiply with A parked in a single ND-digit slot and B
    // read in place (the slot itself for squarings, the window table in global memory, or a
    // per-block constant): ND^2 products more per squaring, no squaring code.
    static constexpr bool ONESLOT = (S >= 128);
    static constexpr bool SQR = RSA_F64_SQR && !ONESLOT;   // dedicated squaring (montsqr) vs montmul(a, a)
    static constexpr bool SQRSLOT = ONESLOT && RSA_F64_SQR128;   // ONESLOT squarings by montsqr_slot
    static constexpr bool ASMEM = ONESLOT || ((S >= 64) && RSA_F64_ASMEM && SQR);   // montmul's A parked in smem
};

template <int S>
__global__ void __launch_bounds__(F64Cfg<S>::BLOCK, F64Cfg<S>::MINB)
modexp_f64_kernel(const __grid_constant__ ModexpF64Params<S> p) {
    constexpr int ND = F64Cfg<S>::ND;
    constexpr int NP = ND / 2;
    static_assert(ND % 2 == 0, "digit pairs");
    extern __shared__ __align__(16) double bsm_raw[];
    double* const bsm = bsm_raw + threadIdx.x;
    const int stride = blockDim.x;
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned nthr = gridDim.x * blockDim.x;
    double2* const table = reinterpret_cast<double2*>(p.ip.table);
    const ModexpParams<S>& ip = p.ip;
    // n's digits, one shared copy per block (read by the volatile pair loads
    // of mont_f64.cuh)
    __shared__ __align__(16) double nds[ND];
    __shared__ __align__(16) double cst[F64Cfg<S>::ONESLOT ? 2 * ND : 1];   // R^2 mod n, 1 (ONESLOT)
    for (int k = threadIdx.x; k < ND; k += blockDim.x) {
        nds[k] = p.nd[k];
        if constexpr (F64Cfg<S>::ONESLOT) {
            cst[k] = p.r2d[k];
            cst[ND + k] = (k == 0) ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    // RSA_F64_NCONST: n's digits are read from the parameter block (constant
    // bank); 2^104 then lives in an ordinary (non-uniform) register so the
    // DFMA's one constant-bank operand slot is left to the digit of n
    const double* const nsrc = RSA_F64_NCONST ? p.nd : nds;
    double c104 = p.c104;
    if constexpr (RSA_F64_NCONST != 0) {
        unsigned z;
        asm volatile("mov.u32 %0, %%laneid;\n\tand.b32 %0, %0, 0;" : "=r"(z));
        c104 = __longlong_as_double(__double_as_longlong(c104) + z);
    }

    // Every thread runs the same number of trips (uniform barriers in the
    // lockstep configurations); an out-of-range trip recomputes the last packet
    // and skips the store.  Measured alternatives: guarding the arithmetic of
    // such a trip (582K vs 591K at 2048 bits, and no faster on a partial last
    // wave, whose packets sit on the first SMs anyway); stopping those threads
    // in the non-lockstep 1024-bit class (RSA_F64_EARLYEXIT: CRT-2048 2.14M vs
    // 2.19M).
    const unsigned long long trips = (ip.count + nthr - 1) / nthr;
    for (unsigned long long tr = 0; tr < trips; tr++) {
        const unsigned long long pkt0 = gtid + tr * nthr;
        const bool valid = pkt0 < ip.count;
        if (RSA_F64_EARLYEXIT && !F64Cfg<S>::LOCKSTEP && !valid) break;
        const unsigned long long pkt = valid ? pkt0 : ip.count - 1;
        const uint32_t* src = ip.base + pkt * (unsigned long long)ip.s_io;
        auto load_input = [&](double (&x)[ND]) {
            uint32_t l[S];
            if (ip.s_io == S) {
#pragma unroll
                for (int k = 0; k < S; k += 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + k));
                    l[k] = v.x; l[k + 1] = v.y; l[k + 2] = v.z; l[k + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < S; k++) l[k] = (k < ip.s_io) ? __ldg(src + k) : 0u;
            }
            f64::limbs_to_digits<S, ND>(l, x);
        };
        double a[ND];
        uint64_t t[ND];
        if constexpr (F64Cfg<S>::ONESLOT) {
            // A lives in this thread's slot
            double x[ND];
            load_input(x);
#pragma unroll
            for (int k = 0; k < ND; k++) bsm[k * stride] = x[k];
        } else {
            load_input(a);
        }
        auto from_smem = [&](int i) { return bsm[i * stride]; };

        for (int i = 0; i < ip.nops; i++) {
            const RsaOp op = ip.ops[i];
            if (op.flags & RSA_F_LOADA) {
#pragma unroll
                for (int g = 0; g < NP; g++) {
                    const double2 v = table[((size_t)op.lidx * NP + g) * nthr + gtid];
                    if constexpr (F64Cfg<S>::ONESLOT) {
                        bsm[(2 * g) * stride] = v.x;
                        bsm[(2 * g + 1) * stride] = v.y;
                    } else {
                        a[2 * g] = v.x; a[2 * g + 1] = v.y;
                    }
                }
            }
            if constexpr (F64Cfg<S>::ONESLOT) {
                // b(i) = bp[i * bs]: generic loads from the A slot (squaring), this
                // thread's table entry (global), or the per-block constants
                // digit i at bp[(i >> 1) * P + (i & 1) * Q]: one formula for the
                // digit-major slot, the pair-interleaved table and the constants
                const double* bp;
                size_t P, Q;
                if (op.kind == RSA_OP_SQR) { bp = bsm; P = 2 * (size_t)stride; Q = stride; }
                else if (op.kind == RSA_OP_MUL) {
                    bp = reinterpret_cast<const double*>(table) + (size_t)op.bidx * ND * nthr + 2 * (size_t)gtid;
                    P = 2 * (size_t)nthr; Q = 1;
                } else if (op.kind == RSA_OP_R2) { bp = cst; P = 2; Q = 1; }
                else { bp = cst + ND; P = 2; Q = 1; }   // RSA_OP_ONE (plans for this class carry no MULX)
                auto bget = [&](int i) -> double { return bp[(size_t)(i >> 1) * P + (i & 1) * Q]; };
                if (F64Cfg<S>::SQRSLOT && op.kind == RSA_OP_SQR) {
                    // dedicated squaring: ND (ND+1)/2 + ND^2 digit products, A stays in the slot
                    for (int r = 0; r < op.rep; r++) {
                        if constexpr (F64Cfg<S>::LOCKSTEP) __syncthreads();
                        f64::montsqr_slot<ND>(nsrc, p.np52, c104, t, bsm, stride);
                    }
                } else if (RSA_F64_SQRSMEM && op.kind == RSA_OP_SQR) {
                    // squarings (the bulk): b is the slot itself, read with explicit
                    // shared-memory loads instead of generic ones
                    auto bsq = [&](int i) -> double { return f64::ld_digit(bsm + (size_t)i * stride); };
                    for (int r = 0; r < op.rep; r++)
                        f64::montmul<ND, true, decltype(bsq), true, RSA_F64_FUSEJ>(a, bsq, nsrc, p.np52, c104, t,
                                                                                  bsm, stride);
                } else {
                    for (int r = 0; r < op.rep; r++) {
                        if constexpr (F64Cfg<S>::LOCKSTEP) __syncthreads();
                        f64::montmul<ND, true, decltype(bget), true, RSA_F64_FUSEJ>(a, bget, nsrc, p.np52, c104, t,
                                                                                   bsm, stride);
                    }
                }
            } else
            for (int r = 0; r < op.rep; r++) {
                if constexpr (F64Cfg<S>::LOCKSTEP) __syncthreads();
                // stage the b operand in this thread's slot; one montmul call site
                // keeps the kernel's code (and its register allocation) single
                if (op.kind == RSA_OP_SQR) {
                    if constexpr (F64Cfg<S>::SQR) {
                        // the square's 2 ND digits go to this thread's slot
                        f64::montsqr<ND>(a, nsrc, p.np52, c104, t, reinterpret_cast<uint64_t*>(bsm), stride);
                        continue;
                    } else {
#pragma unroll
                        for (int k = 0; k < ND; k++) bsm[k * stride] = a[k];
                    }
                } else if (op.kind == RSA_OP_MUL) {
#pragma unroll
                    for (int g = 0; g < NP; g++) {
                        const double2 v = table[((size_t)op.bidx * NP + g) * nthr + gtid];
                        bsm[(2 * g) * stride] = v.x;
                        bsm[(2 * g + 1) * stride] = v.y;
                    }
                } else if (op.kind == RSA_OP_R2) {
#pragma unroll
                    for (int k = 0; k < ND; k++) bsm[k * stride] = p.r2d[k];
                } else if (op.kind == RSA_OP_MULX) {
                    double x[ND];
                    load_input(x);
#pragma unroll
                    for (int k = 0; k < ND; k++) bsm[k * stride] = x[k];
                } else {  // RSA_OP_ONE
#pragma unroll
                    for (int k = 0; k < ND; k++) bsm[k * stride] = (k == 0) ? 1.0 : 0.0;
                }
                // b occupies digits [0, ND) of the slot; A is parked in [ND, 2 ND)
                f64::montmul<ND, F64Cfg<S>::ASMEM, decltype(from_smem), false, RSA_F64_FUSEJ64 != 0>(
                    a, from_smem, nsrc, p.np52, c104, t, bsm + ND * stride, stride);
            }
            if (op.flags & RSA_F_STORE) {
#pragma unroll
                for (int g = 0; g < NP; g++) {
                    if constexpr (F64Cfg<S>::ONESLOT)
                        table[((size_t)op.sidx * NP + g) * nthr + gtid] =
                            make_double2(bsm[(2 * g) * stride], bsm[(2 * g + 1) * stride]);
                    else
                        table[((size_t)op.sidx * NP + g) * nthr + gtid] = make_double2(a[2 * g], a[2 * g + 1]);
                }
            }
        }

        // the last op (RSA_OP_ONE or RSA_OP_MULX) left the digits in t, < 2n
        f64::canonicalise<ND>(t, reinterpret_cast<const uint64_t*>(p.nu));
        uint32_t l[S];
        f64::digits_to_limbs<S, ND>(t, l);
        uint32_t* dst = ip.out + pkt * (unsigned long long)ip.s_io;
        if (!valid) {
        } else if (ip.s_io == S) {
#pragma unroll
            for (int k = 0; k < S; k += 4)
                *reinterpret_cast<uint4*>(dst + k) = make_uint4(l[k], l[k + 1], l[k + 2], l[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < S; k++)
                if (k < ip.s_io) dst[k] = l[k];
        }
    }
}

template <int S>
static cudaError_t launch_f64(const void* params, int sms, cudaStream_t stream, int* grid_out, int* block_out,
                              size_t* slots_out, bool query_only) {
    const int block = F64Cfg<S>::BLOCK;
    const size_t smem = sizeof(double) * F64Cfg<S>::ND * ((F64Cfg<S>::SQR || F64Cfg<S>::ASMEM) && !F64Cfg<S>::ONESLOT ? 2 : 1) * block;
    static OccCache cache;
    int occ = 0;
    cudaError_t ce = cached_occupancy(
        cache, [&](int* o) { return occupancy_with_smem(modexp_f64_kernel<S>, block, smem, o); }, &occ);
    if (ce != cudaSuccess) return ce;
    int grid = sms * occ;
    if (grid_out) *grid_out = grid;
    if (block_out) *block_out = block;
    if (slots_out) *slots_out = (size_t)grid * block;
    if (query_only) return cudaSuccess;
    const ModexpF64Params<S>& prm = *static_cast<const ModexpF64Params<S>*>(params);
    const unsigned long long need = (prm.ip.count + block - 1) / block;
    if (need < (unsigned long long)grid) grid = (int)need;
    modexp_f64_kernel<S><<<grid, block, smem, stream>>>(prm);
    return cudaGetLastError();
}

}  // namespace rsa_b200

// host entry points (C++ linkage) used by modexp.cu's dispatch

// 1 if the FP64 kernel of class S squares with a dedicated squaring
// (ND (ND+1)/2 + ND^2 digit products), 0 if with the CIOS multiply (2 ND^2)
int rsa_b200_f64_sqr(int S) {
    using namespace rsa_b200;
    switch (S) {
    case 32: return F64Cfg<32>::SQR ? 1 : 0;
    case 64: return F64Cfg<64>::SQR ? 1 : 0;
    case 128: return F64Cfg<128>::SQRSLOT ? 1 : 0;
    default: return 0;
    }
}
cudaError_t rsa_b200_launch_f64(int S, const void* params, int sms, cudaStream_t stream, int* grid, int* block,
                                size_t* slots, bool query_only) {
    using namespace rsa_b200;
    switch (S) {
    case 32: return launch_f64<32>(params, sms, stream, grid, block, slots, query_only);
    case 64: return launch_f64<64>(params, sms, stream, grid, block, slots, query_only);
    case 128: return launch_f64<128>(params, sms, stream, grid, block, slots, query_only);
    default: return cudaErrorInvalidValue;
    }
}
