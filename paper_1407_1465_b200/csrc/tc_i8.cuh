// tc_i8.cuh -- the tcgen05 (5th-generation tensor core) pieces used by the
// tensor-core Montgomery reduction (mont_tc.cuh): u8 x u8 -> s32 MMAs with
// operands in shared memory and the accumulator in tensor memory (TMEM).
//
// Why a tensor core in a carry-propagating product: Montgomery reduction of
// a batch under ONE modulus n is two products with a CONSTANT operand,
//   m = (T mod R) n' mod R   and   (T + m n) / R,
// i.e. [packets x K] x [K x N] matrix products against Toeplitz matrices of
// n' and n (byte digits: column j of x n = sum_k x_k n_{j-k}).  The tensor
// core returns the exact column sums (< 2^24 for 256-byte operands) and the
// CUDA cores resolve the carries.  PAPER.md:357 (sec. 9) names the modular
// multiply as the hot spot; this takes two thirds of a squaring's digit
// products off the CUDA cores.
//
// Layout (SWIZZLE_NONE, K-major, PTX "canonical layout"): an operand is a set
// of core matrices of 8 rows x 16 bytes (128 contiguous bytes); rows within a
// core matrix are 16 bytes apart, 8-row groups SBO bytes apart, the two
// 16-byte K chunks of one K = 32 MMA step LBO bytes apart.  Every operand
// here keeps its rows consecutive (SBO = 128) inside one region per 16-byte
// K chunk, so a window starting at ANY row is again canonical: that is what
// lets one "strip" hold every Toeplitz block (block (J, I) of the n matrix is
// the strip's rows starting at 32 (J - I)).
#pragma once
#include <stdint.h>

namespace rsa_b200 {
namespace tc {

// instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B unsigned 8-bit
// (formats 0), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// shared-memory matrix descriptor, SWIZZLE_NONE: start, LBO and SBO in
// 16-byte units (bits 0-13, 16-29, 32-45), version 1 at bit 46 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// D[tmem] (+)= A[smem] B[smem]^T, issued by one thread for the CTA
__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// arrive (once) on the mbarrier when every MMA this thread issued has completed
__device__ __forceinline__ void commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}

// Wait for the phase with the given parity to complete.  Bounded: a phase that
// never completes (a malformed descriptor, a lost commit) traps after ~2^26
// polls (seconds) instead of hanging the GPU; the launch then fails with an
// error the host reports as RSA_ECUDA.
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t tries = 0;; tries++) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(mbar), "r"(parity)
            : "memory");
        if (done) return;
        if (tries > (1u << 26)) __trap();
    }
}

// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// named barrier over `count` threads (a 128-thread tile: id 1 + tile)
__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMEM allocation (one warp; result address written to shared memory)
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 consecutive columns of this thread's TMEM lane (32x32b shape: warp w of
// a warpgroup reads lanes 32 (w % 4) .. + 31, thread i lane 32 (w % 4) + i)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tc
}  // namespace rsa_b200
