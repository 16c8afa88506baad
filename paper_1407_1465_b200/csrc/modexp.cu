// modexp.cu -- batched modular exponentiation kernels for sm_100a.
//
// out[i] = base[i]^exp mod n for every packet i (sec. 2;
// PAPER.md:65, sec. 3.3; "same kernel code will work for decryption too",
// PAPER.md:489).  One thread owns one packet, as in the paper's kernel
// (Alg 1) -- but the per-packet work is a windowed
// Montgomery exponentiation on S-limb numbers instead of Fig 12's O(e) loop.
//
// Grid: persistent, gridDim = SMs x resident CTAs; each thread walks packets
// tid, tid + nthreads, ...  so the per-thread window table (global memory,
// limb-group-major across threads -> coalesced) is sized by resident threads,
// not by the batch, and stays mostly L2-resident.
//
// Every thread executes the same operation list (the exponent is shared by
// the batch), so control flow is warp-uniform: no divergence.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mont.cuh"
#include "plan.h"

namespace rsa_b200 {

template <int S>
struct KCfg {
    static constexpr int BLOCK = 128;
    static constexpr int MINB = (S >= 64) ? 2 : (S >= 32 ? 3 : 4);
};

template <int S>
__global__ void __launch_bounds__(KCfg<S>::BLOCK, KCfg<S>::MINB)
modexp_kernel(const __grid_constant__ ModexpParams<S> p) {
    using V = typename BVec<S>::T;
    constexpr int G = BVec<S>::G;
    constexpr int NG = S / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* const bslot = reinterpret_cast<V*>(smem_raw) + threadIdx.x;
    const int stride = blockDim.x;
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned nthr = gridDim.x * blockDim.x;
    V* const table = reinterpret_cast<V*>(p.table);

    for (unsigned long long pkt = gtid; pkt < p.count; pkt += nthr) {
        uint32_t a[S];
        // a2: load the packet (packet-major at the boundary), zero padded
        const uint32_t* src = p.base + pkt * (unsigned long long)p.s_io;
        if (p.s_io == S && (S % 4) == 0) {
#pragma unroll
            for (int k = 0; k < S; k += 4) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + k));
                a[k] = v.x; a[k + 1] = v.y; a[k + 2] = v.z; a[k + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < S; k++) a[k] = (k < p.s_io) ? __ldg(src + k) : 0u;
        }

        for (int i = 0; i < p.nops; i++) {
            const RsaOp op = p.ops[i];
            if (op.flags & RSA_F_LOADA) {
#pragma unroll
                for (int g = 0; g < NG; g++) {
                    const V v = table[((size_t)op.lidx * NG + g) * nthr + gtid];
                    a[G * g] = v.x; a[G * g + 1] = v.y;
                    if constexpr (G == 4) { a[G * g + 2] = v.z; a[G * g + 3] = v.w; }
                }
            }
            for (int r = 0; r < op.rep; r++) {
                // stage the b operand in this thread's shared-memory slot
                if (op.kind == RSA_OP_SQR) {
#pragma unroll
                    for (int g = 0; g < NG; g++) {
                        V v; v.x = a[G * g]; v.y = a[G * g + 1];
                        if constexpr (G == 4) { v.z = a[G * g + 2]; v.w = a[G * g + 3]; }
                        bslot[g * stride] = v;
                    }
                } else if (op.kind == RSA_OP_MUL) {
#pragma unroll
                    for (int g = 0; g < NG; g++)
                        bslot[g * stride] = table[((size_t)op.bidx * NG + g) * nthr + gtid];
                } else if (op.kind == RSA_OP_R2) {
#pragma unroll
                    for (int g = 0; g < NG; g++) {
                        V v; v.x = p.r2[G * g]; v.y = p.r2[G * g + 1];
                        if constexpr (G == 4) { v.z = p.r2[G * g + 2]; v.w = p.r2[G * g + 3]; }
                        bslot[g * stride] = v;
                    }
                } else {  // RSA_OP_ONE
#pragma unroll
                    for (int g = 0; g < NG; g++) {
                        V v; v.x = (g == 0) ? 1u : 0u; v.y = 0u;
                        if constexpr (G == 4) { v.z = 0u; v.w = 0u; }
                        bslot[g * stride] = v;
                    }
                }
                montmul<S>(a, bslot, stride, p.n, p.n0inv);
            }
            if (op.flags & RSA_F_STORE) {
#pragma unroll
                for (int g = 0; g < NG; g++) {
                    V v; v.x = a[G * g]; v.y = a[G * g + 1];
                    if constexpr (G == 4) { v.z = a[G * g + 2]; v.w = a[G * g + 3]; }
                    table[((size_t)op.sidx * NG + g) * nthr + gtid] = v;
                }
            }
        }

        // a8: store the canonical result
        uint32_t* dst = p.out + pkt * (unsigned long long)p.s_io;
        if (p.s_io == S && (S % 4) == 0) {
#pragma unroll
            for (int k = 0; k < S; k += 4)
                *reinterpret_cast<uint4*>(dst + k) = make_uint4(a[k], a[k + 1], a[k + 2], a[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < S; k++)
                if (k < p.s_io) dst[k] = a[k];
        }
    }
}

// exp == 0: every output is 1 mod n = 1 (n >= 3), reading Z12
__global__ void fill_one_kernel(uint32_t* out, unsigned long long count, int s_io) {
    const unsigned long long total = count * (unsigned long long)s_io;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = (i % s_io) == 0 ? 1u : 0u;
}

template <int S>
static cudaError_t launch_class(const void* params, int sms, cudaStream_t stream, int* grid_out,
                                int* block_out, size_t* tab_stride_out, bool query_only) {
    using V = typename BVec<S>::T;
    const int block = KCfg<S>::BLOCK;
    const size_t smem = sizeof(V) * (S / BVec<S>::G) * block;
    static int occ = -1;
    if (occ < 0) {
        cudaError_t e = cudaFuncSetAttribute(modexp_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, modexp_kernel<S>, block, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int grid = sms * occ;
    if (grid_out) *grid_out = grid;
    if (block_out) *block_out = block;
    if (tab_stride_out) *tab_stride_out = (size_t)grid * block;
    if (query_only) return cudaSuccess;
    modexp_kernel<S><<<grid, block, smem, stream>>>(*static_cast<const ModexpParams<S>*>(params));
    return cudaGetLastError();
}

}  // namespace rsa_b200

// Host entry points used by rsa_abi.cpp (C++ linkage, not part of the C-ABI).
cudaError_t rsa_b200_launch(int S, const void* params, int sms, cudaStream_t stream) {
    using namespace rsa_b200;
    switch (S) {
    case 2: return launch_class<2>(params, sms, stream, nullptr, nullptr, nullptr, false);
    case 4: return launch_class<4>(params, sms, stream, nullptr, nullptr, nullptr, false);
    case 8: return launch_class<8>(params, sms, stream, nullptr, nullptr, nullptr, false);
    case 16: return launch_class<16>(params, sms, stream, nullptr, nullptr, nullptr, false);
    case 32: return launch_class<32>(params, sms, stream, nullptr, nullptr, nullptr, false);
    case 64: return launch_class<64>(params, sms, stream, nullptr, nullptr, nullptr, false);
    default: return cudaErrorInvalidValue;
    }
}

// threads of the persistent grid for class S (sizes the table workspace)
cudaError_t rsa_b200_grid(int S, int sms, int* grid, int* block, size_t* nthreads) {
    using namespace rsa_b200;
    switch (S) {
    case 2: return launch_class<2>(nullptr, sms, 0, grid, block, nthreads, true);
    case 4: return launch_class<4>(nullptr, sms, 0, grid, block, nthreads, true);
    case 8: return launch_class<8>(nullptr, sms, 0, grid, block, nthreads, true);
    case 16: return launch_class<16>(nullptr, sms, 0, grid, block, nthreads, true);
    case 32: return launch_class<32>(nullptr, sms, 0, grid, block, nthreads, true);
    case 64: return launch_class<64>(nullptr, sms, 0, grid, block, nthreads, true);
    default: return cudaErrorInvalidValue;
    }
}

size_t rsa_b200_params_size(int S) {
    using namespace rsa_b200;
    switch (S) {
    case 2: return sizeof(ModexpParams<2>);
    case 4: return sizeof(ModexpParams<4>);
    case 8: return sizeof(ModexpParams<8>);
    case 16: return sizeof(ModexpParams<16>);
    case 32: return sizeof(ModexpParams<32>);
    case 64: return sizeof(ModexpParams<64>);
    default: return 0;
    }
}

cudaError_t rsa_b200_fill_one(uint32_t* out, unsigned long long count, int s_io, int sms, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    rsa_b200::fill_one_kernel<<<sms * 4, 256, 0, stream>>>(out, count, s_io);
    return cudaGetLastError();
}
