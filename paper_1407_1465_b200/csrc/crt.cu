// crt.cu -- CRT decryption (beyond the paper).
//
// M = C^d mod n computed from the key material the Fig 1 check
// already has (p, q):  m1 = C^dp mod p, m2 = C^dq mod q  (dp = d mod (p-1),
// dq = d mod (q-1)), h = qinv (m1 - m2) mod p, M = m2 + h q  (Garner).  Two
// half-width exponentiations instead of one full-width: ~4x fewer limb
// products.  Kernels here:
//   crt_split   : C (2SH limbs) -> C mod p, C mod q  (wide Montgomery reduction
//                 T R^-1, then one Montgomery multiply by R^2: T R^-1 R^2 R^-1 = T)
//   crt_combine : (m1, m2) -> M
// The half exponentiations run on modexp.cu's kernels (class SH).
#include <cuda_runtime.h>
#include <stdint.h>

#include "devcache.h"
#include "mont.cuh"
#include "mont_sqr.cuh"

namespace rsa_b200 {

template <int SH>
struct CrtParams {
    const uint32_t* c;       // [count][s_io]        (split)
    uint32_t* cp;            // [count][sh_io]       (split out; combine in as m1)
    uint32_t* cq;            // [count][sh_io]       (split out; combine in as m2)
    uint32_t* out;           // [count][s_io]        (combine)
    unsigned long long count;
    int s_io, sh_io;
    uint32_t pinv, qinv32;   // -p^-1, -q^-1 mod 2^32
    uint32_t p[SH], q[SH];
    uint32_t r2p[SH], r2q[SH];   // R^2 mod p, R^2 mod q (R = 2^(32 SH))
    uint32_t qinvR[SH];          // (q^-1 mod p) R mod p
};

template <int SH>
__device__ __forceinline__ void stage_const(uint4* bslot, int stride, const uint32_t (&v)[SH]) {
#pragma unroll
    for (int g = 0; g < SH / 4; g++) bslot[g * stride] = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
}

template <int SH>
__global__ void __launch_bounds__(128) crt_split_kernel(const __grid_constant__ CrtParams<SH> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint4* const bslot = reinterpret_cast<uint4*>(smem_raw) + threadIdx.x;
    const int stride = blockDim.x;
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= p.count) return;
    uint32_t T[2 * SH];
    const uint32_t* src = p.c + i * (unsigned long long)p.s_io;
#pragma unroll
    for (int k = 0; k < 2 * SH; k++) T[k] = (k < p.s_io) ? __ldg(src + k) : 0u;
    uint32_t a[SH];
    // C mod p: T R^-1 mod p, then * R^2 R^-1
    reduce_wide<SH>(a, T, p.p, p.pinv);
    stage_const<SH>(bslot, stride, p.r2p);
    montmul<SH>(a, reinterpret_cast<const uint4*>(bslot), stride, p.p, p.pinv);
    uint32_t* dp_ = p.cp + i * (unsigned long long)p.sh_io;
#pragma unroll
    for (int k = 0; k < SH; k++)
        if (k < p.sh_io) dp_[k] = a[k];
    // C mod q
    reduce_wide<SH>(a, T, p.q, p.qinv32);
    stage_const<SH>(bslot, stride, p.r2q);
    montmul<SH>(a, reinterpret_cast<const uint4*>(bslot), stride, p.q, p.qinv32);
    uint32_t* dq_ = p.cq + i * (unsigned long long)p.sh_io;
#pragma unroll
    for (int k = 0; k < SH; k++)
        if (k < p.sh_io) dq_[k] = a[k];
}

template <int SH>
__global__ void __launch_bounds__(128) crt_combine_kernel(const __grid_constant__ CrtParams<SH> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint4* const bslot = reinterpret_cast<uint4*>(smem_raw) + threadIdx.x;
    const int stride = blockDim.x;
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= p.count) return;
    uint32_t m1[SH], m2[SH], t[SH];
    const uint32_t* s1 = p.cp + i * (unsigned long long)p.sh_io;
    const uint32_t* s2 = p.cq + i * (unsigned long long)p.sh_io;
#pragma unroll
    for (int k = 0; k < SH; k++) {
        m1[k] = (k < p.sh_io) ? s1[k] : 0u;
        m2[k] = (k < p.sh_io) ? s2[k] : 0u;
    }
    // m2' = m2 mod p  (m2 < q < 2p)
    sub_cc(t[0], m2[0], p.p[0]);
#pragma unroll
    for (int k = 1; k < SH; k++) subc_cc(t[k], m2[k], p.p[k]);
    uint32_t keep;
    subc(keep, 0u, 0u);                      // 0xFFFFFFFF if m2 < p
#pragma unroll
    for (int k = 0; k < SH; k++) t[k] = (m2[k] & keep) | (t[k] & ~keep);
    // diff = m1 - m2' mod p
    sub_cc(m1[0], m1[0], t[0]);
#pragma unroll
    for (int k = 1; k < SH; k++) subc_cc(m1[k], m1[k], t[k]);
    uint32_t neg;
    subc(neg, 0u, 0u);
    add_cc(m1[0], m1[0], p.p[0] & neg);
#pragma unroll
    for (int k = 1; k < SH; k++) addc_cc(m1[k], m1[k], p.p[k] & neg);
    // h = diff * qinv mod p  (Montgomery multiply by qinv R)
    stage_const<SH>(bslot, stride, p.qinvR);
    montmul<SH>(m1, reinterpret_cast<const uint4*>(bslot), stride, p.p, p.pinv);
    // M = m2 + h q  (schoolbook; M < p q = n)
    uint32_t M[2 * SH];
#pragma unroll
    for (int k = 0; k < 2 * SH; k++) M[k] = (k < SH) ? m2[k] : 0u;
#pragma unroll
    for (int j = 0; j < SH; j++) {
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < SH; k++) {
            const uint64_t v = (uint64_t)m1[j] * p.q[k] + M[j + k] + c;
            M[j + k] = (uint32_t)v;
            c = (uint32_t)(v >> 32);
        }
#pragma unroll
        for (int k = j + SH; k < 2 * SH; k++) {
            const uint64_t v = (uint64_t)M[k] + c;
            M[k] = (uint32_t)v;
            c = (uint32_t)(v >> 32);
        }
    }
    uint32_t* dst = p.out + i * (unsigned long long)p.s_io;
#pragma unroll
    for (int k = 0; k < 2 * SH; k++)
        if (k < p.s_io) dst[k] = M[k];
}

template <int SH>
static cudaError_t crt_launch(const void* raw, int which, unsigned long long count, cudaStream_t st) {
    const int block = 128;
    const size_t smem = sizeof(uint4) * (SH / 4) * block;
    const unsigned grid = (unsigned)((count + block - 1) / block);
    const CrtParams<SH>& prm = *static_cast<const CrtParams<SH>*>(raw);
    static AttrCache cache;
    cudaError_t e = cached_attr(cache, [&]() {
        cudaError_t r = cudaFuncSetAttribute(crt_split_kernel<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (r != cudaSuccess) return r;
        return cudaFuncSetAttribute(crt_combine_kernel<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (e != cudaSuccess) return e;
    if (which == 0) crt_split_kernel<SH><<<grid, block, smem, st>>>(prm);
    else crt_combine_kernel<SH><<<grid, block, smem, st>>>(prm);
    return cudaGetLastError();
}

}  // namespace rsa_b200

size_t rsa_b200_crt_params_size(int SH) {
    using namespace rsa_b200;
    switch (SH) {
    case 4: return sizeof(CrtParams<4>);
    case 8: return sizeof(CrtParams<8>);
    case 16: return sizeof(CrtParams<16>);
    case 32: return sizeof(CrtParams<32>);
    case 64: return sizeof(CrtParams<64>);
    default: return 0;
    }
}

// fill a CrtParams<SH> blob: pointers + scalars + the limb arrays (SH limbs each)
void rsa_b200_crt_fill(int SH, void* raw, const uint32_t* c, uint32_t* cp, uint32_t* cq, uint32_t* out,
                       unsigned long long count, int s_io, int sh_io, uint32_t pinv, uint32_t qinv32,
                       const uint32_t* p, const uint32_t* q, const uint32_t* r2p, const uint32_t* r2q,
                       const uint32_t* qinvR) {
    using namespace rsa_b200;
#define FILL(N)                                                                      \
    case N: {                                                                        \
        CrtParams<N>* x = static_cast<CrtParams<N>*>(raw);                           \
        x->c = c; x->cp = cp; x->cq = cq; x->out = out; x->count = count;            \
        x->s_io = s_io; x->sh_io = sh_io; x->pinv = pinv; x->qinv32 = qinv32;        \
        for (int k = 0; k < N; k++) {                                                \
            x->p[k] = p[k]; x->q[k] = q[k]; x->r2p[k] = r2p[k]; x->r2q[k] = r2q[k];  \
            x->qinvR[k] = qinvR[k];                                                  \
        }                                                                            \
        break;                                                                       \
    }
    switch (SH) {
        FILL(4)
        FILL(8)
        FILL(16)
        FILL(32)
        FILL(64)
    }
#undef FILL
}

cudaError_t rsa_b200_crt_launch(int SH, const void* raw, int which, unsigned long long count, cudaStream_t st) {
    using namespace rsa_b200;
    switch (SH) {
    case 4: return crt_launch<4>(raw, which, count, st);
    case 8: return crt_launch<8>(raw, which, count, st);
    case 16: return crt_launch<16>(raw, which, count, st);
    case 32: return crt_launch<32>(raw, which, count, st);
    case 64: return crt_launch<64>(raw, which, count, st);
    default: return cudaErrorInvalidValue;
    }
}
