// tc_redc.cu -- standalone check + timing of the tensor-core Montgomery
// reduction (mont_tc.cuh) on one B200.  Reads in.bin written by
// tools/tc_redc_check.py (n, n' = -n^-1 mod 2^2048, T per packet), runs
// U = T R^-1 mod n for every packet, writes out.bin (U and m per packet);
// the script checks both against Python integers.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc_redc tc_redc.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../mont_tc.cuh"

using namespace rsa_b200;
using namespace rsa_b200::tc;

__global__ void __launch_bounds__(256, 1)
tc_redc_test(const uint32_t* __restrict__ T, uint32_t* __restrict__ U, uint32_t* __restrict__ M,
             const uint8_t* __restrict__ npb, const uint8_t* __restrict__ nb, int reps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    using Sh = TcShared<256, 2>;
    constexpr int NW = Geom<256>::NW;
    Sh& sh = *reinterpret_cast<Sh*>(smem_raw);
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(smem_u32(&sh.tmem_base), 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; i++) mbar_init(smem_u32(&sh.mbar[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    build_strips(sh, npb, nb);
    for (int i = threadIdx.x; i < NW; i += blockDim.x)
        sh.nw[i] = nb[4 * i] | (nb[4 * i + 1] << 8) | (nb[4 * i + 2] << 16) | ((uint32_t)nb[4 * i + 3] << 24);
    fence_before();
    __syncthreads();
    fence_after();
    TcTile tt;
    tt.tile = threadIdx.x / TILE;
    tt.r = threadIdx.x % TILE;
    tt.tmem = sh.tmem_base + 256 * tt.tile;
    tt.tlane = (uint32_t)(32 * (warp % 4)) << 16;
    tt.mbar = smem_u32(&sh.mbar[tt.tile]);
    tt.phase = 0;
    const size_t pkt = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t* t = T + pkt * 128;
    uint32_t th[NW];
    uint32_t t63 = 0;
    for (int rep = 0; rep < reps; rep++) {
#pragma unroll
        for (int c = 0; c < 16; c++) {
            const uint4 v = *reinterpret_cast<const uint4*>(t + 4 * c);
            *stage_chunk(sh, tt.tile, tt.r, c) = v;
            if (c == 15) t63 = v.w;
        }
#pragma unroll
        for (int w = 0; w < NW; w++) th[w] = t[64 + w];
        redc(sh, tt, t63, th);
    }
#pragma unroll
    for (int w = 0; w < NW; w++) U[pkt * NW + w] = th[w];
    // m is still in the staging buffer
#pragma unroll
    for (int c = 0; c < 16; c++) {
        const uint4 v = *stage_chunk(sh, tt.tile, tt.r, c);
        M[pkt * NW + 4 * c] = v.x;
        M[pkt * NW + 4 * c + 1] = v.y;
        M[pkt * NW + 4 * c + 2] = v.z;
        M[pkt * NW + 4 * c + 3] = v.w;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        tmem_dealloc(sh.tmem_base, 512);
    }
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(int argc, char** argv) {
    const char* in = argc > 1 ? argv[1] : "in.bin";
    const char* out = argc > 2 ? argv[2] : "out.bin";
    const int reps = argc > 3 ? atoi(argv[3]) : 1;
    FILE* f = fopen(in, "rb");
    if (!f) { perror(in); return 1; }
    int count = 0;
    if (fread(&count, 4, 1, f) != 1) return 1;
    std::vector<uint8_t> n(256), np(256);
    std::vector<uint32_t> T((size_t)count * 128);
    if (fread(n.data(), 1, 256, f) != 256 || fread(np.data(), 1, 256, f) != 256 ||
        fread(T.data(), 4, T.size(), f) != T.size()) return 1;
    fclose(f);
    if (count % 256) { fprintf(stderr, "count must be a multiple of 256\n"); return 1; }
    uint32_t *dT, *dU, *dM;
    uint8_t *dn, *dnp;
    CK(cudaMalloc(&dT, T.size() * 4));
    CK(cudaMalloc(&dU, (size_t)count * 64 * 4));
    CK(cudaMalloc(&dM, (size_t)count * 64 * 4));
    CK(cudaMalloc(&dn, 256));
    CK(cudaMalloc(&dnp, 256));
    CK(cudaMemcpy(dT, T.data(), T.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dn, n.data(), 256, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dnp, np.data(), 256, cudaMemcpyHostToDevice));
    const int smem = sizeof(TcShared<256, 2>) + 1024;
    CK(cudaFuncSetAttribute(tc_redc_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_redc_test<<<count / 256, 256, smem>>>(dT, dU, dM, dnp, dn, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> U((size_t)count * 64), M((size_t)count * 64);
    CK(cudaMemcpy(U.data(), dU, U.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(M.data(), dM, M.size() * 4, cudaMemcpyDeviceToHost));
    f = fopen(out, "wb");
    fwrite(U.data(), 4, U.size(), f);
    fwrite(M.data(), 4, M.size(), f);
    fclose(f);
    if (reps > 1) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        tc_redc_test<<<count / 256, 256, smem>>>(dT, dU, dM, dnp, dn, reps);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"count\": %d, \"reps\": %d, \"ms\": %.3f, \"redc_per_s\": %.4g}\n", count, reps, ms,
               (double)count * reps / (ms * 1e-3));
    }
    printf("smem %d bytes\n", smem);
    return 0;
}
