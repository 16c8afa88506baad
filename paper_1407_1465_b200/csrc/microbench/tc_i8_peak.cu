// tc_i8_peak.cu -- issue rate of tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32)
// on one B200, the tensor-core peak behind bench.py's roofline.tensor: one
// CTA per SM, one thread issues back-to-back MMAs of M = 128, K = 32 and
// N = 128 / 256 from shared-memory operands (SWIZZLE_NONE, the layout of
// mont_tc.cuh) into TMEM, with a commit + mbarrier wait every `batch` MMAs.
// Prints one JSON line per shape: int8 ops/s (2 per MAC) over the whole GPU.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc_i8_peak tc_i8_peak.cu
#include <cstdio>

#include "../tc_i8.cuh"

using namespace rsa_b200::tc;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int batch, unsigned long long* sink) {
    __shared__ __align__(1024) uint8_t a[128 * 32];
    __shared__ __align__(1024) uint8_t b[N * 32];
    __shared__ unsigned long long mbar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) a[i] = (uint8_t)(i * 7 + 1);
    for (int i = threadIdx.x; i < N * 32; i += blockDim.x) b[i] = (uint8_t)(i * 13 + 3);
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&tbase), 512);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&mbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint64_t ad = sdesc(smem_u32(a), 128 * 16, 128);   // rows 16 B apart, K chunks 2 KB apart
    const uint64_t bd = sdesc(smem_u32(b), N * 16, 128);
    constexpr uint32_t id = idesc_u8(128, N);
    uint32_t phase = 0;
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; it += batch) {
            for (int k = 0; k < batch; k++) mma_u8(tbase + (k & 1) * (512 - N), ad, bd, id, k > 0);
            commit(smem_u32(&mbar));
            mbar_wait(smem_u32(&mbar), phase);
            phase ^= 1;
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    uint32_t v[32];
    tmem_ld32(tbase + ((uint32_t)(32 * (threadIdx.x / 32)) << 16), v);
    tmem_ld_wait();
    if (v[0] == 0x12345678u) sink[0] = v[1];   // keep the result observable
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        fence_after();
        tmem_dealloc(tbase, 512);
    }
}

template <int N>
static void run(int sms) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int iters = 1 << 16;
    for (int batch : {8, 64}) {
        mma_loop<N><<<sms, 128>>>(256, batch, sink);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        mma_loop<N><<<sms, 128>>>(iters, batch, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const cudaError_t err = cudaGetLastError();
        const double ops = 2.0 * 128 * N * 32 * (double)iters * sms;
        printf("{\"shape\": \"u8 M=128 N=%d K=32\", \"batch\": %d, \"sms\": %d, \"ms\": %.3f, "
               "\"int8_tops\": %.1f, \"macs_per_clk_per_sm_at_1965\": %.0f, \"err\": \"%s\"}\n",
               N, batch, sms, ms, ops / (ms * 1e-3) / 1e12, ops / 2 / (ms * 1e-3) / sms / 1.965e9,
               cudaGetErrorString(err));
    }
    cudaFree(sink);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<128>(sms);
    run<256>(sms);
    return 0;
}
