// imad_latency.cu -- dependent-issue latency of the Montgomery chain forms on
// sm_100a: one warp per SMSP (4 warps per SM, one CTA per SM), C independent
// carry chains per thread (C = 1, 2, 4, 8); cycles per chained IMAD.WIDE.U32.X
// = measured cycles / (iterations * products per chain).  With C = 1 this is
// the chain latency; the C at which cycles/product reaches 4 (the half-rate
// issue interval per SMSP) is the parallelism the kernels need per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int C>
__global__ void chain_kernel(uint32_t* out, uint32_t a0, unsigned long long* clk) {
    uint32_t acc[C][9], av[8];
#pragma unroll
    for (int k = 0; k < 8; k++) av[k] = a0 * (k + 3) + threadIdx.x;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int k = 0; k < 9; k++) acc[c][k] = k + c;
    uint32_t b = a0 ^ threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            asm volatile(
                "mad.lo.cc.u32 %0, %9, %17, %0;\n\t"
                "madc.hi.cc.u32 %1, %9, %17, %1;\n\t"
                "madc.lo.cc.u32 %2, %10, %17, %2;\n\t"
                "madc.hi.cc.u32 %3, %10, %17, %3;\n\t"
                "madc.lo.cc.u32 %4, %11, %17, %4;\n\t"
                "madc.hi.cc.u32 %5, %11, %17, %5;\n\t"
                "madc.lo.cc.u32 %6, %12, %17, %6;\n\t"
                "madc.hi.cc.u32 %7, %12, %17, %7;\n\t"
                "addc.u32 %8, %8, 0;\n\t"
                : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3]), "+r"(acc[c][4]),
                  "+r"(acc[c][5]), "+r"(acc[c][6]), "+r"(acc[c][7]), "+r"(acc[c][8])
                : "r"(av[0]), "r"(av[1]), "r"(av[2]), "r"(av[3]), "r"(av[4]), "r"(av[5]), "r"(av[6]),
                  "r"(av[7]), "r"(b));
        }
        b ^= acc[0][7];
    }
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int k = 0; k < 9; k++) s ^= acc[c][k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = (unsigned long long)(t1 - t0);
}

template <int C>
static void run(int sms, int warps_per_smsp) {
    uint32_t* out; unsigned long long* clk;
    const int threads = 128 * warps_per_smsp;
    cudaMalloc(&out, sizeof(uint32_t) * sms * threads);
    cudaMalloc(&clk, 8);
    chain_kernel<C><<<sms, threads>>>(out, 7, clk);
    cudaDeviceSynchronize();
    chain_kernel<C><<<sms, threads>>>(out, 7, clk);
    unsigned long long h;
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / ((double)ITERS * 4.0 * C);    // 4 wide products per chain per iter
    printf("{\"chains_per_thread\": %d, \"warps_per_smsp\": %d, \"cycles_per_chained_product_per_warp\": %.2f, "
           "\"smsp_products_per_cycle\": %.3f}\n", C, warps_per_smsp, per, warps_per_smsp * 32.0 / per / 32.0);
    cudaFree(out); cudaFree(clk);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {1, 2, 3, 4}) {
        run<1>(sms, w); run<2>(sms, w); run<4>(sms, w); run<8>(sms, w);
    }
    return 0;
}
