// dfma_latency.cu -- issue cost of the FP64-pipe digit product on sm_100a
// (csrc/mont_f64.cuh): h = DFMA.RZ(x, y, 2^104); s = DADD(2^104 + 2^52, -h);
// l = DFMA.RZ(x, y, s); acc += bits(l) + bits(h) (IADD3 + IADD3.X).
// W warps per SM sub-partition (one CTA of 4 W warps per SM), C independent
// product chains per thread; reports cycles per digit product per warp and
// FP64 ops/clk/SM.  C = 1, W = 1 is the chain latency; the (C, W) at which the
// FP64 pipe saturates is the parallelism a Montgomery kernel needs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

// MODE 0: the kernel's mix; 1: without the 64-bit column adds; 2: the column adds as
// add.cc (IADD3, ALU) + madc by a runtime 1 (IMAD.X, the IMAD pipe) for the high words
template <int C, int MODE>
__global__ void chain_kernel(unsigned long long* out, double x0, unsigned long long* clk, unsigned one) {
    double x[C], y = 1234567.0 + threadIdx.x;
    unsigned long long acc[C];
#pragma unroll
    for (int c = 0; c < C; c++) { x[c] = x0 + 7.0 * c + threadIdx.x; acc[c] = c; }
    const double c104 = 20282409603651670423947251286016.0, c2 = 20282409603651674927546878656512.0;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            const double h = __fma_rz(x[c], y, c104);
            const double l = __fma_rz(x[c], y, __dsub_rn(c2, h));
            if (MODE == 0) {
                acc[c] += (unsigned long long)__double_as_longlong(l) + (unsigned long long)__double_as_longlong(h);
            } else if (MODE == 2) {
                const unsigned long long bl = __double_as_longlong(l), bh = __double_as_longlong(h);
                unsigned lo = (unsigned)acc[c], hi = (unsigned)(acc[c] >> 32);
                asm volatile("add.cc.u32 %0, %0, %2;\n\tmadc.lo.u32 %1, %3, %6, %1;\n\t"
                             "add.cc.u32 %0, %0, %4;\n\tmadc.lo.u32 %1, %5, %6, %1;"
                             : "+r"(lo), "+r"(hi)
                             : "r"((unsigned)bl), "r"((unsigned)(bl >> 32)), "r"((unsigned)bh),
                               "r"((unsigned)(bh >> 32)), "r"(one));
                acc[c] = ((unsigned long long)hi << 32) | lo;
            }
            // the next product of this chain depends on this one: x <- l (an integer
            // in [2^52, 2^53); with y < 2^21 the product stays < 2^104, the split exact)
            x[c] = l;
        }
    }
    const long long t1 = clock64();
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < C; c++) s += acc[c] + (unsigned long long)__double_as_longlong(x[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = (unsigned long long)(t1 - t0);
}

template <int C, int MODE = 0>
static int run(int sms, int w) {
    unsigned long long *out, *clk;
    const int block = 128 * w;   // W warps per SMSP
    cudaMalloc(&out, sizeof(unsigned long long) * sms * block);
    cudaMalloc(&clk, sizeof(unsigned long long));
    chain_kernel<C, MODE><<<sms, block>>>(out, 3.0, clk, 1u);
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 3; r++) {
        chain_kernel<C, MODE><<<sms, block>>>(out, 3.0, clk, 1u);
        cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, clk, sizeof c, cudaMemcpyDeviceToHost);
        if (c < best) best = (double)c;
    }
    const double products = (double)ITERS * C;   // per warp
    printf("{\"mix\": \"%s\", \"chains_per_thread\": %d, \"warps_per_smsp\": %d, "
           "\"cycles_per_product_per_warp\": %.2f, \"fp64_ops_per_clk_per_sm\": %.1f}\n",
           MODE == 0 ? "dfma+dadd+dfma+iadd3x2" : (MODE == 1 ? "dfma+dadd+dfma" : "dfma+dadd+dfma+(iadd3+imad.x)x2"),
           C, w, best / products,
           3.0 * products * 32 * 4 * w / best);
    cudaFree(out);
    cudaFree(clk);
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {1, 2, 4}) {
        run<1>(sms, w); run<2>(sms, w); run<4>(sms, w); run<8>(sms, w);
    }
    for (int w : {2, 4}) { run<2, 1>(sms, w); run<4, 1>(sms, w); run<8, 1>(sms, w); }
    for (int w : {2, 4}) { run<2, 2>(sms, w); run<4, 2>(sms, w); run<8, 2>(sms, w); }
    return 0;
}
