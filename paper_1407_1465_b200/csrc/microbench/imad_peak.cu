// imad_peak.cu -- integer-multiply issue-rate microbenchmark for sm_100a.
//
// Fixes the roofline denominator of DESIGN.md "Roofline": how many 32x32->64
// limb products per clock per SM the fmaheavy pipe sustains, in the exact
// instruction forms a Montgomery kernel can use.  Every multiplier operand is
// loop-carried (b ^= previous result) so ptxas cannot hoist or
// strength-reduce the products.
//   wide     : mad.wide.u32                      -> IMAD.WIDE.U32 (no carries)
//   wide_co  : mad.lo.cc + madc.hi.cc + addc     -> IMAD.WIDE.U32 (carry-out) + IADD3.X
//   chain    : mad.lo.cc / madc.lo.cc / madc.hi.cc row chains -> IMAD.WIDE.U32.X
//   lo / hi  : mad.lo.u32 / mad.hi.u32           -> IMAD / IMAD.HI.U32
//   dfma     : fma.rn.f64                        -> DFMA
// The SM clock is measured in-kernel (%clock64 vs %globaltimer).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

#define PROLOGUE \
    uint64_t c0 = clock64(), t0 = gtimer();
#define EPILOGUE(S) \
    uint64_t c1 = clock64(), t1 = gtimer(); \
    out[blockIdx.x * blockDim.x + threadIdx.x] = (S); \
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }

// 8 independent 64-bit accumulators, mad.wide.u32
__global__ void k_wide(uint32_t* out, uint32_t a0, uint32_t b0, unsigned long long* clk) {
    uint64_t acc[8]; uint32_t av[8];
    uint32_t b = b0 ^ threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; k++) { acc[k] = k; av[k] = a0 * (2 * k + 1) + threadIdx.x; }
    PROLOGUE
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[k]) : "r"(av[k]), "r"(b));
        b ^= (uint32_t)(acc[it & 7] >> 7);
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += acc[k];
    EPILOGUE((uint32_t)s ^ (uint32_t)(s >> 32))
}

// 8 independent 64-bit MACs each with carry-out captured into a third word
__global__ void k_wide_co(uint32_t* out, uint32_t a0, uint32_t b0, unsigned long long* clk) {
    uint32_t lo[8], hi[8], tp[8], av[8];
    uint32_t b = b0 ^ threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; k++) { lo[k] = k; hi[k] = 0; tp[k] = 0; av[k] = a0 * (2 * k + 1) + threadIdx.x; }
    PROLOGUE
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                         : "+r"(lo[k]), "+r"(hi[k]), "+r"(tp[k]) : "r"(av[k]), "r"(b));
        b ^= hi[it & 7];
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s ^= lo[k] ^ hi[k] ^ tp[k];
    EPILOGUE(s)
}

// row chain: acc[0..8) += a[0..4) * b with carry propagation (1 plain + 3 .X)
__device__ __forceinline__ void row4(uint32_t* acc, const uint32_t* av, uint32_t b) {
    asm volatile(
        "mad.lo.cc.u32 %0, %9, %13, %0;\n\t"
        "madc.hi.cc.u32 %1, %9, %13, %1;\n\t"
        "madc.lo.cc.u32 %2, %10, %13, %2;\n\t"
        "madc.hi.cc.u32 %3, %10, %13, %3;\n\t"
        "madc.lo.cc.u32 %4, %11, %13, %4;\n\t"
        "madc.hi.cc.u32 %5, %11, %13, %5;\n\t"
        "madc.lo.cc.u32 %6, %12, %13, %6;\n\t"
        "madc.hi.cc.u32 %7, %12, %13, %7;\n\t"
        "addc.u32 %8, %8, 0;\n\t"
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
          "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8])
        : "r"(av[0]), "r"(av[1]), "r"(av[2]), "r"(av[3]), "r"(b));
}

__global__ void k_chain(uint32_t* out, uint32_t a0, uint32_t b0, unsigned long long* clk) {
    uint32_t ev[4][9], av[4][4];
    uint32_t b = b0 ^ threadIdx.x;
#pragma unroll
    for (int c = 0; c < 4; c++) {
#pragma unroll
        for (int k = 0; k < 4; k++) av[c][k] = a0 * (k + 1 + 4 * c) + threadIdx.x;
#pragma unroll
        for (int k = 0; k < 9; k++) ev[c][k] = k;
    }
    PROLOGUE
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < 4; c++) row4(ev[c], av[c], b);   // 4 independent chains x 4 products
        b ^= ev[it & 3][7];
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int k = 0; k < 9; k++) s ^= ev[c][k];
    EPILOGUE(s)
}

template <int MODE>   // 0: mad.lo, 1: mad.hi, 3: fma.rn.f64
__global__ void k_simple(uint32_t* out, uint32_t a0, uint32_t b0, unsigned long long* clk) {
    uint32_t acc[8], av[8];
    double dacc[8];
    uint32_t b = b0 ^ threadIdx.x;
    double db = 0.999999 + threadIdx.x * 1e-9;
#pragma unroll
    for (int k = 0; k < 8; k++) { acc[k] = k; dacc[k] = k; av[k] = a0 * (2 * k + 1) + threadIdx.x; }
    PROLOGUE
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (MODE == 0) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[k]) : "r"(av[k]), "r"(b));
            if (MODE == 1) asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[k]) : "r"(av[k]), "r"(b));
            if (MODE == 3) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dacc[k]) : "d"(db), "d"(1e-300));
        }
        if (MODE != 3) b ^= acc[it & 7];
        else db = dacc[it & 7] * 1e-30 + 0.999999;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s ^= acc[k] ^ (uint32_t)(long long)dacc[k];
    EPILOGUE(s)
}

typedef void (*kfn)(uint32_t*, uint32_t, uint32_t, unsigned long long*);

static int run(const char* name, kfn f, double ops_per_thread_iter, const char* unit,
               int sms, int blocks_per_sm, int threads) {
    uint32_t* out; unsigned long long* clk;
    int grid = sms * blocks_per_sm;
    CK(cudaMalloc(&out, sizeof(uint32_t) * grid * threads));
    CK(cudaMalloc(&clk, 16));
    f<<<grid, threads>>>(out, 3, 5, clk);   // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        f<<<grid, threads>>>(out, 3, 5, clk);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    unsigned long long hc[2];
    CK(cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost));
    double mhz = (double)hc[0] / (double)hc[1] * 1e3;
    double total = ops_per_thread_iter * (double)ITERS * grid * threads;
    double per_s = total / (best * 1e-3);
    double per_clk_sm = per_s / (mhz * 1e6) / sms;
    printf("{\"form\": \"%s\", \"blocks_per_sm\": %d, \"threads\": %d, \"ms\": %.4f, \"sm_mhz\": %.0f, "
           "\"%s_per_s\": %.4e, \"%s_per_clk_per_sm\": %.2f}\n",
           name, blocks_per_sm, threads, best, mhz, unit, per_s, unit, per_clk_sm);
    cudaFree(out); cudaFree(clk);
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int bps : {2, 4, 8}) {
        run("mad.wide.u32", k_wide, 8, "products", sms, bps, 256);
        run("mad.lo.cc+madc.hi.cc+addc (carry-out)", k_wide_co, 8, "products", sms, bps, 256);
        run("madc row chain (IMAD.WIDE.U32.X)", k_chain, 16, "products", sms, bps, 256);
        run("mad.lo.u32", k_simple<0>, 8, "imad", sms, bps, 256);
        run("mad.hi.u32", k_simple<1>, 8, "imad_hi", sms, bps, 256);
        run("fma.rn.f64", k_simple<3>, 8, "dfma", sms, bps, 256);
    }
    return 0;
}
