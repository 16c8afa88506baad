// dfma_mix.cu -- what an extra instruction costs beside the FP64-pipe digit
// product on sm_100a (csrc/mont_f64.cuh).  Every variant runs the exact split
// h = DFMA.RZ(x, y, 2^104); s = DADD(2^104 + 2^52, -h); l = DFMA.RZ(x, y, s)
// on C independent chains per thread (x <- l), W warps per SM sub-partition,
// plus MODE's extra work per product; reports cycles per product per warp,
// FP64 ops/clk/SM and warp instructions issued per clk per SMSP.  The question
// it answers: which auxiliary instruction classes (64-bit integer add, 32-bit
// add, LOP3, IMAD, FP32, shared-memory load) are "free" beside the FP64 pipe
// and which take dispatch slots from it -- the design input for cutting the
// integer work per digit product (FP64 section).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

#define MODES(X)                                                        \
    X(0, "fp64 only (dfma dadd dfma)", 0)                               \
    X(1, "+ 64-bit add of l and h (iadd3 + iadd3.x)", 2)                \
    X(2, "+ one 32-bit 3-input add (iadd3)", 1)                         \
    X(3, "+ two 32-bit 2-input adds (2 iadd3)", 2)                      \
    X(4, "+ one lop3", 1)                                               \
    X(5, "+ one 32-bit imad", 1)                                        \
    X(6, "+ one fp32 ffma", 1)                                          \
    X(7, "+ two fp32 ffma", 2)                                          \
    X(8, "fp64 only, constants in registers", 0)                        \
    X(9, "+ 64-bit add of l only (iadd3 + iadd3.x)", 2)                 \
    X(10, "+ two 64-bit adds (4 alu)", 4)                               \
    X(11, "+ one lds.64 + one iadd3 consuming it", 2)                                            \
    X(12, "+ one lds.128 per 2 products + one iadd3 consuming it", 2)                            \
    X(13, "+ 64-bit add (iadd3 + iadd3.x) + one lds.64 + one iadd3", 4)             \
    X(14, "+ one 32-bit 3-input add + one lop3", 2)

template <int C, int MODE>
__global__ void mix_kernel(unsigned long long* out, double x0, unsigned long long* clk, double rc104, double rc2) {
    __shared__ __align__(16) double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)(i * 3 + 1);
    __syncthreads();
    double x[C], y = 1234567.0 + threadIdx.x;
    unsigned long long acc[C], acc2[C];
    unsigned a32[C], b32[C];
    float f[C], g[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
        x[c] = x0 + 7.0 * c + threadIdx.x;
        acc[c] = c;
        acc2[c] = 3 * c;
        a32[c] = c;
        b32[c] = 5 * c;
        f[c] = 1.0f + c;
        g[c] = 2.0f + c;
    }
    const double c104 = (MODE == 8) ? rc104 : 20282409603651670423947251286016.0;
    const double c2 = (MODE == 8) ? rc2 : 20282409603651674927546878656512.0;
    unsigned soff = threadIdx.x & 31;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            const double h = __fma_rz(x[c], y, c104);
            const double l = __fma_rz(x[c], y, __dsub_rn(c2, h));
            const unsigned long long bl = __double_as_longlong(l), bh = __double_as_longlong(h);
            if (MODE == 1 || MODE == 13) acc[c] += bl + bh;
            if (MODE == 2 || MODE == 14) a32[c] += (unsigned)bl + (unsigned)bh;
            if (MODE == 3) { a32[c] += (unsigned)bl; b32[c] += (unsigned)bh; }
            if (MODE == 4 || MODE == 14) b32[c] = (b32[c] & (unsigned)bl) ^ (unsigned)bh;
            if (MODE == 5) a32[c] = a32[c] * (unsigned)bl + (unsigned)bh;
            if (MODE == 6 || MODE == 7) f[c] = fmaf(f[c], __uint_as_float((unsigned)bl | 0x3f800000u), 1.0f);
            if (MODE == 7) g[c] = fmaf(g[c], __uint_as_float((unsigned)bh | 0x3f800000u), 1.0f);
            if (MODE == 9) acc[c] += bl;
            if (MODE == 10) { acc[c] += bl; acc2[c] += bh; }
            if (MODE == 11 || MODE == 13) {
                double v;
                asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v)
                             : "r"((unsigned)__cvta_generic_to_shared(sm + ((soff + 8 * c + it) & 1023))));
                const unsigned long long bv = __double_as_longlong(v);
                b32[c] += (unsigned)bv + (unsigned)(bv >> 32);      // consume: one 3-input IADD3
            }
            if (MODE == 12 && (c & 1) == 0) {
                double v, w;
                asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(w)
                             : "r"((unsigned)__cvta_generic_to_shared(sm + ((2 * (soff + 8 * c + it)) & 1022))));
                const unsigned long long bv = __double_as_longlong(v), bw = __double_as_longlong(w);
                a32[c] += (unsigned)bv + (unsigned)(bv >> 32);
                b32[c] += (unsigned)bw + (unsigned)(bw >> 32);
            }
            const double nx = l;
            x[c] = nx;
        }
    }
    const long long t1 = clock64();
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < C; c++)
        s += acc[c] + acc2[c] + a32[c] + b32[c] + (unsigned long long)__double_as_longlong(x[c]) +
             __float_as_uint(f[c]) + __float_as_uint(g[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = (unsigned long long)(t1 - t0);
}

template <int C, int MODE>
static void run(int sms, int w, const char* name, int extra) {
    unsigned long long *out, *clk;
    const int block = 128 * w;
    cudaMalloc(&out, sizeof(unsigned long long) * sms * block);
    cudaMalloc(&clk, sizeof(unsigned long long));
    const double c104 = 20282409603651670423947251286016.0, c2 = 20282409603651674927546878656512.0;
    mix_kernel<C, MODE><<<sms, block>>>(out, 3.0, clk, c104, c2);
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 3; r++) {
        mix_kernel<C, MODE><<<sms, block>>>(out, 3.0, clk, c104, c2);
        cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, clk, sizeof c, cudaMemcpyDeviceToHost);
        if (c < best) best = (double)c;
    }
    const double products = (double)ITERS * C;   // per warp
    const double cyc = best / products;           // cycles per product per warp
    printf("{\"mode\": %d, \"mix\": \"%s\", \"extra_instr_per_product\": %d, \"chains_per_thread\": %d, "
           "\"warps_per_smsp\": %d, \"cycles_per_product_per_warp\": %.2f, \"fp64_ops_per_clk_per_sm\": %.1f, "
           "\"smsp_cycles_per_product\": %.2f}\n",
           MODE, name, extra, C, w, cyc, 3.0 * 32 * 4 * w / cyc, cyc / w);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define RUN(M, NAME, EXTRA)           \
    run<8, M>(sms, 2, NAME, EXTRA);   \
    run<8, M>(sms, 4, NAME, EXTRA);
    MODES(RUN)
    return 0;
}
