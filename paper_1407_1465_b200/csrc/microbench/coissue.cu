// coissue.cu -- which instruction classes issue side by side on sm_100a.
// Each kernel runs NCH independent dependency chains per thread of class A
// and (optionally) NCH of class B, interleaved, W warps per SM sub-partition;
// it reports SMSP cycles per (A [+ B]) warp-instruction group.  If A alone
// costs a and B alone b cycles, a pair costing max(a, b) means the two
// classes issue in parallel; a + b means they share an issue resource.  The
// design question (FP64 section): what the integer column adds
// beside the FP64 digit products really cost, and which cheaper instruction
// class could carry them.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 512;
constexpr int NCH = 16;

enum Op { NONE, DFMA, DADD, FFMA, FADD, IADD3, IADD64, LOP3, IMAD, IMADWIDE, SHF, LDS64, LDS128, PRMT, IADD3X };

static const char* opname(int o) {
    switch (o) {
    case NONE: return "none";
    case DFMA: return "dfma";
    case DADD: return "dadd";
    case FFMA: return "ffma";
    case FADD: return "fadd";
    case IADD3: return "iadd3";
    case IADD64: return "iadd3+iadd3.x (64-bit add)";
    case LOP3: return "lop3";
    case IMAD: return "imad";
    case IMADWIDE: return "imad.wide.u32";
    case SHF: return "shf";
    case LDS64: return "lds.64";
    case LDS128: return "lds.128";
    case PRMT: return "prmt";
    case IADD3X: return "iadd3 3-input";
    default: return "?";
    }
}

template <int OP>
__device__ __forceinline__ void step(double& sd, float& sf, unsigned& su, unsigned long long& sw,
                                     unsigned long long k64, int c, const double* sm, unsigned k) {
    if constexpr (OP == DFMA) asm volatile("fma.rn.f64 %0, %0, 0d3FF0000100000000, 0d3FE0000000000000;" : "+d"(sd));
    if constexpr (OP == DADD) asm volatile("add.rn.f64 %0, %0, 0d3FE0000000000000;" : "+d"(sd));
    if constexpr (OP == FFMA) asm volatile("fma.rn.f32 %0, %0, 0f3F800347, 0f3F000000;" : "+f"(sf));
    if constexpr (OP == FADD) asm volatile("add.rn.f32 %0, %0, 0f3F000000;" : "+f"(sf));
    if constexpr (OP == IADD3) asm volatile("add.u32 %0, %0, %1;" : "+r"(su) : "r"(k));
    if constexpr (OP == IADD3X) {
        unsigned t;
        asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(t) : "r"(su), "r"(k), "r"(k ^ 5u));
        su = t;
    }
    if constexpr (OP == IADD64) asm volatile("add.u64 %0, %0, %1;" : "+l"(sw) : "l"(k64));
    if constexpr (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(su) : "r"(k), "r"(k + 7));
    if constexpr (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(su) : "r"(k | 1), "r"(k));
    if constexpr (OP == IMADWIDE) {
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(sw) : "r"((unsigned)sw), "r"(k | 1));
    }
    if constexpr (OP == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, 3;" : "+r"(su) : "r"(k));
    if constexpr (OP == PRMT) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(su) : "r"(k));
    if constexpr (OP == LDS64) {
        double v;
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(sm + 8 * c + (threadIdx.x & 31))));
        sd = v;
    }
    if constexpr (OP == LDS128) {
        double v, x;
        asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(x)
                     : "r"((unsigned)__cvta_generic_to_shared(sm + 16 * c + 2 * (threadIdx.x & 31))));
        sd = v;
        sw = (unsigned long long)__double_as_longlong(x);
    }
}

template <int A, int B>
__global__ void co_kernel(unsigned long long* out, unsigned long long* clk, unsigned seed) {
    __shared__ __align__(16) double sm[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sm[i] = (double)i;
    __syncthreads();
    double d[NCH];
    float f[NCH];
    unsigned u[NCH];
    unsigned long long w[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        d[c] = 1.0 + c + threadIdx.x;
        f[c] = 1.0f + c;
        u[c] = seed + c;
        w[c] = seed * 3ull + c;
    }
    unsigned k = seed ^ threadIdx.x;
    const unsigned long long k64 = ((unsigned long long)seed << 32) | k;
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            step<A>(d[c], f[c], u[c], w[c], k64, c, sm, k);
            step<B>(d[c], f[c], u[c], w[c], k64, c, sm, k);
        }
    }
    const long long t1 = clock64();
    unsigned long long r = 0;
#pragma unroll
    for (int c = 0; c < NCH; c++)
        r += (unsigned long long)__double_as_longlong(d[c]) + __float_as_uint(f[c]) + u[c] + w[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = (unsigned long long)(t1 - t0);
}

template <int A, int B>
static void run(int sms, int w) {
    unsigned long long *out, *clk;
    const int block = 128 * w;
    cudaMalloc(&out, sizeof(unsigned long long) * sms * block);
    cudaMalloc(&clk, sizeof(unsigned long long));
    co_kernel<A, B><<<sms, block>>>(out, clk, 12345u);
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 3; r++) {
        co_kernel<A, B><<<sms, block>>>(out, clk, 12345u);
        cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, clk, sizeof c, cudaMemcpyDeviceToHost);
        if (c < best) best = (double)c;
    }
    const double groups = (double)ITERS * NCH;   // per warp
    printf("{\"a\": \"%s\", \"b\": \"%s\", \"warps_per_smsp\": %d, \"smsp_cycles_per_group\": %.3f}\n", opname(A),
           opname(B), w, best / groups / w);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int w = 4;
#define SINGLE(X) run<X, NONE>(sms, w);
    SINGLE(DFMA) SINGLE(DADD) SINGLE(FFMA) SINGLE(FADD) SINGLE(IADD3) SINGLE(IADD3X) SINGLE(IADD64) SINGLE(LOP3)
    SINGLE(IMAD) SINGLE(IMADWIDE) SINGLE(SHF) SINGLE(PRMT) SINGLE(LDS64) SINGLE(LDS128)
#define PAIR(X, Y) run<X, Y>(sms, w);
    PAIR(DFMA, FFMA) PAIR(DFMA, FADD) PAIR(DFMA, IADD3) PAIR(DFMA, LOP3) PAIR(DFMA, IMAD) PAIR(DFMA, IMADWIDE)
    PAIR(DFMA, SHF) PAIR(DFMA, PRMT) PAIR(DFMA, LDS64) PAIR(DFMA, LDS128) PAIR(DFMA, IADD64) PAIR(DFMA, DADD)
    PAIR(IADD3, FFMA) PAIR(IADD3, IMAD) PAIR(IADD3, LOP3) PAIR(IMAD, FFMA) PAIR(IMADWIDE, IADD3)
    PAIR(IMADWIDE, FFMA) PAIR(LDS128, IADD3) PAIR(FFMA, FADD)
    run<DFMA, NONE>(sms, 2);
    run<DFMA, IADD3>(sms, 2);
    run<IADD3, NONE>(sms, 2);
    return 0;
}
