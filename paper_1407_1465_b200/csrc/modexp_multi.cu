// modexp_multi.cu -- per-packet moduli and exponents (SURVEY.md sec. 8(f)
// row f1): multi-key batches and the Miller-Rabin test that drives the GPU
// prime search for key generation (Fig 1, "choose two different random prime
// numbers").
//
// One thread per packet.  Everything per-key is derived on the device:
//   n'  = -n^-1 mod 2^32             (Newton, 5 steps)
//   r1  = R mod n                    (2^b - n, then 32S - b modular doublings)
//   R^2 mod n = Mont(2^KD)^(2^J)     (KD more doublings, then J Montgomery
//                                     squarings, KD 2^J = 32 S; plan.h)
// The exponent is scanned with a FIXED window of w bits over a uniform bit
// length (exp_bits), so every thread executes the same op sequence and only
// the table index (its own digit) differs: no divergence despite per-packet
// exponents.  T[0] = Mont(1) makes a zero digit a plain multiply.
//   mode 0: out[i] = base[i]^exp[i] mod mod[i]
//   mode 1: Miller-Rabin to base `mr_base` on candidate mod[i]:
//           n - 1 = 2^r d;  x = a^d;  prime-ish iff x == 1 or some
//           x^(2^j) == n - 1, j < r;  out[i] = 1 (probable prime) / 0.
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

#include "devcache.h"
#include "mont_multi.cuh"
#include "plan.h"

namespace rsa_b200 {

struct MultiParams {
    const uint32_t* base;     // [count][s_io] (mode 0)
    const uint32_t* exps;     // [count][s_io] (mode 0)
    const uint32_t* mods;     // [count][s_io]
    uint32_t* out;            // [count][s_io] (mode 0) or [count] flags (mode 1)
    int32_t* status;          // [count] or null: 0 ok, -3 (RSA_EEVEN) bad modulus
    uint4* table;             // workspace: 2^w entries x S limbs x nthreads
    unsigned long long count;
    int s_io;
    int exp_bits;             // bits scanned (mode 0); mode 1 uses nbits - 1
    int window;               // fixed window width w (1..6)
    int mode;
    uint32_t mr_base;
};

template <int S>
#ifndef RSA_MMINB32
#define RSA_MMINB32 2
#endif
#ifndef RSA_MMINB16
#define RSA_MMINB16 4
#endif
#ifndef RSA_MULTI_SKIP0
#define RSA_MULTI_SKIP0 1
#endif
#ifndef RSA_MULTI_NREG_MAX
#define RSA_MULTI_NREG_MAX 32
#endif
struct MCfg {
    static constexpr int BLOCK = (S >= 64) ? 256 : 128;
    static constexpr bool NREG = (S <= RSA_MULTI_NREG_MAX);   // n in registers (else shared memory)
    static constexpr int MINB = (S >= 64) ? 1 : (S >= 32 ? RSA_MMINB32 : RSA_MMINB16);
};

// w bits of a packet's exponent at bit position pos (bits beyond the packet are 0)
__device__ __forceinline__ uint32_t exp_bits_at(const uint32_t* e, int s_io, int pos, int w) {
    const int li = pos >> 5, sh = pos & 31;
    uint64_t v = (li < s_io) ? __ldg(e + li) : 0u;
    if (li + 1 < s_io) v |= (uint64_t)__ldg(e + li + 1) << 32;
    return (uint32_t)(v >> sh) & ((1u << w) - 1u);
}

template <int S>
__global__ void __launch_bounds__(MCfg<S>::BLOCK, MCfg<S>::MINB)
modexp_multi_kernel(const __grid_constant__ MultiParams p) {
    constexpr int NG = S / 4;
    constexpr int NQ = S / 8;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int stride = MCfg<S>::BLOCK;       // launched with exactly this block size
    constexpr bool NREG = MCfg<S>::NREG;
    using NS = std::conditional_t<NREG, NRegsT<S, stride>, NSharedT<stride>>;
    uint4* const bslot = reinterpret_cast<uint4*>(smem_raw) + threadIdx.x;
    uint4* const nodd = reinterpret_cast<uint4*>(smem_raw) + NG * stride + threadIdx.x;
    uint4* const neven = nodd + NQ * stride;
    uint32_t nreg[S];
    const NS nsh = [&] {
        if constexpr (NREG) return NS{nreg};
        else return NS{nodd, neven};
    }();
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned nthr = gridDim.x * blockDim.x;
    const int w = p.window;
    const int nent = 1 << w;
    const unsigned long long trips = (p.count + nthr - 1) / nthr;
    // per-thread contiguous entries: with per-packet exponents the lanes of a
    // warp read different entries, so each entry is one thread's 16*S bytes
    // (whole lines) rather than striped across threads
    auto tab = [&](int entry, int g) -> uint4& { return p.table[((size_t)gtid * nent + entry) * NG + g]; };
    auto store_a = [&](int entry, const uint32_t (&v)[S]) {
#pragma unroll
        for (int g = 0; g < NG; g++) tab(entry, g) = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    };
    auto load_a = [&](int entry, uint32_t (&v)[S]) {
#pragma unroll
        for (int g = 0; g < NG; g++) {
            const uint4 x = tab(entry, g);
            v[4 * g] = x.x; v[4 * g + 1] = x.y; v[4 * g + 2] = x.z; v[4 * g + 3] = x.w;
        }
    };
    auto stage = [&](const uint32_t (&v)[S]) {
#pragma unroll
        for (int g = 0; g < NG; g++) bslot[g * stride] = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    };

    for (unsigned long long t = 0; t < trips; t++) {
        const unsigned long long pkt0 = gtid + t * nthr;
        const bool valid = pkt0 < p.count;
        const unsigned long long pkt = valid ? pkt0 : p.count - 1;
        const uint32_t* nsrc = p.mods + pkt * (unsigned long long)p.s_io;
        uint32_t a[S];
        // ---- the modulus into this thread's smem slot (odd / even limbs)
#pragma unroll
        for (int k = 0; k < S; k++) a[k] = (k < p.s_io) ? __ldg(nsrc + k) : 0u;
        if constexpr (NREG) {
#pragma unroll
            for (int k = 0; k < S; k++) nreg[k] = a[k];
        } else {
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                nodd[q * stride] = make_uint4(a[8 * q + 1], a[8 * q + 3], a[8 * q + 5], a[8 * q + 7]);
                neven[q * stride] = make_uint4(a[8 * q], a[8 * q + 2], a[8 * q + 4], a[8 * q + 6]);
            }
        }
        bool small = a[0] < 3;
#pragma unroll
        for (int k = 1; k < S; k++) small = small && a[k] == 0;
        const bool bad = ((a[0] & 1u) == 0) || small;
        // n' = -n^-1 mod 2^32
        uint32_t inv = a[0];
#pragma unroll
        for (int i = 0; i < 5; i++) inv *= 2u - a[0] * inv;
        const uint32_t n0inv = 0u - inv;
        // bit length b of n; v = 2^b - n (< n), then 32S - b doublings -> R mod n
        int b = 0;
#pragma unroll
        for (int k = 0; k < S; k++)
            if (a[k]) b = 32 * k + 32 - __clz(a[k]);
        {
            // two's complement of n restricted to b bits
            uint32_t c = 1;
#pragma unroll
            for (int k = 0; k < S; k++) {
                const uint64_t v = (uint64_t)(~a[k]) + c;
                a[k] = (uint32_t)v;
                c = (uint32_t)(v >> 32);
                const int lo = 32 * k;
                if (lo >= b) a[k] = 0;
                else if (b - lo < 32) a[k] &= (1u << (b - lo)) - 1u;
            }
        }
        // v = 2v mod n, (32S - b) + KD times: the last KD give Mont(2^KD) = 2^KD R mod n
        constexpr int KD = MultiR2<S>::KD;
        for (int d = 0; d < 32 * S - b + KD; d++) {
            if (d == 32 * S - b) store_a(0, a);          // T[0] = R mod n = Mont(1)
            uint32_t top = a[S - 1] >> 31;
            uint32_t sh[S];
#pragma unroll
            for (int k = S - 1; k > 0; k--) sh[k] = (a[k] << 1) | (a[k - 1] >> 31);
            sh[0] = a[0] << 1;
            const NS& nn = nsh;
            uint32_t dd[S];
            sub_cc(dd[0], sh[0], nn.limb(0));
#pragma unroll
            for (int k = 1; k < S; k++) subc_cc(dd[k], sh[k], nn.limb(k));
            uint32_t keep;
            subc(keep, top, 0u);                          // 0 if 2v >= n (use dd)
#pragma unroll
            for (int k = 0; k < S; k++) a[k] = (sh[k] & keep) | (dd[k] & ~keep);
        }
        // ---- exponent source
        const uint32_t* esrc;
        int ebits, eoff;
        if (p.mode == 0) {
            esrc = p.exps + pkt * (unsigned long long)p.s_io;
            ebits = p.exp_bits;
            eoff = 0;
        } else {
            // d = (n - 1) >> r: the bits of n above position r (n odd)
            int r = 1;
            while (r < 32 * p.s_io && ((__ldg(nsrc + (r >> 5)) >> (r & 31)) & 1u) == 0) r++;
            esrc = nsrc;
            eoff = r;
            ebits = 32 * p.s_io - 1;                       // uniform upper bound on bits(d)
        }
        const int nwin = (ebits + w - 1) / w;
        // ---- step machine (one call site each for montsqr_sm / montmul_sm):
        //  [0, K)                 SQR: Mont(2^KD) -> R^2 mod n  (K = J, plan.h)
        //  K                      MUL: x * R^2 -> T[1] = Mont(x)
        //  K+1 .. K+nent-2        MUL: T[j] = T[j-1] * T[1]
        //  scan                   per window below the top: w SQR + 1 MUL by T[digit]
        //  mode 0: 1 MUL by 1 (from Montgomery);  mode 1: r-1 SQR, compare with Mont(-1)
        constexpr int K = MultiR2<S>::SQ;
        const int s_tab = K + 1, s_scan = K + 1 + (nent - 2);
        const int s_fin = s_scan + (nwin - 1) * (w + 1);
        // lockstep (S >= 64): a barrier per step keeps the CTA's warps on the
        // same code lines; the Miller-Rabin tail runs to the block's largest r
        // (extra squarings of a thread past its own r do not change its verdict)
        int tail = (p.mode == 0 ? 1 : eoff - 1);
        if constexpr (S >= 64) {
            __shared__ int s_tail;
            if (threadIdx.x == 0) s_tail = 0;
            __syncthreads();
            atomicMax(&s_tail, tail);
            __syncthreads();
            tail = s_tail;
            __syncthreads();
        }
        const int total = s_fin + tail;
        const int my_total = s_fin + (p.mode == 0 ? 1 : eoff - 1);
        uint32_t mone[S];
        bool prime = false;
        for (int st = 0; st < total; st++) {
            if constexpr (S >= 64) __syncthreads();
            bool sqr;
            if (st < K) {
                sqr = true;
            } else if (st == K) {
                stage(a);                                   // b = R^2 mod n
                if (p.mode == 0) {
                    const uint32_t* bsrc = p.base + pkt * (unsigned long long)p.s_io;
#pragma unroll
                    for (int k = 0; k < S; k++) a[k] = (k < p.s_io) ? __ldg(bsrc + k) : 0u;
                } else {
#pragma unroll
                    for (int k = 0; k < S; k++) a[k] = 0u;
                    a[0] = p.mr_base;
                }
                sqr = false;
            } else if (st < s_scan) {
                if (st == s_tab) stage(a);                  // b = T[1] for the table chain
                sqr = false;
            } else if (st < s_fin) {
                const int rel = st - s_scan;
                const int wi = nwin - 2 - rel / (w + 1);
                const int ph = rel % (w + 1);
                if (rel == 0) {                              // A = T[top digit]
                    const int pos = (nwin - 1) * w;
                    load_a((int)exp_bits_at(esrc, p.s_io, pos + eoff, ebits - pos), a);
                }
                sqr = ph < w;
                if (!sqr) {
                    const uint32_t dig = exp_bits_at(esrc, p.s_io, wi * w + eoff, w);
                    // the multiply by T[0] = Mont(1) is the identity (mod n): a CTA (the
                    // lockstep classes) or warp whose digits are all 0 skips it.  Sparse
                    // exponents (e = 65537: 7 of 8 windows below the top at w = 2) gain
                    // the most; the result is unchanged (RSA_MULTI_SKIP0 = 0 for A/B).
                    if constexpr (RSA_MULTI_SKIP0 != 0) {
                        bool any;
                        if constexpr (S >= 64) any = __syncthreads_or(dig != 0u) != 0;
                        else any = __any_sync(__activemask(), dig != 0u);
                        if (!any) continue;
                    }
#pragma unroll
                    for (int g = 0; g < NG; g++) bslot[g * stride] = tab(dig, g);
                }
            } else if (p.mode == 0) {
                if (st == s_fin && s_fin == s_scan) load_a((int)exp_bits_at(esrc, p.s_io, eoff, ebits), a);
                uint32_t one[S];
#pragma unroll
                for (int k = 0; k < S; k++) one[k] = 0u;
                one[0] = 1u;
                stage(one);
                sqr = false;
            } else {
                sqr = true;
            }
            // MR: before the first post-scan squaring, test x = a^d against +-1
            if (p.mode == 1 && st == s_fin) {
                if (s_fin == s_scan) load_a((int)exp_bits_at(esrc, p.s_io, eoff, ebits), a);
                uint32_t one[S];
                load_a(0, one);                              // Mont(1) = R mod n
                sub_cc(mone[0], nsh.limb(0), one[0]);        // Mont(n-1) = n - Mont(1)
#pragma unroll
                for (int k = 1; k < S; k++) subc_cc(mone[k], nsh.limb(k), one[k]);
                bool eq1 = true, eqm = true;
#pragma unroll
                for (int k = 0; k < S; k++) { eq1 = eq1 && a[k] == one[k]; eqm = eqm && a[k] == mone[k]; }
                prime = eq1 || eqm;
            }
            if (sqr) montsqr_sm<S, NS>(a, nsh, n0inv);
            else montmul_sm<S, NS>(a, bslot, stride, nsh, n0inv);
            if (st >= K && st < s_scan) store_a(st - K + 1, a);   // T[1] .. T[nent-1]
            if (p.mode == 1 && st >= s_fin && st < my_total) {
                bool e = true;
#pragma unroll
                for (int k = 0; k < S; k++) e = e && a[k] == mone[k];
                prime = prime || e;
            }
        }
        if (p.mode == 1 && my_total == s_fin && total == s_fin) {   // r == 1 everywhere: no squaring after the scan
            if (s_fin == s_scan) load_a((int)exp_bits_at(esrc, p.s_io, eoff, ebits), a);
            uint32_t one[S];
            load_a(0, one);
            sub_cc(mone[0], nsh.limb(0), one[0]);
#pragma unroll
            for (int k = 1; k < S; k++) subc_cc(mone[k], nsh.limb(k), one[k]);
            bool eq1 = true, eqm = true;
#pragma unroll
            for (int k = 0; k < S; k++) { eq1 = eq1 && a[k] == one[k]; eqm = eqm && a[k] == mone[k]; }
            prime = eq1 || eqm;
        }
        if (valid) {
            if (p.mode == 0) {
                uint32_t* dst = p.out + pkt * (unsigned long long)p.s_io;
#pragma unroll
                for (int k = 0; k < S; k++)
                    if (k < p.s_io) dst[k] = bad ? 0u : a[k];
            } else {
                p.out[pkt] = (prime && !bad) ? 1u : 0u;
            }
        }
        if (valid && p.status) p.status[pkt] = bad ? -3 : 0;
    }
}


// ---------------------------------------------------------------------------
// Prime-search helpers.  Candidate i of a search (seed): limb pair j is the
// splitmix64 finaliser of seed + (i * 2^16 + j + 1) * 0x9E3779B97F4A7C15;
// the value is masked to nbits, bits nbits-1 and nbits-2 set (so p*q has
// exactly 2*nbits bits), bit 0 set.  workload/ re-implements this generator
// independently for the tests.
__device__ __forceinline__ uint64_t splitmix_mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void prime_candidates_kernel(uint64_t seed, unsigned long long first, unsigned long long count,
                                        int nbits, int s_io, uint32_t* __restrict__ out) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const unsigned long long idx = first + i;
    uint32_t* o = out + i * (unsigned long long)s_io;
    for (int j = 0; 2 * j < s_io; j++) {
        const uint64_t z = splitmix_mix(seed + ((idx << 16) + (uint64_t)j + 1ull) * 0x9E3779B97F4A7C15ull);
        for (int h = 0; h < 2 && 2 * j + h < s_io; h++) {
            const int k = 2 * j + h;
            uint32_t v = (uint32_t)(z >> (32 * h));
            const int lo = 32 * k;
            if (lo >= nbits) v = 0;
            else if (nbits - lo < 32) v &= (1u << (nbits - lo)) - 1u;
            if (k == (nbits - 1) / 32) v |= 1u << ((nbits - 1) % 32);
            if (k == (nbits - 2) / 32) v |= 1u << ((nbits - 2) % 32);
            if (k == 0) v |= 1u;
            o[k] = v;
        }
    }
}

// verdict[i] = 0 if candidate i has a prime factor < 2^12 (and is not that
// prime), else 1.  Horner with 64-bit remainders.
struct SmallPrimes {
    int count;
    uint16_t p[564];
};
// the odd primes < 2^12, computed once on the host (a kernel parameter: no
// per-device __constant__ upload to keep in sync)
static const SmallPrimes& small_primes() {
    static const SmallPrimes sp = [] {
        SmallPrimes s{};
        for (uint32_t x = 3; x < 4096 && s.count < 564; x += 2) {
            bool is = true;
            for (uint32_t f = 3; f * f <= x; f += 2)
                if (x % f == 0) { is = false; break; }
            if (is) s.p[s.count++] = (uint16_t)x;
        }
        return s;
    }();
    return sp;
}
__global__ void sieve_kernel(const uint32_t* __restrict__ cand, unsigned long long count, int s_io,
                             const __grid_constant__ SmallPrimes sp, uint32_t* __restrict__ verdict) {
    const int nprimes = sp.count;
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t* c = cand + i * (unsigned long long)s_io;
    bool one_limb = true;
    for (int k = 1; k < s_io; k++) one_limb = one_limb && c[k] == 0;
    uint32_t ok = 1;
    for (int t = 0; t < nprimes && ok; t++) {
        const uint32_t pr = sp.p[t];
        uint64_t r = 0;
        for (int k = s_io - 1; k >= 0; k--) r = ((r << 32) | c[k]) % pr;
        if (r == 0 && !(one_limb && c[0] == pr)) ok = 0;
    }
    verdict[i] = ok;
}

// stable compaction helper: out_index[i] = running count of flags (exclusive
// scan done on the host for the small survivor sets of a search)

template <int S>
static cudaError_t launch_multi(const MultiParams& prm, int sms, cudaStream_t stream, size_t* slots_out,
                                bool query_only) {
    const int block = MCfg<S>::BLOCK;
    const size_t smem = sizeof(uint4) * (S / 2) * block;
    static OccCache cache;
    int occ = 0;
    cudaError_t ce = cached_occupancy(
        cache, [&](int* o) { return occupancy_with_smem(modexp_multi_kernel<S>, block, smem, o); }, &occ);
    if (ce != cudaSuccess) return ce;
    const int grid = sms * occ;
    if (slots_out) *slots_out = (size_t)grid * block;
    if (query_only) return cudaSuccess;
    modexp_multi_kernel<S><<<grid, block, smem, stream>>>(prm);
    return cudaGetLastError();
}

}  // namespace rsa_b200

// Host entry (C++ linkage) used by rsa_abi.cpp.  S in {8, 16, 32, 64}.
cudaError_t rsa_b200_multi(int S, const uint32_t* base, const uint32_t* exps, const uint32_t* mods, uint32_t* out,
                           int32_t* status, void* table, unsigned long long count, int s_io, int exp_bits,
                           int window, int mode, uint32_t mr_base, int sms, cudaStream_t stream, size_t* slots,
                           bool query_only) {
    using namespace rsa_b200;
    MultiParams p;
    p.base = base;
    p.exps = exps;
    p.mods = mods;
    p.out = out;
    p.status = status;
    p.table = reinterpret_cast<uint4*>(table);
    p.count = count;
    p.s_io = s_io;
    p.exp_bits = exp_bits;
    p.window = window;
    p.mode = mode;
    p.mr_base = mr_base;
    switch (S) {
    case 8: return launch_multi<8>(p, sms, stream, slots, query_only);
    case 16: return launch_multi<16>(p, sms, stream, slots, query_only);
    case 32: return launch_multi<32>(p, sms, stream, slots, query_only);
    case 64: return launch_multi<64>(p, sms, stream, slots, query_only);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t rsa_b200_prime_candidates(uint64_t seed, unsigned long long first, unsigned long long count, int nbits,
                                      int s_io, uint32_t* out, cudaStream_t stream) {
    if (!count) return cudaSuccess;
    const unsigned blocks = (unsigned)((count + 255) / 256);
    rsa_b200::prime_candidates_kernel<<<blocks, 256, 0, stream>>>(seed, first, count, nbits, s_io, out);
    return cudaGetLastError();
}

cudaError_t rsa_b200_sieve(const uint32_t* cand, unsigned long long count, int s_io, uint32_t* verdict,
                           cudaStream_t stream) {
    if (!count) return cudaSuccess;
    const unsigned blocks = (unsigned)((count + 127) / 128);
    rsa_b200::sieve_kernel<<<blocks, 128, 0, stream>>>(cand, count, s_io, rsa_b200::small_primes(), verdict);
    return cudaGetLastError();
}
