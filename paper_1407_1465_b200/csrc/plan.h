// plan.h -- the launch plan shared by the host C-ABI (rsa_abi.cpp) and the
// sm_100a kernels (modexp.cu).  Product code only; the oracle never sees it.
//
// A plan is the host-side key precompute of SURVEY.md sec. 8(a) step a1:
//   n' = -n^-1 mod 2^32, R^2 mod n (R = 2^(32*S)), and the exponent recoded
//   into a flat list of Montgomery-multiply operations (to-Montgomery, window
//   table precompute, the left-to-right window scan, from-Montgomery).
// The scan follows Fig 7 (sliding window) with reading Z6
// (longest window ending in a 1-bit; A starts at the top window's entry);
// w = 1 is exactly Fig 5 left-to-right binary.
#pragma once
#include <stdint.h>

#define RSA_MAX_OPS 2048          // ops per plan (8 B each, kernel params)

// Op capacity of class S.  A 32S-bit exponent needs at most 2 ops per bit at
// w = 1 (a squaring run + a multiply), plus the table precompute (<= 65) and
// the conversions, so small classes carry a small op array: the parameter
// block (copied into every launch) shrinks from 16 KB to 1.2 KB at S = 2.
// Plans that do not fit a window's op list skip that window (build_ops).
constexpr int rsa_ops_cap(int S) { return (64 * S + 160 < RSA_MAX_OPS) ? 64 * S + 160 : RSA_MAX_OPS; }

enum RsaOpKind : uint8_t {
    RSA_OP_SQR = 0,    // A <- A * A * R^-1
    RSA_OP_MUL = 1,    // A <- A * T[bidx] * R^-1   (T = per-thread window table)
    RSA_OP_R2 = 2,     // A <- A * (R^2 mod n) * R^-1   (to Montgomery form)
    RSA_OP_ONE = 3,    // A <- A * 1 * R^-1              (from Montgomery form)
    RSA_OP_MULX = 4,   // A <- A * x * R^-1, x = the packet's input as given (not in
                       // Montgomery form): the last multiply by g and the conversion
                       // from Montgomery form in one.  A < n and x < R keep
                       // A x + m n < 2 n R, so one conditional subtraction suffices
                       // for any input x (also x >= n).
};

enum RsaOpFlags : uint8_t {
    RSA_F_LOADA = 1,   // before the op: A <- T[lidx]
    RSA_F_STORE = 2,   // after the op:  T[sidx] <- A
};

struct __align__(8) RsaOp {
    uint16_t rep;      // number of times the montmul is applied (>= 1)
    uint8_t kind;      // RsaOpKind
    uint8_t flags;     // RsaOpFlags
    uint8_t bidx;      // table entry used as the b operand of RSA_OP_MUL
    uint8_t lidx;      // table entry loaded into A (RSA_F_LOADA)
    uint8_t sidx;      // table entry written from A (RSA_F_STORE)
    uint8_t pad;
};

// Kernel parameters for width class S (32-bit limbs).  Passed by value as a
// __grid_constant__ so n[] and r2[] are constant-bank operands of the IMADs.
template <int S>
struct ModexpParams {
    const uint32_t* base;         // device, [count][s_io] LE limbs (or text bytes, codec mode)
    uint32_t* out;                // device, [count][s_io] (or text bytes, codec mode)
    int* status;                  // device, [count] per-packet codec status, or null
    void* table;                  // device workspace: ntab entries x S limbs x nthreads
    unsigned long long count;
    int s_io;                     // limbs per packet at the boundary (ceil(nbits/32))
    int nops;
    int ntab;                     // table entries (odd powers + g^2)
    uint32_t n0inv;               // -n^-1 mod 2^32
    uint32_t n[S];                // modulus, zero padded to S limbs
    uint32_t r2[S];               // R^2 mod n, R = 2^(32 S)
    RsaOp ops[rsa_ops_cap(S)];
};

// FP64-pipe kernel (mont_f64.cuh) for class S: digits of 52 bits, R = 2^(52 ND)
// with 4n < R.  The integer params come first, so the blob also serves the
// IMAD kernel of the same class (patch_params casts it to ModexpParams<S>).
// (rounded up to an even count: table entries move as digit pairs)
constexpr int rsa_f64_digits(int S) { return ((32 * S + 2 + 51) / 52 + 1) / 2 * 2; }

template <int S>
struct ModexpF64Params {
    ModexpParams<S> ip;
    unsigned long long np52;                 // -n^-1 mod 2^52
    double c104;                             // 2^104 (a runtime value: see mont_f64.cuh montmul)
    double nd[rsa_f64_digits(S)];            // n, digits as doubles (DFMA constant-bank operands)
    double r2d[rsa_f64_digits(S)];           // R^2 mod n, R = 2^(52 ND), digits as doubles
    unsigned long long nu[rsa_f64_digits(S)];  // n, digits as integers (final subtraction)
};

// Tensor-core reduction kernel (modexp_tc.cu, class S = 64): R = 2^(32 S)
// (ip.r2 is R^2 mod n for that R), the full-width quotient multiplier
// n' = -n^-1 mod R as bytes for the tensor-core Toeplitz operand.  The FP64
// params come first (same op list, same table entry format: digits as doubles).
template <int S>
struct ModexpTcParams {
    ModexpF64Params<S> f;
    uint8_t npb[4 * S];                      // -n^-1 mod 2^(32 S), little-endian bytes
};

// Multi-key kernel (modexp_multi.cu) per-key R^2 mod n: Mont(2^KD) = 2^KD R mod
// n by modular doublings of R mod n, then RSA_MULTI_R2SQ Montgomery squarings
// ((2^KD R)^(2^J) R^-(2^J - 1) = 2^(KD 2^J) R = R^2 with KD 2^J = 32 S).  A
// doubling is ~1/36 of a 2048-bit squaring, so J = 4 (KD = 128 at S = 64)
// instead of J = log2(32 S) = 11 (KD = 1).
#ifndef RSA_MULTI_R2SQ
#define RSA_MULTI_R2SQ 4    // A/B multi-key RSA-2048 encrypt: J = 11 / 6 / 5 / 4 -> 23.2M / 26.1M / 26.6M / 26.8M
#endif
constexpr int rsa_log2_bits(int S) { return S <= 1 ? 5 : 1 + rsa_log2_bits(S / 2); }   // log2(32 S)
constexpr int rsa_multi_r2_squarings(int S) {
    return rsa_log2_bits(S) < RSA_MULTI_R2SQ ? rsa_log2_bits(S) : RSA_MULTI_R2SQ;
}
constexpr int rsa_multi_r2_doublings(int S) { return 1 << (rsa_log2_bits(S) - rsa_multi_r2_squarings(S)); }
static_assert(rsa_log2_bits(64) == 11 && rsa_multi_r2_doublings(64) << rsa_multi_r2_squarings(64) == 2048, "R^2 schedule");
template <int S>
struct MultiR2 {   // the same, as compile-time constants usable in device code
    static constexpr int SQ = rsa_multi_r2_squarings(S), KD = rsa_multi_r2_doublings(S);
};

// host-visible summary of a plan (also exported through the C-ABI)
struct RsaPlanInfo {
    int width_class;              // S
    int s_io;
    int window;                   // sliding-window width w (1 = binary)
    int table_entries;            // 2^(w-1) odd powers (+1 for g^2 when w > 1)
    int nops;
    long long montmuls;           // Montgomery multiplications per packet
    long long squarings;          // of which squarings
    int exp_bits;
};
