/*
 * rsa_b200.h -- C-ABI of the B200-native batched RSA library (librsa_b200.so).
 *
 * Method: arXiv 1407.1465, "Analysis of RSA Algorithm using GPU Programming"
 * (PAPER.md = the paper's text).  The library implements the paper's
 * data-parallel hot path -- C = M^e mod n for encryption and M = C^d mod n
 * for decryption, applied independently to every packet (sec. 2;
 * PAPER.md:65, sec. 3.3; sec. 11) -- for moduli from the
 * paper's toy key (n = 17947) to 4096-bit keys, plus the key-generation check
 * of Fig 1 and the packetisation of sec. 2.
 *
 * Conventions for every call:
 *   - big integers are little-endian arrays of uint32_t limbs (limb 0 least
 *     significant); a packet of an nbits-bit modulus has s = ceil(nbits/32)
 *     limbs; a batch is packet-major: packet i occupies limbs [i*s, (i+1)*s);
 *   - return value: RSA_OK (0) or a negative RSA_E* status; no call aborts,
 *     prints or throws; rsa_strerror() names a status;
 *   - no call keeps a pointer past its return except the asynchronous device
 *     work of rsa_modexp_batch, which reads `base` and writes `out` in stream
 *     order on `stream`.
 */
#ifndef RSA_B200_H
#define RSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define RSA_OK            0
#define RSA_EINVAL       -1   /* null pointer, bad size/length argument, partial overlap */
#define RSA_ERANGE       -2   /* nbits out of [2, 4096], n >= 2^nbits, or e not in (1, phi) */
#define RSA_EEVEN        -3   /* modulus even or < 3 (Montgomery needs gcd(n, 2) = 1) */
#define RSA_ENOTPRIME    -4   /* p or q not prime (Fig 1: "random prime numbers") */
#define RSA_EEQUAL       -5   /* p == q (Fig 1: "two different ... prime numbers") */
#define RSA_ENOTCOPRIME  -6   /* gcd(e, phi) != 1 (Fig 1) */
#define RSA_ECHAR        -7   /* encode: character outside a..z (after stripping spaces) */
#define RSA_EODD         -8   /* encode: odd number of letters */
#define RSA_ENOSPC       -9   /* output capacity too small */
#define RSA_EPACKET     -10   /* decode: a digit pair > 25 */
#define RSA_EBADKEY     -11   /* validate: d*e != 1 (mod phi) */
#define RSA_ECUDA       -12   /* CUDA launch / allocation / copy failure */

/* Largest modulus the GPU path accepts in this build (bits). */
#define RSA_MAX_NBITS 4096

const char* rsa_strerror(int status);

/* ---- key generation check: Fig 1, PAPER.md:48-55 ---------------------
 * Given p, q (pq_limbs limbs each, pq_limbs in [1, 64]) and e (e_limbs limbs,
 * e_limbs in [1, 128]):  checks p and q prime (Miller-Rabin, deterministic
 * below 2^64) and p != q; computes n = p*q and phi = (p-1)(q-1)
 * (PAPER.md:53); checks 1 < e < phi and gcd(e, phi) = 1; computes
 * d = e^-1 mod phi with 0 < d < phi ("d . e = 1 (mod phi(n))").
 * Outputs are host buffers of 2*pq_limbs limbs each, caller-allocated.
 * n_out and phi_out are written before the e checks (so ERANGE/ENOTCOPRIME
 * still report them); d_out only on RSA_OK.  Synchronous, host only.
 * Errors: RSA_EINVAL, RSA_ENOTPRIME, RSA_EEQUAL, RSA_ERANGE, RSA_ENOTCOPRIME. */
int rsa_keygen_check(const uint32_t* p, const uint32_t* q, int pq_limbs,
                     const uint32_t* e, int e_limbs,
                     uint32_t* n_out, uint32_t* phi_out, uint32_t* d_out);

/* ---- key validity: PAPER.md:33 ---------------------------------------
 * residue_out (2*limbs limbs) = (d*e) mod phi, phi = (p-1)(q-1).  Returns
 * RSA_OK when the residue is 1, RSA_EBADKEY otherwise (the paper's own sec. 2
 * pair e=131, d=137, n=17947 gives residue 267).  All inputs
 * have `limbs` limbs, limbs in [1, 64].  Synchronous, host only. */
int rsa_validate_key(const uint32_t* e, const uint32_t* d, const uint32_t* p,
                     const uint32_t* q, int limbs, uint32_t* residue_out);

/* ---- batched modular exponentiation: the hot path ---------------------
 * out[i] = base[i]^exp mod n for i < count  (C = M^e mod n, M = C^d mod n,
 * PAPER.md:35; the same call serves encryption and decryption).
 *   base, out : DEVICE pointers, [count][s] packet-major uint32 limbs,
 *               s = ceil(nbits/32); caller-owned; out == base (exact
 *               in-place) is allowed, any other overlap is RSA_EINVAL.
 *               Any base[i] < 2^(32 s) is accepted (it is reduced mod n);
 *               outputs are canonical, in [0, n).
 *   exp, n    : HOST pointers of s limbs each; read before the call returns
 *               (the caller may free them immediately).  exp = 0 gives 1.
 *   nbits     : modulus width in bits, 2 <= nbits <= RSA_MAX_NBITS, and
 *               n < 2^nbits; n must be odd and >= 3.
 *   stream    : a cudaStream_t (NULL = legacy default stream).  The call is
 *               asynchronous: it enqueues the kernel (and a stream-ordered
 *               workspace allocation) and returns; completion is observed
 *               through the stream.  count == 0 is a no-op returning RSA_OK.
 * Kernels (results identical; chosen by measurement): moduli of
 * 513..4096 bits run the tensor-core path (the product A B on the FP64 pipe,
 * 52-bit digits with exact DFMA.RZ products; the Montgomery reduction by the
 * batch's modulus as u8 tcgen05 matrix products), narrower ones the integer
 * (IMAD) pipe; rsa_set_kernel_path (below) selects the alternates per width
 * class for A/B measurement.  The tensor-core kernels hold all 512 TMEM
 * columns of their SM while resident.
 * Errors: RSA_EINVAL, RSA_ERANGE, RSA_EEVEN, RSA_ECUDA. */
int rsa_modexp_batch(const uint32_t* base, const uint32_t* exp, const uint32_t* n,
                     int nbits, size_t count, uint32_t* out, void* stream);

/* Same operation end to end from HOST memory: copies base_host to the device,
 * exponentiates, and copies the result back to out_host, pipelining chunks
 * so copies overlap compute (two streams, created once per calling host
 * thread and device and reused; one stream for a single-chunk call).
 * base_host/out_host may be pageable or pinned (pinned is faster).
 * Synchronous: returns when out_host is written.  Errors: as rsa_modexp_batch. */
int rsa_modexp_batch_host(const uint32_t* base_host, const uint32_t* exp, const uint32_t* n,
                          int nbits, size_t count, uint32_t* out_host);

/* CRT decryption (beyond the paper): the same
 * M = C^d mod n as rsa_modexp_batch with exp = d, computed from
 * the primes: m1 = C^(d mod p-1) mod p, m2 = C^(d mod q-1) mod q, M = m2 + q *
 * (q^-1 (m1 - m2) mod p).  ~4x fewer limb products than the full-width path.
 *   c, out : DEVICE, [count][s], s = ceil(nbits/32), 8 <= nbits <= 4096; each
 *            c[i] < n = p q (as for decryption); out != c unless equal.
 *   p, q   : HOST, pq_limbs limbs each (1..64), odd, distinct, p q < 2^nbits;
 *   d      : HOST, s limbs.  Asynchronous on `stream` (4 launches).
 * Errors: RSA_EINVAL, RSA_ERANGE, RSA_EEVEN, RSA_EEQUAL, RSA_ENOTCOPRIME,
 * RSA_ECUDA. */
int rsa_decrypt_crt_batch(const uint32_t* c, const uint32_t* p, const uint32_t* q, int pq_limbs, const uint32_t* d,
                          int nbits, size_t count, uint32_t* out, void* stream);

/* The paper's own GPU kernel, for comparison:
 * Alg 1 / Fig 11 + Alg 2 / Fig 12, one thread
 * per packet, 64 threads per block, O(key) loop: result[i] = num[i]^key mod
 * den computed as floor(key/2) multiplications by (num mod den)^2 and one by
 * (num mod den) if key is odd.  Exact integers (see modexp.cu).
 *   num, result : DEVICE pointers, `count` uint32 values each.
 *   key < 2^32, 1 <= den < 2^31 (the kernel's single-word envelope);
 *   faithful != 0 keeps the paper's key == 0 -> num mod den,
 *   faithful == 0 returns 1 mod den.  Asynchronous on `stream`.
 * Errors: RSA_ERANGE (den or key out of range), RSA_EINVAL, RSA_ECUDA. */
int rsa_modexp_batch_paper(const uint32_t* num, uint64_t key, uint32_t den, size_t count,
                           uint32_t* result, int faithful, void* stream);

/* The paper's exponentiation schedules as selectable single-word GPU kernels
 * (SURVEY.md sec. 8(f) row f2), one thread per packet, 64-bit exact products
 * (den < 2^32), for replaying the paper's toy keys on B200 beside the
 * Montgomery path:
 *   RSA_SCHED_NAIVE            Fig 4: c = g mod m, then
 *                              exp - 1 times c = c g mod m (O(exp));
 *   RSA_SCHED_R2L              Fig 5a: right-to-left binary;
 *   RSA_SCHED_L2R              Fig 5b: left-to-right binary;
 *   RSA_SCHED_HALVING          Fig 12, exact, exp = 0 -> 1;
 *   RSA_SCHED_HALVING_FAITHFUL Fig 12 with its exp = 0 -> g mod m (reading Z5).
 *   num, out : DEVICE pointers, `count` uint32 values each (out may be num);
 *   1 <= den < 2^32 (Fig 12: < 2^31); exp < 2^32 for NAIVE and the Fig 12
 *   schedules (their loops are O(exp)), any 64-bit exp for R2L / L2R.
 * Every schedule returns num^exp mod den (0^0 = 1 mod den), except the
 * faithful Fig 12 at exp = 0.  Asynchronous on `stream`.
 * Errors: RSA_ERANGE (den or exp out of range), RSA_EINVAL (null pointer,
 * unknown schedule), RSA_ECUDA. */
#define RSA_SCHED_NAIVE             1
#define RSA_SCHED_R2L               2
#define RSA_SCHED_L2R               3
#define RSA_SCHED_HALVING           4
#define RSA_SCHED_HALVING_FAITHFUL  5
int rsa_modexp_batch_schedule(const uint32_t* num, uint64_t exp, uint32_t den, size_t count, uint32_t* out,
                              int schedule, void* stream);

/* ---- multi-key batches and GPU prime search ----
 * rsa_modexp_batch_multi: out[i] = base[i]^exps[i] mod mods[i], every packet
 * with its own exponent and modulus (e.g. encrypting to many recipients).
 *   base, exps, mods, out: DEVICE, [count][s] limbs, s = ceil(nbits/32),
 *   2 <= nbits <= 2048; exps are scanned over their low exp_bits bits
 *   (1 <= exp_bits <= 32 s) with a fixed window; every mods[i] must be odd and
 *   >= 3 -- packets whose modulus is not get out = 0 and, if `status` (DEVICE,
 *   count int32, may be NULL) is given, status[i] = RSA_EEVEN (else 0).
 *   n', R mod n and R^2 mod n are derived per packet on the device.
 *   Asynchronous on `stream`.  Errors: RSA_ERANGE, RSA_EINVAL, RSA_ECUDA. */
int rsa_modexp_batch_multi(const uint32_t* base, const uint32_t* exps, const uint32_t* mods, int nbits,
                           int exp_bits, size_t count, uint32_t* out, int32_t* status, void* stream);

/* One Miller-Rabin round to base `base` (>= 2) on every candidate (DEVICE,
 * [count][s], odd, > base): verdict[i] (DEVICE, uint32) = 1 if cand[i] is a
 * strong probable prime to that base, else 0.  4 <= nbits <= 2048.  Async. */
int rsa_miller_rabin_batch(const uint32_t* cand, int nbits, size_t count, uint32_t base, uint32_t* verdict,
                           void* stream);

/* The prime search's candidate generator (counter based, reproducible):
 * candidate `first + i` -> out[i] (DEVICE, [count][s]); exactly nbits bits
 * with the top two bits and bit 0 set.  Async. */
int rsa_prime_candidates(int nbits, uint64_t seed, unsigned long long first, size_t count, uint32_t* out,
                         void* stream);

/* Small-prime sieve: verdict[i] = 0 if cand[i] has a prime factor < 4096
 * other than itself, else 1 (DEVICE arrays).  Async. */
int rsa_prime_sieve(const uint32_t* cand, int nbits, size_t count, uint32_t* verdict, void* stream);

/* Find `want` primes of nbits bits (16 <= nbits <= 2048): generator + sieve +
 * `rounds` (1..16) Miller-Rabin rounds, bases 2, 3, 5, ..., all on the GPU.
 * primes_out: HOST, want * s limbs, in candidate order; *tried_out (may be
 * NULL) = candidates examined.  Synchronous.  Errors: RSA_ERANGE, RSA_EINVAL,
 * RSA_ECUDA. */
int rsa_prime_search(int nbits, uint64_t seed, int want, int rounds, uint32_t* primes_out,
                     unsigned long long* tried_out);

/* Key generation, Fig 1: p, q from rsa_prime_search (seeded),
 * then rsa_keygen_check (host Miller-Rabin re-test, gcd(e, phi) = 1, d).
 * 32 <= nbits <= 4096; p has nbits/2 bits, q nbits - nbits/2 bits, so n has
 * exactly nbits bits.  HOST outputs: p_out, q_out with h = ceil((nbits -
 * nbits/2)/32) limbs; n_out, phi_out, d_out with 2h limbs.  Synchronous. */
int rsa_keygen(int nbits, const uint32_t* e, int e_limbs, uint64_t seed, uint32_t* p_out, uint32_t* q_out,
               uint32_t* n_out, uint32_t* phi_out, uint32_t* d_out);

/* Plan summary for (exp, n, nbits): the width class, window and the number
 * of Montgomery multiplications each packet costs (for the roofline). */
typedef struct {
    int width_class;      /* S: limbs of the kernel's Montgomery arithmetic */
    int s_io;             /* ceil(nbits/32): limbs per packet at this ABI */
    int window;           /* sliding-window width (1 = binary, Fig 5) */
    int table_entries;    /* per-packet window table entries */
    int nops;             /* operations in the kernel's op list */
    long long montmuls;   /* Montgomery multiplications per packet */
    long long squarings;  /* of which squarings */
    int exp_bits;         /* bit length of exp */
    int grid;             /* persistent grid (CTAs) */
    int block;            /* threads per CTA */
    int sqr_kernel;       /* 1 if squarings use the dedicated squaring (1.5S^2+1.5S products) */
    long long products;   /* algorithmic 32x32->64 limb products per packet: squarings x
                             (1.5S^2+1.5S or 2S^2+S) + other montmuls x (2S^2+S) */
    int fp64_digits;      /* 0: the class runs on the integer (IMAD) pipe; else ND, the
                             number of 52-bit digits of the FP64-pipe arithmetic (mont_f64.cuh;
                             also the product half of the tensor-core path) */
    long long digit_products; /* 52x52-bit digit products per packet on the FP64 pipe, each
                             2 DFMA + 1 DADD.  FP64 kernel: squarings x (ND(ND+1)/2 + ND^2) +
                             other montmuls x 2 ND^2.  Tensor-core path (RSA_PATH_TC): the
                             product T = A B only, squarings x ND(ND+1)/2 (x ND^2 at S = 128,
                             sqr_kernel 0) + other montmuls x ND^2 (the reduction runs on the
                             tensor core).  0 for
                             integer-pipe classes */
} rsa_plan_info_t;

int rsa_plan_info(const uint32_t* exp, const uint32_t* n, int nbits, rsa_plan_info_t* info);

/* Work summary of rsa_modexp_batch_multi (mr = 0) / rsa_miller_rabin_batch
 * (mr = 1) per packet: window, Montgomery multiplications, products. */
int rsa_multi_plan_info(int nbits, int exp_bits, int mr, rsa_plan_info_t* info);

/* Force a sliding-window width for subsequent calls on this thread
 * (0 = automatic, the default; 1..7 = fixed).  For tests and benchmarks. */
int rsa_set_window(int w);

/* ---- kernel path per width class (measurement and A/B only) -----------
 * A batch of an nbits-bit modulus runs in width class S = the smallest of
 * 2, 4, 8, 16, 32, 64, 128 limbs >= ceil(nbits/32).  Each class runs, by
 * default, the kernel measured fastest on B200 (DESIGN.md "Shapes chosen by
 * measurement"); every path computes the same, bit-exact result (the Montgomery
 * multiply of Fig 3), only the number representation and the
 * thread shape differ.  Paths:
 *   RSA_PATH_DEFAULT    the measured default of the class (see below)
 *   RSA_PATH_FP64       S = 32, 64, 128: 52-bit digits on the FP64 pipe
 *   RSA_PATH_INT        32-bit limbs, IMAD carry chains, one thread per packet
 *                       (default for S = 8, 16; for S = 128 it means the
 *                       2-lane pair kernel)
 *   RSA_PATH_INT_GROUP  S = 64: 2 lanes per packet; S = 128: 4 lanes
 *   RSA_PATH_INT_PAIR   S = 128: 2 lanes per packet
 *   RSA_PATH_INT_MULTI  S = 2, 4: several packets per thread (default there)
 *   RSA_PATH_TC         S = 32, 64, 128: the product A B on the FP64 pipe,
 *                       the Montgomery reduction (m = T n' mod R, T + m n) as
 *                       u8 matrix products on the tensor core (tcgen05, TMEM),
 *                       R = 2^(32 S); 128-packet tiles, one CTA per SM
 *                       (default for S = 32, 64, 128)
 * rsa_set_kernel_path sets the path of class `width_class` for subsequent
 * calls of every thread (process-wide, thread-safe; a call in flight keeps the
 * path it started with).  RSA_PATH_DEFAULT restores the default, under which
 * the RSA_B200_F64 / _F64_4096 / _TC / _SHAPE64 / _TPI128 / _SMALL environment
 * switches of the A/B tools are honoured (read per call).
 * Errors: RSA_EINVAL (no such class, or the class has no such kernel).
 * rsa_get_kernel_path returns the path the class resolves to now (never
 * RSA_PATH_DEFAULT), or RSA_EINVAL for an unknown class. */
#define RSA_PATH_DEFAULT    0
#define RSA_PATH_FP64       1
#define RSA_PATH_INT        2
#define RSA_PATH_INT_GROUP  3
#define RSA_PATH_INT_PAIR   4
#define RSA_PATH_INT_MULTI  5
#define RSA_PATH_TC         6
int rsa_set_kernel_path(int width_class, int path);
int rsa_get_kernel_path(int width_class);

/* ---- packet codec: sec. 2, PAPER.md:39-40 -----------------------------
 * rsa_encode: strips ASCII spaces, maps a=00 .. z=25 and packs consecutive
 * letter pairs as hi*100 + lo ("parallel encryption" ->
 * 1500 1700 1111 0411 0413 0217 2415 1908 1413).  `packets` holds `cap`
 * values; *count_out receives the packet count (or, on RSA_ECHAR, the index
 * of the offending character in `text`; on RSA_ENOSPC, the count needed).
 * rsa_decode: inverse (spaces are not recovered); `text` has `cap` bytes
 * including the terminating NUL (needs 2*count + 1).
 * Errors: RSA_EINVAL, RSA_ECHAR, RSA_EODD, RSA_ENOSPC, RSA_EPACKET. */
int rsa_encode(const char* text, uint32_t* packets, size_t cap, size_t* count_out);
int rsa_decode(const uint32_t* packets, size_t count, char* text, size_t cap);

/* ---- codec fused with the exponentiation ----
 * rsa_encrypt_text: DEVICE `text` of nletters lowercase letters a..z (spaces
 * already stripped, nletters even) -> cipher[i] = packet_i^e mod n, packet_i =
 * hi*100 + lo of letters 2i, 2i+1, in one kernel.  cipher:
 * DEVICE [nletters/2][s] limbs, s = ceil(nbits/32).  Single-word keys only:
 * 2 <= nbits <= 64 and n > 2525 (every packet must be < n).
 * rsa_decrypt_text: DEVICE cipher [count][s] -> packet = c^d mod n -> two
 * letters per packet into DEVICE `text` (2*count bytes, no terminator).
 * status (DEVICE int32 per packet, may be NULL): 0, RSA_ECHAR (a letter
 * outside a..z; that packet encrypts 0) or RSA_EPACKET (a result that is not a
 * packet; its letters are "??").  Asynchronous.  Errors: RSA_EINVAL,
 * RSA_ERANGE, RSA_EEVEN, RSA_EODD, RSA_ECUDA. */
int rsa_encrypt_text(const char* text, size_t nletters, const uint32_t* e, const uint32_t* n, int nbits,
                     uint32_t* cipher, int* status, void* stream);
int rsa_decrypt_text(const uint32_t* cipher, size_t count, const uint32_t* d, const uint32_t* n, int nbits,
                     char* text, int* status, void* stream);

/* Number of kernels this library has launched since load (for the bench's
 * gpu_launches accounting). */
unsigned long long rsa_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* RSA_B200_H */
