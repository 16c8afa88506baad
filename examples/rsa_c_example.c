/* rsa_c_example.c -- the C-ABI used from plain C (no Python, no torch):
 * the paper's sec. 2 example end to end.  Build (see tests/test_gpu_c_abi.py):
 *   gcc -I include examples/rsa_c_example.c -L paper_1407_1465_b200 -lrsa_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o rsa_c_example
 * Prints the ciphertexts and the decoded text; exits non-zero on any error. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <cuda_runtime.h>

#include "rsa_b200.h"

#define CHECK(x) do { int rc_ = (x); if (rc_ != RSA_OK) { \
    fprintf(stderr, "%s: %s\n", #x, rsa_strerror(rc_)); return 1; } } while (0)

int main(void) {
    /* Fig 1 on the sec. 2 primes: p = 131, q = 137, e = 131 */
    uint32_t p = 131, q = 137, e = 131, n[2], phi[2], d[2], residue[2];
    CHECK(rsa_keygen_check(&p, &q, 1, &e, 1, n, phi, d));
    uint32_t paper_d = 137;
    int v = rsa_validate_key(&e, &paper_d, &p, &q, 1, residue);
    printf("paper's d=137: %s (d*e mod phi = %u)\n", v == RSA_OK ? "valid" : "INVALID", residue[0]);
    printf("n=%u phi=%u d=%u\n", n[0], phi[0], d[0]);

    /* sec. 2 packetisation */
    uint32_t packets[16];
    size_t count = 0;
    CHECK(rsa_encode("parallel encryption", packets, 16, &count));

    /* C = M^e mod n, M = C^d mod n on the GPU (device buffers, default stream) */
    uint32_t *dm = NULL, *dc = NULL;
    if (cudaMalloc((void**)&dm, count * 4) != cudaSuccess || cudaMalloc((void**)&dc, count * 4) != cudaSuccess) return 2;
    cudaMemcpy(dm, packets, count * 4, cudaMemcpyHostToDevice);
    CHECK(rsa_modexp_batch(dm, &e, n, 15, count, dc, NULL));
    uint32_t cipher[16], back[16];
    cudaMemcpy(cipher, dc, count * 4, cudaMemcpyDeviceToHost);
    CHECK(rsa_modexp_batch(dc, d, n, 15, count, dm, NULL));
    cudaMemcpy(back, dm, count * 4, cudaMemcpyDeviceToHost);
    printf("cipher:");
    for (size_t i = 0; i < count; i++) printf(" %u", cipher[i]);
    printf("\n");
    char text[64];
    CHECK(rsa_decode(back, count, text, sizeof text));
    printf("decoded: %s\n", text);

    /* the same through the host-buffer entry */
    uint32_t cipher2[16];
    CHECK(rsa_modexp_batch_host(packets, &e, n, 15, count, cipher2));
    if (memcmp(cipher, cipher2, count * 4) != 0) { fprintf(stderr, "host path differs\n"); return 3; }
    cudaFree(dm);
    cudaFree(dc);
    return strcmp(text, "parallelencryption") == 0 ? 0 : 4;
}
