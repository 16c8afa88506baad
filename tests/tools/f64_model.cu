// f64_model.cu -- host build of paper_1407_1465_b200/csrc/mont_f64.cuh for the
// CPU design check tests/test_f64_model.py (the same template code the kernel
// runs, executed on the CPU with the FP rounding mode set toward zero, which
// is what the device's __fma_rz does).  Not product code.
//
// stdin lines:  "M <S> <n> <a> <b>"  -> montmul(a, b) digits, printed as hex
//               "S <S> <n> <a> <a>"  -> montsqr(a) (the second a is ignored)
//               "Q <S> <n> <a> <a>"  -> montsqr_slot(a): A in a strided slot
//               "C <S> <n> <r>"      -> canonicalise(r)
//               "L <S> <x>"          -> limbs -> digits -> limbs round trip
// numbers in hex; n' and the digit split are computed here.
#include <cfenv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_1407_1465_b200/csrc/mont_f64.cuh"

using namespace rsa_b200::f64;

static std::vector<uint32_t> parse_hex(const char* s, int S) {
    std::vector<uint32_t> x(S, 0);
    int len = (int)strlen(s);
    for (int i = 0; i < len; i++) {
        const char c = s[len - 1 - i];
        const int v = (c >= '0' && c <= '9') ? c - '0' : (c | 32) - 'a' + 10;
        if (i / 8 < S) x[i / 8] |= (uint32_t)v << (4 * (i % 8));
    }
    return x;
}

template <int S>
static void run(char op, char** tok) {
    constexpr int ND = Digits<S>::ND;
    uint32_t nl[S], al[S], bl[S];
    auto load = [&](uint32_t (&dst)[S], const char* s) {
        auto v = parse_hex(s, S);
        for (int k = 0; k < S; k++) dst[k] = v[k];
    };
    if (op == 'L') {
        load(al, tok[0]);
        double ad[ND];
        limbs_to_digits<S, ND>(al, ad);
        uint64_t di[ND];
        for (int k = 0; k < ND; k++) di[k] = (uint64_t)ad[k];
        uint32_t back[S];
        digits_to_limbs<S, ND>(di, back);
        for (int k = S - 1; k >= 0; k--) printf("%08x", back[k]);
        printf("\n");
        return;
    }
    load(nl, tok[0]);
    double nd[ND];
    limbs_to_digits<S, ND>(nl, nd);
    uint64_t nu[ND];
    for (int k = 0; k < ND; k++) nu[k] = (uint64_t)nd[k];
    // np = -n^-1 mod 2^52 (Newton on 64 bits)
    uint64_t inv = 1;
    for (int it = 0; it < 7; it++) inv *= 2 - nu[0] * inv;
    const uint64_t np = (0 - inv) & M52;
    uint64_t r[ND];
    if (op == 'M' || op == 'S' || op == 'Q' || op == 'A' || op == 'I' || op == 'F') {
        // a, b may be up to 2n: given as digits-of-hex over ND*52 bits
        constexpr int SW = (52 * ND + 31) / 32;
        auto av = parse_hex(tok[1], SW), bv = parse_hex(tok[2], SW);
        double ad[ND], bd[ND];
        auto split = [&](const std::vector<uint32_t>& v, double* d) {
            for (int k = 0; k < ND; k++) {
                uint64_t x = 0;
                for (int b = 0; b < 52; b++) {
                    const int o = 52 * k + b;
                    if (o / 32 < SW && ((v[o / 32] >> (o % 32)) & 1)) x |= 1ull << b;
                }
                d[k] = (double)x;
            }
        };
        split(av, ad);
        split(bv, bd);
        if (op == 'S') {
            uint64_t th[2 * ND];
            montsqr<ND>(ad, nd, np, C104, r, th, 1);
        } else if (op == 'Q') {           // squaring with A living in one strided slot (4096-bit kernel)
            double slot[3 * ND];
            for (int k = 0; k < ND; k++) slot[1 + 3 * k] = ad[k];
            montsqr_slot<ND>(nd, np, C104, r, slot + 1, 3);
            for (int k = 0; k < ND; k++) ad[k] = slot[1 + 3 * k];
        } else {
            if (op == 'A') {              // the ASMEM variant (A parked in a strided slot)
                double slot[3 * ND];
                montmul<ND, true>(ad, [&](int i) { return bd[i]; }, nd, np, C104, r, slot + 1, 3);
            } else if (op == 'I' || op == 'F') {   // A lives in the slot (the 4096-bit kernel)
                double slot[3 * ND], dummy[ND];
                for (int k = 0; k < ND; k++) { slot[1 + 3 * k] = ad[k]; dummy[k] = -1.0; }
                auto bf = [&](int i) { return bd[i]; };
                if (op == 'F') montmul<ND, true, decltype(bf), true, true>(dummy, bf, nd, np, C104, r, slot + 1, 3);
                else montmul<ND, true, decltype(bf), true>(dummy, bf, nd, np, C104, r, slot + 1, 3);
                for (int k = 0; k < ND; k++) ad[k] = slot[1 + 3 * k];
            } else {
                montmul<ND>(ad, [&](int i) { return bd[i]; }, nd, np, C104, r);
            }
        }
        for (int k = 0; k < ND; k++)
            if ((uint64_t)ad[k] != r[k]) { printf("MISMATCH\n"); return; }
    } else {
        constexpr int SW = (52 * ND + 31) / 32;
        auto rv = parse_hex(tok[1], SW);
        for (int k = 0; k < ND; k++) {
            uint64_t x = 0;
            for (int b = 0; b < 52; b++) {
                const int o = 52 * k + b;
                if (o / 32 < SW && ((rv[o / 32] >> (o % 32)) & 1)) x |= 1ull << b;
            }
            r[k] = x;
        }
        canonicalise<ND>(r, nu);
    }
    // print as one hex number, most significant digit first (13 hex chars per digit)
    for (int k = ND - 1; k >= 0; k--) printf("%013llx", (unsigned long long)r[k]);
    printf("\n");
}

// "Z <ND> v_0 ... v_{ND-1}" (hex columns < 2^62) -> normalize() digits (hex, top first)
template <int ND>
static void run_norm(char** tok) {
    uint64_t t[ND];
    for (int k = 0; k < ND; k++) t[k] = strtoull(tok[k], nullptr, 16);
    normalize<ND>(t);
    for (int k = ND - 1; k >= 0; k--) printf("%013llx", (unsigned long long)t[k]);
    printf("\n");
}

int main() {
    fesetround(FE_TOWARDZERO);
    char line[65536];
    while (fgets(line, sizeof line, stdin)) {
        char* tok[96];
        int nt = 0;
        for (char* p = strtok(line, " \n"); p && nt < 96; p = strtok(nullptr, " \n")) tok[nt++] = p;
        if (nt > 2 && tok[0][0] == 'Z') {
            const int nd = atoi(tok[1]);
            if (nd == 20) run_norm<20>(tok + 2);
            else if (nd == 40) run_norm<40>(tok + 2);
            else if (nd == 80) run_norm<80>(tok + 2);
            fflush(stdout);
            continue;
        }
        if (nt < 3) continue;
        const int S = atoi(tok[1]);
        switch (S) {
        case 8: run<8>(tok[0][0], tok + 2); break;
        case 16: run<16>(tok[0][0], tok + 2); break;
        case 32: run<32>(tok[0][0], tok + 2); break;
        case 64: run<64>(tok[0][0], tok + 2); break;
        case 128: run<128>(tok[0][0], tok + 2); break;
        default: printf("BAD\n");
        }
        fflush(stdout);
    }
    return 0;
}
