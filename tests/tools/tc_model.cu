// tc_model.cu -- host build of the CUDA-core half of the tensor-core
// Montgomery multiply (paper_1407_1465_b200/csrc/tc_digits.cuh, and
// f64::sqr_scan from mont_f64.cuh) for tests/test_tc_model.py.  Compiled with
// nvcc for the host; the rounding mode is set toward zero (the DFMA.RZ split).
// Protocol (one line per command, hex numbers, stdout one hex line):
//   M a b   T = A B through mul_rows + Packer (128 words)
//   Q a     T = A^2 through sqr_scan + Packer
//   R a     T = A^2 through sqr_col (compile-time-expanded scan, batch 2: the 2048-bit TC kernel)
//   H a     the 1024-bit class (ND = 20, a < 2^1024): T = A^2 through sqr_col (batch 4), 64 words
//   W x     x (64 words) -> 40 digits (words_to_digits) -> back to words (Packer)
//   E x     x (64 words) -> 40 digits -> words again through the run-time WordEmitter
//   P a b   A B as two row halves (mul_rows_f with NR = 20 on b_0..19 and b_20..39), summed
//   B a     T = A^2 through sqr_blocks (rolled block triangle), ND = 40, blocks of 10 / 8 (B / C)
//   N a b   T = A B through mul_blocks, ND = 40, blocks of 10
//   O a b   mul_blocks at ND = 80 (4096-bit operands, high digits over A's dead blocks)
//   G a     the 4096-bit class (ND = 80, a < 2^4096, 256 output words): sqr_blocks, blocks of 10
#include <cfenv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>

#include "../../paper_1407_1465_b200/csrc/tc_digits.cuh"

using namespace rsa_b200;
constexpr int ND = 40, NW = 64;

static void parse_words(const std::string& hex, uint32_t* w, int n) {
    for (int i = 0; i < n; i++) w[i] = 0;
    int bit = 0;
    for (int i = (int)hex.size() - 1; i >= 0 && bit < 32 * n; i--, bit += 4) {
        const char c = hex[i];
        const uint32_t v = (c >= '0' && c <= '9') ? c - '0' : (c >= 'a' && c <= 'f') ? c - 'a' + 10 : c - 'A' + 10;
        w[bit / 32] |= v << (bit % 32);
    }
}

static void print_words(const uint32_t* w, int n) {
    int top = n - 1;
    while (top > 0 && w[top] == 0) top--;
    printf("%x", w[top]);
    for (int i = top - 1; i >= 0; i--) printf("%08x", w[i]);
    printf("\n");
    fflush(stdout);
}

int main() {
    fesetround(FE_TOWARDZERO);
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream is(line);
        std::string op, x, y;
        is >> op >> x >> y;
        uint32_t aw[2 * NW], bw[2 * NW], out[4 * NW];
        const bool big = op == "G" || op == "O";
        parse_words(x, aw, big ? 2 * NW : NW);
        parse_words(y.empty() ? "0" : y, bw, big ? 2 * NW : NW);
        double a[ND], b[ND];
        tcd::words_to_digits<ND>([&](int w) -> uint32_t { return w < NW ? aw[w] : 0u; }, a);
        tcd::words_to_digits<ND>([&](int w) -> uint32_t { return w < NW ? bw[w] : 0u; }, b);
        memset(out, 0, sizeof(out));
        auto word = [&](int w, uint32_t v) { out[w] = v; };
        tcd::Packer<2 * NW, decltype(word)> pk{word, 0};
        auto put = [&](int k, uint64_t d) { pk.put(k, d); };
        if (op == "M") {
            uint64_t low[ND];
            double bs[ND];
            memcpy(bs, b, sizeof(b));
            tcd::mul_rows<ND>(
                a, [&](int j) { return bs[j]; },
                [&](int j, uint64_t d) { memcpy(&bs[j], &d, 8); low[j] = d; },   // overwrites b_j, like the kernel
                [&](int j) { return low[j]; }, put);
        } else if (op == "Q") {
            f64::sqr_scan<ND>(a, put);
        } else if (op == "R") {
            f64::sqr_col<ND, 0, 2, 0>(a, 0, 0, 0, put);
        } else if (op == "H") {
            double h[20];
            tcd::words_to_digits<20>([&](int w) -> uint32_t { return w < 32 ? aw[w] : 0u; }, h);
            f64::sqr_col<20, 0, 4, 0>(h, 0, 0, 0, put);
        } else if (op == "P") {
            // rows split in two: P0 = A (b_0..b_19), P1 = A (b_20..b_39); T = P0 + P1 2^(52 * 20)
            constexpr int NR = 20;
            uint64_t dig[2][ND + NR];
            for (int hf = 0; hf < 2; hf++) {
                auto ag = [&](int i) { return a[i]; };
                auto bg = [&](int j) { return b[hf * NR + j]; };
                auto lo = [&](int j, uint64_t d) { dig[hf][j] = d; };
                auto li = [&](int) -> uint64_t { return 0; };
                auto pt = [&](int k, uint64_t d) { dig[hf][k] = d; };
                tcd::mul_rows_f<ND, false, decltype(ag), decltype(bg), decltype(lo), decltype(li), decltype(pt), NR>(
                    ag, bg, lo, li, pt);
            }
            uint64_t sum[2 * ND + 1] = {0}, c = 0;
            for (int k = 0; k < 2 * ND; k++) {
                uint64_t v = c;
                if (k < ND + NR) v += dig[0][k];
                if (k >= NR && k - NR < ND + NR) v += dig[1][k - NR];
                sum[k] = v & f64::M52;
                c = v >> 52;
            }
            for (int k = 0; k < 2 * ND; k++) put(k, sum[k]);
        } else if (op == "E" || op == "F") {
            int ew = 0;
            auto emit = [&](uint32_t v) { if (ew < 2 * NW) out[ew] = v; ew++; };
            auto emit_sel = [&](uint32_t v, bool valid) { if (valid && ew < 2 * NW) out[ew] = v; ew += valid; };
            tcd::WordEmitter<decltype(emit)> we{emit, 0, 0};
            tcd::WordEmitter<decltype(emit_sel), true> wes{emit_sel, 0, 0};
            for (int k = 0; k < ND; k++) {
                if (op == "E") we.digit((uint64_t)a[k]);
                else wes.digit((uint64_t)a[k]);
            }
        } else if (op == "B" || op == "C") {
            uint64_t low[ND], high[ND];
            auto ag = [&](int i) { return a[i]; };
            auto lo = [&](int c, uint64_t d) { low[c] = d; };
            auto ho = [&](int k, uint64_t d) { high[k] = d; };
            auto hi = [&](int k) { return high[k]; };
            if (op == "B") tcd::sqr_blocks<ND, 10>(ag, lo, ho, hi, put);
            else tcd::sqr_blocks<ND, 8>(ag, lo, ho, hi, put);
            // put got columns ND.. only: the low columns through the packer first
            tcd::Packer<2 * NW, decltype(word)> pk2{word, 0};
            for (int k = 0; k < ND; k++) pk2.put(k, low[k]);
            for (int k = ND; k < 2 * ND; k++) pk2.put(k, high[k - ND]);
        } else if (op == "G") {
            constexpr int N4 = 80;
            double a4[N4];
            uint64_t low[N4], high[N4];
            tcd::words_to_digits<N4>([&](int w) -> uint32_t { return w < 2 * NW ? aw[w] : 0u; }, a4);
            auto word4 = [&](int w, uint32_t v) { out[w] = v; };
            tcd::Packer<4 * NW, decltype(word4)> pk4{word4, 0};
            auto put4 = [&](int, uint64_t) {};
            // high digit k overwrites A's digit k (block s - NB, dead), like the kernel's slot
            tcd::sqr_blocks<N4, 10>([&](int i) { return a4[i]; }, [&](int c, uint64_t d) { low[c] = d; },
                                    [&](int k, uint64_t d) { memcpy(&a4[k], &d, 8); },
                                    [&](int k) { uint64_t d; memcpy(&d, &a4[k], 8); high[k] = d; return d; }, put4);
            for (int k = 0; k < N4; k++) pk4.put(k, low[k]);
            for (int k = N4; k < 2 * N4; k++) pk4.put(k, high[k - N4]);
            print_words(out, 4 * NW);
            continue;
        } else if (op == "N") {
            uint64_t low[ND], high[ND];
            tcd::mul_blocks<ND, 10>([&](int i) { return a[i]; }, [&](int j) { return b[j]; },
                                    [&](int c, uint64_t d) { low[c] = d; }, [&](int k, uint64_t d) { high[k] = d; },
                                    [&](int k) { return high[k]; }, [](int, uint64_t) {});
            for (int k = 0; k < ND; k++) put(k, low[k]);
            for (int k = ND; k < 2 * ND; k++) put(k, high[k - ND]);
        } else if (op == "O") {
            constexpr int N4 = 80;
            double a4[N4], b4[N4];
            uint64_t low[N4], high[N4];
            tcd::words_to_digits<N4>([&](int w) -> uint32_t { return w < 2 * NW ? aw[w] : 0u; }, a4);
            tcd::words_to_digits<N4>([&](int w) -> uint32_t { return w < 2 * NW ? bw[w] : 0u; }, b4);
            auto word4 = [&](int w, uint32_t v) { out[w] = v; };
            tcd::Packer<4 * NW, decltype(word4)> pk4{word4, 0};
            tcd::mul_blocks<N4, 10>([&](int i) { return a4[i]; }, [&](int j) { return b4[j]; },
                                    [&](int c, uint64_t d) { low[c] = d; },
                                    [&](int k, uint64_t d) { memcpy(&a4[k], &d, 8); },
                                    [&](int k) { uint64_t d; memcpy(&d, &a4[k], 8); high[k] = d; return d; },
                                    [](int, uint64_t) {});
            for (int k = 0; k < N4; k++) pk4.put(k, low[k]);
            for (int k = N4; k < 2 * N4; k++) pk4.put(k, high[k - N4]);
            print_words(out, 4 * NW);
            continue;
        } else if (op == "W") {
            for (int k = 0; k < ND; k++) put(k, (uint64_t)a[k]);
            for (int k = ND; k < 2 * ND; k++) put(k, 0);
        } else {
            printf("?\n");
            fflush(stdout);
            continue;
        }
        print_words(out, 2 * NW);
    }
    return 0;
}
