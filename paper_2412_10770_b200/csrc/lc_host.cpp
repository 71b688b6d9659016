// lc_host.cpp -- host side of the C ABI (include/lc.h): encoder, validator, view setup.
//
// The encoder is the greedy anchored integer cone of FORMAT F4-F6 (the eps-PLA of Def. 2,
// PAPER.md:171-181, fitted greedily per the north star instead of O'Rourke's optimal fit,
// PAPER.md:188), with residual packing per PAPER.md:184-186.  It is written independently of
// oracle/ (which tests compare byte for byte) and optimised for throughput: the
// cone is tested with 64x64->128 multiplications and divides only when a bound tightens.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lc.h"
#include "lc_internal.h"

namespace {

using u128 = unsigned __int128;
constexpr uint64_t kSlopeMax = 0x7fffffffffffffffULL;  // guard G = 2^63 - 1 (FORMAT F2)

// floor(x / d) for a quotient known to be < 2^64
inline uint64_t div_q64(u128 x, uint64_t d) {
#if defined(__x86_64__)
    uint64_t q, r;
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    __asm__("divq %4" : "=a"(q), "=d"(r) : "a"(lo), "d"(hi), "rm"(d));
    return q;
#else
    return (uint64_t)(x / d);
#endif
}

inline uint64_t rup(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Layout {
    uint64_t H, n_hint, W, o_starts, o_params, o_hint, o_words, total;
};

Layout layout_of(uint64_t n, uint64_t L, uint32_t b) {
    Layout y;
    y.H = (n + 1023) >> 10;
    y.n_hint = y.H + 1;
    y.W = rup((n * b + 31) / 32 + 1, 4);
    y.o_starts = 256;
    y.o_params = rup(y.o_starts + 4 * (L + 1), 256);
    y.o_hint = rup(y.o_params + 16 * L, 256);
    y.o_words = rup(y.o_hint + 4 * y.n_hint, 256);
    y.total = y.o_words + 4 * y.W;
    return y;
}

template <typename K>
int32_t check_sorted(const K* k, uint64_t n) {
    for (uint64_t i = 1; i < n; ++i)
        if (k[i] <= k[i - 1]) return LC_ERR_UNSORTED;
    return LC_OK;
}

// One greedy segment anchored at s (FORMAT F4): returns its end e and slope (F5).
template <typename K>
inline uint64_t fit_segment(const K* k, uint64_t n, uint64_t s, uint64_t eps, uint64_t* slope) {
    const uint64_t base = k[s];
    uint64_t lo = 0, hi = kSlopeMax;  // current cone [lo, hi] of slope * 2^32
    uint64_t e = s + 1;
    for (; e < n; ++e) {
        const uint64_t d = e - s;
        const uint64_t D = (uint64_t)k[e] - base;
        const u128 lod = (u128)lo * d, hid = (u128)hi * d;
        const u128 X = ((((u128)D + eps + 1) << 32) - 1);  // slope <= floor(X / d)
        if (lod > X || lod > (u128)kSlopeMax) break;       // lo above the upper bound or guard
        uint64_t nlo = lo, nhi = hi;
        if (D > eps) {
            const u128 Y = (u128)(D - eps) << 32;          // slope >= ceil(Y / d)
            if (Y > hid) break;                            // lower bound above hi
            if (Y > lod) nlo = div_q64(Y + d - 1, d);
        }
        if (X < hid) nhi = div_q64(X, d);
        if ((u128)kSlopeMax < hid) {
            const uint64_t g = kSlopeMax / d;
            if (g < nhi) nhi = g;
        }
        if (nlo > nhi) break;  // F6
        lo = nlo;
        hi = nhi;
    }
    *slope = (e - s == 1) ? 0 : lo + (hi - lo) / 2;
    return e;
}

template <typename K>
int32_t encode_t(const K* keys, uint64_t n, uint32_t key_bits, uint32_t eps, void** out_blob,
                 uint64_t* out_bytes) {
    int32_t st = check_sorted(keys, n);
    if (st) return st;
    if (key_bits == 32 && (uint64_t)keys[n - 1] > 0xffffffffULL) return LC_ERR_TOO_LARGE;
    std::vector<uint32_t> starts;
    std::vector<uint64_t> params;  // interleaved base, slope
    starts.reserve(n / 8 + 16);
    params.reserve(n / 4 + 32);
    for (uint64_t s = 0; s < n;) {
        uint64_t slope;
        uint64_t e = fit_segment(keys, n, s, eps, &slope);
        starts.push_back((uint32_t)s);
        params.push_back((uint64_t)keys[s]);
        params.push_back(slope);
        s = e;
    }
    const uint64_t L = starts.size();
    const uint32_t b = lc_detail::res_bits(eps);
    const Layout y = layout_of(n, L, b);
    uint8_t* blob = (uint8_t*)std::calloc(1, y.total);
    if (!blob) return LC_ERR_ALLOC;

    lc_header h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "LCG1", 4);
    h.version = 1;
    h.key_bits = (uint8_t)key_bits;
    h.res_bits = (uint8_t)b;
    h.eps = eps;
    h.hint_log2 = 10;
    h.n = n;
    h.n_seg = L;
    h.n_hint = y.n_hint;
    h.n_words = y.W;
    h.off_starts = y.o_starts;
    h.off_params = y.o_params;
    h.off_hint = y.o_hint;
    h.off_words = y.o_words;
    h.total_bytes = y.total;
    std::memcpy(blob, &h, sizeof h);

    uint32_t* S = (uint32_t*)(blob + y.o_starts);
    std::memcpy(S, starts.data(), 4 * L);
    S[L] = (uint32_t)n;
    std::memcpy(blob + y.o_params, params.data(), 16 * L);

    // hint[q] = segment holding key 1024 q; hint[H] = L - 1
    uint32_t* Hn = (uint32_t*)(blob + y.o_hint);
    for (uint64_t q = 0, j = 0; q < y.H; ++q) {
        const uint64_t key = q << 10;
        while (j + 1 < L && S[j + 1] <= key) ++j;
        Hn[q] = (uint32_t)j;
    }
    Hn[y.H] = (uint32_t)(L - 1);

    // residual fields u = K[i] - floor(f(i)) + eps, LSB-first into 32-bit words
    if (b) {
        uint32_t* Wd = (uint32_t*)(blob + y.o_words);
        uint64_t acc = 0;
        uint32_t nbits = 0;
        uint64_t w = 0;
        for (uint64_t j = 0; j < L; ++j) {
            const uint64_t s = S[j], e = S[j + 1];
            const uint64_t base = params[2 * j], slope = params[2 * j + 1];
            uint64_t run = 0;  // slope * d, < 2^63 by the guard
            for (uint64_t i = s; i < e; ++i, run += slope) {
                const uint64_t u = (uint64_t)keys[i] - base - (run >> 32) + eps;
                acc |= u << nbits;
                nbits += b;
                if (nbits >= 32) {
                    Wd[w++] = (uint32_t)acc;
                    acc >>= 32;
                    nbits -= 32;
                }
            }
        }
        if (nbits) Wd[w++] = (uint32_t)acc;
    }
    *out_blob = blob;
    *out_bytes = y.total;
    return LC_OK;
}

std::atomic<uint64_t> g_launches{0};

}  // namespace

namespace lc_detail {

uint32_t res_bits(uint64_t eps) {
    uint32_t b = 0;
    while ((1ULL << b) < 2 * eps + 1) ++b;  // eps <= 2^31 - 1 so 2 eps + 1 < 2^32
    return b;
}

int32_t check_header(const lc_header* h, uint64_t blob_bytes) {
    if (std::memcmp(h->magic, "LCG1", 4) != 0 || h->version != 1) return LC_ERR_FORMAT;
    if (h->key_bits != 32 && h->key_bits != 64) return LC_ERR_FORMAT;
    if (h->eps > 0x7fffffffu || h->res_bits != res_bits(h->eps)) return LC_ERR_FORMAT;
    if (h->hint_log2 != 10) return LC_ERR_FORMAT;
    if (h->n == 0 || h->n >= (1ULL << 32) || h->n_seg == 0 || h->n_seg > h->n)
        return LC_ERR_FORMAT;
    for (int i = 0; i < 40; ++i)
        if (h->reserved[i]) return LC_ERR_FORMAT;
    const Layout y = layout_of(h->n, h->n_seg, h->res_bits);
    if (h->n_hint != y.n_hint || h->n_words != y.W || h->off_starts != y.o_starts ||
        h->off_params != y.o_params || h->off_hint != y.o_hint || h->off_words != y.o_words ||
        h->total_bytes != y.total)
        return LC_ERR_FORMAT;
    if (blob_bytes < y.total) return LC_ERR_FORMAT;
    return LC_OK;
}

void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace lc_detail

extern "C" {

int32_t lc_encode(const void* keys, uint64_t n, uint32_t key_bits, uint32_t eps, void** blob,
                  uint64_t* blob_bytes) {
    if (!blob || !blob_bytes) return LC_ERR_ARG;
    if (key_bits != 32 && key_bits != 64) return LC_ERR_ARG;
    if (eps > 0x7fffffffu) return LC_ERR_ARG;
    if (n == 0) return LC_ERR_EMPTY;
    if (!keys) return LC_ERR_ARG;
    if (n >= (1ULL << 32)) return LC_ERR_TOO_LARGE;
    if (key_bits == 32)
        return encode_t((const uint32_t*)keys, n, key_bits, eps, blob, blob_bytes);
    return encode_t((const uint64_t*)keys, n, key_bits, eps, blob, blob_bytes);
}

void lc_free(void* blob) { std::free(blob); }

int32_t lc_validate(const void* blob, uint64_t blob_bytes) {
    if (!blob || blob_bytes < sizeof(lc_header)) return blob ? LC_ERR_FORMAT : LC_ERR_ARG;
    lc_header h;
    std::memcpy(&h, blob, sizeof h);
    int32_t st = lc_detail::check_header(&h, blob_bytes);
    if (st) return st;
    const uint8_t* B = (const uint8_t*)blob;
    const uint64_t n = h.n, L = h.n_seg, b = h.res_bits, eps = h.eps;
    // zero filler between header/sections
    const uint64_t sec_beg[4] = {h.off_starts, h.off_params, h.off_hint, h.off_words};
    const uint64_t sec_end[4] = {h.off_starts + 4 * (L + 1), h.off_params + 16 * L,
                                 h.off_hint + 4 * h.n_hint, h.total_bytes};
    for (uint64_t p = sizeof(lc_header); p < sec_beg[0]; ++p)
        if (B[p]) return LC_ERR_FORMAT;
    for (int s = 0; s < 3; ++s)
        for (uint64_t p = sec_end[s]; p < sec_beg[s + 1]; ++p)
            if (B[p]) return LC_ERR_FORMAT;
    const uint32_t* S = (const uint32_t*)(B + h.off_starts);
    const uint64_t* P = (const uint64_t*)(B + h.off_params);
    const uint32_t* Hn = (const uint32_t*)(B + h.off_hint);
    const uint32_t* Wd = (const uint32_t*)(B + h.off_words);
    if (S[0] != 0 || S[L] != n) return LC_ERR_FORMAT;
    for (uint64_t j = 0; j < L; ++j) {
        if (S[j + 1] <= S[j]) return LC_ERR_FORMAT;
        const uint64_t slope = P[2 * j + 1];
        if (slope > kSlopeMax) return LC_ERR_FORMAT;
        if ((u128)slope * (S[j + 1] - 1 - S[j]) > (u128)kSlopeMax) return LC_ERR_FORMAT;
    }
    for (uint64_t q = 0, j = 0; q < h.n_hint - 1; ++q) {
        while (j + 1 < L && S[j + 1] <= (q << 10)) ++j;
        if (Hn[q] != j) return LC_ERR_FORMAT;
    }
    if (Hn[h.n_hint - 1] != L - 1) return LC_ERR_FORMAT;
    // residual fields <= 2 eps, decoded keys strictly increasing and within key_bits,
    // stream bits past n*b zero
    const uint64_t kmax = h.key_bits == 32 ? 0xffffffffULL : ~0ULL;
    uint64_t prev = 0;
    for (uint64_t j = 0; j < L; ++j) {
        const uint64_t base = P[2 * j], slope = P[2 * j + 1];
        uint64_t run = 0;
        for (uint64_t i = S[j]; i < S[j + 1]; ++i, run += slope) {
            uint64_t u = 0;
            if (b) {
                const uint64_t p = i * b;
                const uint64_t two = (uint64_t)Wd[p >> 5] | ((uint64_t)Wd[(p >> 5) + 1] << 32);
                u = (two >> (p & 31)) & ((1ULL << b) - 1);
            }
            if (u > 2 * eps) return LC_ERR_FORMAT;
            if (i == S[j] && u != eps) return LC_ERR_FORMAT;  // anchor: base_j = K[s_j]
            const u128 full = (u128)base + (run >> 32) + u;
            if (full < eps || full - eps > kmax) return LC_ERR_FORMAT;
            const uint64_t key = (uint64_t)(full - eps);
            if (i > 0 && key <= prev) return LC_ERR_FORMAT;
            prev = key;
        }
    }
    const uint64_t used = n * b;
    for (uint64_t w = used >> 5; w < h.n_words; ++w) {
        uint32_t v = Wd[w];
        if (w == (used >> 5)) v &= (used & 31) ? ~((1u << (used & 31)) - 1) : ~0u;
        if (v) return LC_ERR_FORMAT;
    }
    return LC_OK;
}

int32_t lc_view_init(lc_view* v, const void* host_header128, const void* d_blob,
                     uint64_t blob_bytes) {
    if (!v || !host_header128 || !d_blob) return LC_ERR_ARG;
    if ((uintptr_t)d_blob % 256) return LC_ERR_ARG;
    lc_header h;
    std::memcpy(&h, host_header128, sizeof h);
    int32_t st = lc_detail::check_header(&h, blob_bytes);
    if (st) return st;
    v->h = h;
    v->d_blob = d_blob;
    return LC_OK;
}

const char* lc_status_str(int32_t s) {
    switch (s) {
        case LC_OK: return "LC_OK";
        case LC_ERR_ARG: return "LC_ERR_ARG";
        case LC_ERR_EMPTY: return "LC_ERR_EMPTY";
        case LC_ERR_UNSORTED: return "LC_ERR_UNSORTED";
        case LC_ERR_TOO_LARGE: return "LC_ERR_TOO_LARGE";
        case LC_ERR_FORMAT: return "LC_ERR_FORMAT";
        case LC_ERR_ALLOC: return "LC_ERR_ALLOC";
        case LC_ERR_CUDA: return "LC_ERR_CUDA";
        default: return "LC_ERR_UNKNOWN";
    }
}

uint64_t lc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
