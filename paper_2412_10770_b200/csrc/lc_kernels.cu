// lc_kernels.cu -- sm_100a kernels and launchers for lc_decode / lc_decode_span / lc_access /
// lc_range_decode / lc_decode_host (include/lc.h).
//
// What is computed (FORMAT F3; PAPER.md:105 K[i] = floor(f(i)) + Delta[i]; Eq. 1):
//     key_i = base_j + floor(slope_j * (i - s_j) / 2^32) + u_i - eps,  j = max{t : s_t <= i}.
//
// Design:
//  * Full decode: one WARP per 1024-key hint block ("chunk"), persistent over chunks.  The
//    hint array gives the chunk's segment range [hint[h], hint[h+1]] with no search
//    (PAPER.md:286's auxiliary localisation structure).  Lane 0 stages the chunk's starts,
//    params and residual words into the warp's shared-memory page with cp.async.bulk (TMA 1D)
//    on an mbarrier; dense chunks are paged.  The chunk is decoded as 32 windows of 32 keys,
//    lane = key: a warp OR-reduction (REDUX) of the next 32 segment starts gives a bitmask of
//    segment boundaries inside the window, so each lane gets its segment with POPC/CLZ —
//    branch-free, no per-key search and no serial walk ("reduce the data
//    dependencies ... to maximize parallelism").  The prediction is exact 32-bit integer
//    math: floor(slope*d/2^32) = umulhi(slope_lo, d) + slope_hi*d (it is < 2^31 by the
//    slope guard).  Residual fields are funnel-shifted out of the staged words.  Each warp
//    store writes 32 consecutive keys (coalesced, streaming hint).
//  * Random access: one thread per query (hint bracket + binary search over starts).
//  * Range decode: one warp per range; cooperative bracket search, then the same window
//    scheme reading through L1.
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <utility>

#include "lc.h"
#include "lc_internal.h"

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr uint32_t kSegCap = 128;  // segments per staged page (per warp)
constexpr uint32_t kFull = 0xffffffffu;

struct Sections {
    const uint32_t* starts;
    const ulonglong2* params;  // {base, slope_fx}
    const uint32_t* hint;
    const uint32_t* words;
};

Sections sections_of(const lc_view* v) {
    const uint8_t* B = (const uint8_t*)v->d_blob;
    Sections s;
    s.starts = (const uint32_t*)(B + v->h.off_starts);
    s.params = (const ulonglong2*)(B + v->h.off_params);
    s.hint = (const uint32_t*)(B + v->h.off_hint);
    s.words = (const uint32_t*)(B + v->h.off_words);
    return s;
}

// ------------------------------------------------------------------ PTX helpers (sm_90+/100a)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
// TMA 1D bulk copy global -> shared, completion counted on the mbarrier (16-B aligned, 16-B
// multiple; FORMAT F2 + the 1024-key chunking make every slice satisfy both)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// floor(slope * d / 2^32) for slope * d < 2^63 (FORMAT F2 guard): exact in 32 bits.
__device__ __forceinline__ uint32_t pred_delta(uint64_t slope, uint32_t d) {
    return __umulhi((uint32_t)slope, d) + (uint32_t)(slope >> 32) * d;
}
// t = floor(slope * d / 2^32) + v  (v = u - eps): mul.hi + mad.lo + add, kept as 3 ops
__device__ __forceinline__ uint32_t pred_plus(uint64_t slope, uint32_t d, uint32_t v) {
    uint32_t t;
    asm("{\n.reg .u32 h;\nmul.hi.u32 h, %1, %2;\nmad.lo.u32 h, %3, %2, h;\nadd.u32 %0, h, %4;\n}"
        : "=r"(t)
        : "r"((uint32_t)slope), "r"(d), "r"((uint32_t)(slope >> 32)), "r"(v));
    return t;
}

template <bool K64>
__device__ __forceinline__ void store_key(void* out, uint64_t pos, uint64_t base, uint32_t delta,
                                          uint32_t u, uint32_t eps) {
    if (K64) {
        __stcs((unsigned long long*)out + pos, (unsigned long long)(base + delta + u - eps));
    } else {
        __stcs((unsigned int*)out + pos, (unsigned int)((uint32_t)base + delta + u - eps));
    }
}

// --------------------------------------------------------------------------- full decode
struct DecodeArgs {
    Sections sec;
    void* out;         // receives keys [i0, i1)
    uint32_t i0, i1;   // i0 % 1024 == 0
    uint32_t chunk0;   // i0 / 1024
    uint32_t nchunks;  // ceil((i1 - i0) / 1024)
    uint32_t eps;
    uint32_t warp_bytes;  // shared memory per warp
};

// Per-warp shared-memory page: [mbarrier | starts (kSegCap+4) | params kSegCap | words]
__host__ __device__ constexpr uint32_t page_starts_off() { return 16; }
__host__ __device__ constexpr uint32_t page_params_off() { return 16 + 4 * (kSegCap + 4); }
__host__ __device__ constexpr uint32_t page_words_off() { return page_params_off() + 16 * kSegCap; }
__host__ __device__ constexpr uint32_t warp_bytes_for(uint32_t b) {
    return (page_words_off() + 4 * (b ? 32 * b + 4 : 0) + 127) & ~127u;
}

struct Page {
    uint64_t* bar;
    uint32_t* sS;         // starts[pj .. pj + cs)
    ulonglong2* sP;       // params[pj .. pj + cp)
    uint32_t* sW;         // the chunk's residual words
    uint32_t pj, cp;
    uint32_t phase;
};

// Stage starts[pj, pj + cs) and params[pj, pj + cp) (plus, when wbytes != 0, the chunk's words)
// with TMA bulk copies; cs covers one start past the params so every window candidate
// (clamped at jlast + 1) is a real start.  Lane 0 issues, the warp waits on the mbarrier.
__device__ __forceinline__ void stage(Page& pg, const Sections& sec, uint32_t from, uint32_t jlast,
                                      const uint32_t* wsrc, uint32_t wbytes, uint32_t lane) {
    __syncwarp();  // every lane is done reading the previous contents
    pg.pj = from & ~3u;
    pg.cp = min(kSegCap, jlast + 1 - pg.pj);
    if (lane == 0) {
        const uint32_t cs = min(kSegCap + 4, jlast + 2 - pg.pj);
        const uint32_t sbytes = ((cs + 3) & ~3u) * 4, pbytes = pg.cp * 16;
        mbar_expect_tx(pg.bar, sbytes + pbytes + wbytes);
        bulk_g2s(pg.sS, sec.starts + pg.pj, sbytes, pg.bar);
        bulk_g2s(pg.sP, sec.params + pg.pj, pbytes, pg.bar);
        if (wbytes) bulk_g2s(pg.sW, wsrc, wbytes, pg.bar);
    }
    mbar_wait(pg.bar, pg.phase);
    pg.phase ^= 1;
}

// Decode one 32-key window [wb, wb + 32) of a chunk, lane = key.  w is the window index in
// the chunk (selects the residual words).  Segment j of each lane: boundaries inside the
// window form a bitmask (REDUX.OR over the next 32 segment starts); popc/clz give the
// segment and the offset d = i - s_j with no search.  key = base + t with
// t = floor(slope d / 2^32) + u - eps = K[i] - K[s_j] in [0, 2^32) (FORMAT F2 anchor + guard).
template <uint32_t B>
__device__ __forceinline__ uint32_t field(const uint32_t* sW, uint32_t w, uint32_t lw, uint32_t ls) {
    if (!B) return 0;
    constexpr uint32_t mask = B >= 32 ? 0xffffffffu : ((1u << (B & 31)) - 1);
    const uint32_t* wp = sW + w * B + lw;
    return __funnelshift_r(wp[0], wp[1], ls) & mask;
}

template <bool K64>
__device__ __forceinline__ void put(void* outl, uint64_t base, uint32_t t) {  // outl: lane's slot
    if (K64) __stcs((unsigned long long*)outl, (unsigned long long)(base + t));
    else __stcs((unsigned int*)outl, (unsigned int)base + t);
}

__device__ __forceinline__ uint32_t bit_or_zero(uint32_t x) {  // 1 << x, 0 when x >= 32
    uint32_t r;
    asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(x));
    return r;
}

template <bool K64, uint32_t B, bool CHECK, bool FULL>
__device__ __forceinline__ void decode_window(Page& pg, const Sections& sec, uint32_t& jb,
                                              uint32_t& sb, uint32_t jlast, uint32_t wb,
                                              uint32_t w, uint32_t lane, uint32_t lmask,
                                              uint32_t lw, uint32_t ls, uint32_t eps,
                                              void* outw, uint32_t valid) {
    if (CHECK && min(jb + 31, jlast) >= pg.pj + pg.cp)  // warp-uniform: re-page a dense chunk
        stage(pg, sec, jb, jlast, nullptr, 0, lane);
    const uint32_t cand = min(jb + 1 + lane, jlast + 1);
    const uint32_t x = pg.sS[cand - pg.pj] - wb;  // > 0: position of the next start
    const uint32_t P = __reduce_or_sync(kFull, bit_or_zero(x));
    const uint32_t adv = __popc(__ballot_sync(kFull, x <= 32));
    const uint32_t m = P & lmask;  // boundaries at or before this lane's key
    const uint32_t seg = jb + __popc(m);
    const uint32_t d = m ? lane - (31 - __clz(m)) : (wb - sb) + lane;
    const ulonglong2 pr = pg.sP[seg - pg.pj];
    const uint32_t t = pred_plus(pr.y, d, field<B>(pg.sW, w, lw, ls) - eps);
    if (FULL || lane < valid) put<K64>(outw, pr.x, t);
    jb += adv;
    sb = pg.sS[jb - pg.pj];
}

// Two windows at once: keys [wb, wb + 64), lane handles wb + lane and wb + 32 + lane.  One
// candidate load / vote serves both halves when fewer than 32 segment starts fall inside;
// otherwise it falls back to two single windows.  w2 = pair index (windows 2 w2, 2 w2 + 1).
template <bool K64, uint32_t B, bool CHECK>
__device__ __forceinline__ void decode_pair(Page& pg, const Sections& sec, uint32_t& jb,
                                            uint32_t& sb, uint32_t jlast, uint32_t wb,
                                            uint32_t w2, uint32_t lane, uint32_t lmask,
                                            uint32_t lw, uint32_t ls, uint32_t eps, void* outw) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    if (CHECK && min(jb + 31, jlast) >= pg.pj + pg.cp)
        stage(pg, sec, jb, jlast, nullptr, 0, lane);
    const uint32_t cand = min(jb + 1 + lane, jlast + 1);
    const uint32_t x = pg.sS[cand - pg.pj] - wb;
    const uint32_t inside = __ballot_sync(kFull, x < 64);
    if (inside == kFull) {  // >= 32 boundaries in 64 keys: not enough candidates, go window-wise
        decode_window<K64, B, CHECK, true>(pg, sec, jb, sb, jlast, wb, 2 * w2, lane, lmask, lw,
                                           ls, eps, outw, 32);
        decode_window<K64, B, CHECK, true>(pg, sec, jb, sb, jlast, wb + 32, 2 * w2 + 1, lane,
                                           lmask, lw, ls, eps, (uint8_t*)outw + 32 * kw, 32);
        return;
    }
    const uint32_t PA = __reduce_or_sync(kFull, bit_or_zero(x));       // starts in (wb, wb+32)
    const uint32_t PB = __reduce_or_sync(kFull, bit_or_zero(x - 32));  // starts in [wb+32, wb+64)
    const uint32_t adv = __popc(__ballot_sync(kFull, x <= 64));
    const uint32_t off0 = wb - sb;                                      // uniform
    const uint32_t offB = PA ? __clz(PA) + 1 : off0 + 32;               // uniform
    const uint32_t jB = jb + __popc(PA);                                // uniform
    const uint32_t mA = PA & lmask;
    const uint32_t dA = mA ? lane - (31 - __clz(mA)) : off0 + lane;
    const ulonglong2 pA = pg.sP[jb + __popc(mA) - pg.pj];
    const uint32_t mB = PB & lmask;
    const uint32_t dB = mB ? lane - (31 - __clz(mB)) : offB + lane;
    const ulonglong2 pB = pg.sP[jB + __popc(mB) - pg.pj];
    const uint32_t tA = pred_plus(pA.y, dA, field<B>(pg.sW, 2 * w2, lw, ls) - eps);
    const uint32_t tB = pred_plus(pB.y, dB, field<B>(pg.sW, 2 * w2 + 1, lw, ls) - eps);
    put<K64>(outw, pA.x, tA);
    put<K64>((uint8_t*)outw + 32 * kw, pB.x, tB);
    jb += adv;
    sb = pg.sS[jb - pg.pj];
}

template <bool K64, uint32_t B>
__global__ void __launch_bounds__(kThreads) lc_decode_kernel(const DecodeArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = smem + warp * a.warp_bytes;
    Page pg;
    pg.bar = (uint64_t*)base;
    pg.sS = (uint32_t*)(base + page_starts_off());
    pg.sP = (ulonglong2*)(base + page_params_off());
    pg.sW = (uint32_t*)(base + page_words_off());
    pg.phase = 0;
    if (lane == 0) mbar_init(pg.bar);
    __syncwarp();

    constexpr uint32_t kw = K64 ? 8 : 4;
    const uint32_t lw = (lane * B) >> 5, ls = (lane * B) & 31;  // lane's field in a window
    const uint32_t lmask = lanemask_le();
    const uint32_t nwarps = gridDim.x * kWarpsPerCta;
    const Sections sec = a.sec;

    uint32_t c = blockIdx.x * kWarpsPerCta + warp;
    // hint pair of the warp's next chunk, loaded one chunk ahead (hides a DRAM round trip)
    uint32_t nj0 = 0, njl = 0;
    if (c < a.nchunks) {
        nj0 = __ldg(sec.hint + a.chunk0 + c);
        njl = __ldg(sec.hint + a.chunk0 + c + 1);
    }
    for (; c < a.nchunks; c += nwarps) {
        const uint32_t h = a.chunk0 + c;
        const uint32_t key0 = h << 10;
        const uint32_t nk = min(1024u, a.i1 - key0);
        const uint32_t j0 = nj0;
        const uint32_t jlast = njl;  // last segment the chunk can touch
        if (c + nwarps < a.nchunks) {
            nj0 = __ldg(sec.hint + h + nwarps);
            njl = __ldg(sec.hint + h + nwarps + 1);
        }
        const uint32_t wbytes = B ? ((((nk * B + 31) >> 5) + 1 + 3) & ~3u) * 4 : 0;
        stage(pg, sec, j0, jlast, sec.words + (size_t)h * 32 * B, wbytes, lane);
        uint32_t jb = j0;                // segment holding the window's first key
        uint32_t sb = pg.sS[j0 - pg.pj];  // its start
        uint8_t* outl = (uint8_t*)a.out + ((size_t)(key0 - a.i0) + lane) * kw;  // lane's slot
        if (nk == 1024 && jlast < pg.pj + pg.cp) {  // whole chunk staged: no re-page checks
#pragma unroll 1
            for (uint32_t g = 0; g < 16; g += 4, outl += 4 * 64 * kw) {
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k)
                    decode_pair<K64, B, false>(pg, sec, jb, sb, jlast, key0 + 64 * (g + k), g + k,
                                               lane, lmask, lw, ls, a.eps, outl + 64 * kw * k);
            }
        } else if (nk == 1024) {  // dense chunk: paged
#pragma unroll 1
            for (uint32_t g = 0; g < 16; g += 4, outl += 4 * 64 * kw) {
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k)
                    decode_pair<K64, B, true>(pg, sec, jb, sb, jlast, key0 + 64 * (g + k), g + k,
                                              lane, lmask, lw, ls, a.eps, outl + 64 * kw * k);
            }
        } else {  // ragged tail chunk
            for (uint32_t w = 0; 32 * w < nk; ++w)
                decode_window<K64, B, true, false>(pg, sec, jb, sb, jlast, key0 + 32 * w, w, lane,
                                                   lmask, lw, ls, a.eps, outl + 32 * kw * w,
                                                   nk - 32 * w);
        }
    }
}

// ------------------------------------------------------------------------- random access
struct AccessArgs {
    Sections sec;
    const uint64_t* idx;
    void* out;
    uint32_t* err;
    uint64_t q;
    uint32_t n, b, eps, mask;
};

template <bool K64>
__global__ void __launch_bounds__(256) lc_access_kernel(const AccessArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= a.q) return;
    const uint64_t i64 = __ldcs(a.idx + t);
    if (i64 >= a.n) {
        if (a.err) atomicOr(a.err, 1u);
        if (K64) __stcs((unsigned long long*)a.out + t, 0ull);
        else __stcs((unsigned int*)a.out + t, 0u);
        return;
    }
    const uint32_t i = (uint32_t)i64;
    uint32_t lo = __ldg(a.sec.hint + (i >> 10)), hi = __ldg(a.sec.hint + (i >> 10) + 1);
    while (lo < hi) {  // j = max{t in [lo, hi] : starts[t] <= i}
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(a.sec.starts + mid) <= i) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t s = __ldg(a.sec.starts + lo);
    const ulonglong2 pr = __ldg(a.sec.params + lo);
    uint32_t u = 0;
    if (a.b) {
        const uint64_t bit = (uint64_t)i * a.b;
        const uint32_t* wp = a.sec.words + (bit >> 5);
        u = __funnelshift_r(__ldg(wp), __ldg(wp + 1), (uint32_t)bit & 31) & a.mask;
    }
    store_key<K64>(a.out, t, pr.x, pred_delta(pr.y, i - s), u, a.eps);
}

// -------------------------------------------------------------------------- range decode
struct RangeArgs {
    Sections sec;
    const uint64_t* start;
    void* out;
    uint32_t* err;
    uint64_t q;
    uint32_t len, n, L, b, eps, mask;
};

template <bool K64>
__global__ void __launch_bounds__(256) lc_range_kernel(const RangeArgs a) {
    const uint64_t r = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (r >= a.q) return;  // warp-uniform
    const uint64_t rs64 = __ldg(a.start + r);
    const uint64_t obase = r * a.len;
    if (rs64 > a.n || a.len > a.n - rs64) {
        if (lane == 0 && a.err) atomicOr(a.err, 1u);
        for (uint32_t k = lane; k < a.len; k += 32) store_key<K64>(a.out, obase + k, 0, 0, 0, 0);
        return;
    }
    const uint32_t rs = (uint32_t)rs64;
    // warp-cooperative search for j = max{t : starts[t] <= rs} inside the hint bracket
    uint32_t lo = __ldg(a.sec.hint + (rs >> 10)), hi = __ldg(a.sec.hint + (rs >> 10) + 1);
    while (hi - lo + 1 > 32) {
        const uint32_t step = (hi - lo + 32) >> 5;  // ceil((hi - lo + 1) / 32)
        const uint32_t p = lo + lane * step;
        const bool ok = p <= hi && __ldg(a.sec.starts + p) <= rs;
        const uint32_t c = __popc(__ballot_sync(kFull, ok));  // >= 1: starts[lo] <= rs
        lo += (c - 1) * step;
        hi = min(hi, lo + step - 1);
    }
    {
        const uint32_t p = lo + lane;
        const bool ok = p <= hi && __ldg(a.sec.starts + p) <= rs;
        lo += __popc(__ballot_sync(kFull, ok)) - 1;
    }
    uint32_t jb = lo, sb = __ldg(a.sec.starts + lo);
    const uint32_t lmask = lanemask_le();
    const uint32_t jmax = a.L - 1;
    for (uint32_t w0 = 0; w0 < a.len; w0 += 32) {
        const uint32_t wb = rs + w0;
        const uint32_t cand = jb + 1 + lane;
        const uint32_t x = (cand <= jmax) ? __ldg(a.sec.starts + cand) - wb : kFull;
        const uint32_t P = __reduce_or_sync(kFull, x < 32 ? (1u << x) : 0u);
        const uint32_t adv = __popc(__ballot_sync(kFull, x <= 32));
        const uint32_t m = P & lmask;
        const uint32_t seg = jb + __popc(m);
        const uint32_t d = m ? lane - (31 - __clz(m)) : wb + lane - sb;
        const uint32_t k = w0 + lane;
        if (k < a.len) {
            const ulonglong2 pr = __ldg(a.sec.params + seg);
            uint32_t u = 0;
            if (a.b) {
                const uint64_t bit = (uint64_t)(wb + lane) * a.b;
                const uint32_t* wp = a.sec.words + (bit >> 5);
                u = __funnelshift_r(__ldg(wp), __ldg(wp + 1), (uint32_t)bit & 31) & a.mask;
            }
            store_key<K64>(a.out, obase + k, pr.x, pred_delta(pr.y, d), u, a.eps);
        }
        jb += adv;
        if (adv) sb = __ldg(a.sec.starts + jb);
    }
}

// ------------------------------------------------------------------------------ launchers
uint32_t mask_of(uint32_t b) { return b >= 32 ? 0xffffffffu : ((1u << b) - 1); }

int32_t cuda_status() { return cudaGetLastError() == cudaSuccess ? LC_OK : LC_ERR_CUDA; }

using DecodeFn = void (*)(DecodeArgs);

template <bool K64, uint32_t... Bs>
constexpr std::array<DecodeFn, sizeof...(Bs)> decode_table(std::integer_sequence<uint32_t, Bs...>) {
    return {{&lc_decode_kernel<K64, Bs>...}};
}
// one instantiation per residual width b = 0..32 (compile-time field offsets and masks)
const std::array<DecodeFn, 33> kDecode[2] = {
    decode_table<false>(std::make_integer_sequence<uint32_t, 33>{}),
    decode_table<true>(std::make_integer_sequence<uint32_t, 33>{})};

struct GridCache {
    std::mutex mu;
    int dev = -1;
    int sms = 0;
    int occ[2][33] = {};  // [K64][res_bits] -> resident CTAs per SM
};
GridCache g_grid;

// persistent grid size for the decode kernel: SMs x resident CTAs at this smem footprint
int persistent_grid(bool k64, uint32_t b) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_grid.mu);
    if (g_grid.dev != dev) {
        g_grid.dev = dev;
        cudaDeviceGetAttribute(&g_grid.sms, cudaDevAttrMultiProcessorCount, dev);
        std::memset(g_grid.occ, 0, sizeof g_grid.occ);
    }
    int& occ = g_grid.occ[k64][b];
    if (occ == 0) {
        const void* fn = (const void*)kDecode[k64][b];
        const int smem = (int)(warp_bytes_for(b) * kWarpsPerCta);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem);
        if (occ < 1) occ = 1;
    }
    return occ * g_grid.sms;
}

int32_t launch_decode(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out, cudaStream_t st) {
    DecodeArgs a;
    a.sec = sections_of(v);
    a.out = d_out;
    a.i0 = (uint32_t)i0;
    a.i1 = (uint32_t)i1;
    a.chunk0 = (uint32_t)(i0 >> 10);
    a.nchunks = (uint32_t)((i1 - i0 + 1023) >> 10);
    a.eps = v->h.eps;
    const uint32_t b = v->h.res_bits;
    a.warp_bytes = warp_bytes_for(b);
    const uint32_t smem = a.warp_bytes * kWarpsPerCta;
    const bool k64 = v->h.key_bits == 64;
    const int full = persistent_grid(k64, b);
    const uint32_t need = (a.nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
    const uint32_t grid = need < (uint32_t)full ? need : (uint32_t)full;
    kDecode[k64][b]<<<grid, kThreads, smem, st>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

struct HostPipe {
    std::mutex mu;
    int dev = -1;
    cudaStream_t copy = nullptr;
    cudaEvent_t ev[17] = {};
};
HostPipe g_pipe;

}  // namespace

extern "C" {

int32_t lc_decode_span(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (i0 > i1 || i1 > v->h.n || (i0 & 1023)) return LC_ERR_ARG;
    if (i0 == i1) return LC_OK;
    if (!d_out || ((uintptr_t)d_out & 15)) return LC_ERR_ARG;
    return launch_decode(v, i0, i1, d_out, (cudaStream_t)stream);
}

int32_t lc_decode(const lc_view* v, void* d_out, lc_stream stream) {
    if (!v) return LC_ERR_ARG;
    return lc_decode_span(v, 0, v->h.n, d_out, stream);
}

int32_t lc_access(const lc_view* v, const uint64_t* d_idx, uint64_t q, void* d_out,
                  uint32_t* d_err, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (q == 0) return LC_OK;
    if (!d_idx || !d_out) return LC_ERR_ARG;
    AccessArgs a;
    a.sec = sections_of(v);
    a.idx = d_idx;
    a.out = d_out;
    a.err = d_err;
    a.q = q;
    a.n = (uint32_t)v->h.n;
    a.b = v->h.res_bits;
    a.eps = v->h.eps;
    a.mask = mask_of(a.b);
    const uint64_t grid = (q + 255) / 256;
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    if (v->h.key_bits == 64)
        lc_access_kernel<true><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    else
        lc_access_kernel<false><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

int32_t lc_range_decode(const lc_view* v, const uint64_t* d_start, uint64_t q, uint32_t len,
                        void* d_out, uint32_t* d_err, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (len == 0 || len > (1u << 20)) return LC_ERR_ARG;
    if (q == 0) return LC_OK;
    if (!d_start || !d_out) return LC_ERR_ARG;
    RangeArgs a;
    a.sec = sections_of(v);
    a.start = d_start;
    a.out = d_out;
    a.err = d_err;
    a.q = q;
    a.len = len;
    a.n = (uint32_t)v->h.n;
    a.L = (uint32_t)v->h.n_seg;
    a.b = v->h.res_bits;
    a.eps = v->h.eps;
    a.mask = mask_of(a.b);
    const uint64_t grid = (q + 7) / 8;
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    if (v->h.key_bits == 64)
        lc_range_kernel<true><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    else
        lc_range_kernel<false><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

int32_t lc_decode_host(const void* h_blob, uint64_t blob_bytes, void* d_blob, void* d_out,
                       void* h_out, lc_stream stream) {
    if (!h_blob || !d_blob || !d_out || !h_out) return LC_ERR_ARG;
    if (blob_bytes < sizeof(lc_header)) return LC_ERR_FORMAT;
    lc_view v;
    int32_t st = lc_view_init(&v, h_blob, d_blob, blob_bytes);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(d_blob, h_blob, v.h.total_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return LC_ERR_CUDA;
    // decode in spans; each span's device->host copy runs on a side stream and overlaps the
    // next span's decode
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_pipe.mu);
    if (g_pipe.dev != dev) {
        if (cudaStreamCreateWithFlags(&g_pipe.copy, cudaStreamNonBlocking) != cudaSuccess)
            return LC_ERR_CUDA;
        for (auto& e : g_pipe.ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return LC_ERR_CUDA;
        g_pipe.dev = dev;
    }
    const uint64_t n = v.h.n, w = v.h.key_bits / 8;
    const uint64_t spans = 16;
    const uint64_t per = ((n + spans - 1) / spans + 1023) & ~1023ULL;
    uint32_t k = 0;
    for (uint64_t i0 = 0; i0 < n; i0 += per, ++k) {
        const uint64_t i1 = i0 + per < n ? i0 + per : n;
        st = launch_decode(&v, i0, i1, (uint8_t*)d_out + i0 * w, s);
        if (st) return st;
        cudaEventRecord(g_pipe.ev[k], s);
        cudaStreamWaitEvent(g_pipe.copy, g_pipe.ev[k], 0);
        if (cudaMemcpyAsync((uint8_t*)h_out + i0 * w, (uint8_t*)d_out + i0 * w, (i1 - i0) * w,
                            cudaMemcpyDeviceToHost, g_pipe.copy) != cudaSuccess)
            return LC_ERR_CUDA;
    }
    cudaEventRecord(g_pipe.ev[16], g_pipe.copy);
    cudaStreamWaitEvent(s, g_pipe.ev[16], 0);
    return cuda_status();
}

}  // extern "C"
