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
//    on an mbarrier (dense chunks are paged) and prefetches the next chunk into L2.  The chunk
//    is decoded as 16 pair-windows of 64 keys (2 keys per lane): warp OR-reductions (REDUX) of
//    the next 32 segment starts give the boundary bitmasks, so each key gets its segment and
//    offset with POPC/CLZ -- no per-key search and no serial walk ("reduce the
//    data dependencies ... to maximize parallelism").  The prediction is exact 32-bit integer
//    math (see pred_plus).  Each warp store writes 32 consecutive keys (coalesced, streaming).
//  * Random access / quantiles: hint bracket + binary search, two interleaved queries per
//    thread, L2 evict_last for the search structures and evict_first for the gathers.
//  * Range decode: one warp per 32 ranges (lane-parallel search); len == 64 gathers each
//    range's slices through a per-warp cp.async ring and decodes from shared memory.
//  * Successor search / intersection: binary search over the anchored segment bases
//    (segments as skip pointers), then inside one segment.
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <type_traits>
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
    uint32_t L, W;  // segments, residual words (bounds of params / words)
};

Sections sections_of(const lc_view* v) {
    const uint8_t* B = (const uint8_t*)v->d_blob;
    Sections s;
    s.starts = (const uint32_t*)(B + v->h.off_starts);
    s.params = (const ulonglong2*)(B + v->h.off_params);
    s.hint = (const uint32_t*)(B + v->h.off_hint);
    s.words = (const uint32_t*)(B + v->h.off_words);
    s.L = (uint32_t)v->h.n_seg;
    s.W = (uint32_t)v->h.n_words;
    return s;
}

// Bounds-checked build (-DLC_DEBUG_BOUNDS, tests/test_gpu_bounds.py): every shared-memory page
// / ring-slot index and every section index is checked; a violation is counted in
// g_lc_violations (read by lc_debug_violations) and the access is clamped instead of faulting.
#ifdef LC_DEBUG_BOUNDS
__device__ uint32_t g_lc_violations;
__device__ uint32_t g_lc_where[3];  // source line, index, limit of the last violation
__device__ __forceinline__ uint32_t lc_bound(bool live, uint32_t i, uint32_t n, uint32_t line) {
    if (live && i >= n) {
        atomicAdd(&g_lc_violations, 1u);
        g_lc_where[0] = line;
        g_lc_where[1] = i;
        g_lc_where[2] = n;
        return 0;
    }
    return i;
}
#define LC_BOUND(live, i, n) lc_bound((live), (i), (n), __LINE__)
#define LC_CHECK(live, i, n) ((void)lc_bound((live), (i), (n), __LINE__))
#else
#define LC_BOUND(live, i, n) (i)
#define LC_CHECK(live, i, n) ((void)0)
#endif

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
// L2 cache policies for the gather kernels: the search structures (hint, starts: 0.4 + 30 MB
// on config 5) stay resident (evict_last) while the one-touch params/words gathers are
// marked evict_first, so the binary-search probes keep hitting L2.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ldh(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ ulonglong2 ldh(const ulonglong2* p, uint64_t pol) {
    ulonglong2 v;
    asm("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// TMA bulk prefetch of [src, src + bytes) into L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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

// t = floor(slope * d / 2^32) + v  (v = u - eps), with floor(slope * d / 2^32) =
// umulhi(slope_lo, d) + slope_hi * d exact in 32 bits because slope * d < 2^63 (FORMAT F2
// guard): mul.hi + mad.lo + add, kept as 3 ops
__device__ __forceinline__ uint32_t pred_plus(uint64_t slope, uint32_t d, uint32_t v) {
    uint32_t t;
    asm("{\n.reg .u32 h;\nmul.hi.u32 h, %1, %2;\nmad.lo.u32 h, %3, %2, h;\nadd.u32 %0, h, %4;\n}"
        : "=r"(t)
        : "r"((uint32_t)slope), "r"(d), "r"((uint32_t)(slope >> 32)), "r"(v));
    return t;
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
    uint32_t nwords;      // W (words section length)
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
#ifdef LC_DEBUG_BOUNDS
    uint32_t cs, nw;  // staged starts / words entries
#endif
};

// Stage starts[pj, pj + cs) and params[pj, pj + cp) (plus, when wbytes != 0, the chunk's words)
// with TMA bulk copies; cs covers one start past the params so every window candidate
// (clamped at jlast + 1) is a real start.  Lane 0 issues, the warp waits on the mbarrier.
__device__ __forceinline__ void stage(Page& pg, const Sections& sec, uint32_t from, uint32_t jlast,
                                      const uint32_t* wsrc, uint32_t wbytes, uint32_t lane) {
    __syncwarp();  // every lane is done reading the previous contents
    pg.pj = from & ~3u;
    pg.cp = min(kSegCap, jlast + 1 - pg.pj);
#ifdef LC_DEBUG_BOUNDS
    pg.cs = (min(kSegCap + 4, jlast + 2 - pg.pj) + 3) & ~3u;
    if (wbytes) pg.nw = wbytes / 4;
#endif
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
    const uint32_t x = pg.sS[LC_BOUND(true, cand - pg.pj, pg.cs)] - wb;  // next start
    const uint32_t P = __reduce_or_sync(kFull, bit_or_zero(x));
    const uint32_t adv = __popc(__ballot_sync(kFull, x <= 32));
    const uint32_t m = P & lmask;  // boundaries at or before this lane's key
    const uint32_t seg = jb + __popc(m);
    const uint32_t d = m ? lane - (31 - __clz(m)) : (wb - sb) + lane;
    const ulonglong2 pr = pg.sP[LC_BOUND(FULL || lane < valid, seg - pg.pj, pg.cp)];
    LC_CHECK(B && (FULL || lane < valid), w * B + lw + 1, pg.nw);
    const uint32_t t = pred_plus(pr.y, d, field<B>(pg.sW, w, lw, ls) - eps);
    if (FULL || lane < valid) put<K64>(outw, pr.x, t);
    // candidates clamped at jlast + 1 repeat the list's final start N in the last chunk: cap
    // the advance there so jb stays a valid staged index
    jb = min(jb + adv, jlast + 1);
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
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
    const uint32_t x = pg.sS[LC_BOUND(true, cand - pg.pj, pg.cs)] - wb;
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
    const ulonglong2 pA = pg.sP[LC_BOUND(true, jb + __popc(mA) - pg.pj, pg.cp)];
    const uint32_t mB = PB & lmask;
    const uint32_t dB = mB ? lane - (31 - __clz(mB)) : offB + lane;
    const ulonglong2 pB = pg.sP[LC_BOUND(true, jB + __popc(mB) - pg.pj, pg.cp)];
    LC_CHECK(B, (2 * w2 + 1) * B + lw + 1, pg.nw);
    const uint32_t tA = pred_plus(pA.y, dA, field<B>(pg.sW, 2 * w2, lw, ls) - eps);
    const uint32_t tB = pred_plus(pB.y, dB, field<B>(pg.sW, 2 * w2 + 1, lw, ls) - eps);
    put<K64>(outw, pA.x, tA);
    put<K64>((uint8_t*)outw + 32 * kw, pB.x, tB);
    jb = min(jb + adv, jlast + 1);  // see decode_window
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
}

// Four windows at once: keys [wb, wb + 128), lane handles wb + 32 q + lane (q = 0..3).  One
// candidate load / advance vote serves four quarters when fewer than 32 segment starts fall
// inside; otherwise two pair steps.  w4 = quad index (windows 4 w4 .. 4 w4 + 3).
template <bool K64, uint32_t B, bool CHECK>
__device__ __forceinline__ void decode_quad(Page& pg, const Sections& sec, uint32_t& jb,
                                            uint32_t& sb, uint32_t jlast, uint32_t wb,
                                            uint32_t w4, uint32_t lane, uint32_t lmask,
                                            uint32_t lw, uint32_t ls, uint32_t eps, void* outw) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    if (CHECK && min(jb + 31, jlast) >= pg.pj + pg.cp)
        stage(pg, sec, jb, jlast, nullptr, 0, lane);
    const uint32_t cand = min(jb + 1 + lane, jlast + 1);
    const uint32_t x = pg.sS[LC_BOUND(true, cand - pg.pj, pg.cs)] - wb;
    if (__ballot_sync(kFull, x < 128) == kFull) {  // >= 32 boundaries in 128 keys
        decode_pair<K64, B, CHECK>(pg, sec, jb, sb, jlast, wb, 2 * w4, lane, lmask, lw, ls, eps,
                                   outw);
        decode_pair<K64, B, CHECK>(pg, sec, jb, sb, jlast, wb + 64, 2 * w4 + 1, lane, lmask, lw,
                                   ls, eps, (uint8_t*)outw + 64 * kw);
        return;
    }
    const uint32_t adv = __popc(__ballot_sync(kFull, x <= 128));
    uint32_t off = wb - sb, jq = jb;  // uniform: distance to the last start, segment base
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t P = __reduce_or_sync(kFull, bit_or_zero(x - 32 * q));  // starts in quarter q
        const uint32_t m = P & lmask;
        const uint32_t d = m ? lane - (31 - __clz(m)) : off + lane;
        const ulonglong2 pr = pg.sP[LC_BOUND(true, jq + __popc(m) - pg.pj, pg.cp)];
        LC_CHECK(B, (4 * w4 + q) * B + lw + 1, pg.nw);
        put<K64>((uint8_t*)outw + 32 * kw * q, pr.x,
                 pred_plus(pr.y, d, field<B>(pg.sW, 4 * w4 + q, lw, ls) - eps));
        off = P ? __clz(P) + 1 : off + 32;
        jq += __popc(P);
    }
    jb = min(jb + adv, jlast + 1);  // see decode_window
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
}

// SPARSE: lists with fewer than one segment per 64 keys (config 4) read < 1 B per key, so the
// kernel is issue-bound: cap registers at 40 for 6 resident CTAs and skip the L2 prefetch
// (A/B on B200: -4.7% time on config 4, +0.5-0.8% on dense configs, hence the switch);
// dense lists keep 5 resident CTAs (<= 48 registers).
template <bool K64, uint32_t B, bool SPARSE>
__global__ void __launch_bounds__(kThreads, SPARSE ? 6 : 5) lc_decode_kernel(const DecodeArgs a) {
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
        const bool has_next = !SPARSE && c + nwarps < a.nchunks;
        if (B && has_next && lane == 0)  // next chunk's residual words -> L2 now
            bulk_prefetch_l2(sec.words + (size_t)(h + nwarps) * 32 * B,
                             min(32 * B * 4 + 16, (a.nwords - (h + nwarps) * 32 * B) * 4));
        uint32_t jb = j0;                // segment holding the window's first key
        uint32_t sb = pg.sS[LC_BOUND(true, j0 - pg.pj, pg.cs)];  // its start
        uint8_t* outl = (uint8_t*)a.out + ((size_t)(key0 - a.i0) + lane) * kw;  // lane's slot
        if (nk == 1024 && jlast < pg.pj + pg.cp) {  // whole chunk staged: no re-page checks
#pragma unroll 1
            for (uint32_t g = 0; g < 8; g += 2, outl += 2 * 128 * kw) {
#pragma unroll
                for (uint32_t k = 0; k < 2; ++k)
                    decode_quad<K64, B, false>(pg, sec, jb, sb, jlast, key0 + 128 * (g + k), g + k,
                                               lane, lmask, lw, ls, a.eps, outl + 128 * kw * k);
                if (g == 2 && has_next && lane == 0) {  // next chunk's hint pair has landed:
                    const uint32_t npj = nj0 & ~3u;     // its segment slices -> L2
                    const uint32_t ncs = min(kSegCap + 4, njl + 2 - npj);
                    bulk_prefetch_l2(sec.starts + npj, ((ncs + 3) & ~3u) * 4);
                    bulk_prefetch_l2(sec.params + npj, min(kSegCap, njl + 1 - npj) * 16);
                }
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

// -------------------------------------------------------------------------- range decode
struct RangeArgs {
    Sections sec;
    const uint64_t* start;
    void* out;
    uint32_t* err;
    uint64_t q;
    uint32_t len, n, L, b, eps, mask;
    uint32_t nwords;  // W
};

// j = max{t in [hint[i>>10], hint[(i>>10)+1]] : starts[t] <= i} (Table I caption)
__device__ __forceinline__ uint32_t seg_search(const Sections& sec, uint32_t i, uint64_t keep) {
    uint32_t lo = ldh(sec.hint + (i >> 10), keep), hi = ldh(sec.hint + (i >> 10) + 1, keep);
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (ldh(sec.starts + mid, keep) <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// residual field of key i read from global words (two loads + funnel shift)
__device__ __forceinline__ uint2 field_words(const Sections& sec, uint32_t i, uint32_t b,
                                             uint64_t pol) {
    const uint64_t bit = (uint64_t)i * b;
    uint32_t wi = (uint32_t)(bit >> 5);
    if (LC_BOUND(true, wi + 1, sec.W) == 0) wi = 0;  // (only a checked build can take this)
    const uint32_t* wp = sec.words + wi;
    return make_uint2(ldh(wp, pol), ldh(wp + 1, pol));
}
__device__ __forceinline__ uint32_t field_of(uint2 w, uint32_t i, uint32_t b, uint32_t mask) {
    return __funnelshift_r(w.x, w.y, (i * b) & 31) & mask;
}

// One warp decodes 32 ranges.  Phase 1: lane r binary-searches the segment of range r's first
// key (32 independent searches in flight).  Phase 2: the warp decodes the ranges one after
// another with the window scheme of the full decode (64 keys per step, 2 keys per lane); the
// next range's candidate starts and residual words are fetched while the current range is
// decoded, so each range waits on a single dependent load (the params gather).
template <bool K64>
__global__ void __launch_bounds__(256) lc_range_kernel(const RangeArgs a) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t r0 = ((uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
    if (r0 >= a.q) return;  // warp-uniform
    const Sections sec = a.sec;
    const uint32_t len = a.len, b = a.b, mask = a.mask, L = a.L, eps = a.eps;
    const uint32_t lmask = lanemask_le();
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();

    // ---- phase 1: lane-parallel search
    uint32_t rs = 0, j = 0, sj = 0, ok = 0;
    if (r0 + lane < a.q) {
        const uint64_t s64 = __ldg(a.start + r0 + lane);
        if (s64 <= a.n && len <= a.n - s64) {
            ok = 1;
            rs = (uint32_t)s64;
            j = seg_search(sec, rs, keep);
            sj = ldh(sec.starts + j, keep);
        } else if (a.err) {
            atomicOr(a.err, 1u);
        }
    }
    const uint32_t nr = (uint32_t)min((uint64_t)32, a.q - r0);

    // candidate starts and first-step residual words of range k
    uint32_t nx;
    uint2 nwA = make_uint2(0, 0), nwB = make_uint2(0, 0);
    auto fetch = [&](uint32_t k) {
        const uint32_t rk = __shfl_sync(kFull, rs, k), jk = __shfl_sync(kFull, j, k);
        nx = ldh(sec.starts + min(jk + 1 + lane, L), keep) - rk;
        if (b && len >= 64) {
            nwA = field_words(sec, rk + lane, b, once);
            nwB = field_words(sec, rk + 32 + lane, b, once);
        }
    };
    fetch(0);
    for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t rk = __shfl_sync(kFull, rs, k);
        uint32_t jb = __shfl_sync(kFull, j, k);
        uint32_t sb = __shfl_sync(kFull, sj, k);
        const uint32_t okk = __shfl_sync(kFull, ok, k);
        const uint32_t x = nx;
        const uint2 wA = nwA, wB = nwB;
        if (k + 1 < nr) fetch(k + 1);
        uint8_t* outk = (uint8_t*)a.out + (size_t)(r0 + k) * len * kw;
        if (!okk) {
            for (uint32_t e = lane; e < len; e += 32) {
                if (K64) __stcs((unsigned long long*)outk + e, 0ull);
                else __stcs((unsigned int*)outk + e, 0u);
            }
            continue;
        }
        uint32_t w0 = 0;
        // first 64 keys as one pair step, from the prefetched candidates and words
        if (len >= 64 && __ballot_sync(kFull, x < 64) != kFull) {
            const uint32_t PA = __reduce_or_sync(kFull, bit_or_zero(x));
            const uint32_t PB = __reduce_or_sync(kFull, bit_or_zero(x - 32));
            const uint32_t adv = __popc(__ballot_sync(kFull, x <= 64));
            const uint32_t off0 = rk - sb;
            const uint32_t offB = PA ? __clz(PA) + 1 : off0 + 32;
            const uint32_t mA = PA & lmask, mB = PB & lmask;
            const uint32_t dA = mA ? lane - (31 - __clz(mA)) : off0 + lane;
            const uint32_t dB = mB ? lane - (31 - __clz(mB)) : offB + lane;
            const ulonglong2 pA = ldh(sec.params + LC_BOUND(true, jb + __popc(mA), L), once);
            const ulonglong2 pB =
                ldh(sec.params + LC_BOUND(true, jb + __popc(PA) + __popc(mB), L), once);
            const uint32_t uA = b ? field_of(wA, rk + lane, b, mask) : 0;
            const uint32_t uB = b ? field_of(wB, rk + 32 + lane, b, mask) : 0;
            put<K64>(outk + lane * kw, pA.x, pred_plus(pA.y, dA, uA - eps));
            put<K64>(outk + (32 + lane) * kw, pB.x, pred_plus(pB.y, dB, uB - eps));
            if (len == 64) continue;
            jb += adv;
            sb = ldh(sec.starts + min(jb, L), keep);
            w0 = 64;
        }
        while (w0 < len) {  // remaining keys: 32-key windows through L1/L2
            const uint32_t wb = rk + w0, rem = len - w0;
            const uint32_t xw = ldh(sec.starts + min(jb + 1 + lane, L), keep) - wb;
            const uint32_t P = __reduce_or_sync(kFull, bit_or_zero(xw));
            const uint32_t adv = __popc(__ballot_sync(kFull, xw <= 32));
            const uint32_t m = P & lmask;
            const uint32_t d = m ? lane - (31 - __clz(m)) : wb - sb + lane;
            if (lane < rem) {
                const ulonglong2 pr = ldh(sec.params + LC_BOUND(true, jb + __popc(m), L), once);
                const uint32_t u =
                    b ? field_of(field_words(sec, wb + lane, b, once), wb + lane, b, mask) : 0;
                put<K64>(outk + (w0 + lane) * kw, pr.x, pred_plus(pr.y, d, u - eps));
            }
            jb += adv;
            sb = ldh(sec.starts + min(jb, L), keep);
            w0 += 32;
        }
    }
}

// ---------------------------------------------------------------- range decode, len == 64
// cp.async (LDGSTS) 16-byte copy with zero fill when `valid` is false
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}

#ifndef LC_R64_SEGS
#define LC_R64_SEGS 8
#endif
// params staged per range: 1 + boundaries in 64 keys is <= 8 for 99.6% of config-5 ranges
// (max 10); a range needing more is decoded through L2
constexpr uint32_t kR64Segs = LC_R64_SEGS;
constexpr uint32_t kR64StartGroups = (kR64Segs + 3 + 3) / 4;  // starts[j+1 .. j+kR64Segs] from a 16-B boundary
#ifndef LC_R64_SLOTS
#define LC_R64_SLOTS 4
#endif
constexpr uint32_t kR64Slots = LC_R64_SLOTS;  // ring depth per warp (ranges gathered ahead)
__host__ __device__ constexpr uint32_t r64_words(uint32_t b) {  // staged residual words
    return ((((64 * b + 31) >> 5) + 2 + 3) + 3) & ~3u;
}
__host__ __device__ constexpr uint32_t r64_bytes(uint32_t b) {  // per slot: params|starts|words
    return 16 * kR64Segs + 16 * kR64StartGroups + 4 * r64_words(b);
}

// 64-key ranges (BASELINE config 5).  Phase 1: lane r binary-searches range r's first segment
// (32 independent searches).  Phase 2: the warp walks its 32 ranges through a 4-slot shared-
// memory ring: the lanes gather range k+3's params[j..j+8), starts[j+1..j+9) and residual
// words with cp.async (one 16-byte copy per lane) while range k is decoded from smem with the
// pair-window scheme, so the decode never waits on a dependent global load.  A range crossing
// more than 7 segment starts is decoded through L2 instead.
template <bool K64>
__global__ void __launch_bounds__(256) lc_range64_kernel(const RangeArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t kw = K64 ? 8 : 4;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r0 = ((uint64_t)blockIdx.x * 8 + warp) * 32;
    if (r0 >= a.q) return;  // warp-uniform
    const Sections sec = a.sec;
    const uint32_t b = a.b, mask = a.mask, L = a.L, eps = a.eps;
    const uint32_t RB = r64_bytes(b), nw16 = r64_words(b) / 4;
    uint8_t* ring = smem + warp * kR64Slots * RB;
    const uint32_t lmask = lanemask_le();
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();

    // ---- phase 1: lane-parallel search
    uint32_t rs = 0, j = 0, sj = 0, ok = 0;
    if (r0 + lane < a.q) {
        const uint64_t s64 = __ldg(a.start + r0 + lane);
        if (s64 <= a.n && 64 <= a.n - s64) {
            ok = 1;
            rs = (uint32_t)s64;
            j = seg_search(sec, rs, keep);
            sj = ldh(sec.starts + j, keep);
        } else if (a.err) {
            atomicOr(a.err, 1u);
        }
    }
    const uint32_t nr = (uint32_t)min((uint64_t)32, a.q - r0);

    // gather range k into ring slot k % kR64Slots: copy groups 0..11 = params, 12..16 = starts,
    // then words; group g is done by lane g % 32.  Each lane's role (source section, offset in
    // the slot) is fixed, so per range it only adds the range's uniform section offset.
    const uint32_t ngroups = kR64Segs + kR64StartGroups + nw16;
    struct Role {
        const uint8_t* src;  // section base + 16 t
        uint32_t dst, kind, t;
    };
    auto role_of = [&](uint32_t g) {
        Role r;
        const uint32_t gw = kR64Segs + kR64StartGroups;
        if (g < kR64Segs) r = {(const uint8_t*)(sec.params + g), 16 * g, 0, g};
        else if (g < gw)
            r = {(const uint8_t*)(sec.starts + 4 * (g - kR64Segs)), 16 * g, 1, g - kR64Segs};
        else
            r = {(const uint8_t*)(sec.words + 4 * (g - gw)), 16 * g, 2, g - gw};
        return r;
    };
    const Role ra = role_of(lane), rb = role_of(lane + 32);
    const bool has_a = lane < ngroups, has_b = lane + 32 < ngroups;
    auto copy = [&](const Role& r, uint8_t* slot, uint32_t jk, uint32_t s0, uint32_t w0) {
        const uint64_t off = r.kind == 0 ? (uint64_t)jk * 16 : r.kind == 1 ? (uint64_t)s0 * 4
                                                                            : (uint64_t)w0 * 4;
        const bool valid = r.kind == 0 ? jk + r.t < L
                                       : (r.kind == 1 || w0 + 4 * r.t + 4 <= a.nwords);
        cp16(slot + r.dst, r.src + off, valid);
    };
    auto issue = [&](uint32_t k) {
        if (k < nr) {
            const uint32_t rk = __shfl_sync(kFull, rs, k), jk = __shfl_sync(kFull, j, k);
            const uint32_t okk = __shfl_sync(kFull, ok, k);
            uint8_t* slot = ring + (k % kR64Slots) * RB;
            if (okk) {
                const uint32_t s0 = (jk + 1) & ~3u;
                const uint32_t w0 = (uint32_t)(((uint64_t)rk * b) >> 5) & ~3u;
                if (has_a) copy(ra, slot, jk, s0, w0);
                if (has_b) copy(rb, slot, jk, s0, w0);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // one group per range (maybe empty)
    };
    for (uint32_t k = 0; k + 1 < kR64Slots; ++k) issue(k);

    for (uint32_t k = 0; k < nr; ++k) {
        issue(k + kR64Slots - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kR64Slots - 1) : "memory");
        __syncwarp();
        const uint32_t rk = __shfl_sync(kFull, rs, k);
        const uint32_t jk = __shfl_sync(kFull, j, k);
        const uint32_t sb = __shfl_sync(kFull, sj, k);
        const uint32_t okk = __shfl_sync(kFull, ok, k);
        uint8_t* outk = (uint8_t*)a.out + (size_t)(r0 + k) * 64 * kw;
        if (!okk) {
            put<K64>(outk + lane * kw, 0, 0);
            put<K64>(outk + (32 + lane) * kw, 0, 0);
            __syncwarp();
            continue;
        }
        const uint8_t* rsm = ring + (k % kR64Slots) * RB;
        const ulonglong2* P = (const ulonglong2*)rsm;
        const uint32_t* S = (const uint32_t*)(rsm + 16 * kR64Segs) + ((jk + 1) & 3);  // starts[jk+1+t]
        const uint32_t x = (lane < kR64Segs && jk + 1 + lane <= L) ? S[lane] - rk : kFull;
        const uint32_t inside = __ballot_sync(kFull, x < 64);
        if (__popc(inside) < kR64Segs) {
            const uint32_t PA = __reduce_or_sync(kFull, bit_or_zero(x));
            const uint32_t PB = __reduce_or_sync(kFull, bit_or_zero(x - 32));
            const uint32_t off0 = rk - sb;
            const uint32_t offB = PA ? __clz(PA) + 1 : off0 + 32;
            const uint32_t mA = PA & lmask, mB = PB & lmask;
            const uint32_t dA = mA ? lane - (31 - __clz(mA)) : off0 + lane;
            const uint32_t dB = mB ? lane - (31 - __clz(mB)) : offB + lane;
            const ulonglong2 pA = P[LC_BOUND(true, __popc(mA), kR64Segs)];
            const ulonglong2 pB = P[LC_BOUND(true, __popc(PA) + __popc(mB), kR64Segs)];
            uint32_t uA = 0, uB = 0;
            if (b) {
                const uint32_t* Wd = (const uint32_t*)(rsm + 16 * (kR64Segs + kR64StartGroups));
                const uint64_t wbase = ((((uint64_t)rk * b) >> 5) & ~3ull) << 5;
                const uint32_t bA = (uint32_t)((uint64_t)(rk + lane) * b - wbase);
                const uint32_t bB = bA + 32 * b;
                LC_CHECK(true, (bB >> 5) + 1, r64_words(b));
                uA = __funnelshift_r(Wd[bA >> 5], Wd[(bA >> 5) + 1], bA & 31) & mask;
                uB = __funnelshift_r(Wd[bB >> 5], Wd[(bB >> 5) + 1], bB & 31) & mask;
            }
            put<K64>(outk + lane * kw, pA.x, pred_plus(pA.y, dA, uA - eps));
            put<K64>(outk + (32 + lane) * kw, pB.x, pred_plus(pB.y, dB, uB - eps));
        } else {  // dense range: two 32-key windows through L2
            uint32_t jb = jk, sbw = sb;
            for (uint32_t w0 = 0; w0 < 64; w0 += 32) {
                const uint32_t wb = rk + w0;
                const uint32_t xw = ldh(sec.starts + min(jb + 1 + lane, L), keep) - wb;
                const uint32_t Pm = __reduce_or_sync(kFull, bit_or_zero(xw));
                const uint32_t adv = __popc(__ballot_sync(kFull, xw <= 32));
                const uint32_t m = Pm & lmask;
                const uint32_t d = m ? lane - (31 - __clz(m)) : wb - sbw + lane;
                const ulonglong2 pr = ldh(sec.params + LC_BOUND(true, jb + __popc(m), L), once);
                const uint32_t u =
                    b ? field_of(field_words(sec, wb + lane, b, once), wb + lane, b, mask) : 0;
                put<K64>(outk + (w0 + lane) * kw, pr.x, pred_plus(pr.y, d, u - eps));
                jb += adv;
                sbw = ldh(sec.starts + min(jb, L), keep);
            }
        }
        __syncwarp();  // the slot is refilled by the next issue()
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
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

constexpr uint32_t kAccessPerThread = 2;

// Dec(K^c)[i] per query (Table I): hint bracket, binary search
// over starts, one params gather, one residual field.  Each thread serves kAccessPerThread
// queries whose dependent load chains are interleaved; the residual words do not depend on
// the segment and are fetched before the search.
template <bool K64>
__global__ void __launch_bounds__(256) lc_access_kernel(const AccessArgs a) {
    const uint64_t t0 = (uint64_t)blockIdx.x * (256 * kAccessPerThread) + threadIdx.x;
    const Sections sec = a.sec;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    uint32_t i[kAccessPerThread], lo[kAccessPerThread], hi[kAccessPerThread];
    bool live[kAccessPerThread];
    uint2 w[kAccessPerThread];
#pragma unroll
    for (uint32_t k = 0; k < kAccessPerThread; ++k) {
        const uint64_t t = t0 + 256 * k;
        live[k] = false;
        i[k] = 0;
        lo[k] = hi[k] = 0;
        w[k] = make_uint2(0, 0);
        if (t < a.q) {
            const uint64_t i64 = __ldcs(a.idx + t);
            if (i64 < a.n) {
                live[k] = true;
                i[k] = (uint32_t)i64;
            } else {
                if (a.err) atomicOr(a.err, 1u);
                if (K64) __stcs((unsigned long long*)a.out + t, 0ull);
                else __stcs((unsigned int*)a.out + t, 0u);
            }
        }
    }
#pragma unroll
    for (uint32_t k = 0; k < kAccessPerThread; ++k) {
        if (live[k]) {
            lo[k] = ldh(sec.hint + (i[k] >> 10), keep);
            hi[k] = ldh(sec.hint + (i[k] >> 10) + 1, keep);
            if (a.b) w[k] = field_words(sec, i[k], a.b, once);
        }
    }
    for (;;) {  // interleaved binary searches: j = max{t in [lo, hi] : starts[t] <= i}
        bool any = false;
        uint32_t mid[kAccessPerThread], v[kAccessPerThread];
#pragma unroll
        for (uint32_t k = 0; k < kAccessPerThread; ++k) {
            mid[k] = (lo[k] + hi[k] + 1) >> 1;
            v[k] = 0;
            if (lo[k] < hi[k]) {
                v[k] = ldh(sec.starts + mid[k], keep);
                any = true;
            }
        }
        if (!any) break;
#pragma unroll
        for (uint32_t k = 0; k < kAccessPerThread; ++k) {
            if (lo[k] < hi[k]) {
                if (v[k] <= i[k]) lo[k] = mid[k];
                else hi[k] = mid[k] - 1;
            }
        }
    }
#pragma unroll
    for (uint32_t k = 0; k < kAccessPerThread; ++k) {
        if (!live[k]) continue;
        const uint32_t s = ldh(sec.starts + lo[k], keep);
        const ulonglong2 pr = ldh(sec.params + LC_BOUND(true, lo[k], sec.L), once);
        const uint32_t u = a.b ? field_of(w[k], i[k], a.b, a.mask) : 0;
        const uint64_t t = t0 + 256 * k;
        put<K64>((uint8_t*)a.out + t * (K64 ? 8 : 4), pr.x, pred_plus(pr.y, i[k] - s, u - a.eps));
    }
}

// ----------------------------------------------------------------------------- quantiles
struct QuantArgs {
    Sections sec;
    const uint64_t* k;
    void* out;
    uint32_t* err;
    uint64_t m, q;
    uint32_t n, b, eps, mask;
};

// The k-th q-quantile K[min(floor(N k / q), N - 1)] (§III-C; Table I): exact =
// f(i) + Delta[i] through the hint bracket + binary search; approximate (EXACT = false) =
// floor(f(i)) from the segment alone, no residual read, error <= eps.
template <bool K64, bool EXACT>
__global__ void __launch_bounds__(256) lc_quantile_kernel(const QuantArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= a.m) return;
    const Sections sec = a.sec;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    const uint64_t k = __ldg(a.k + t);
    uint8_t* o = (uint8_t*)a.out + t * (K64 ? 8 : 4);
    if (k > a.q) {
        if (a.err) atomicOr(a.err, 1u);
        put<K64>(o, 0, 0);
        return;
    }
    const uint32_t i = (uint32_t)min((uint64_t)a.n * k / a.q, (uint64_t)a.n - 1);  // N k < 2^64
    const uint32_t j = seg_search(sec, i, keep);
    const uint32_t s = ldh(sec.starts + j, keep);
    const ulonglong2 pr = ldh(sec.params + j, once);
    if (EXACT) {
        const uint32_t v = (a.b ? field_of(field_words(sec, i, a.b, once), i, a.b, a.mask) : 0) - a.eps;
        put<K64>(o, pr.x, pred_plus(pr.y, i - s, v));
    } else {  // floor(f(i)) can exceed the key width by up to eps: saturate (L24)
        const uint32_t t = pred_plus(pr.y, i - s, 0);
        const uint64_t f = pr.x + t;
        if (K64) __stcs((unsigned long long*)o, f < pr.x ? ~0ull : (unsigned long long)f);
        else __stcs((unsigned int*)o, f > 0xffffffffull ? 0xffffffffu : (unsigned int)f);
    }
}

// ------------------------------------------------------ successor search and intersection
// Key-space search uses the segments as skip pointers (Fig. 4b): with the
// FORMAT F2 anchor, base_j = K[s_j] and the bases are strictly increasing, so segment j covers
// exactly the keys [base_j, base_{j+1}).  next_geq(x) = binary search over the bases, then a
// binary search inside the one segment, decoding only the probed keys (never a whole segment).
__device__ __forceinline__ uint64_t key_at(const Sections& sec, uint32_t i, uint32_t s,
                                           ulonglong2 pr, uint32_t b, uint32_t mask, uint32_t eps,
                                           uint64_t once) {
    const uint32_t u = b ? field_of(field_words(sec, i, b, once), i, b, mask) : 0;
    return pr.x + pred_plus(pr.y, i - s, u - eps);
}

struct SuccResult {
    uint32_t idx;  // first index with K[idx] >= x, n if none
    uint64_t key;  // K[idx], 0 if none
};

__device__ SuccResult next_geq_one(const Sections& sec, uint32_t n, uint32_t L, uint32_t b,
                                   uint32_t mask, uint32_t eps, uint64_t x, uint64_t keep,
                                   uint64_t once) {
    const uint64_t* bases = (const uint64_t*)sec.params;  // base_j at bases[2 j]
    const uint64_t b0 = __ldg(bases);
    if (x <= b0) return {0u, b0};
    uint32_t lo = 0, hi = L - 1;  // max{j : base_j <= x}
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(bases + 2 * (size_t)mid) <= x) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t j = lo;
    const uint32_t s = ldh(sec.starts + j, keep), e = ldh(sec.starts + j + 1, keep);
    const ulonglong2 pr = ldh(sec.params + j, once);
    uint32_t l = s + 1, r = e;  // K[s] = base_j <= x; answer in (s, e]
    if (pr.x == x) return {s, x};
    uint64_t kr = 0;
    bool have = false;
    while (l < r) {
        const uint32_t mid = (l + r) >> 1;
        const uint64_t km = key_at(sec, mid, s, pr, b, mask, eps, once);
        if (km >= x) {
            r = mid;
            kr = km;
            have = true;
        } else {
            l = mid + 1;
        }
    }
    if (l < e) {
        if (!have || r != l) kr = key_at(sec, l, s, pr, b, mask, eps, once);
        return {l, kr};
    }
    if (e >= n) return {n, 0};
    return {e, __ldg(bases + 2 * (size_t)(j + 1))};  // K[e] = base_{j+1} > x
}

struct SuccArgs {
    Sections sec;
    const uint64_t* x;
    uint64_t* out_idx;
    void* out_key;
    uint64_t m;
    uint32_t n, L, b, eps, mask;
};

template <bool K64>
__global__ void __launch_bounds__(256) lc_next_geq_kernel(const SuccArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= a.m) return;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    const uint64_t x = __ldg(a.x + t);
    SuccResult r;
    if (!K64 && x > 0xffffffffull) r = {a.n, 0};
    else r = next_geq_one(a.sec, a.n, a.L, a.b, a.mask, a.eps, x, keep, once);
    if (a.out_idx) a.out_idx[t] = r.idx;
    if (a.out_key) put<K64>((uint8_t*)a.out_key + t * (K64 ? 8 : 4), r.key, 0);
}

// Intersection A ∩ B (AND query): A is decoded into scratch, each key of A is looked up in B
// with next_geq (segments of B holding no key of A are never touched), matches are flagged
// with warp ballots and compacted in order (per-CTA counts, one-CTA scan, scatter).
struct IsectArgs {
    Sections sb;            // list B (searched)
    const void* a_keys;     // decoded list A
    uint32_t* flags;        // ceil(na / 32) match bitmap
    uint32_t* counts;       // per-CTA match counts, then exclusive offsets; [nblk] = total
    void* out;
    uint64_t* d_count;
    uint32_t na, nb, Lb, b, eps, mask, nblk;
};

template <bool K64>
__global__ void __launch_bounds__(256) lc_isect_flag_kernel(const IsectArgs a) {
    __shared__ uint32_t warp_cnt[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    bool hit = false;
    if (t < a.na) {
        const uint64_t x = K64 ? ((const uint64_t*)a.a_keys)[t] : ((const uint32_t*)a.a_keys)[t];
        const SuccResult r = next_geq_one(a.sb, a.nb, a.Lb, a.b, a.mask, a.eps, x, keep, once);
        hit = r.idx < a.nb && r.key == x;
    }
    const uint32_t bal = __ballot_sync(kFull, hit);
    if (lane == 0) {
        if (t < a.na) a.flags[t >> 5] = bal;
        warp_cnt[warp] = __popc(bal);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (int w = 0; w < 8; ++w) c += warp_cnt[w];
        a.counts[blockIdx.x] = c;
    }
}

// exclusive scan of the per-CTA counts in one CTA of 1024 threads; counts[nblk] = total
__global__ void __launch_bounds__(1024) lc_isect_scan_kernel(const IsectArgs a) {
    __shared__ uint32_t part[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < a.nblk; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < a.nblk ? a.counts[i] : 0;
        uint32_t x = v;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) part[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t p = part[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, p, o);
                if (lane >= (uint32_t)o) p += y;
            }
            part[lane] = p;  // inclusive over warps
        }
        __syncthreads();
        const uint32_t excl = carry + (warp ? part[warp - 1] : 0) + x - v;
        if (i < a.nblk) a.counts[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.counts[a.nblk] = carry;
        *a.d_count = carry;
    }
}

template <bool K64>
__global__ void __launch_bounds__(256) lc_isect_write_kernel(const IsectArgs a) {
    __shared__ uint32_t warp_off[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bal = t < a.na ? a.flags[t >> 5] : 0;  // whole warp reads the same word
    if (lane == 0) warp_off[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = a.counts[blockIdx.x];
        for (int w = 0; w < 8; ++w) {
            const uint32_t v = warp_off[w];
            warp_off[w] = c;
            c += v;
        }
    }
    __syncthreads();
    if ((bal >> lane) & 1) {
        const uint32_t pos = warp_off[warp] + __popc(bal & ((1u << lane) - 1));
        if (K64) ((uint64_t*)a.out)[pos] = ((const uint64_t*)a.a_keys)[t];
        else ((uint32_t*)a.out)[pos] = ((const uint32_t*)a.a_keys)[t];
    }
}

// Union (OR query): both lists are decoded into scratch; the keys of the shorter
// list that are absent from the longer one are flagged (binary search in the decoded longer
// list) and compacted in order with the intersection's scan/scatter kernels; then one
// merge-path pass merges the two disjoint sorted lists straight into the output.
template <bool K64>
__global__ void __launch_bounds__(256) lc_union_flag_kernel(const IsectArgs a, const void* a_sorted,
                                                            uint32_t n_sorted) {
    __shared__ uint32_t warp_cnt[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bool keep = false;
    if (t < a.na) {  // a.a_keys = decoded B; keep keys of B not in A
        const uint64_t x = K64 ? ((const uint64_t*)a.a_keys)[t] : ((const uint32_t*)a.a_keys)[t];
        uint32_t lo = 0, hi = n_sorted;  // first A[i] >= x
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            const uint64_t v = K64 ? __ldg((const uint64_t*)a_sorted + mid)
                                   : __ldg((const uint32_t*)a_sorted + mid);
            if (v < x) lo = mid + 1;
            else hi = mid;
        }
        const uint64_t v = lo < n_sorted ? (K64 ? __ldg((const uint64_t*)a_sorted + lo)
                                                : __ldg((const uint32_t*)a_sorted + lo))
                                         : ~0ull;
        keep = lo == n_sorted || v != x;
    }
    const uint32_t bal = __ballot_sync(kFull, keep);
    if (lane == 0) {
        if (t < a.na) a.flags[t >> 5] = bal;
        warp_cnt[warp] = __popc(bal);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (int w = 0; w < 8; ++w) c += warp_cnt[w];
        a.counts[blockIdx.x] = c;
    }
}

constexpr uint32_t kMergeItems = 8;                 // output keys per thread
constexpr uint32_t kMergeTile = 256 * kMergeItems;  // output keys per CTA

// number of A keys among the first `diag` keys of merge(A, C) (disjoint sorted lists)
template <typename K>
__device__ __forceinline__ uint32_t merge_split(const K* a, uint32_t na, const K* c, uint32_t nc,
                                                uint32_t diag) {
    uint32_t lo = diag > nc ? diag - nc : 0, hi = min(diag, na);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < c[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Tiled merge path: CTA t produces outputs [t*2048, (t+1)*2048).  One thread finds the tile's
// split on each input, the tile's slices of A and C are loaded coalesced into shared memory,
// each thread merges 8 outputs from shared memory, and the tile is stored coalesced.
template <bool K64>
__global__ void __launch_bounds__(256) lc_merge_kernel(const void* A, uint32_t na, const void* C,
                                                       const uint32_t* nc_ptr, void* out,
                                                       uint64_t* d_count) {
    using K = typename std::conditional<K64, uint64_t, uint32_t>::type;
    __shared__ K sm[kMergeTile];   // A slice then C slice
    __shared__ K so[kMergeTile];   // merged tile
    __shared__ uint32_t bounds[4];
    const K* a = (const K*)A;
    const K* c = (const K*)C;
    const uint32_t nc = *nc_ptr, total = na + nc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_count = total;
    const uint64_t t0 = (uint64_t)blockIdx.x * kMergeTile;
    if (t0 >= total) return;
    const uint32_t d0 = (uint32_t)t0, d1 = (uint32_t)min(t0 + kMergeTile, (uint64_t)total);
    if (threadIdx.x < 2) {
        const uint32_t d = threadIdx.x ? d1 : d0;
        const uint32_t i = merge_split(a, na, c, nc, d);
        bounds[2 * threadIdx.x] = i;
        bounds[2 * threadIdx.x + 1] = d - i;
    }
    __syncthreads();
    const uint32_t a0 = bounds[0], c0 = bounds[1], a1 = bounds[2], c1 = bounds[3];
    const uint32_t la = a1 - a0, lcn = c1 - c0;  // la + lcn = d1 - d0
    for (uint32_t k = threadIdx.x; k < la; k += 256) sm[k] = __ldg(a + a0 + k);
    for (uint32_t k = threadIdx.x; k < lcn; k += 256) sm[la + k] = __ldg(c + c0 + k);
    __syncthreads();
    const uint32_t n = la + lcn;
    const uint32_t dd = min(threadIdx.x * kMergeItems, n);
    uint32_t i = merge_split(sm, la, sm + la, lcn, dd), j = dd - i;
    for (uint32_t k = 0; k < kMergeItems && dd + k < n; ++k) {
        const bool take_a = j >= lcn || (i < la && sm[i] < sm[la + j]);
        so[dd + k] = take_a ? sm[i++] : sm[la + j++];
    }
    __syncthreads();
    K* o = (K*)out + d0;
    for (uint32_t k = threadIdx.x; k < n; k += 256) __stcs(o + k, so[k]);
}

// ------------------------------------------------------------------------------ launchers
uint32_t mask_of(uint32_t b) { return b >= 32 ? 0xffffffffu : ((1u << b) - 1); }

int32_t cuda_status() { return cudaGetLastError() == cudaSuccess ? LC_OK : LC_ERR_CUDA; }

using DecodeFn = void (*)(DecodeArgs);

template <bool K64, bool SPARSE, uint32_t... Bs>
constexpr std::array<DecodeFn, sizeof...(Bs)> decode_table(std::integer_sequence<uint32_t, Bs...>) {
    return {{&lc_decode_kernel<K64, Bs, SPARSE>...}};
}
// one instantiation per residual width b = 0..32 (compile-time field offsets and masks),
// key width and segment density: kDecode[sparse][k64][b]
const std::array<DecodeFn, 33> kDecode[2][2] = {
    {decode_table<false, false>(std::make_integer_sequence<uint32_t, 33>{}),
     decode_table<true, false>(std::make_integer_sequence<uint32_t, 33>{})},
    {decode_table<false, true>(std::make_integer_sequence<uint32_t, 33>{}),
     decode_table<true, true>(std::make_integer_sequence<uint32_t, 33>{})}};

struct GridCache {
    std::mutex mu;
    int dev = -1;
    int sms = 0;
    int occ[2][2][33] = {};  // [sparse][K64][res_bits] -> resident CTAs per SM
};
GridCache g_grid;

// persistent grid size for the decode kernel: SMs x resident CTAs at this smem footprint
int persistent_grid(bool sparse, bool k64, uint32_t b) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_grid.mu);
    if (g_grid.dev != dev) {
        g_grid.dev = dev;
        cudaDeviceGetAttribute(&g_grid.sms, cudaDevAttrMultiProcessorCount, dev);
        std::memset(g_grid.occ, 0, sizeof g_grid.occ);
    }
    int& occ = g_grid.occ[sparse][k64][b];
    if (occ == 0) {
        const void* fn = (const void*)kDecode[sparse][k64][b];
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
    a.nwords = (uint32_t)v->h.n_words;
    const uint32_t b = v->h.res_bits;
    a.warp_bytes = warp_bytes_for(b);
    const uint32_t smem = a.warp_bytes * kWarpsPerCta;
    const bool k64 = v->h.key_bits == 64;
    const bool sparse = v->h.n_seg * 64 < v->h.n;  // < 1 segment per 64 keys
    const int full = persistent_grid(sparse, k64, b);
    const uint32_t need = (a.nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
    const uint32_t grid = need < (uint32_t)full ? need : (uint32_t)full;
    kDecode[sparse][k64][b]<<<grid, kThreads, smem, st>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

// lc_decode_host pipeline resources, created once per device: an H2D and a D2H copy stream and
// one event per span and stage.
constexpr uint32_t kMaxSpans = 64;
struct HostPipe {
    std::mutex mu;
    int dev = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t up[kMaxSpans] = {}, dec[kMaxSpans] = {}, done = nullptr;
};
HostPipe g_pipe;

int32_t pipe_init() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_pipe.dev == dev) return LC_OK;
    if (cudaStreamCreateWithFlags(&g_pipe.h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g_pipe.d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_pipe.done, cudaEventDisableTiming) != cudaSuccess)
        return LC_ERR_CUDA;
    for (uint32_t k = 0; k < kMaxSpans; ++k)
        if (cudaEventCreateWithFlags(&g_pipe.up[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g_pipe.dec[k], cudaEventDisableTiming) != cudaSuccess)
            return LC_ERR_CUDA;
    g_pipe.dev = dev;
    return LC_OK;
}

// host->device copy of blob bytes [a, b) (same offsets on both sides)
int32_t up_bytes(const void* h, void* d, uint64_t a, uint64_t b, cudaStream_t st) {
    if (b <= a) return LC_OK;
    return cudaMemcpyAsync((uint8_t*)d + a, (const uint8_t*)h + a, b - a, cudaMemcpyHostToDevice,
                           st) == cudaSuccess
               ? LC_OK
               : LC_ERR_CUDA;
}

}  // namespace

extern "C" {

int32_t lc_decode_span(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (i0 > i1 || i1 > v->h.n) return LC_ERR_ARG;
    if (i0 == i1) return LC_OK;  // an empty span (e.g. a shard past the end) is a no-op
    if (i0 & 1023) return LC_ERR_ARG;
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
    const uint64_t grid = (q + 256 * kAccessPerThread - 1) / (256 * kAccessPerThread);
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
    a.nwords = (uint32_t)v->h.n_words;
    const uint64_t grid = (q + 255) / 256;  // 8 warps x 32 ranges per CTA
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    const bool k64 = v->h.key_bits == 64;
    cudaStream_t st = (cudaStream_t)stream;
    if (len == 64) {  // the config-5 shape: cp.async ring kernel
        const uint32_t smem = 8 * kR64Slots * r64_bytes(a.b);
        const void* fn = k64 ? (const void*)lc_range64_kernel<true> : (const void*)lc_range64_kernel<false>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (k64) lc_range64_kernel<true><<<(unsigned)grid, 256, smem, st>>>(a);
        else lc_range64_kernel<false><<<(unsigned)grid, 256, smem, st>>>(a);
        lc_detail::count_launch(1);
        return cuda_status();
    }
    if (k64) lc_range_kernel<true><<<(unsigned)grid, 256, 0, st>>>(a);
    else lc_range_kernel<false><<<(unsigned)grid, 256, 0, st>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

int32_t lc_quantile(const lc_view* v, const uint64_t* d_k, uint64_t m, uint64_t q,
                    int32_t exact, void* d_out, uint32_t* d_err, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (q == 0 || q > 0xffffffffULL) return LC_ERR_ARG;
    if (m == 0) return LC_OK;
    if (!d_k || !d_out) return LC_ERR_ARG;
    QuantArgs a;
    a.sec = sections_of(v);
    a.k = d_k;
    a.out = d_out;
    a.err = d_err;
    a.m = m;
    a.q = q;
    a.n = (uint32_t)v->h.n;
    a.b = v->h.res_bits;
    a.eps = v->h.eps;
    a.mask = mask_of(a.b);
    const uint64_t grid = (m + 255) / 256;
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const bool k64 = v->h.key_bits == 64;
    if (exact) {
        if (k64) lc_quantile_kernel<true, true><<<(unsigned)grid, 256, 0, st>>>(a);
        else lc_quantile_kernel<false, true><<<(unsigned)grid, 256, 0, st>>>(a);
    } else {
        if (k64) lc_quantile_kernel<true, false><<<(unsigned)grid, 256, 0, st>>>(a);
        else lc_quantile_kernel<false, false><<<(unsigned)grid, 256, 0, st>>>(a);
    }
    lc_detail::count_launch(1);
    return cuda_status();
}

int32_t lc_next_geq(const lc_view* v, const uint64_t* d_x, uint64_t m, uint64_t* d_out_idx,
                    void* d_out_key, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (m == 0) return LC_OK;
    if (!d_x || (!d_out_idx && !d_out_key)) return LC_ERR_ARG;
    SuccArgs a;
    a.sec = sections_of(v);
    a.x = d_x;
    a.out_idx = d_out_idx;
    a.out_key = d_out_key;
    a.m = m;
    a.n = (uint32_t)v->h.n;
    a.L = (uint32_t)v->h.n_seg;
    a.b = v->h.res_bits;
    a.eps = v->h.eps;
    a.mask = mask_of(a.b);
    const uint64_t grid = (m + 255) / 256;
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    if (v->h.key_bits == 64) lc_next_geq_kernel<true><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    else lc_next_geq_kernel<false><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    lc_detail::count_launch(1);
    return cuda_status();
}

uint64_t lc_intersect_scratch_bytes(const lc_view* a) {
    if (!a) return 0;
    const uint64_t na = a->h.n, kw = a->h.key_bits / 8;
    const uint64_t nblk = (na + 255) / 256;
    auto r256 = [](uint64_t x) { return (x + 255) & ~255ULL; };
    return r256(na * kw) + r256(4 * ((na + 31) / 32)) + r256(4 * (nblk + 1));
}

int32_t lc_intersect(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                     void* d_out, uint64_t* d_count, lc_stream stream) {
    if (!a || !b || !a->d_blob || !b->d_blob || !d_scratch || !d_out || !d_count) return LC_ERR_ARG;
    if (a->h.key_bits != b->h.key_bits) return LC_ERR_ARG;
    if (scratch_bytes < lc_intersect_scratch_bytes(a) || ((uintptr_t)d_scratch & 255)) return LC_ERR_ARG;
    const uint64_t na = a->h.n, kw = a->h.key_bits / 8;
    auto r256 = [](uint64_t x) { return (x + 255) & ~255ULL; };
    uint8_t* sc = (uint8_t*)d_scratch;
    IsectArgs g;
    g.sb = sections_of(b);
    g.a_keys = sc;
    g.flags = (uint32_t*)(sc + r256(na * kw));
    g.counts = (uint32_t*)(sc + r256(na * kw) + r256(4 * ((na + 31) / 32)));
    g.out = d_out;
    g.d_count = d_count;
    g.na = (uint32_t)na;
    g.nb = (uint32_t)b->h.n;
    g.Lb = (uint32_t)b->h.n_seg;
    g.b = b->h.res_bits;
    g.eps = b->h.eps;
    g.mask = mask_of(g.b);
    g.nblk = (uint32_t)((na + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    int32_t rc = launch_decode(a, 0, na, sc, st);
    if (rc) return rc;
    if (kw == 8) lc_isect_flag_kernel<true><<<g.nblk, 256, 0, st>>>(g);
    else lc_isect_flag_kernel<false><<<g.nblk, 256, 0, st>>>(g);
    lc_isect_scan_kernel<<<1, 1024, 0, st>>>(g);
    if (kw == 8) lc_isect_write_kernel<true><<<g.nblk, 256, 0, st>>>(g);
    else lc_isect_write_kernel<false><<<g.nblk, 256, 0, st>>>(g);
    lc_detail::count_launch(3);
    return cuda_status();
}

uint64_t lc_union_scratch_bytes(const lc_view* a, const lc_view* b) {
    if (!a || !b) return 0;
    const uint64_t na = a->h.n, nb = b->h.n, kw = a->h.key_bits / 8;
    const uint64_t ns = na < nb ? na : nb;  // the shorter list is flagged and compacted
    auto r256 = [](uint64_t x) { return (x + 255) & ~255ULL; };
    return r256(na * kw) + r256(nb * kw) + r256(ns * kw) + r256(4 * ((ns + 31) / 32)) +
           r256(4 * ((ns + 255) / 256 + 1));
}

int32_t lc_union(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                 void* d_out, uint64_t* d_count, lc_stream stream) {
    if (!a || !b || !a->d_blob || !b->d_blob || !d_scratch || !d_out || !d_count) return LC_ERR_ARG;
    if (a->h.key_bits != b->h.key_bits) return LC_ERR_ARG;
    if (scratch_bytes < lc_union_scratch_bytes(a, b) || ((uintptr_t)d_scratch & 255)) return LC_ERR_ARG;
    // union = long ∪ (short \ long): only the shorter list is searched and compacted
    const lc_view* lg = a->h.n >= b->h.n ? a : b;
    const lc_view* sh = a->h.n >= b->h.n ? b : a;
    const uint64_t nl = lg->h.n, ns = sh->h.n, kw = a->h.key_bits / 8;
    auto r256 = [](uint64_t x) { return (x + 255) & ~255ULL; };
    uint8_t* sL = (uint8_t*)d_scratch;
    uint8_t* sS = sL + r256(nl * kw);
    uint8_t* sC = sS + r256(ns * kw);  // short \ long
    uint32_t* flags = (uint32_t*)(sC + r256(ns * kw));
    uint32_t* counts = (uint32_t*)((uint8_t*)flags + r256(4 * ((ns + 31) / 32)));
    IsectArgs g{};
    g.a_keys = sS;
    g.flags = flags;
    g.counts = counts;
    g.out = sC;
    g.d_count = d_count;  // overwritten by the merge with the union size
    g.na = (uint32_t)ns;
    g.nblk = (uint32_t)((ns + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    int32_t rc = launch_decode(lg, 0, nl, sL, st);
    if (!rc) rc = launch_decode(sh, 0, ns, sS, st);
    if (rc) return rc;
    const bool k64 = kw == 8;
    if (k64) lc_union_flag_kernel<true><<<g.nblk, 256, 0, st>>>(g, sL, (uint32_t)nl);
    else lc_union_flag_kernel<false><<<g.nblk, 256, 0, st>>>(g, sL, (uint32_t)nl);
    lc_isect_scan_kernel<<<1, 1024, 0, st>>>(g);
    if (k64) lc_isect_write_kernel<true><<<g.nblk, 256, 0, st>>>(g);
    else lc_isect_write_kernel<false><<<g.nblk, 256, 0, st>>>(g);
    const unsigned mgrid = (unsigned)((nl + ns + kMergeTile - 1) / kMergeTile);
    if (k64) lc_merge_kernel<true><<<mgrid, 256, 0, st>>>(sL, (uint32_t)nl, sC, counts + g.nblk, d_out, d_count);
    else lc_merge_kernel<false><<<mgrid, 256, 0, st>>>(sL, (uint32_t)nl, sC, counts + g.nblk, d_out, d_count);
    lc_detail::count_launch(6);
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
    std::lock_guard<std::mutex> lk(g_pipe.mu);
    if ((st = pipe_init())) return st;
    // order the pipeline after whatever the caller queued on its stream
    cudaEventRecord(g_pipe.done, s);
    cudaStreamWaitEvent(g_pipe.h2d, g_pipe.done, 0);
    cudaStreamWaitEvent(g_pipe.d2h, g_pipe.done, 0);

    const lc_header& h = v.h;
    const uint8_t* B = (const uint8_t*)h_blob;
    const uint32_t* hint = (const uint32_t*)(B + h.off_hint);
    const uint64_t n = h.n, w = h.key_bits / 8, L = h.n_seg, b = h.res_bits;
    const uint64_t H = h.n_hint - 1;
    // spans of >= 4 Mi keys (multiples of 1024), at most kMaxSpans
    uint64_t per = (n + kMaxSpans - 1) / kMaxSpans;
    if (per < (4u << 20)) per = 4u << 20;
    per = (per + 1023) & ~1023ULL;
    uint32_t k = 0;
    for (uint64_t i0 = 0; i0 < n; i0 += per, ++k) {
        const uint64_t i1 = i0 + per < n ? i0 + per : n;
        const uint64_t c0 = i0 >> 10, c1 = (i1 + 1023) >> 10;  // chunks [c0, c1)
        const uint64_t j0 = hint[c0], j1 = hint[c1 < H ? c1 : H];
        // exactly the slices the span's kernel stages (FORMAT F2 sections, 16-byte rounded)
        const uint64_t s_lo = (j0 & ~3ULL), s_hi = ((j1 + 2 + 3) & ~3ULL) < ((L + 1 + 3) & ~3ULL)
                                                     ? ((j1 + 2 + 3) & ~3ULL)
                                                     : ((L + 1 + 3) & ~3ULL);
        const uint64_t w_lo = c0 * 32 * b, w_hi = (c1 * 32 * b + 4) < h.n_words ? c1 * 32 * b + 4
                                                                                  : h.n_words;
        if ((st = up_bytes(B, d_blob, h.off_hint + 4 * c0, h.off_hint + 4 * (c1 + 1), g_pipe.h2d)) ||
            (st = up_bytes(B, d_blob, h.off_starts + 4 * s_lo, h.off_starts + 4 * s_hi, g_pipe.h2d)) ||
            (st = up_bytes(B, d_blob, h.off_params + 16 * (j0 & ~3ULL), h.off_params + 16 * (j1 + 1),
                           g_pipe.h2d)) ||
            (b && (st = up_bytes(B, d_blob, h.off_words + 4 * w_lo, h.off_words + 4 * w_hi,
                                 g_pipe.h2d))))
            return st;
        cudaEventRecord(g_pipe.up[k], g_pipe.h2d);
        cudaStreamWaitEvent(s, g_pipe.up[k], 0);
        if ((st = launch_decode(&v, i0, i1, (uint8_t*)d_out + i0 * w, s))) return st;
        cudaEventRecord(g_pipe.dec[k], s);
        cudaStreamWaitEvent(g_pipe.d2h, g_pipe.dec[k], 0);
        if (cudaMemcpyAsync((uint8_t*)h_out + i0 * w, (uint8_t*)d_out + i0 * w, (i1 - i0) * w,
                            cudaMemcpyDeviceToHost, g_pipe.d2h) != cudaSuccess)
            return LC_ERR_CUDA;
    }
    cudaEventRecord(g_pipe.done, g_pipe.d2h);
    cudaStreamWaitEvent(s, g_pipe.done, 0);
    return cuda_status();
}

#ifdef LC_DEBUG_BOUNDS
// bounds-checked builds only: violations counted since the previous call (and reset)
uint32_t lc_debug_violations(void) {
    uint32_t v = 0, z = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&v, g_lc_violations, sizeof v);
    cudaMemcpyToSymbol(g_lc_violations, &z, sizeof z);
    return v;
}
// source line / index / limit of the last violation
void lc_debug_where(uint32_t* out3) { cudaMemcpyFromSymbol(out3, g_lc_where, 3 * sizeof(uint32_t)); }
#endif

}  // extern "C"
