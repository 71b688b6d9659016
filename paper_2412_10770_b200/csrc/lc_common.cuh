// lc_common.cuh -- constants, section pointers, PTX helpers, exact prediction
// Internal part of lc_kernels.cu: included inside its anonymous namespace (one translation
// unit, so the launch tables and the bounds-check counter keep internal linkage).
#pragma once


constexpr int kWarpsPerCta = 8;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr uint32_t kSegCap = 128;  // segments per staged page (per warp)
constexpr uint32_t kFull = 0xffffffffu;

struct Sections {
    const uint32_t* starts;
    const ulonglong2* params;  // {base, slope_fx}
    const uint32_t* hint;
    const uint32_t* words;
    const uint64_t* first;  // optional successor-search index (lc_view.d_first), may be null
    // optional access layout (lc_view.d_acc, lc_access_layout_build), null when absent: per
    // 32 keys {start bitmap, rank | dist << 11}, then the segment-major records
    const uint2* dir;
    const ulonglong2* acc;
    uint32_t L;  // segments (bound of params)
    uint64_t W;  // residual words (bound of words; up to 2^32 + 4 at N = 2^32 - 1, b = 32)
};

bool is_shard(const lc_view* v) { return v->span_hi != 0; }

Sections sections_of(const lc_view* v) {
    const uint8_t* B = (const uint8_t*)v->d_blob;
    Sections s;
    if (is_shard(v)) {  // lc_shard_upload: rebased slice pointers (only the span's slices exist)
        s.starts = (const uint32_t*)(uintptr_t)v->sec_base[0];
        s.params = (const ulonglong2*)(uintptr_t)v->sec_base[1];
        s.hint = (const uint32_t*)(uintptr_t)v->sec_base[2];
        s.words = (const uint32_t*)(uintptr_t)v->sec_base[3];
    } else {
        s.starts = (const uint32_t*)(B + v->h.off_starts);
        s.params = (const ulonglong2*)(B + v->h.off_params);
        s.hint = (const uint32_t*)(B + v->h.off_hint);
        s.words = (const uint32_t*)(B + v->h.off_words);
    }
    s.first = v->d_first;
    const uint64_t H = v->h.n_hint - 1;
    const uint8_t* A = (const uint8_t*)v->d_acc;
    s.dir = A ? (const uint2*)A : nullptr;
    s.acc = A ? (const ulonglong2*)(A + 256 * H) : nullptr;
    s.L = (uint32_t)v->h.n_seg;
    s.W = v->h.n_words;
    return s;
}

// FORMAT F3 decode bias c: eps for anchored blobs, 0 for free-intercept blobs (F7)
bool is_free(const lc_view* v) { return v->h.flags & LC_FLAG_FREE_INTERCEPT; }
uint32_t bias_of(const lc_view* v) { return is_free(v) ? 0u : v->h.eps; }
uint32_t bias_of_header(const lc_header& h) { return (h.flags & LC_FLAG_FREE_INTERCEPT) ? 0u : h.eps; }

// Bounds-checked build (-DLC_DEBUG_BOUNDS, tests/test_gpu_bounds.py): every shared-memory page
// / ring-slot index and every section index is checked; a violation is counted in
// g_lc_violations (read by lc_debug_violations) and the access is clamped instead of faulting.
#ifdef LC_DEBUG_BOUNDS
__device__ uint32_t g_lc_violations;
__device__ uint32_t g_lc_where[3];  // source line, index, limit of the last violation
template <typename T>
__device__ __forceinline__ T lc_bound(bool live, T i, uint64_t n, uint32_t line) {
    if (live && (uint64_t)i >= n) {
        atomicAdd(&g_lc_violations, 1u);
        g_lc_where[0] = line;
        g_lc_where[1] = (uint32_t)i;
        g_lc_where[2] = (uint32_t)n;
        return 0;
    }
    return i;
}
#define LC_BOUND(live, i, n) lc_bound((live), (i), (n), __LINE__)
#define LC_CHECK(live, i, n) ((void)lc_bound((live), (i), (n), __LINE__))
// this translation unit's violation count since the previous call (reset), and where3 = line,
// index, limit of its last violation (each .cu file has its own counter)
uint32_t debug_take(uint32_t* where3) {
    uint32_t v = 0, z = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&v, g_lc_violations, sizeof v);
    cudaMemcpyToSymbol(g_lc_violations, &z, sizeof z);
    if (v && where3) cudaMemcpyFromSymbol(where3, g_lc_where, 3 * sizeof(uint32_t));
    return v;
}
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
__device__ __forceinline__ uint64_t ldh(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ldh(const uint2* p, uint64_t pol) {
    uint2 v;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
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

// t = floor(slope * d / 2^32) + v  (v = u - c, c the decode bias), with floor(slope * d / 2^32) =
// umulhi(slope_lo, d) + slope_hi * d exact in 32 bits because slope * d < 2^63 (FORMAT F2
// guard): mul.hi + mad.lo + add, kept as 3 ops
__device__ __forceinline__ uint32_t pred_plus(uint64_t slope, uint32_t d, uint32_t v) {
    uint32_t t;
    asm("{\n.reg .u32 h;\nmul.hi.u32 h, %1, %2;\nmad.lo.u32 h, %3, %2, h;\nadd.u32 %0, h, %4;\n}"
        : "=r"(t)
        : "r"((uint32_t)slope), "r"(d), "r"((uint32_t)(slope >> 32)), "r"(v));
    return t;
}

// ------------------------------------------------------------ shared per-key helpers
// Residual of lane's key in staged window w (lw, ls: the lane's word and bit offset in a
// window).  Widths dividing 32 never straddle a word: one load, and for b = 8 / 16 one byte
// permute (PRMT) instead of shift + mask.
template <uint32_t B>
__device__ __forceinline__ uint32_t field(const uint32_t* sW, uint32_t w, uint32_t lw, uint32_t ls) {
    if (!B) return 0;
    constexpr uint32_t mask = B >= 32 ? 0xffffffffu : ((1u << (B & 31)) - 1);
    const uint32_t* wp = sW + w * B + lw;
    if (B == 8) return __byte_perm(wp[0], 0, 0x4440 | (ls >> 3));
    if (B == 16) return __byte_perm(wp[0], 0, 0x4400 | (((ls >> 3) + 1) << 4) | (ls >> 3));
    if (32 % (B ? B : 1) == 0) return (wp[0] >> ls) & mask;
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

