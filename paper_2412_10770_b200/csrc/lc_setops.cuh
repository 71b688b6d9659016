// lc_setops.cuh -- successor search, intersection, union (fused into the long list's decode)
// Internal part of lc_kernels.cu: included inside its anonymous namespace (one translation
// unit, so the launch tables and the bounds-check counter keep internal linkage).
#pragma once

// ------------------------------------------------------ successor search and intersection
// successor-search index layout (lc_search_index_build): L first keys, padded to a 256-byte
// multiple, then ceil(L / 16) sampled first keys (one per 128-byte line of the first array)
constexpr uint32_t kIdxStride = 16;  // A/B: 8 measured 2-4% slower for next_geq
__host__ __device__ constexpr uint64_t idx_sample_off(uint64_t L) { return (L + 31) & ~31ull; }

// Key-space search uses the segments as skip pointers (Fig. 4b): segment j
// covers exactly the keys [K[s_j], K[s_{j+1}]).  With the FORMAT F2 anchor K[s_j] = base_j (one
// load per search step); F7 blobs decode K[s_j] = base_j + u(s_j).  next_geq(x) = binary search
// over the first keys, then a binary search inside the one segment, decoding only the probed
// keys (never a whole segment).

struct SuccResult {
    uint32_t idx;  // first index with K[idx] >= x, n if none
    uint64_t key;  // K[idx], 0 if none
};

// K[s_j]: base_j for anchored blobs (F2); base_j + u(s_j) for F7 blobs (bias 0, the base is
// the band floor, not a key), one more dependent load (the starts and params loads overlap)
// IDX: read it from the successor-search index (lc_search_index_build) instead
template <bool FREE, bool IDX = false>
__device__ __forceinline__ uint64_t seg_first(const Sections& sec, uint32_t j, uint32_t b,
                                              uint32_t mask, uint64_t keep, uint64_t once) {
    if (IDX) return __ldg(sec.first + LC_BOUND(true, j, sec.L));
    const uint64_t base = __ldg((const uint64_t*)sec.params + 2 * (size_t)j);
    if (!FREE) return base;
    const uint32_t s = ldh(sec.starts + j, keep);
    return base + (b ? field_of(field_words(sec, s, b, once), s, b, mask) : 0);
}

// next_geq(x) for Q independent probes per thread: a key-space binary search over the
// segments' first keys (strictly increasing in both formats), then a binary search inside the
// one segment.  For F7 blobs K[s_j] lies in [base_j, base_j + 2 eps] (the residual u <= 2 eps,
// bias 0), so a search step decodes the first key only when x falls inside that band
// (band = 2 eps).  Level-synchronous: each level issues the Q probes' loads before consuming
// any of them, so a thread can keep Q dependent chains in flight (Q = 1 by default: the
// searches are DRAM-gather bound, see kSuccQ).  Probes with live[q] false are skipped.
template <bool FREE, bool IDX, int Q>
__device__ __forceinline__ void next_geq_q(const Sections& sec, uint32_t n, uint32_t L, uint32_t b,
                                           uint32_t mask, uint32_t bias, uint64_t band,
                                           const uint64_t (&x)[Q], const bool (&live)[Q],
                                           SuccResult (&res)[Q], uint64_t keep, uint64_t once,
                                           uint64_t spol) {
    const uint64_t k0 = seg_first<FREE, IDX>(sec, 0, b, mask, keep, once);
    bool go[Q];
    uint32_t lo[Q], hi[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        go[q] = live[q] && x[q] > k0;
        lo[q] = 0;
        hi[q] = go[q] ? L - 1 : 0;
    }
    // 1. j = max{t : K[s_t] <= x} over the segments' first keys.  With the index: first over
    // its sample (every 16th first key, L2-resident), then inside one 128-byte line of it
    if (IDX) {
        const uint32_t S = (L + kIdxStride - 1) / kIdxStride;
        const uint64_t* sample = sec.first + idx_sample_off(L);
#pragma unroll
        for (int q = 0; q < Q; ++q) hi[q] = go[q] ? S - 1 : 0;
        for (;;) {
            bool act[Q], any = false;
            uint32_t mid[Q];
            uint64_t v[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                act[q] = lo[q] < hi[q];
                any |= act[q];
                mid[q] = (lo[q] + hi[q] + 1) >> 1;
                v[q] = act[q] ? ldh(sample + LC_BOUND(true, mid[q], S), keep) : 0;
            }
            if (!any) break;
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (act[q]) {
                    if (v[q] <= x[q]) lo[q] = mid[q];
                    else hi[q] = mid[q] - 1;
                }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            lo[q] *= kIdxStride;
            hi[q] = go[q] ? min(lo[q] + kIdxStride - 1, L - 1) : lo[q];
        }
    }
    for (;;) {
        bool act[Q], any = false;
        uint32_t mid[Q];
        uint64_t v[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            act[q] = lo[q] < hi[q];
            any |= act[q];
            mid[q] = (lo[q] + hi[q] + 1) >> 1;
            if (IDX) v[q] = act[q] ? __ldg(sec.first + LC_BOUND(true, mid[q], sec.L)) : 0;
            else v[q] = act[q] ? __ldg((const uint64_t*)sec.params + 2 * (size_t)mid[q]) : 0;
        }
        if (!any) break;
        if (FREE && !IDX) {  // first key = base + u(s) only matters when x lies in [base, base + 2 eps)
            bool nd[Q];
            uint32_t sm[Q];
            uint2 w[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                nd[q] = act[q] && v[q] <= x[q] && x[q] - v[q] < band;
                sm[q] = nd[q] ? ldh(sec.starts + mid[q], keep) : 0;
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) w[q] = nd[q] && b ? field_words(sec, sm[q], b, once) : make_uint2(0, 0);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (nd[q]) v[q] += b ? field_of(w[q], sm[q], b, mask) : 0;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (act[q]) {
                if (v[q] <= x[q]) lo[q] = mid[q];
                else hi[q] = mid[q] - 1;
            }
    }
    // 2. inside segment j: first index in (s_j, s_{j+1}] with K >= x (K[s_j] <= x)
    uint32_t s[Q], e[Q], l[Q], r[Q];
    ulonglong2 pr[Q];
    uint64_t ks[Q], kr[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        s[q] = go[q] ? ldh(sec.starts + lo[q], spol) : 0;
        e[q] = go[q] ? ldh(sec.starts + lo[q] + 1, spol) : 0;
        pr[q] = go[q] ? ldh(sec.params + lo[q], once) : make_ulonglong2(0, 0);
    }
    if (IDX) {
#pragma unroll
        for (int q = 0; q < Q; ++q) ks[q] = go[q] ? __ldg(sec.first + lo[q]) : 0;
    } else if (FREE) {
        uint2 w[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) w[q] = go[q] && b ? field_words(sec, s[q], b, once) : make_uint2(0, 0);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            ks[q] = pr[q].x + pred_plus(pr[q].y, 0, (b ? field_of(w[q], s[q], b, mask) : 0) - bias);
    } else {
#pragma unroll
        for (int q = 0; q < Q; ++q) ks[q] = pr[q].x;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        l[q] = s[q] + 1;
        r[q] = go[q] && ks[q] != x[q] ? e[q] : l[q];  // no search when K[s_j] == x
        kr[q] = 0;
    }
    for (;;) {
        bool act[Q], any = false;
        uint32_t mid[Q];
        uint2 w[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            act[q] = l[q] < r[q];
            any |= act[q];
            mid[q] = (l[q] + r[q]) >> 1;
            w[q] = act[q] && b ? field_words(sec, mid[q], b, once) : make_uint2(0, 0);
        }
        if (!any) break;
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (act[q]) {
                const uint32_t u = b ? field_of(w[q], mid[q], b, mask) : 0;
                const uint64_t km = pr[q].x + pred_plus(pr[q].y, mid[q] - s[q], u - bias);
                if (km >= x[q]) {
                    r[q] = mid[q];
                    kr[q] = km;  // = K[r]: at the end l == r, so K[l] when l < e
                } else {
                    l[q] = mid[q] + 1;
                }
            }
    }
    // 3. results; x in the gap after segment j's last key: K[e] = first key of segment j + 1
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (!live[q]) continue;
        if (!go[q]) res[q] = {0u, k0};
        else if (ks[q] == x[q]) res[q] = {s[q], x[q]};
        else if (l[q] < e[q]) res[q] = {l[q], kr[q]};
        else if (e[q] >= n) res[q] = {n, 0};
        else res[q] = {e[q], seg_first<FREE, IDX>(sec, lo[q] + 1, b, mask, keep, once)};
    }
}

struct SuccArgs {
    Sections sec;
    const uint64_t* x;
    uint64_t* out_idx;
    void* out_key;
    uint64_t m;
    uint64_t band;  // 2 eps (F7 first-key band)
    uint32_t n, L, b, bias, mask;
};

// Probes per thread.  A/B on B200 (config 5, tools/prof_setops.py; Q = 1 / 2 / 4):
// next_geq 1e7 random probes 0.974 / 1.05 / 1.16 ms, intersect 1e6 x 1e8 0.106 / 0.105 /
// 0.119 ms, union 0.367 / 0.366 / 0.382 ms.  More chains per thread do not help: both run at
// ~2.7e11 probe loads/s whatever Q (a cache request-rate limit, not chain latency), and
// Q = 4 needs 80 registers.  Compile-time knobs for such A/B builds.
#ifndef LC_NEXT_GEQ_Q
#define LC_NEXT_GEQ_Q 1
#endif
#ifndef LC_ISECT_Q
#define LC_ISECT_Q 1
#endif
constexpr int kSuccQ = LC_NEXT_GEQ_Q;   // lc_next_geq (random probes)
constexpr int kIsectQ = LC_ISECT_Q;     // intersect / union ranks (sorted probes)

// CTA c, thread t handles probes c * 256 Q + 256 q + t (q < Q): coalesced per q
template <bool K64, bool FREE, bool IDX>
__global__ void __launch_bounds__(256) lc_next_geq_kernel(const SuccArgs a) {
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    const uint64_t t0 = (uint64_t)blockIdx.x * 256 * kSuccQ + threadIdx.x;
    uint64_t x[kSuccQ];
    bool live[kSuccQ];
    SuccResult r[kSuccQ];
#pragma unroll
    for (int q = 0; q < kSuccQ; ++q) {
        const uint64_t t = t0 + 256 * q;
        x[q] = t < a.m ? __ldg(a.x + t) : 0;
        live[q] = t < a.m && (K64 || x[q] <= 0xffffffffull);
        r[q] = {a.n, 0};
    }
    next_geq_q<FREE, IDX, kSuccQ>(a.sec, a.n, a.L, a.b, a.mask, a.bias, a.band, x, live, r, keep, once,
                                  keep);
#pragma unroll
    for (int q = 0; q < kSuccQ; ++q) {
        const uint64_t t = t0 + 256 * q;
        if (t >= a.m) continue;
        if (a.out_idx) a.out_idx[t] = r[q].idx;
        if (a.out_key) put<K64>((uint8_t*)a.out_key + t * (K64 ? 8 : 4), r[q].key, 0);
    }
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
    uint64_t band;          // 2 eps of list B (F7 first-key band)
    uint32_t na, nb, Lb, b, bias, mask, nblk;
};

// Probe flags of the searched list a against list b, Q probes per thread: CTA c covers the
// 256-probe groups c Q .. c Q + Q - 1 (thread t: probe 256 (c Q + q) + t), so flags words and
// per-group counts keep the layout the scan / write kernels expect (one count per 256 probes).
// HIT = true: flag keys found in b (intersect); false: flag keys absent from b and store
// rank[t] = their next_geq index (union).
template <bool K64, bool FREE, bool IDX, bool HIT>
__device__ __forceinline__ void flag_probes(const IsectArgs& a, uint32_t* rank) {
    __shared__ uint32_t warp_cnt[kIsectQ][8];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    uint64_t x[kIsectQ];
    bool live[kIsectQ];
    SuccResult r[kIsectQ];
#pragma unroll
    for (int q = 0; q < kIsectQ; ++q) {
        const uint32_t t = (blockIdx.x * kIsectQ + q) * 256 + threadIdx.x;
        live[q] = t < a.na;
        x[q] = live[q] ? (K64 ? ((const uint64_t*)a.a_keys)[t] : ((const uint32_t*)a.a_keys)[t]) : 0;
        r[q] = {a.nb, 0};
    }
    // sorted probes: with the index, the segment's starts pair is a one-touch gather
    // (evict_first: intersect 0.097 -> 0.086 ms on config 5; random next_geq prefers evict_last)
    next_geq_q<FREE, IDX, kIsectQ>(a.sb, a.nb, a.Lb, a.b, a.mask, a.bias, a.band, x, live, r, keep,
                                   once, IDX ? once : keep);
#pragma unroll
    for (int q = 0; q < kIsectQ; ++q) {
        const uint32_t g = blockIdx.x * kIsectQ + q, t = g * 256 + threadIdx.x;
        const bool found = live[q] && r[q].idx < a.nb && r[q].key == x[q];
        const bool flag = HIT ? found : live[q] && !found;
        if (!HIT && live[q]) rank[t] = r[q].idx;
        const uint32_t bal = __ballot_sync(kFull, flag);
        if (lane == 0) {
            if (t < a.na) a.flags[t >> 5] = bal;
            warp_cnt[q][warp] = __popc(bal);
        }
    }
    __syncthreads();
    if (threadIdx.x < kIsectQ) {
        const uint32_t g = blockIdx.x * kIsectQ + threadIdx.x;
        uint32_t c = 0;
        for (int w = 0; w < 8; ++w) c += warp_cnt[threadIdx.x][w];
        if (g < a.nblk) a.counts[g] = c;
    }
}

template <bool K64, bool FREE, bool IDX>
__global__ void __launch_bounds__(256) lc_isect_flag_kernel(const IsectArgs a) {
    flag_probes<K64, FREE, IDX, true>(a, nullptr);
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

// Union (OR query) of a short list s and a long list l, fused into l's decode:
// no decoded copy of l and no merge pass.  Each key x of s (decoded into scratch) gets rank =
// next_geq index in l (the number of l keys below x) from l's segments (skip pointers); the
// keys absent from l are compacted in order (C, with rho_m = rank) and written straight to
// their union slot m + rho_m; then l is decoded once with every key i stored at
// i + #{m : rho_m <= i} (lc_decode_kernel<..., UNI>, Ins).
template <bool K64, bool FREE, bool IDX>
__global__ void __launch_bounds__(256) lc_union_rank_kernel(const IsectArgs a, uint32_t* rank) {
    flag_probes<K64, FREE, IDX, false>(a, rank);
}

// successor-search index: first[j] = K[s_j] = base_j + u(s_j) - c (FORMAT F3 at d = 0) for
// j < L, then (from idx_sample_off(L)) the sample first[kIdxStride * k]
template <bool FREE>
__global__ void __launch_bounds__(256) lc_first_kernel(const Sections sec, uint64_t* first,
                                                       uint32_t b, uint32_t mask, uint32_t bias) {
    const uint32_t j = blockIdx.x * 256 + threadIdx.x;
    if (j >= sec.L) return;
    uint64_t k = __ldg((const uint64_t*)sec.params + 2 * (size_t)j);
    if (FREE) {  // F2 anchor: u(s_j) = eps = c, so K[s_j] = base_j; F7: base_j + u(s_j)
        const uint32_t s = __ldg(sec.starts + j);
        const uint64_t pol = policy_evict_first();
        const uint32_t u = b ? field_of(field_words(sec, s, b, pol), s, b, mask) : 0;
        k += (uint32_t)(u - bias);
    }
    first[j] = k;
    if (j % kIdxStride == 0) first[idx_sample_off(sec.L) + j / kIdxStride] = k;
}

// absent key t of s -> C position m (flags + scanned counts, as lc_isect_write_kernel):
// rho[m] = rank[t], out[m + rank[t]] = key
template <bool K64>
__global__ void __launch_bounds__(256) lc_union_place_kernel(const IsectArgs a,
                                                             const uint32_t* rank, uint32_t* rho) {
    __shared__ uint32_t warp_off[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bal = t < a.na ? a.flags[t >> 5] : 0;
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
        const uint32_t m = warp_off[warp] + __popc(bal & ((1u << lane) - 1));
        const uint32_t r = rank[t];
        rho[m] = r;
        const size_t slot = (size_t)m + r;
        if (K64) ((uint64_t*)a.out)[slot] = ((const uint64_t*)a.a_keys)[t];
        else ((uint32_t*)a.out)[slot] = ((const uint32_t*)a.a_keys)[t];
    }
}

// coff[h] = #{m : rho_m < 1024 h} for h = 0..H (chunk insertion offsets); *d_count = nl + |C|
__global__ void __launch_bounds__(256) lc_union_coff_kernel(const uint32_t* rho,
                                                            const uint32_t* nc_ptr, uint32_t H,
                                                            uint32_t* coff, uint64_t nl,
                                                            uint64_t* d_count) {
    const uint32_t h = blockIdx.x * 256 + threadIdx.x;
    const uint32_t nc = *nc_ptr;
    if (h == 0) *d_count = nl + nc;
    if (h > H) return;
    const uint64_t x = (uint64_t)h << 10;
    uint32_t lo = 0, hi = nc;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(rho + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    coff[h] = lo;
}
