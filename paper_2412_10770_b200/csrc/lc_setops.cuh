// lc_setops.cuh -- successor search, intersection, union (merge path)
// Internal part of lc_kernels.cu: included inside its anonymous namespace (one translation
// unit, so the launch tables and the bounds-check counter keep internal linkage).
#pragma once

// ------------------------------------------------------ successor search and intersection
// Key-space search uses the segments as skip pointers (Fig. 4b): segment j
// covers exactly the keys [K[s_j], K[s_{j+1}]).  With the FORMAT F2 anchor K[s_j] = base_j (one
// load per search step); F7 blobs decode K[s_j] = base_j + u(s_j).  next_geq(x) = binary search
// over the first keys, then a binary search inside the one segment, decoding only the probed
// keys (never a whole segment).
__device__ __forceinline__ uint64_t key_at(const Sections& sec, uint32_t i, uint32_t s,
                                           ulonglong2 pr, uint32_t b, uint32_t mask, uint32_t bias,
                                           uint64_t once) {
    const uint32_t u = b ? field_of(field_words(sec, i, b, once), i, b, mask) : 0;
    return pr.x + pred_plus(pr.y, i - s, u - bias);
}

struct SuccResult {
    uint32_t idx;  // first index with K[idx] >= x, n if none
    uint64_t key;  // K[idx], 0 if none
};

// K[s_j]: base_j for anchored blobs (F2); base_j + u(s_j) for F7 blobs (bias 0, the base is
// the band floor, not a key), one more dependent load (the starts and params loads overlap)
template <bool FREE>
__device__ __forceinline__ uint64_t seg_first(const Sections& sec, uint32_t j, uint32_t b,
                                              uint32_t mask, uint64_t keep, uint64_t once) {
    const uint64_t base = __ldg((const uint64_t*)sec.params + 2 * (size_t)j);
    if (!FREE) return base;
    const uint32_t s = ldh(sec.starts + j, keep);
    return base + (b ? field_of(field_words(sec, s, b, once), s, b, mask) : 0);
}

// Key-space search over the segments' first keys (strictly increasing in both formats), then
// a binary search inside the one segment.
// For F7 blobs K[s_j] lies in [base_j, base_j + 2 eps] (the residual u <= 2 eps, bias 0), so
// a search step decodes the first key only when x falls inside that band (band = 2 eps).
template <bool FREE>
__device__ SuccResult next_geq_one(const Sections& sec, uint32_t n, uint32_t L, uint32_t b,
                                   uint32_t mask, uint32_t bias, uint64_t band, uint64_t x,
                                   uint64_t keep, uint64_t once) {
    const uint64_t k0 = seg_first<FREE>(sec, 0, b, mask, keep, once);
    if (x <= k0) return {0u, k0};
    uint32_t lo = 0, hi = L - 1;  // max{j : K[s_j] <= x}
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        bool le;
        if (FREE) {
            const uint64_t base = __ldg((const uint64_t*)sec.params + 2 * (size_t)mid);
            if (base > x) le = false;
            else if (x - base >= band) le = true;
            else le = seg_first<FREE>(sec, mid, b, mask, keep, once) <= x;
        } else {
            le = seg_first<FREE>(sec, mid, b, mask, keep, once) <= x;
        }
        if (le) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t j = lo;
    const uint32_t s = ldh(sec.starts + j, keep), e = ldh(sec.starts + j + 1, keep);
    const ulonglong2 pr = ldh(sec.params + j, once);
    uint32_t l = s + 1, r = e;  // K[s] <= x; answer in (s, e]
    if ((FREE ? key_at(sec, s, s, pr, b, mask, bias, once) : pr.x) == x) return {s, x};
    uint64_t kr = 0;
    bool have = false;
    while (l < r) {
        const uint32_t mid = (l + r) >> 1;
        const uint64_t km = key_at(sec, mid, s, pr, b, mask, bias, once);
        if (km >= x) {
            r = mid;
            kr = km;
            have = true;
        } else {
            l = mid + 1;
        }
    }
    if (l < e) {
        if (!have || r != l) kr = key_at(sec, l, s, pr, b, mask, bias, once);
        return {l, kr};
    }
    if (e >= n) return {n, 0};
    return {e, seg_first<FREE>(sec, j + 1, b, mask, keep, once)};  // K[e] = K[s_{j+1}] > x
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

template <bool K64, bool FREE>
__global__ void __launch_bounds__(256) lc_next_geq_kernel(const SuccArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= a.m) return;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    const uint64_t x = __ldg(a.x + t);
    SuccResult r;
    if (!K64 && x > 0xffffffffull) r = {a.n, 0};
    else r = next_geq_one<FREE>(a.sec, a.n, a.L, a.b, a.mask, a.bias, a.band, x, keep, once);
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
    uint64_t band;          // 2 eps of list B (F7 first-key band)
    uint32_t na, nb, Lb, b, bias, mask, nblk;
};

template <bool K64, bool FREE>
__global__ void __launch_bounds__(256) lc_isect_flag_kernel(const IsectArgs a) {
    __shared__ uint32_t warp_cnt[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    bool hit = false;
    if (t < a.na) {
        const uint64_t x = K64 ? ((const uint64_t*)a.a_keys)[t] : ((const uint32_t*)a.a_keys)[t];
        const SuccResult r =
            next_geq_one<FREE>(a.sb, a.nb, a.Lb, a.b, a.mask, a.bias, a.band, x, keep, once);
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

