// lc_setops.cuh -- successor search, intersection, union (fused into the long list's decode)
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

// Union (OR query) of a short list s and a long list l, fused into l's decode:
// no decoded copy of l and no merge pass.  Each key x of s (decoded into scratch) gets rank =
// next_geq index in l (the number of l keys below x) from l's segments (skip pointers); the
// keys absent from l are compacted in order (C, with rho_m = rank) and written straight to
// their union slot m + rho_m; then l is decoded once with every key i stored at
// i + #{m : rho_m <= i} (lc_decode_kernel<..., UNI>, Ins).
template <bool K64, bool FREE>
__global__ void __launch_bounds__(256) lc_union_rank_kernel(const IsectArgs a, uint32_t* rank) {
    __shared__ uint32_t warp_cnt[8];
    const uint32_t t = blockIdx.x * 256 + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    bool absent = false;
    if (t < a.na) {
        const uint64_t x = K64 ? ((const uint64_t*)a.a_keys)[t] : ((const uint32_t*)a.a_keys)[t];
        const SuccResult r =
            next_geq_one<FREE>(a.sb, a.nb, a.Lb, a.b, a.mask, a.bias, a.band, x, keep, once);
        absent = !(r.idx < a.nb && r.key == x);
        rank[t] = r.idx;
    }
    const uint32_t bal = __ballot_sync(kFull, absent);
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
