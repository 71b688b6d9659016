// lc_batchops.cuh -- AND / OR of many list pairs of a batch in a fixed number of launches
// Internal part of lc_kernels.cu: included inside its anonymous namespace.
//
// The paper's inverted-index queries (§III-A, Fig. 4) over a batch of posting
// lists (lc_batch_init): for each pair p of lists, the shorter s_p and the longer l_p.
//  * AND: s_p's keys are decoded (one batch decode of a selection of chunk records), each is
//    searched in the COMPRESSED l_p with next_geq (segments as skip pointers: segments of l_p
//    holding no key of s_p are never read), matches flagged, counted, scanned and written
//    packed; pair p's result is out[out_off[p] .. out_off[p + 1]).
//  * OR: both lists are decoded into scratch; every key gets its union slot from ranks:
//    slot(x in s, index i) = i + #{l < x} - #{matched s keys before i} and
//    slot(y in l, index j) = j + #{s < y} - #{matched s keys below y} (a key present in both
//    lists gets the same slot from both sides), so no merge pass runs; pair p's result is
//    out[out_off[p] .. out_off[p] + count[p]) with out_off[p] = sum over earlier pairs of
//    n_s + n_l (capacity).

struct SetopArgs {
    const BatchList* lists;
    const uint32_t* sl;       // [2 p] short list, [2 p + 1] long list
    const uint64_t* s_off;    // P + 1: short keys of pair p at keys_s[s_off[p] .. s_off[p + 1])
    const uint64_t* l_off;    // P + 1: long keys of pair p at keys_l[l_off[p] ..) (OR)
    const uint64_t* cap_off;  // P + 1: OR output capacity offsets
    const void* keys_s;
    const void* keys_l;
    uint32_t* flags;          // match bit per short key (ceil(S / 32) + 1 words, zeroed)
    uint32_t* counts;         // matches per 256 short keys, then exclusive offsets; [nblk] total
    uint32_t* mw;             // matches before each flags word
    uint32_t* rank;           // OR: #{l < x} per short key
    uint64_t* total;          // scan total (device scalar)
    void* out;
    uint64_t* d_out_off;      // P + 1 result offsets
    uint64_t* d_counts;       // P result sizes
    const uint32_t* blk_s;    // pair holding short key 1024 g (or the pair before it)
    const uint32_t* blk_l;    // pair holding long key 1024 g (OR)
    uint64_t S, Lt;
    uint32_t P, nblk, nwords;
};

template <bool K64>
__device__ __forceinline__ uint64_t key_at(const void* base, uint64_t i) {
    return K64 ? __ldg((const uint64_t*)base + i) : (uint64_t)__ldg((const uint32_t*)base + i);
}

// pair of element g: max{p : off[p] <= g} over the P + 1 offsets (off[0] = 0), from the pair
// recorded for g's 1024-element block (blk[g / 1024] <= the answer) and a short forward walk
__device__ __forceinline__ uint32_t pair_of(const uint32_t* blk, const uint64_t* off, uint64_t g) {
    uint32_t p = __ldg(blk + (g >> 10));
    while (__ldg(off + p + 1) <= g) ++p;
    return p;
}

// #{t < n : keys[t] < x} over decoded keys
template <bool K64>
__device__ __forceinline__ uint64_t lower_bound_keys(const void* keys, uint64_t lo, uint64_t n,
                                                     uint64_t x) {
    uint64_t l = 0, r = n;
    while (l < r) {
        const uint64_t mid = (l + r) >> 1;
        if (key_at<K64>(keys, lo + mid) < x) l = mid + 1;
        else r = mid;
    }
    return l;
}

// matches among short keys [0, g)
__device__ __forceinline__ uint64_t matches_before(const SetopArgs& a, uint64_t g) {
    const uint32_t w = (uint32_t)(g >> 5);
    return __ldg(a.mw + w) + __popc(__ldg(a.flags + w) & ((1u << (g & 31)) - 1));
}

__device__ __forceinline__ Sections list_sections(const BatchList& e) {
    const uint8_t* B = (const uint8_t*)e.blob;
    Sections s;
    s.starts = (const uint32_t*)(B + 256);
    s.params = (const ulonglong2*)(B + e.off_params);
    s.hint = (const uint32_t*)(B + e.off_hint);
    s.words = (const uint32_t*)(B + e.off_words);
    s.first = nullptr;
    s.dir = nullptr;
    s.acc = nullptr;
    s.L = e.L;
    s.W = 0;
    return s;
}

// one thread per short key: found in its pair's long list?  AND searches the compressed list
// (next_geq), OR the decoded one (and keeps the rank)
template <bool K64, bool OR>
__global__ void __launch_bounds__(256) lc_bprobe_kernel(const SetopArgs a) {
    __shared__ uint32_t warp_cnt[8];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t g = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    const bool live = g < a.S;
    bool found = false;
    if (live) {
        const uint64_t x = key_at<K64>(a.keys_s, g);
        const uint32_t p = pair_of(a.blk_s, a.s_off, g);
        if (OR) {
            const uint64_t lo = __ldg(a.l_off + p), nl = __ldg(a.l_off + p + 1) - lo;
            const uint64_t r = lower_bound_keys<K64>(a.keys_l, lo, nl, x);
            found = r < nl && key_at<K64>(a.keys_l, lo + r) == x;
            a.rank[g] = (uint32_t)r;
        } else {
            const BatchList e = a.lists[__ldg(a.sl + 2 * p + 1)];
            const Sections sec = list_sections(e);
            const uint64_t keep = policy_evict_last(), once = policy_evict_first();
            const uint64_t xs[1] = {x};
            const bool lv[1] = {true};
            SuccResult r[1] = {{e.n, 0}};
            const uint32_t mask = e.b >= 32 ? kFull : (1u << e.b) - 1;
            if (e.flags & LC_FLAG_FREE_INTERCEPT)
                next_geq_q<true, false, 1>(sec, e.n, e.L, e.b, mask, e.bias, 2 * (uint64_t)e.eps,
                                           xs, lv, r, keep, once, once);
            else
                next_geq_q<false, false, 1>(sec, e.n, e.L, e.b, mask, e.bias, 2 * (uint64_t)e.eps,
                                            xs, lv, r, keep, once, once);
            found = r[0].idx < e.n && r[0].key == x;
        }
    }
    const uint32_t bal = __ballot_sync(kFull, found);
    if (lane == 0) {
        if (g < a.S) a.flags[g >> 5] = bal;
        warp_cnt[warp] = __popc(bal);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (int w = 0; w < 8; ++w) c += warp_cnt[w];
        a.counts[blockIdx.x] = c;
    }
}

// mw[w] = matches before flags word w (counts hold the exclusive per-256 offsets)
__global__ void __launch_bounds__(256) lc_bmw_kernel(const SetopArgs a) {
    const uint32_t w = blockIdx.x * 256 + threadIdx.x;
    if (w >= a.nwords) return;
    uint32_t m = a.counts[min(w >> 3, a.nblk)];
    for (uint32_t v = w & ~7u; v < w; ++v) m += __popc(a.flags[v]);
    a.mw[w] = m;
}

// AND: matched short keys to their packed slot; OR: unmatched short keys to their union slot
template <bool K64, bool OR>
__global__ void __launch_bounds__(256) lc_bwrite_s_kernel(const SetopArgs a) {
    const uint64_t g = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (g >= a.S) return;
    const bool found = (__ldg(a.flags + (g >> 5)) >> (g & 31)) & 1;
    if (found == OR) return;
    const uint64_t x = key_at<K64>(a.keys_s, g);
    uint64_t pos;
    if (!OR) {
        pos = matches_before(a, g);
    } else {
        const uint32_t p = pair_of(a.blk_s, a.s_off, g);
        const uint64_t s0 = __ldg(a.s_off + p);
        pos = __ldg(a.cap_off + p) + (g - s0) + __ldg(a.rank + g) -
              (matches_before(a, g) - matches_before(a, s0));
    }
    if (K64) ((uint64_t*)a.out)[pos] = x;
    else ((uint32_t*)a.out)[pos] = (uint32_t)x;
}

// OR: every long key to its union slot
constexpr uint32_t kWlKeys = 512;  // long keys per warp in lc_bwrite_l_kernel (16 per lane; A/B on the corpus OR: 256 1.10 ms, 512 1.04, 1024 1.03, 2048 1.06)
template <bool K64>
__global__ void __launch_bounds__(256) lc_bwrite_l_kernel(const SetopArgs a) {
    // A warp places 256 consecutive long keys.  They usually belong to one pair and share one
    // rank in its (much shorter) short list: the ranks of the range's first and last keys are
    // searched once per warp, and a key only searches when they differ (between them).
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t g0 = ((uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * kWlKeys;
    if (g0 >= a.Lt) return;
    const uint64_t g1 = min(g0 + kWlKeys, a.Lt) - 1;  // last key of the warp's range
    const uint32_t pa = pair_of(a.blk_l, a.l_off, g0), pb = pair_of(a.blk_l, a.l_off, g1);
    if (pa == pb) {
        const uint64_t s0 = __ldg(a.s_off + pa), ns = __ldg(a.s_off + pa + 1) - s0;
        uint64_t r = 0;
        if (lane < 2) r = lower_bound_keys<K64>(a.keys_s, s0, ns, key_at<K64>(a.keys_l, lane ? g1 : g0));
        const uint64_t r0 = __shfl_sync(kFull, r, 0), r1 = __shfl_sync(kFull, r, 1);
        const uint64_t m0 = matches_before(a, s0);
        const uint64_t base = __ldg(a.cap_off + pa) - __ldg(a.l_off + pa) + m0;  // + gl + ra - M(s0 + ra)
        const uint64_t c0 = base + r0 - matches_before(a, s0 + r0);
#pragma unroll 4
        for (uint32_t q = 0; q < kWlKeys / 32; ++q) {
            const uint64_t gl = g0 + 32 * q + lane;
            if (gl > g1) break;
            const uint64_t y = key_at<K64>(a.keys_l, gl);
            uint64_t pos;
            if (r0 == r1) {
                pos = c0 + gl;
            } else {  // a short key falls inside the range: rank between r0 and r1
                uint64_t l = r0, h = r1;
                while (l < h) {
                    const uint64_t mid = (l + h) >> 1;
                    if (key_at<K64>(a.keys_s, s0 + mid) < y) l = mid + 1;
                    else h = mid;
                }
                pos = base + gl + l - matches_before(a, s0 + l);
            }
            if (K64) ((uint64_t*)a.out)[pos] = y;
            else ((uint32_t*)a.out)[pos] = (uint32_t)y;
        }
        return;
    }
    // the range spans pairs: every key on its own
    for (uint32_t q = 0; q < kWlKeys / 32; ++q) {
        const uint64_t gl = g0 + 32 * q + lane;
        if (gl > g1) break;
        const uint32_t p = pair_of(a.blk_l, a.l_off, gl);
        const uint64_t y = key_at<K64>(a.keys_l, gl);
        const uint64_t s0 = __ldg(a.s_off + p), ns = __ldg(a.s_off + p + 1) - s0;
        const uint64_t ra = lower_bound_keys<K64>(a.keys_s, s0, ns, y);
        const uint64_t pos = __ldg(a.cap_off + p) + (gl - __ldg(a.l_off + p)) + ra -
                             (matches_before(a, s0 + ra) - matches_before(a, s0));
        if (K64) ((uint64_t*)a.out)[pos] = y;
        else ((uint32_t*)a.out)[pos] = (uint32_t)y;
    }
}

// per pair: result offset and size
template <bool OR>
__global__ void __launch_bounds__(256) lc_bpairs_kernel(const SetopArgs a) {
    const uint32_t p = blockIdx.x * 256 + threadIdx.x;
    if (p > a.P) return;
    const uint64_t m0 = matches_before(a, __ldg(a.s_off + p));
    a.d_out_off[p] = OR ? __ldg(a.cap_off + p) : m0;
    if (p == a.P) return;
    const uint64_t m1 = matches_before(a, __ldg(a.s_off + p + 1));
    a.d_counts[p] = OR ? (__ldg(a.s_off + p + 1) - __ldg(a.s_off + p)) +
                             (__ldg(a.l_off + p + 1) - __ldg(a.l_off + p)) - (m1 - m0)
                       : m1 - m0;
}

// ---- device-side plan (no host pass over the batch, no upload): per pair the short / long
// list, then exclusive scans of the key and unit counts, then the chunk records to decode
struct PlanArgs {
    const BatchList* lists;
    const uint32_t* pairs;  // 2 P list indices (device)
    uint32_t* sl;           // [2 p] short, [2 p + 1] long
    uint64_t* s_off;        // P + 1 (counts, then exclusive offsets; [P] = total)
    uint64_t* l_off;
    uint64_t* cap_off;
    uint64_t* u_off;
    uint32_t* sel;          // U chunk-record indices ...
    uint64_t* sel_out;      // ... and output element offsets (short keys, then S + long keys)
    uint32_t* blk_s;        // pair of short key 1024 g, for g < ceil(S / 1024)
    uint32_t* blk_l;        // pair of long key 1024 g (OR)
    uint32_t* err;          // bit 0: a pair index >= m
    uint64_t U, S;          // the host plan's totals (capacities)
    uint32_t P, m, n_chunks, OR;
};

__device__ __forceinline__ uint32_t list_chunks(uint32_t n) { return (n + 1023) >> 10; }

__global__ void __launch_bounds__(256) lc_bplan_kernel(const PlanArgs a) {
    const uint32_t p = blockIdx.x * 256 + threadIdx.x;
    if (p >= a.P) return;
    uint32_t x = __ldg(a.pairs + 2 * p), y = __ldg(a.pairs + 2 * p + 1);
    if (x >= a.m || y >= a.m) {
        atomicOr(a.err, 1u);
        x = min(x, a.m - 1);
        y = min(y, a.m - 1);
    }
    const uint32_t nx = a.lists[x].n, ny = a.lists[y].n;
    const uint32_t sh = nx <= ny ? x : y, lg = nx <= ny ? y : x;
    const uint32_t ns = min(nx, ny), nl = max(nx, ny);
    a.sl[2 * p] = sh;
    a.sl[2 * p + 1] = lg;
    a.s_off[p] = ns;
    a.l_off[p] = a.OR ? nl : 0;
    a.cap_off[p] = ns + (a.OR ? nl : 0);
    a.u_off[p] = list_chunks(ns) + (a.OR ? list_chunks(nl) : 0);
}

// exclusive scans of the four count arrays in one CTA ([P] receives the total)
__global__ void __launch_bounds__(1024) lc_bscan_kernel(const PlanArgs a) {
    __shared__ uint64_t part[32];
    uint64_t* arr[4] = {a.s_off, a.l_off, a.cap_off, a.u_off};
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = (a.P + 1023) / 1024, lo = threadIdx.x * per, hi = min(lo + per, a.P);
    for (int k = 0; k < 4; ++k) {
        uint64_t* v = arr[k];
        uint64_t sum = 0;
        for (uint32_t i = lo; i < hi; ++i) sum += v[i];
        uint64_t x = sum;  // inclusive scan of the thread sums
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) part[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint64_t q = part[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(kFull, q, o);
                if (lane >= (uint32_t)o) q += y;
            }
            part[lane] = q;
        }
        __syncthreads();
        uint64_t run = (warp ? part[warp - 1] : 0) + x - sum;
        for (uint32_t i = lo; i < hi; ++i) {
            const uint64_t c = v[i];
            v[i] = run;
            run += c;
        }
        if (threadIdx.x == 1023) v[a.P] = run;
        __syncthreads();
    }
}

// the chunk records of pair p's short list (and long list for OR), in key order
__global__ void __launch_bounds__(256) lc_bexpand_kernel(const PlanArgs a) {
    const uint32_t p = blockIdx.x * 256 + threadIdx.x;
    if (p >= a.P) return;
    // block tables: every 1024-key block starting inside this pair's keys names it
    for (uint64_t g = (a.s_off[p] + 1023) >> 10; (g << 10) < a.s_off[p + 1]; ++g) a.blk_s[g] = p;
    if (p == 0) a.blk_s[0] = 0;
    if (a.OR) {
        for (uint64_t g = (a.l_off[p] + 1023) >> 10; (g << 10) < a.l_off[p + 1]; ++g) a.blk_l[g] = p;
        if (p == 0) a.blk_l[0] = 0;
    }
    uint64_t u = a.u_off[p];
    for (int side = 0; side < (a.OR ? 2 : 1); ++side) {
        const BatchList e = a.lists[a.sl[2 * p + side]];
        const uint32_t H = list_chunks(e.n);
        const bool small = e.pad[0] != 0xffffffffu;
        const uint64_t dst = side ? a.S + a.l_off[p] : a.s_off[p];
        for (uint32_t q = 0; q < H && u < a.U; ++q, ++u) {
            a.sel[u] = small && q == H - 1 ? e.pad[0] : e.chunk0 + q;
            a.sel_out[u] = dst + ((uint64_t)q << 10);
        }
    }
}
