// lc_gather.cuh -- range decode (generic + cp.async ring for 64 keys), access, quantiles
// Internal part of lc_kernels.cu: included inside its anonymous namespace (one translation
// unit, so the launch tables and the bounds-check counter keep internal linkage).
#pragma once

// -------------------------------------------------------------------------- range decode
struct RangeArgs {
    Sections sec;
    const uint64_t* start;
    void* out;
    uint32_t* err;
    uint64_t q;
    uint32_t len, n, L, b, bias, mask;
    uint64_t nwords;  // W
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
    uint64_t wi = bit >> 5;
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
    const uint32_t len = a.len, b = a.b, mask = a.mask, L = a.L, bias = a.bias;
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
            put<K64>(outk + lane * kw, pA.x, pred_plus(pA.y, dA, uA - bias));
            put<K64>(outk + (32 + lane) * kw, pB.x, pred_plus(pB.y, dB, uB - bias));
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
                put<K64>(outk + (w0 + lane) * kw, pr.x, pred_plus(pr.y, d, u - bias));
            }
            jb += adv;
            sb = ldh(sec.starts + min(jb, L), keep);
            w0 += 32;
        }
    }
}

// ---------------------------------------------------------------- range decode, len <= 64
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

// Ranges of up to 64 keys (written for the 64 of BASELINE config 5; shorter ones mask the
// tail).  Phase 1: lane r binary-searches range r's first segment
// (32 independent searches) and parks {start, segment, segment start, first word} in shared
// memory.  Phase 2: the warp walks its 32 ranges through a 4-slot shared-memory ring: lane g
// gathers 16-byte group g of range k+3's slot (params[j..j+8), starts[j+1..j+9), residual
// words) with cp.async while range k is decoded from smem with the pair-window scheme, so the
// decode never waits on a dependent global load.  A range crossing more than 7 segment starts
// is decoded through L2 instead.  Each lane's copy role (section, stride, bound) is fixed for
// the whole warp walk, so a range costs it one address computation and one cp.async.
constexpr uint32_t kR64Info = 32 * 16;  // per-warp range info: 32 x {rk, jk (~0: invalid), sb, wlo}
static_assert(kR64Segs + kR64StartGroups + (((64 * 32 + 31) >> 5) + 2 + 3 + 3) / 4 <= 32,
              "one 16-byte copy group per lane for every residual width");
__host__ __device__ constexpr uint32_t r64_smem_per_warp(uint32_t b) {
    return kR64Slots * r64_bytes(b) + kR64Info;
}

// FULL: len == 64 (no tail predicates, the tuned config-5 kernel); otherwise len < 64.
template <bool K64, bool FULL>
__global__ void __launch_bounds__(256) lc_range64_kernel(const RangeArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t kw = K64 ? 8 : 4;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r0 = ((uint64_t)blockIdx.x * 8 + warp) * 32;
    if (r0 >= a.q) return;  // warp-uniform
    const Sections sec = a.sec;
    const uint32_t b = a.b, mask = a.mask, L = a.L, bias = a.bias;
    const uint32_t len = FULL ? 64 : a.len;  // len <= 64
    const uint32_t RB = r64_bytes(b), nw16 = r64_words(b) / 4;
    uint8_t* wbase = smem + warp * r64_smem_per_warp(b);
    uint4* info = (uint4*)(wbase + kR64Slots * RB);
    uint8_t* ring = wbase;
    const uint32_t lmask = lanemask_le();
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();

    // ---- phase 1: lane-parallel search, results parked in shared memory
    {
        uint32_t rs = 0, j = kFull, sj = 0;
        if (r0 + lane < a.q) {
            const uint64_t s64 = __ldg(a.start + r0 + lane);
            if (s64 <= a.n && len <= a.n - s64) {
                rs = (uint32_t)s64;
                j = seg_search(sec, rs, keep);
                sj = ldh(sec.starts + j, keep);
            } else if (a.err) {
                atomicOr(a.err, 1u);
            }
        }
        // first residual word of the range's staged words (16-byte aligned)
        info[lane] = make_uint4(rs, j, sj, (uint32_t)(((uint64_t)rs * b) >> 5) & ~3u);
    }
    __syncwarp();
    const uint32_t nr = (uint32_t)min((uint64_t)32, a.q - r0);

    // ---- this lane's copy role: 16-byte group `lane` of every slot
    //   lanes [0, S8): params[j + lane]           (valid while j + lane < L)
    //   lanes [S8, S8 + SG): starts[4 ((j+1)/4) + 4 (lane - S8) ..]   (inside the section padding)
    //   next nw16 lanes: words[wlo + 4 t ..]     (valid while wlo + 4 t + 4 <= W)
    const uint32_t gs = kR64Segs, gw = kR64Segs + kR64StartGroups;
    const bool has = lane < gw + nw16;
    const int kind = lane < gs ? 0 : lane < gw ? 1 : 2;
    const uint32_t t = kind == 0 ? lane : kind == 1 ? lane - gs : lane - gw;
    const uint8_t* src0 = kind == 0 ? (const uint8_t*)(sec.params + t)
                        : kind == 1 ? (const uint8_t*)(sec.starts + 4 * t)
                                    : (const uint8_t*)(sec.words + 4 * t);
    const uint32_t mul = kind == 0 ? 16 : 4;
    // valid iff v < lim (v = the range's j or wlo)
    const uint64_t lim = kind == 0 ? (uint64_t)L - t : kind == 1 ? ~0ull
                       : (a.nwords >= 4 * (uint64_t)t + 4 ? a.nwords - 4 * (uint64_t)t - 3 : 0);
    auto issue = [&](uint32_t k) {
        if (k < nr && has) {
            const uint4 ri = info[k];
            if (ri.y != kFull) {
                const uint32_t v = kind == 0 ? ri.y : kind == 1 ? ((ri.y + 1) & ~3u) : ri.w;
                cp16(ring + (k % kR64Slots) * RB + 16 * lane, src0 + (uint64_t)v * mul, v < lim);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // one group per range (maybe empty)
    };
    for (uint32_t k = 0; k + 1 < kR64Slots; ++k) issue(k);
    uint8_t* const out0 = (uint8_t*)a.out + ((size_t)r0 * len + lane) * kw;  // lane's slot, range 0
    // ranges shorter than 64 keys: the slot still stages the slices of 64 keys (zero-filled past
    // the sections), the tail is not stored
    const bool liveA = FULL || lane < len, liveB = FULL || 32 + lane < len;

    for (uint32_t k = 0; k < nr; ++k) {
        issue(k + kR64Slots - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kR64Slots - 1) : "memory");
        __syncwarp();
        const uint4 ri = info[k];
        const uint32_t rk = ri.x, jk = ri.y, sb = ri.z;
        uint8_t* outk = out0 + (size_t)k * len * kw;
        if (jk == kFull) {
            if (liveA) put<K64>(outk, 0, 0);
            if (liveB) put<K64>(outk + 32 * kw, 0, 0);
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
                // bit offset inside the staged words; exact mod 2^32 (the true value is small)
                const uint32_t bA = (rk + lane) * b - (ri.w << 5);
                const uint32_t bB = bA + 32 * b;
                LC_CHECK(liveB, (bB >> 5) + 1, r64_words(b));
                uA = __funnelshift_r(Wd[bA >> 5], Wd[(bA >> 5) + 1], bA & 31) & mask;
                uB = __funnelshift_r(Wd[bB >> 5], Wd[(bB >> 5) + 1], bB & 31) & mask;
            }
            if (liveA) put<K64>(outk, pA.x, pred_plus(pA.y, dA, uA - bias));
            if (liveB) put<K64>(outk + 32 * kw, pB.x, pred_plus(pB.y, dB, uB - bias));
        } else {  // dense range: 32-key windows through L2
            uint32_t jb = jk, sbw = sb;
            for (uint32_t w0 = 0; w0 < len; w0 += 32) {
                const uint32_t wb = rk + w0;
                const uint32_t xw = ldh(sec.starts + min(jb + 1 + lane, L), keep) - wb;
                const uint32_t Pm = __reduce_or_sync(kFull, bit_or_zero(xw));
                const uint32_t adv = __popc(__ballot_sync(kFull, xw <= 32));
                const uint32_t m = Pm & lmask;
                const uint32_t d = m ? lane - (31 - __clz(m)) : wb - sbw + lane;
                if (w0 + lane < len) {
                    const ulonglong2 pr = ldh(sec.params + LC_BOUND(true, jb + __popc(m), L), once);
                    const uint32_t u =
                        b ? field_of(field_words(sec, wb + lane, b, once), wb + lane, b, mask) : 0;
                    put<K64>(outk + w0 * kw, pr.x, pred_plus(pr.y, d, u - bias));
                }
                jb += adv;
                sbw = ldh(sec.starts + min(jb, L), keep);
            }
        }
        __syncwarp();  // the slot is refilled by the next issue()
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------- random access and quantiles
struct AccessArgs {
    Sections sec;
    const uint64_t* idx;  // indices (kAccess) or quantile ranks k (kQuantile*)
    void* out;
    uint32_t* err;
    uint64_t q;           // number of queries
    uint64_t qdiv;        // quantile denominator q (kQuantile*)
    uint32_t n, b, bias, mask;
    uint32_t center;  // eps - bias: 0 for anchored blobs, eps for F7 (approximate mode)
};

enum AccessMode { kAccess = 0, kQuantileExact = 1, kQuantileApprox = 2 };
// queries per thread: two interleaved chains when a residual gather follows the search (A/B:
// +4% for exact quantiles), one for the params-only approximate quantile (-8% with two)
__host__ __device__ constexpr uint32_t access_per_thread(int mode) {
    return mode == kQuantileApprox ? 1 : 2;
}

// Access layout (lc_access_layout_build), two parts in one buffer:
//  * dir[32 h + w] = {bits, entry} (8 bytes per 32 keys): bit t of `bits` set iff key
//    1024 h + 32 w + t starts a segment (block position 0 excluded: the hint already names the
//    segment holding key 1024 h); entry = rank | dist << 11, rank = set bits in words < w of
//    block h, dist = 32 w - (start of the segment holding key 1024 h + 32 w), kDistNone when
//    >= 2^21 - 1;
//  * records: record j at 16-byte unit 2 j + floor(s_j b / 128) holds {base_j, slope_j} then
//    the residual units floor(s_j b / 128) .. floor(s_{j+1} b / 128) (every unit of the words
//    section holding a bit of the segment's keys); the offset needs only j and s_j.
// A lookup of key i: j = hint[h] + rank + popc(bits at or below i in its word), d = i - s_j
// from the highest such bit (or dist), then params and residual from record j: one L2 round
// trip (hint, bits, entry: independent loads) and one DRAM line instead of a binary search.
constexpr uint32_t kDistNone = 0x1FFFFF;
__host__ __device__ __forceinline__ uint64_t acc_unit(uint32_t j, uint32_t s, uint32_t b) {
    return 2 * (uint64_t)j + (((uint64_t)s * b) >> 7);
}

// segment starts -> block bitmaps (dir zeroed before)
__global__ void __launch_bounds__(256) lc_acc_bits_kernel(const Sections sec, uint2* dir) {
    const uint32_t j = blockIdx.x * 256 + threadIdx.x + 1;  // segment 0 starts at key 0
    if (j >= sec.L) return;
    const uint32_t s = __ldg(sec.starts + j);
    // word (s >> 10) * 32 + ((s >> 5) & 31) = s >> 5
    if (s & 1023) atomicOr(&dir[s >> 5].x, 1u << (s & 31));
}

// one warp per block: rank (exclusive warp scan of the word popcounts) and dist per word
__global__ void __launch_bounds__(256) lc_acc_dir_kernel(const Sections sec, uint2* dir, uint32_t H) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t h = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (h >= H) return;
    const uint32_t bw = dir[32 * h + lane].x;
    uint32_t inc = __popc(bw);  // inclusive scan of popcounts
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += x;
    }
    const uint32_t rank = inc - __popc(bw);
    const uint32_t nz = __ballot_sync(kFull, bw != 0) & ((1u << lane) - 1);  // nonzero words < w
    const uint32_t wl = nz ? 31 - __clz(nz) : 0;
    const uint32_t bl = __shfl_sync(kFull, bw, wl);
    uint64_t dist;
    if (bw & 1) {  // a segment starts at the word's first key
        dist = 0;
    } else if (nz) {
        dist = 32 * lane - (32 * wl + (31 - __clz(bl)));
    } else {
        const uint32_t s0 = __ldg(sec.starts + __ldg(sec.hint + h));
        dist = ((uint64_t)h << 10) + 32 * lane - s0;
    }
    dir[32 * h + lane].y = rank | ((uint32_t)min(dist, (uint64_t)kDistNone) << 11);
}

// records: one warp per segment (grid-stride) copies params[j] and the segment's residual units
__global__ void __launch_bounds__(256) lc_acc_build_kernel(const Sections sec, ulonglong2* acc,
                                                           uint32_t b) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * 8;
    const ulonglong2* W16 = (const ulonglong2*)sec.words;  // 16-byte units of the words
    for (uint32_t j = blockIdx.x * 8 + (threadIdx.x >> 5); j < sec.L; j += nw) {
        const uint32_t s0 = __ldg(sec.starts + j), s1 = __ldg(sec.starts + j + 1);
        const uint64_t u0 = ((uint64_t)s0 * b) >> 7, u1 = ((uint64_t)s1 * b) >> 7;
        ulonglong2* rec = acc + acc_unit(j, s0, b);
        if (lane == 0) rec[0] = __ldg(sec.params + j);
        for (uint64_t u = u0 + lane; u <= u1; u += 32)
            rec[1 + (u - u0)] = __ldg(W16 + LC_BOUND(true, u, (sec.W + 3) / 4));
    }
}

// ------------------------------------------ range decode, len <= 64, through the access layout
// With the access layout attached a range of up to 64 keys (written for the 64 of BASELINE
// config 5) needs no search, no starts and ONE contiguous gather.  The directory bitmaps of its (at most three) 32-key groups, shifted to the range's
// first key, ARE the window boundary masks the ring kernel votes for (PA: starts among keys
// rk + 1 .. rk + 31, PB: among rk + 32 .. rk + 63), and the records of consecutive segments are
// contiguous, so the range's data is the params unit of its first segment jk plus the span
//   [A, E],  A = 2 jk + 1 + floor(rk b / 128)  (the unit holding key rk's residual in record jk),
//            E = 2 je + 1 + floor(((rk + 64) b - 1) / 128)  (je: segment of key rk + 63),
// which holds every later segment's params and all 64 residual fields.  Phase 1 (lane = range):
// hint and directory loads (L2-resident, evict_last); masks, span and addresses parked in shared
// memory.  Phase 2: the warp walks its 32 ranges through a ring of slots; lane 0 copies the
// params unit, lane g >= 1 span unit g - 1 (one 16-byte cp.async each) while an earlier range
// is decoded from its slot with popc / clz on the parked masks (no votes).  A range whose span
// exceeds 31 units goes through L2.
#ifndef LC_RD_SLOTS
#define LC_RD_SLOTS 4
#endif
// Ring depth (ranges gathered ahead + 1) and the shared-memory carve-out (kRdCarveout, set by
// the launcher).  What decides this kernel's speed is how much of the SM's 256 KB stays L1 (the
// in-flight gathers and stores live there): with the driver's default carve-out (228 KB as soon
// as the resident CTAs need > 196 KB) 4 slots / 7 CTAs per SM take 1.65 ms per 1e7 ranges and
// 8 slots / 4 CTAs 1.76 ms; capped at 164 KB (5 CTAs, 92 KB of L1) 4 slots take 1.40 ms, 8 slots
// (3 CTAs) 1.40 ms, 2 slots 1.61 ms; at 196 KB 1.41 / 1.43 ms; at 132 KB 1.44 / 1.67 ms.
constexpr uint32_t kRdSlots = LC_RD_SLOTS;
constexpr int kRdCarveout = 71;  // percent of 228 KB: the 164 KB configuration
#ifndef LC_RD_WARPS
#define LC_RD_WARPS 8
#endif
constexpr uint32_t kRdWarps = LC_RD_WARPS;  // warps per CTA (2 / 4 / 16 measured slower)
static_assert((kRdSlots & (kRdSlots - 1)) == 0, "slot index is k % kRdSlots");
#ifndef LC_RD_UNITS
#define LC_RD_UNITS 32
#endif
constexpr uint32_t kRdUnits = LC_RD_UNITS;  // copy lanes: unit 0 first params, 1..kRdUnits-1 the span
static_assert(kRdUnits <= 32, "one 16-byte copy per lane");
constexpr uint32_t kRdSlotBytes = 16 * (kRdUnits + 1);  // + 1 pad unit (a field's second word)
constexpr uint32_t kRdInfoBytes = 48;       // per range: 3 x uint4, see phase 1
constexpr uint32_t kRdInvalid = 1u << 31, kRdSlow = 1u << 30;  // flags beside the span units
__host__ __device__ constexpr uint32_t rd_smem_per_warp() {
    return kRdSlots * kRdSlotBytes + 32 * kRdInfoBytes;
}
__device__ __forceinline__ void cp16s(uint32_t dst_s, uint64_t src) {  // shared-space address
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_s), "l"(src) : "memory");
}
__device__ __forceinline__ uint32_t sel_nz(uint32_t c, uint32_t a, uint32_t b) {  // c ? a : b
    uint32_t r;
    asm("{\n.reg .pred p;\nsetp.ne.u32 p, %1, 0;\nselp.u32 %0, %2, %3, p;\n}"
        : "=r"(r)
        : "r"(c), "r"(a), "r"(b));
    return r;
}

// FULL: len == 64 (no tail masks: the tuned config-5 kernel); otherwise len < 64.
template <bool K64, bool FULL>
__global__ void __launch_bounds__(32 * kRdWarps, 5) lc_range64_dir_kernel(const RangeArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t kw = K64 ? 8 : 4;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r0 = ((uint64_t)blockIdx.x * kRdWarps + warp) * 32;
    if (r0 >= a.q) return;  // warp-uniform
    const Sections sec = a.sec;
    const uint32_t b = a.b, mask = a.mask, L = a.L, bias = a.bias;
    const uint32_t len = FULL ? 64 : a.len;  // len <= 64
    uint8_t* ring = smem + warp * rd_smem_per_warp();
    uint4* info = (uint4*)(ring + kRdSlots * kRdSlotBytes);
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();

    // ---- phase 1: lane = range.  Parked per range (3 x uint4):
    //   [0] {rk, rk - s_jk, PA, PB}
    //   [1] {address of span unit A (lo, hi), span units | flags, 16 x (A - unit of jk's params)}
    //   [2] {jk, s_jk, -, -}  (the through-L2 path)
    {
        uint32_t rk = 0, jk = 0, sk = 0, PA = 0, PB = 0, units = kRdInvalid, back = 0;
        uint64_t A = (uint64_t)(uintptr_t)sec.acc;  // ranges without copies: lane 0 reads unit 0
        if (r0 + lane < a.q) {
            const uint64_t s64 = __ldg(a.start + r0 + lane);
            if (s64 <= a.n && len <= a.n - s64) {
                rk = (uint32_t)s64;
                const uint32_t e = rk + len - 1, g0 = rk >> 5, r5 = rk & 31;  // e: the last key
                const uint32_t hA = ldh(sec.hint + (rk >> 10), keep);
                const uint2 d0 = ldh(sec.dir + g0, keep);
                const uint2 d1 = ldh(sec.dir + min(g0 + 1, e >> 5), keep);
                const uint2 d2 = ldh(sec.dir + (e >> 5), keep);  // group g0 + 2, or an earlier one again
                const uint32_t m = d0.x & ((2u << r5) - 1);
                jk = hA + (d0.y & 2047) + __popc(m);
                if (m) sk = (rk & ~31u) + (31 - __clz(m));
                else if ((d0.y >> 11) != kDistNone) sk = (rk & ~31u) - (d0.y >> 11);
                else sk = ldh(sec.starts + jk, keep);  // a segment longer than 2^21 keys
                PA = __funnelshift_r(d0.x, d1.x, r5) & ~1u;  // bit t: key rk + t starts a segment
                PB = __funnelshift_r(d1.x, d2.x, r5);
                // only the starts among keys rk + 1 .. rk + len - 1 count
                if (!FULL) {
                    PA &= len >= 32 ? kFull : (1u << len) - 1;
                    PB &= len > 32 ? (1u << (len - 32)) - 1 : 0u;
                }
                // a start exactly at a block's first key is not in the bitmaps (the hint names
                // it): the block's first group has dist 0 then
                const uint32_t tb = 1024 - (rk & 1023);
                if (tb < len && ((((r5 + tb) >> 5) == 1 ? d1.y : d2.y) >> 11) == 0) {
                    if (tb < 32) PA |= 1u << tb;
                    else PB |= 1u << (tb - 32);
                }
                const uint32_t je = jk + __popc(PA) + __popc(PB);
                LC_CHECK(true, je, L);
                const uint64_t ur = ((uint64_t)rk * b) >> 7;
                const uint32_t r0b = (rk * b) & 127;
                // units in [A, E]: 2 (je - jk) + floor((r0b + len b - 1) / 128) + 1 (b = 0: 2 (je - jk))
                const uint32_t span = 2 * (je - jk) + (uint32_t)(((int32_t)(r0b + len * b) - 1) >> 7) + 1;
                if (span < kRdUnits) {
                    units = span;
                    A = (uint64_t)(uintptr_t)(sec.acc + 2 * (uint64_t)jk + 1 + ur);
                    back = 16 * (1 + (uint32_t)(ur - (((uint64_t)sk * b) >> 7)));
                } else {
                    units = kRdSlow;
                }
            } else if (a.err) {
                atomicOr(a.err, 1u);
            }
        }
        // PA's bit 0 is free (a start at rk itself is part of jk): set = not the ring path
        info[3 * lane] = make_uint4(rk, rk - sk, PA | (units >= kRdSlow ? 1u : 0u), PB);
        info[3 * lane + 1] = make_uint4((uint32_t)A, (uint32_t)(A >> 32), units, back);
        info[3 * lane + 2] = make_uint4(jk, sk, 0, 0);
    }
    __syncwarp();
    const uint32_t nr = (uint32_t)min((uint64_t)32, a.q - r0);

    // lane 0 copies the params unit of jk, lane g >= 1 span unit g - 1, into slot unit `lane`.
    // Shared memory is addressed in the shared window (32-bit) throughout the walk.
    const uint32_t ring_s = smem_addr(ring), info_s = ring_s + kRdSlots * kRdSlotBytes;
    const uint32_t dst_lane = ring_s + 16 * lane;
    const int32_t fwd = 16 * ((int32_t)lane - 1);
    auto lds4 = [](uint32_t addr) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(addr));
        return v;
    };
    auto lds1 = [](uint32_t addr) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
        return v;
    };
    auto issue = [&](uint32_t k) {
        if (k < nr) {
            const uint4 q1 = lds4(info_s + 48 * k + 16);
            if (lane <= (q1.z & 63)) {
                const int32_t off = lane ? fwd : -(int32_t)q1.w;
                cp16s(dst_lane + (k % kRdSlots) * kRdSlotBytes,
                      (((uint64_t)q1.y << 32) | q1.x) + (int64_t)off);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // one group per range (maybe empty)
    };
    for (uint32_t k = 0; k + 1 < kRdSlots; ++k) issue(k);
    uint8_t* outk = (uint8_t*)a.out + ((size_t)r0 * len + lane) * kw;  // lane's slot, range 0
    const bool liveA = FULL || lane < len, liveB = FULL || 32 + lane < len;
    const uint32_t lmask = lanemask_le();
    const uint32_t tbA = lane * b, tbB = tbA + 32 * b;  // bit offsets of the lane's two keys
    const bool pow2 = (b & (b - 1)) == 0;               // b in {0, 1, 2, 4, 8, 16, 32}

    for (uint32_t k = 0; k < nr; ++k, outk += (size_t)len * kw) {
        // range k's copies (and those of k + 1, k + 2) are in flight: wait for k's; the warp
        // sync also orders every lane's reads of slot k - 1 before it is refilled just below
        asm volatile("cp.async.wait_group %0;" ::"n"(kRdSlots - 2) : "memory");
        __syncwarp();
        issue(k + kRdSlots - 1);
        const uint4 q0 = lds4(info_s + 48 * k);
        const uint32_t rk = q0.x;
        if (!(q0.z & 1)) {
            const uint32_t slot = ring_s + (k % kRdSlots) * kRdSlotBytes;
            const uint32_t off0 = q0.y, PA = q0.z, PB = q0.w;
            const uint32_t r0b = (rk * b) & 127;
            const uint32_t offB = PA ? __clz(PA) + 1 : off0 + 32;  // uniform
            const uint32_t mA = PA & lmask, mB = PB & lmask;
            const uint32_t djA = __popc(mA), djB = __popc(PA) + __popc(mB);
            const uint32_t dA = sel_nz(mA, (uint32_t)__clz(mA) - 31, off0) + lane;
            const uint32_t dB = sel_nz(mB, (uint32_t)__clz(mB) - 31, offB) + lane;
            // params: slot unit 0 for jk, else 2 dj + floor((r0b + (s - rk) b) / 128)
            const uint32_t puA = sel_nz(djA, 2 * djA + ((r0b + (lane - dA) * b) >> 7), 0);
            const uint32_t puB = sel_nz(djB, 2 * djB + ((r0b + (32 + lane - dB) * b) >> 7), 0);
            LC_CHECK(liveB, puB, kRdUnits);
            const uint4 pA = lds4(slot + 16 * puA), pB = lds4(slot + 16 * puB);
            const uint32_t wbA = r0b + tbA, wbB = r0b + tbB;
            const uint32_t wA = slot + 16 + 32 * djA + ((wbA >> 3) & ~3u);
            const uint32_t wB = slot + 16 + 32 * djB + ((wbB >> 3) & ~3u);
            LC_CHECK(liveB, 4 + 8 * djB + (wbB >> 5) + 1, kRdSlotBytes / 4);
            uint32_t uA, uB;
            if (pow2) {  // widths dividing 32 never straddle a word (warp-uniform)
                uA = (lds1(wA) >> (wbA & 31)) & mask;
                uB = (lds1(wB) >> (wbB & 31)) & mask;
            } else {
                uA = __funnelshift_r(lds1(wA), lds1(wA + 4), wbA & 31) & mask;
                uB = __funnelshift_r(lds1(wB), lds1(wB + 4), wbB & 31) & mask;
            }
            if (liveA)
                put<K64>(outk, ((uint64_t)pA.y << 32) | pA.x,
                         pred_plus(((uint64_t)pA.w << 32) | pA.z, dA, uA - bias));
            if (liveB)
                put<K64>(outk + 32 * kw, ((uint64_t)pB.y << 32) | pB.x,
                         pred_plus(((uint64_t)pB.w << 32) | pB.z, dB, uB - bias));
        } else if (lds1(info_s + 48 * k + 24) & kRdInvalid) {
            if (liveA) put<K64>(outk, 0, 0);
            if (liveB) put<K64>(outk + 32 * kw, 0, 0);
        } else {  // 32-key windows through L2
            const uint4 q2 = info[3 * k + 2];
            uint32_t jb = q2.x, sbw = q2.y;
            for (uint32_t w0 = 0; w0 < len; w0 += 32) {
                const uint32_t wb = rk + w0;
                const uint32_t xw = ldh(sec.starts + min(jb + 1 + lane, L), keep) - wb;
                const uint32_t Pm = __reduce_or_sync(kFull, bit_or_zero(xw));
                const uint32_t adv = __popc(__ballot_sync(kFull, xw <= 32));
                const uint32_t m = Pm & lmask;
                const uint32_t d = m ? lane - (31 - __clz(m)) : wb - sbw + lane;
                if (w0 + lane < len) {
                    const ulonglong2 pr = ldh(sec.params + LC_BOUND(true, jb + __popc(m), L), once);
                    const uint32_t u =
                        b ? field_of(field_words(sec, wb + lane, b, once), wb + lane, b, mask) : 0;
                    put<K64>(outk + w0 * kw, pr.x, pred_plus(pr.y, d, u - bias));
                }
                jb += adv;
                sbw = ldh(sec.starts + min(jb, L), keep);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Q queries per thread through the access layout: all loads of one step are issued for the Q
// queries before any is consumed.
template <bool K64, int MODE, int Q>
__global__ void __launch_bounds__(256) lc_access_dir_kernel(const AccessArgs a) {
    constexpr bool kResidual = MODE != kQuantileApprox;
    const uint64_t t0 = (uint64_t)blockIdx.x * (256 * Q) + threadIdx.x;
    const Sections sec = a.sec;
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    uint32_t i[Q], j[Q], s[Q];
    uint2 de[Q];
    bool live[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        const uint64_t t = t0 + 256 * k;
        live[k] = false;
        i[k] = 0;
        if (t < a.q) {
            const uint64_t v = __ldcs(a.idx + t);
            const bool ok = MODE == kAccess ? v < a.n : v <= a.qdiv;
            if (ok) {
                live[k] = true;
                i[k] = MODE == kAccess ? (uint32_t)v
                                       : (uint32_t)min((uint64_t)a.n * v / a.qdiv, (uint64_t)a.n - 1);
            } else {
                if (a.err) atomicOr(a.err, 1u);
                if (K64) __stcs((unsigned long long*)a.out + t, 0ull);
                else __stcs((unsigned int*)a.out + t, 0u);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {  // one L2 round trip: hint and the word's {bits, entry}
        j[k] = 0;
        de[k] = make_uint2(0, 0);
        if (live[k]) {
            j[k] = ldh(sec.hint + (i[k] >> 10), keep);
            de[k] = ldh(sec.dir + (i[k] >> 5), keep);  // index 32 h + w
        }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        s[k] = 0;
        if (!live[k]) continue;
        const uint32_t t = i[k] & 31;
        const uint32_t m = de[k].x & ((2u << t) - 1);  // starts in the word at or below the key
        j[k] += (de[k].y & 2047) + __popc(m);
        const uint32_t dist = de[k].y >> 11;
        if (m) s[k] = (i[k] & ~31u) + (31 - __clz(m));
        else if (dist != kDistNone) s[k] = (i[k] & ~31u) - dist;
        else s[k] = ldh(sec.starts + j[k], keep);  // segment longer than 2^21 keys
    }
    ulonglong2 pr[Q];
    uint2 w[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {  // one DRAM line (usually): the record's params and field
        pr[k] = make_ulonglong2(0, 0);
        w[k] = make_uint2(0, 0);
        if (!live[k]) continue;
        const ulonglong2* rec = sec.acc + acc_unit(j[k], s[k], a.b);
        pr[k] = ldh(rec, once);
        if (kResidual && a.b) {
            const uint32_t p = (uint32_t)((uint64_t)i[k] * a.b - ((((uint64_t)s[k] * a.b) >> 7) << 7));
            const uint32_t* wp = (const uint32_t*)(rec + 1) + (p >> 5);
            w[k] = make_uint2(ldh(wp, once), ldh(wp + 1, once));
        }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (!live[k]) continue;
        uint8_t* o = (uint8_t*)a.out + (t0 + 256 * k) * (K64 ? 8 : 4);
        if (kResidual) {
            const uint32_t u = a.b ? field_of(w[k], i[k], a.b, a.mask) : 0;
            put<K64>(o, pr[k].x, pred_plus(pr[k].y, i[k] - s[k], u - a.bias));
        } else {
            const uint64_t f = pr[k].x + pred_plus(pr[k].y, i[k] - s[k], a.center);
            if (K64) __stcs((unsigned long long*)o, f < pr[k].x ? ~0ull : (unsigned long long)f);
            else __stcs((unsigned int*)o, f > 0xffffffffull ? 0xffffffffu : (unsigned int)f);
        }
    }
}

// Dec(K^c)[i] per query (Table I): hint bracket, binary search
// over starts, one params gather, one residual field.  Each thread serves access_per_thread()
// queries whose dependent load chains are interleaved; the residual words do not depend on
// the segment and are fetched before the search.  Quantiles use the same
// path with i = min(floor(N k / q), N - 1): exact = f(i) + Delta[i]; approximate = floor(f(i))
// from the segment alone, no residual read, error <= eps, saturated at the key width (L24).
template <bool K64, int MODE>
__global__ void __launch_bounds__(256) lc_access_kernel(const AccessArgs a) {
    constexpr bool kResidual = MODE != kQuantileApprox;
    constexpr uint32_t kAccessPerThread = access_per_thread(MODE);
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
            const uint64_t v = __ldcs(a.idx + t);
            const bool ok = MODE == kAccess ? v < a.n : v <= a.qdiv;
            if (ok) {
                live[k] = true;
                i[k] = MODE == kAccess ? (uint32_t)v
                                       : (uint32_t)min((uint64_t)a.n * v / a.qdiv, (uint64_t)a.n - 1);
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
            if (kResidual && a.b) w[k] = field_words(sec, i[k], a.b, once);
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
    uint32_t s[kAccessPerThread];
    ulonglong2 pr[kAccessPerThread];
#pragma unroll
    for (uint32_t k = 0; k < kAccessPerThread; ++k) {
        s[k] = 0;
        pr[k] = make_ulonglong2(0, 0);
        if (!live[k]) continue;
        s[k] = ldh(sec.starts + lo[k], keep);
        pr[k] = ldh(sec.params + LC_BOUND(true, lo[k], sec.L), once);
    }
#pragma unroll
    for (uint32_t k = 0; k < kAccessPerThread; ++k) {
        if (!live[k]) continue;
        uint8_t* o = (uint8_t*)a.out + (t0 + 256 * k) * (K64 ? 8 : 4);
        if (kResidual) {
            const uint32_t u = a.b ? field_of(w[k], i[k], a.b, a.mask) : 0;
            put<K64>(o, pr[k].x, pred_plus(pr[k].y, i[k] - s[k], u - a.bias));
        } else {  // floor(f(i)) can exceed the key width by up to eps: saturate (L24)
            // floor(f(i)) = base + floor(slope d / 2^32) + (eps - bias): F7 bases sit eps below
            const uint64_t f = pr[k].x + pred_plus(pr[k].y, i[k] - s[k], a.center);
            if (K64) __stcs((unsigned long long*)o, f < pr[k].x ? ~0ull : (unsigned long long)f);
            else __stcs((unsigned int*)o, f > 0xffffffffull ? 0xffffffffu : (unsigned int)f);
        }
    }
}
