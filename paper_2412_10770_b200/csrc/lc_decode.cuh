// lc_decode.cuh -- full decode: staging pages, window / pair / quad steps, kernel
// Internal part of lc_kernels.cu: included inside its anonymous namespace (one translation
// unit, so the launch tables and the bounds-check counter keep internal linkage).
#pragma once

// --------------------------------------------------------------------------- full decode
struct DecodeArgs {
    Sections sec;
    void* out;         // receives keys [i0, i1)
    uint32_t i0, i1;   // i0 % 1024 == 0
    uint32_t chunk0;   // i0 / 1024
    uint32_t nchunks;  // ceil((i1 - i0) / 1024)
    uint32_t bias;
    uint32_t warp_bytes;  // shared memory per warp
    uint64_t nwords;      // W (words section length; > 2^32 possible at N ~ 2^32, b = 32)
    const uint32_t* rho;   // lc_union fused path only (UNI kernels): see Ins
    const uint32_t* coff;  // [h] = #{m : rho_m < 1024 h}
};

// Insertion shifts for lc_union's fused path: the long list's key i goes to output slot
// i + #{m : rho_m <= i}, where rho (sorted) holds, for each short-list key absent from the long
// list, the number of long-list keys below it (its own slot is m + rho_m).  Per chunk the
// entries with rho in the chunk, [coff[h], coff[h+1]), are read in batches of 32 (one per lane,
// v = rho - key0); cur = #{rho < window start} and nxt = the next entry's chunk offset are
// warp-uniform, so a window holding no entry costs one compare.
struct Ins {
    const uint32_t* rho;
    uint32_t key0, cur, end, bat, v, nxt;
    const uint2* desc;  // SH == 1: per-window {insertion bitmask, shift at the window start}
};

// chunk start: [lo, hi) = [coff[h], coff[h+1]) (loaded one chunk ahead); the first batch's
// load is issued here, before the chunk's staging, and consumed by ins_ready after it
__device__ __forceinline__ void ins_begin(Ins& s, uint32_t lo, uint32_t hi, uint32_t key0,
                                          uint32_t lane) {
    s.key0 = key0;
    s.cur = s.bat = lo;
    s.end = hi;
    s.v = lo + lane < hi ? __ldg(s.rho + lo + lane) - key0 : kFull;
}
__device__ __forceinline__ void ins_ready(Ins& s) {
    s.nxt = __reduce_min_sync(kFull, s.v);  // the first entry; kFull when the chunk has none
}

// shift (in keys) of this lane's key wb + lane; the windows of a chunk are asked in order.
// Entries at distinct positions are one bit each in a REDUX.OR mask (add = popc of the bits
// at or below the lane); equal ranks (several absent keys between two long-list keys) count
// one by one.
template <bool UNI>
__device__ __forceinline__ uint32_t ins_shift(Ins& s, uint32_t wb, uint32_t lane) {
    if (!UNI) return 0;
    const uint32_t o = wb - s.key0;
    if (s.nxt - o >= 32) return s.cur;  // warp-uniform: no entry in this window (nxt >= o)
    const uint32_t c0 = s.cur;
    uint32_t add = 0;
    for (;;) {
        const uint32_t x = s.v - o;  // < 32: this batch's entries in the window
        uint32_t in = __ballot_sync(kFull, x < 32);
        const uint32_t n = __popc(in);
        const uint32_t M = __reduce_or_sync(kFull, bit_or_zero(x));
        s.cur += n;
        if (__popc(M) == n) {
            add += __popc(M & ((2u << lane) - 1));  // bits at or below the lane
        } else {
            while (in) {
                const uint32_t k = __ffs(in) - 1;
                in &= in - 1;
                add += __shfl_sync(kFull, x, k) <= lane;
            }
        }
        if (s.cur - s.bat < 32 || s.cur == s.end) break;
        s.bat = s.cur;  // batch used up inside the window: next 32 entries
        s.v = s.bat + lane < s.end ? __ldg(s.rho + s.bat + lane) - s.key0 : kFull;
    }
    // first unconsumed entry: every entry below the window's end has been counted
    s.nxt = __reduce_min_sync(kFull, s.v < o + 32 ? kFull : s.v);
    return c0 + add;
}

// Store shift of the lane's key wb + lane.  SH = 0: none (plain decode); 1: from the chunk's
// window descriptors (built once per chunk, branch-free per window); 2: streamed (Ins), for
// chunks whose insertions do not fit the descriptors (equal ranks, > 32 entries).
template <bool K64, int SH>
__device__ __forceinline__ void* shifted(void* outw, Ins& ins, uint32_t wb, uint32_t lane) {
    if (SH == 0) return outw;
    if (SH == 1) {
        const uint2 d = ins.desc[(wb - ins.key0) >> 5];
        return (uint8_t*)outw + (size_t)(d.y + __popc(d.x & lanemask_le())) * (K64 ? 8 : 4);
    }
    return (uint8_t*)outw + (size_t)ins_shift<true>(ins, wb, lane) * (K64 ? 8 : 4);
}

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
    uint32_t rb, rmask;   // runtime residual width and mask (B == kRtB: batch kernels)
#ifdef LC_DEBUG_BOUNDS
    uint32_t cs, nw;  // staged starts / words entries
#endif
};

// B == kRtB: the residual width is a runtime value (pg.rb), for the batch kernels whose lists
// have different widths; every other B is a compile-time width (lc_decode_kernel).
constexpr uint32_t kRtB = 64;
template <uint32_t B>
__device__ __forceinline__ uint32_t bits_of(const Page& pg) { return B == kRtB ? pg.rb : B; }
template <uint32_t B>
__device__ __forceinline__ uint32_t fld(const Page& pg, uint32_t w, uint32_t lw, uint32_t ls) {
    if (B == kRtB) {
        if (!pg.rb) return 0;
        const uint32_t* wp = pg.sW + w * pg.rb + lw;
        return __funnelshift_r(wp[0], wp[1], ls) & pg.rmask;
    }
    return field<B == kRtB ? 0 : B>(pg.sW, w, lw, ls);
}

// Stage starts[pj, pj + cs) and params[pj, pj + cp) (plus, when wbytes != 0, the chunk's words)
// with TMA bulk copies; cs covers one start past the params so every window candidate
// (clamped at jlast + 1) is a real start.  Lane 0 issues, the warp waits on the mbarrier.
__device__ __forceinline__ void stage(Page& pg, const Sections& sec, uint32_t from, uint32_t jlast,
                                      const uint32_t* wsrc, uint32_t wbytes, uint32_t lane) {
    __syncwarp();  // every lane is done reading the previous contents ...
    // ... and those generic-proxy reads are ordered before the async-proxy (TMA) writes below
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
// t = floor(slope d / 2^32) + u - bias = K[i] - base_j in [0, 2^32) (FORMAT F2 anchor, or the
// F7 band floor with bias 0, plus the guard).
template <bool K64, uint32_t B, bool CHECK, bool FULL, int SH>
__device__ __forceinline__ void decode_window(Page& pg, const Sections& sec, uint32_t& jb,
                                              uint32_t& sb, uint32_t jlast, uint32_t wb,
                                              uint32_t w, uint32_t lane, uint32_t lmask,
                                              uint32_t lw, uint32_t ls, uint32_t bias,
                                              void* outw, uint32_t valid, Ins& ins) {
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
    LC_CHECK(bits_of<B>(pg) && (FULL || lane < valid), w * bits_of<B>(pg) + lw + 1, pg.nw);
    const uint32_t t = pred_plus(pr.y, d, fld<B>(pg, w, lw, ls) - bias);
    outw = shifted<K64, SH>(outw, ins, wb, lane);
    if (FULL || lane < valid) put<K64>(outw, pr.x, t);
    // candidates clamped at jlast + 1 repeat the list's final start N in the last chunk: cap
    // the advance there so jb stays a valid staged index
    jb = min(jb + adv, jlast + 1);
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
}

// Two windows at once: keys [wb, wb + 64), lane handles wb + lane and wb + 32 + lane.  One
// candidate load / vote serves both halves when fewer than 32 segment starts fall inside;
// otherwise it falls back to two single windows.  w2 = pair index (windows 2 w2, 2 w2 + 1).
template <bool K64, uint32_t B, bool CHECK, int SH>
__device__ __forceinline__ void decode_pair(Page& pg, const Sections& sec, uint32_t& jb,
                                            uint32_t& sb, uint32_t jlast, uint32_t wb,
                                            uint32_t w2, uint32_t lane, uint32_t lmask,
                                            uint32_t lw, uint32_t ls, uint32_t bias, void* outw,
                                            Ins& ins) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    if (CHECK && min(jb + 31, jlast) >= pg.pj + pg.cp)
        stage(pg, sec, jb, jlast, nullptr, 0, lane);
    const uint32_t cand = min(jb + 1 + lane, jlast + 1);
    const uint32_t x = pg.sS[LC_BOUND(true, cand - pg.pj, pg.cs)] - wb;
    const uint32_t inside = __ballot_sync(kFull, x < 64);
    if (inside == kFull) {  // >= 32 boundaries in 64 keys: not enough candidates, go window-wise
        decode_window<K64, B, CHECK, true, SH>(pg, sec, jb, sb, jlast, wb, 2 * w2, lane, lmask,
                                                lw, ls, bias, outw, 32, ins);
        decode_window<K64, B, CHECK, true, SH>(pg, sec, jb, sb, jlast, wb + 32, 2 * w2 + 1, lane,
                                                lmask, lw, ls, bias, (uint8_t*)outw + 32 * kw, 32,
                                                ins);
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
    LC_CHECK(bits_of<B>(pg), (2 * w2 + 1) * bits_of<B>(pg) + lw + 1, pg.nw);
    const uint32_t tA = pred_plus(pA.y, dA, fld<B>(pg, 2 * w2, lw, ls) - bias);
    const uint32_t tB = pred_plus(pB.y, dB, fld<B>(pg, 2 * w2 + 1, lw, ls) - bias);
    put<K64>(shifted<K64, SH>(outw, ins, wb, lane), pA.x, tA);
    put<K64>(shifted<K64, SH>((uint8_t*)outw + 32 * kw, ins, wb + 32, lane), pB.x, tB);
    jb = min(jb + adv, jlast + 1);  // see decode_window
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
}

// Four windows at once: keys [wb, wb + 128), lane handles wb + 32 q + lane (q = 0..3).  One
// candidate load / advance vote serves four quarters when fewer than 32 segment starts fall
// inside; otherwise two pair steps.  w4 = quad index (windows 4 w4 .. 4 w4 + 3).
template <bool K64, uint32_t B, bool CHECK, int SH, bool FAST = false>
__device__ __forceinline__ void decode_quad(Page& pg, const Sections& sec, uint32_t& jb,
                                            uint32_t& sb, uint32_t jlast, uint32_t wb,
                                            uint32_t w4, uint32_t lane, uint32_t lmask,
                                            uint32_t lw, uint32_t ls, uint32_t bias, void* outw,
                                            Ins& ins) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    if (CHECK && min(jb + 31, jlast) >= pg.pj + pg.cp)
        stage(pg, sec, jb, jlast, nullptr, 0, lane);
    const uint32_t cand = min(jb + 1 + lane, jlast + 1);
    const uint32_t x = pg.sS[LC_BOUND(true, cand - pg.pj, pg.cs)] - wb;
    const uint32_t inq = __ballot_sync(kFull, x < 128);
    if (FAST && inq == 0) {  // sparse lists: no segment starts inside the 128 keys, one segment
        const ulonglong2 pr = pg.sP[LC_BOUND(true, jb - pg.pj, pg.cp)];
        const uint32_t d0 = (wb - sb) + lane;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            LC_CHECK(bits_of<B>(pg), (4 * w4 + q) * bits_of<B>(pg) + lw + 1, pg.nw);
            put<K64>(shifted<K64, SH>((uint8_t*)outw + 32 * kw * q, ins, wb + 32 * q, lane), pr.x,
                     pred_plus(pr.y, d0 + 32 * q, fld<B>(pg, 4 * w4 + q, lw, ls) - bias));
        }
        jb = min(jb + __popc(__ballot_sync(kFull, x == 128)), jlast + 1);  // a start at wb + 128
        sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
        return;
    }
    if (inq == kFull) {  // >= 32 boundaries in 128 keys
        decode_pair<K64, B, CHECK, SH>(pg, sec, jb, sb, jlast, wb, 2 * w4, lane, lmask, lw, ls,
                                        bias, outw, ins);
        decode_pair<K64, B, CHECK, SH>(pg, sec, jb, sb, jlast, wb + 64, 2 * w4 + 1, lane, lmask,
                                        lw, ls, bias, (uint8_t*)outw + 64 * kw, ins);
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
        LC_CHECK(bits_of<B>(pg), (4 * w4 + q) * bits_of<B>(pg) + lw + 1, pg.nw);
        put<K64>(shifted<K64, SH>((uint8_t*)outw + 32 * kw * q, ins, wb + 32 * q, lane), pr.x,
                 pred_plus(pr.y, d, fld<B>(pg, 4 * w4 + q, lw, ls) - bias));
        off = P ? __clz(P) + 1 : off + 32;
        jq += __popc(P);
    }
    jb = min(jb + adv, jlast + 1);  // see decode_window
    sb = pg.sS[LC_BOUND(true, jb - pg.pj, pg.cs)];
}

// One staged 1024-key chunk (or a ragged tail): quads when every segment is staged, paged
// pairs for dense chunks, windows for the tail.  SH: the store shift (see shifted).
template <bool K64, uint32_t B, bool SPARSE, int SH>
__device__ __forceinline__ void decode_chunk(Page& pg, const Sections& sec, uint32_t j0,
                                             uint32_t jlast, uint32_t key0, uint32_t nk,
                                             uint32_t lane, uint32_t lmask, uint32_t lw,
                                             uint32_t ls, uint32_t bias, uint8_t* outl, Ins& ins,
                                             bool has_next, uint32_t nj0, uint32_t njl) {
    constexpr uint32_t kw = K64 ? 8 : 4;
    uint32_t jb = j0;                                        // segment holding the window's first key
    uint32_t sb = pg.sS[LC_BOUND(true, j0 - pg.pj, pg.cs)];  // its start
    if (nk == 1024 && jlast < pg.pj + pg.cp) {  // whole chunk staged: no re-page checks
#pragma unroll 1
        for (uint32_t g = 0; g < 8; g += 2, outl += 2 * 128 * kw) {
#pragma unroll
            for (uint32_t k = 0; k < 2; ++k)
                decode_quad<K64, B, false, SH, SPARSE>(pg, sec, jb, sb, jlast, key0 + 128 * (g + k),
                                                       g + k, lane, lmask, lw, ls, bias,
                                                       outl + 128 * kw * k, ins);
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
                decode_pair<K64, B, true, SH>(pg, sec, jb, sb, jlast, key0 + 64 * (g + k), g + k,
                                              lane, lmask, lw, ls, bias, outl + 64 * kw * k, ins);
        }
    } else {  // ragged tail chunk
        for (uint32_t w = 0; 32 * w < nk; ++w)
            decode_window<K64, B, true, false, SH>(pg, sec, jb, sb, jlast, key0 + 32 * w, w, lane,
                                                   lmask, lw, ls, bias, outl + 32 * kw * w,
                                                   nk - 32 * w, ins);
    }
}

// lc_union's fused path: the chunk's window descriptors (ins.desc, 32 x {mask, shift}) from its
// insertion entries [cur, end) (ins_begin / ins_ready loaded the first 32; v = rho - key0):
// window w's mask has bit t for an entry at chunk offset 32 w + t, its shift counts the entries
// before the chunk (cur) and in windows < w.  Returns false (use the streamed path) when the
// chunk has more than 32 entries or two entries share a rank (popc would undercount).
__device__ __forceinline__ bool ins_describe(Ins& s, uint32_t lane) {
    const uint32_t n = s.end - s.cur;
    if (n > 32) return false;
    const bool has = lane < n;
    const uint32_t prev = __shfl_up_sync(kFull, s.v, 1);
    if (__ballot_sync(kFull, has && lane > 0 && prev == s.v)) return false;  // equal ranks
    uint2* d = (uint2*)s.desc;
    d[lane] = make_uint2(0, 0);
    __syncwarp();
    if (has) atomicOr(&d[s.v >> 5].x, 1u << (s.v & 31));
    __syncwarp();
    const uint32_t m = d[lane].x, c = __popc(m);
    uint32_t inc = c;  // inclusive scan of the per-window counts
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    d[lane].y = s.cur + inc - c;
    __syncwarp();
    return true;
}

// SPARSE: lists with fewer than one segment per 64 keys (config 4) read < 1 B per key: no L2
// prefetch of the next chunk (A/B: it costs config 4 +1.4% time) and the per-quad
// single-segment fast path (config 4 -2.3%; it costs dense lists, so dense kernels omit it).
// UNI: lc_union's fused path (stores shifted by Ins; dense settings).
// All: <= 64 registers (4 CTAs per SM fit).  A/B on B200 against the former 5 CTAs / 48
// registers (dense) and 6 / 40 (sparse): bench config 2 5370 -> 5430 GB/s (three alternating
// pairs), config 5 -1.4% time, config 3 flat, config 4 5530 -> 5562 GB/s; the union's shifted
// decode spilled at 48 (0.367 -> 0.358 ms).  The persistent grid is smaller than what fits:
// see persistent_grid (2 CTAs per SM for sparse lists, 3 for dense ones).
template <bool K64, uint32_t B, bool SPARSE, bool UNI = false>
__global__ void __launch_bounds__(kThreads, 4)
    lc_decode_kernel(const DecodeArgs a) {
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
    Ins ins;
    ins.rho = a.rho;
    ins.desc = (const uint2*)(base + a.warp_bytes - 256);  // UNI kernels: 256 B per warp

    uint32_t c = blockIdx.x * kWarpsPerCta + warp;
    // hint pair of the warp's next chunk, loaded one chunk ahead (hides a DRAM round trip)
    uint32_t nj0 = 0, njl = 0, nlo = 0, nhi = 0;
    if (c < a.nchunks) {
        nj0 = __ldg(sec.hint + a.chunk0 + c);
        njl = __ldg(sec.hint + a.chunk0 + c + 1);
        if (UNI) {  // the chunk's insertion range, also one chunk ahead
            nlo = __ldg(a.coff + a.chunk0 + c);
            nhi = __ldg(a.coff + a.chunk0 + c + 1);
        }
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
        if (UNI) {
            ins_begin(ins, nlo, nhi, key0, lane);
            if (c + nwarps < a.nchunks) {
                nlo = __ldg(a.coff + h + nwarps);
                nhi = __ldg(a.coff + h + nwarps + 1);
            }
        }
        const uint32_t wbytes = B ? ((((nk * B + 31) >> 5) + 1 + 3) & ~3u) * 4 : 0;
        stage(pg, sec, j0, jlast, sec.words + (size_t)h * 32 * B, wbytes, lane);
        if (UNI) ins_ready(ins);
        const bool has_next = !SPARSE && c + nwarps < a.nchunks;
        if (B && has_next && lane == 0)  // next chunk's residual words -> L2 now
            bulk_prefetch_l2(sec.words + (size_t)(h + nwarps) * 32 * B,
                             (uint32_t)min((uint64_t)(32 * B * 4 + 16),
                                       (a.nwords - (uint64_t)(h + nwarps) * 32 * B) * 4));
        uint8_t* outl = (uint8_t*)a.out + ((size_t)(key0 - a.i0) + lane) * kw;  // lane's slot
        const uint32_t nj0n = nj0, njln = njl;
        if (UNI && !ins_describe(ins, lane)) {  // rare: equal ranks or > 32 entries: streamed
            decode_chunk<K64, B, SPARSE, 2>(pg, sec, j0, jlast, key0, nk, lane, lmask, lw, ls,
                                            a.bias, outl, ins, has_next, nj0n, njln);
        } else {
            decode_chunk<K64, B, SPARSE, UNI ? 1 : 0>(pg, sec, j0, jlast, key0, nk, lane, lmask, lw,
                                                      ls, a.bias, outl, ins, has_next, nj0n, njln);
        }
    }
}

// ------------------------------------------------------------------------ batch decode
// A batch of many lists (lc_batch_init: an inverted index's posting lists)
// decoded in ONE launch: every 1024-key chunk of every list is a work unit, described by a
// host-built 48-byte record, so the persistent warps stream through all lists the same way
// lc_decode_kernel streams through one (short lists are single partial chunks).  The lists'
// residual widths differ (each list has its own eps), so the width is a runtime value
// (B = kRtB).
struct BatchChunk {
    uint64_t blob;        // device address of the list's blob (FORMAT F1: starts at byte 256)
    uint64_t out;         // output element offset of the chunk's first key
    uint32_t off_params, off_words;
    uint32_t j0, jlast;   // hint pair of the chunk (hint[h], hint[h + 1])
    uint32_t key0;        // first key of the chunk in its list (a multiple of 1024)
    uint32_t nk_b;        // keys in the chunk (1..1024) | residual width b << 16
    uint32_t bias;        // FORMAT F3 decode bias
    uint32_t list;        // list index in the batch
};
static_assert(sizeof(BatchChunk) == 48, "BatchChunk is three 16-byte loads");

// One list of a batch (64 bytes): what the set operations need to search it.
struct BatchList {
    uint64_t blob;        // device address of the list's blob
    uint64_t out;         // output element offset of the list's first key
    uint32_t n, L;
    uint32_t off_params, off_hint, off_words;
    uint32_t chunk0;      // the list's first chunk record of more than kSmallUnit keys ...
    uint32_t b, bias, eps, flags;
    uint32_t pad[2];      // [0]: ... and its small (last) chunk record, or 0xffffffff
};
static_assert(sizeof(BatchList) == 64, "BatchList is four 16-byte loads");

struct BatchArgs {
    const BatchChunk* chunks;  // the batch's chunk records
    const uint32_t* sel;       // optional selection: unit c decodes chunk sel[c] ...
    const uint64_t* sel_out;   // ... to output element offset sel_out[c] (both or neither)
    void* out;
    const uint32_t* nunits;    // optional device count of units (overrides `units` when set)
    uint32_t* work;            // work-queue counter, zero at launch
    uint32_t units;            // chunks to decode (the batch's, or the selection's)
    uint32_t small0;           // units [small0, units) are small (<= kSmallUnit keys) ...
    const uint32_t* sk0;       // ... their keys flattened: small unit u holds flat keys
                               //     [sk0[u], sk0[u + 1]), ...
    const uint32_t* sblk;      // ... sblk[f / 32] = the small unit holding flat key f (f % 32 == 0)
    uint32_t small_keys;       // flat small keys (0: no small path)
    uint32_t warp_bytes;       // shared memory per warp (widest b of the batch)
};

// Small units (a posting list of <= 64 keys is one, and most lists of a Zipf vocabulary are
// that short): their keys are flattened into one index space and decoded one THREAD per key
// from global memory (L1 / L2), 256 keys per work item, instead of one staging round trip per
// list.
constexpr uint32_t kSmallUnit = 64;
constexpr uint32_t kSmallItem = 256;  // flat small keys per work item (8 per lane)

__device__ __forceinline__ BatchChunk load_chunk(const BatchChunk* p) {
    BatchChunk r;
    const uint4* q = (const uint4*)p;
    const uint4 x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
    r.blob = ((uint64_t)x.y << 32) | x.x;
    r.out = ((uint64_t)x.w << 32) | x.z;
    r.off_params = y.x;
    r.off_words = y.y;
    r.j0 = y.z;
    r.jlast = y.w;
    r.key0 = z.x;
    r.nk_b = z.y;
    r.bias = z.z;
    r.list = z.w;
    return r;
}

template <bool K64, bool SPARSE>
__global__ void __launch_bounds__(kThreads, 4)
    lc_decode_batch_kernel(const BatchArgs a) {
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
    const uint32_t lmask = lanemask_le();
    const uint32_t nwarps = gridDim.x * kWarpsPerCta;
    const uint32_t units = a.nunits ? *a.nunits : a.units;
    Ins ins;  // unused (no insertions)
    ins.rho = nullptr;

    const uint32_t big = a.sel ? units : min(a.small0, units);
    const uint32_t ngroups = (a.small_keys + kSmallItem - 1) / kSmallItem;  // small-key items
    const uint32_t items = ngroups + big;
    // Work queue (a.work, zeroed before the launch): items [0, ngroups) are 256 flat small keys
    // each, then the big units (one warp each).  Warps take items as they finish.  The small
    // groups (a chain of dependent loads per key, 8 serial steps per group) go FIRST: spread
    // among the chunk units (every k-th item) the last ones land in the tail of the launch
    // (measured 0.176 vs 0.165 ms on the corpus; smaller groups of 32 / 64 / 128 keys, spread
    // or not, 0.166 - 0.176 ms; one group every 2 / 4 / 8 items from the start 0.167 / 0.166 /
    // 0.164 ms against 0.166: the launch is throughput-bound, not start-up bound).
    constexpr uint32_t kSmallFlag = 0x80000000u, kNone = 0xffffffffu;
    auto grab = [&]() -> uint32_t {  // small group g: g | kSmallFlag; big unit: its index; or kNone
        uint32_t v = 0;
        if (lane == 0) v = atomicAdd(a.work, 1u);
        const uint32_t t = __shfl_sync(kFull, v, 0);
        if (t >= items) return kNone;
        return t < ngroups ? (t | kSmallFlag) : t - ngroups;
    };
    auto load_big = [&](uint32_t cc, BatchChunk& rr, uint64_t& oo) {
        rr = load_chunk(a.chunks + (a.sel ? __ldg(a.sel + cc) : cc));
        oo = a.sel ? __ldg(a.sel_out + cc) : rr.out;
    };
    uint32_t item = grab();
    BatchChunk nr;  // the record of `item` when it is a big unit (loaded one item ahead)
    uint64_t nout = 0;
    if (item < kSmallFlag) load_big(item, nr, nout);
    while (item != kNone) {
        const uint32_t nitem = grab();
        if (item & kSmallFlag) {  // ---- 256 flat small keys: 8 per lane, consecutive per warp step
            const uint32_t f0 = (item & ~kSmallFlag) * kSmallItem;
            if (nitem < kSmallFlag) load_big(nitem, nr, nout);
            item = nitem;
            uint32_t u = __ldg(a.sblk + (f0 >> 5));
#pragma unroll 1
            for (uint32_t q = 0; q < kSmallItem / 32; ++q) {
                const uint32_t f = f0 + 32 * q + lane;
                if (f >= a.small_keys) break;
                while (__ldg(a.sk0 + u + 1) <= f) ++u;  // the unit holding flat key f
                const BatchChunk r = load_chunk(a.chunks + big + u);
                const uint32_t k = f - __ldg(a.sk0 + u), i = r.key0 + k;
                const uint8_t* blob = (const uint8_t*)r.blob;
                const uint32_t* S = (const uint32_t*)(blob + 256);
                uint32_t j = r.j0;
                while (j < r.jlast && __ldg(S + j + 1) <= i) ++j;  // its segment (few)
                const ulonglong2 pr = __ldg((const ulonglong2*)(blob + r.off_params) + j);
                const uint32_t b = r.nk_b >> 16;
                uint32_t uf = 0;
                if (b) {
                    const uint64_t bit = (uint64_t)i * b;
                    const uint32_t* wp = (const uint32_t*)(blob + r.off_words) + (bit >> 5);
                    uf = __funnelshift_r(__ldg(wp), __ldg(wp + 1), (uint32_t)bit & 31) &
                         (b >= 32 ? kFull : (1u << b) - 1);
                }
                const uint32_t t = pred_plus(pr.y, i - __ldg(S + j), uf - r.bias);
                uint8_t* o = (uint8_t*)a.out + (r.out + k) * kw;
                if (K64) __stcs((unsigned long long*)o, (unsigned long long)(pr.x + t));
                else __stcs((unsigned int*)o, (unsigned int)pr.x + t);
            }
            continue;
        }
        // ---- a big unit, one warp (1024-key chunks and longer partial chunks)
        const BatchChunk r = nr;
        const uint64_t out0 = nout;
        if (nitem < kSmallFlag) load_big(nitem, nr, nout);
        item = nitem;
        const uint8_t* blob = (const uint8_t*)r.blob;
        Sections sec;
        sec.starts = (const uint32_t*)(blob + 256);
        sec.params = (const ulonglong2*)(blob + r.off_params);
        sec.words = (const uint32_t*)(blob + r.off_words);
        sec.hint = nullptr;
        sec.first = nullptr;
        sec.dir = nullptr;
        sec.acc = nullptr;
        sec.L = r.jlast + 1;
        sec.W = 0;
        const uint32_t nk = r.nk_b & 0xffff, b = r.nk_b >> 16;
        pg.rb = b;
        pg.rmask = b >= 32 ? kFull : (1u << b) - 1;
        const uint32_t lw = (lane * b) >> 5, ls = (lane * b) & 31;
        const uint32_t wbytes = b ? ((((nk * b + 31) >> 5) + 1 + 3) & ~3u) * 4 : 0;
        stage(pg, sec, r.j0, r.jlast, sec.words + (size_t)(r.key0 >> 10) * 32 * b, wbytes, lane);
        uint32_t jb = r.j0, sb = pg.sS[LC_BOUND(true, r.j0 - pg.pj, pg.cs)];
        uint8_t* outl = (uint8_t*)a.out + (out0 + lane) * kw;
        const uint32_t key0 = r.key0, jlast = r.jlast;
        if (jlast < pg.pj + pg.cp) {  // every segment of the unit staged: no re-page checks
            const uint32_t nq = nk >> 7;  // whole 128-key quads
#pragma unroll 1
            for (uint32_t g = 0; g < nq; ++g, outl += 128 * kw)
                decode_quad<K64, kRtB, false, 0, SPARSE>(pg, sec, jb, sb, jlast, key0 + 128 * g,
                                                             g, lane, lmask, lw, ls, r.bias, outl,
                                                             ins);
            for (uint32_t w = 4 * nq; 32 * w < nk; ++w, outl += 32 * kw)
                decode_window<K64, kRtB, false, false, 0>(pg, sec, jb, sb, jlast, key0 + 32 * w,
                                                              w, lane, lmask, lw, ls, r.bias, outl,
                                                              nk - 32 * w, ins);
        } else if (nk == 1024) {  // dense chunk: paged
#pragma unroll 1
            for (uint32_t g = 0; g < 16; g += 4, outl += 4 * 64 * kw) {
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k)
                    decode_pair<K64, kRtB, true, 0>(pg, sec, jb, sb, jlast, key0 + 64 * (g + k),
                                                        g + k, lane, lmask, lw, ls, r.bias,
                                                        outl + 64 * kw * k, ins);
            }
        } else {  // a dense partial chunk (a list's last)
            for (uint32_t w = 0; 32 * w < nk; ++w)
                decode_window<K64, kRtB, true, false, 0>(pg, sec, jb, sb, jlast, key0 + 32 * w,
                                                             w, lane, lmask, lw, ls, r.bias,
                                                             outl + 32 * kw * w, nk - 32 * w, ins);
        }
    }
}
