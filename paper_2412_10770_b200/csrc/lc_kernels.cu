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
//    on an mbarrier (dense chunks are paged) and prefetches the next chunk into L2.  A fully
//    staged chunk is decoded as 8 quad-windows of 128 keys (a paged one as 16 pair-windows of
//    64): warp OR-reductions (REDUX) of the next 32 segment starts give the boundary bitmasks,
//    so each key gets its segment and offset with POPC/CLZ -- no per-key search and no serial
//    walk ("reduce the data dependencies ... to maximize parallelism"); sparse
//    lists take a single-segment fast path per quad.  The prediction is exact 32-bit integer
//    math (see pred_plus).  Each warp store writes 32 consecutive keys (coalesced, streaming).
//  * Random access / quantiles: hint bracket + binary search, two interleaved queries per
//    thread, L2 evict_last for the search structures and evict_first for the gathers; with the
//    access layout, a directory word instead of the search and one record per query.
//  * Batches: one launch for many lists (chunk records + a work queue; short lists' keys one
//    thread each), batched AND / OR over list pairs (lc_batchops.cuh).
//  * Range decode: one warp per 32 ranges (lane-parallel search); len == 64 gathers each
//    range's slices through a per-warp cp.async ring and decodes from shared memory; with the
//    access layout the boundary masks come from the directory bitmaps and a range is one
//    contiguous gather of its record span (no search, no starts).
//  * Successor search / intersection: binary search over the segments' first keys (the
//    anchored bases, or decoded first keys for F7 blobs: segments as skip pointers), then
//    inside one segment.
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "lc.h"
#include "lc_internal.h"

namespace {

#include "lc_common.cuh"
#include "lc_decode.cuh"
#include "lc_gather.cuh"
#include "lc_setops.cuh"
#include "lc_batchops.cuh"

// ------------------------------------------------------------------------------ launchers
uint32_t mask_of(uint32_t b) { return b >= 32 ? 0xffffffffu : ((1u << b) - 1); }

int32_t cuda_status() { return cudaGetLastError() == cudaSuccess ? LC_OK : LC_ERR_CUDA; }

// lc_decode_kernel<K64, b, SPARSE, UNI>: one instantiation per residual width b = 0..32
// (compile-time field offsets and masks), key width and kind (0 dense, 1 sparse, 2 lc_union's
// shifted decode), built in six parallel translation units (lc_decode_inst.cu)
const void* decode_kernel(int kind, bool k64, uint32_t b) {
    using namespace lc_detail;
    switch (kind * 2 + k64) {
        case 0: return decode_kernel_0_0(b);
        case 1: return decode_kernel_0_1(b);
        case 2: return decode_kernel_1_0(b);
        case 3: return decode_kernel_1_1(b);
        case 4: return decode_kernel_2_0(b);
        default: return decode_kernel_2_1(b);
    }
}

struct GridCache {
    std::mutex mu;
    int dev = -1;
    int sms = 0;
    int occ[3][2][33] = {};  // [sparse | 2 = union][K64][res_bits] -> resident CTAs per SM
};
GridCache g_grid;

// Persistent grid of the decode kernel for a launch over `nchunks` chunks: SMs x CTAs per SM.
// Fewer CTAs than fit for long lists: the decode is bound by the HBM read / write mix, and that
// mix runs faster when the offered load stays just below what HBM delivers (16-24 single-
// buffered warps per SM) than when the memory system is over-subscribed (32 warps per SM).
// Measured on B200 (ms per launch at 16 / 24 / 32 warps per SM = 2 / 3 / 4 CTAs): config 4
// (sparse) 0.724 / 0.797 / 0.802 (also -9.5% / -12% at N = 5e7 / 2e8), config 2 0.200 / 0.207 /
// 0.211, config 5 0.200 / 0.199 / 0.205, config 3 0.421 / 0.377 / 0.382 (its tail of 1-key
// segments is paged chunk by chunk: a latency chain that needs the warps), the union's shifted
// decode 0.368 / 0.341 / 0.353 (whole union); 12 warps per SM: 0.81 (config 4).  Short launches
// are latency-bound and keep every CTA that fits (N = 1e7: 4 CTAs 0.030 / 0.035 ms sparse /
// dense against 0.032 / 0.038 at 2; N = 3e7: 0.058 / 0.077 against 0.054 / 0.074 at 2 / 3).
// Only 64-bit lists: see below.
constexpr uint32_t kLongLaunchChunks = 24 * 1024;  // 2.5e7 keys
int persistent_grid(int kind, bool k64, uint32_t b, uint32_t nchunks) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_grid.mu);
    if (g_grid.dev != dev) {
        g_grid.dev = dev;
        cudaDeviceGetAttribute(&g_grid.sms, cudaDevAttrMultiProcessorCount, dev);
        std::memset(g_grid.occ, 0, sizeof g_grid.occ);
    }
    int& occ = g_grid.occ[kind][k64][b];
    if (occ == 0) {
        const void* fn = decode_kernel(kind, k64, b);
        const int smem = (int)((warp_bytes_for(b) + (kind == 2 ? 256 : 0)) * kWarpsPerCta);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem);
        if (occ < 1) occ = 1;
    }
    // u32 lists move half the bytes per key: their decode is issue-bound and keeps every warp
    // (5e7 sparse u32 keys: 0.086 / 0.076 / 0.074 ms at 2 / 3 / 4 CTAs per SM)
    const int want = (nchunks < kLongLaunchChunks || !k64) ? occ : kind == 1 ? 2 : 3;
    return (occ < want ? occ : want) * g_grid.sms;
}

// rho / coff non-null: lc_union's fused path (whole list, stores shifted by the insertions)
int32_t launch_decode(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out, cudaStream_t st,
                      const uint32_t* rho = nullptr, const uint32_t* coff = nullptr) {
    DecodeArgs a;
    a.rho = rho;
    a.coff = coff;
    a.sec = sections_of(v);
    a.out = d_out;
    a.i0 = (uint32_t)i0;
    a.i1 = (uint32_t)i1;
    a.chunk0 = (uint32_t)(i0 >> 10);
    a.nchunks = (uint32_t)((i1 - i0 + 1023) >> 10);
    a.bias = bias_of(v);
    a.nwords = v->h.n_words;
    const uint32_t b = v->h.res_bits;
    a.warp_bytes = warp_bytes_for(b) + (coff ? 256 : 0);  // union: + the window descriptors
    const uint32_t smem = a.warp_bytes * kWarpsPerCta;
    const bool k64 = v->h.key_bits == 64;
    const bool sparse = v->h.n_seg * 64 < v->h.n;  // < 1 segment per 64 keys
    const int kind = coff ? 2 : sparse;
    const int full = persistent_grid(kind, k64, b, a.nchunks);
    const uint32_t need = (a.nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
    const uint32_t grid = need < (uint32_t)full ? need : (uint32_t)full;
    void* args[] = {&a};
    if (cudaLaunchKernel(decode_kernel(kind, k64, b), dim3(grid), dim3(kThreads), args, smem, st) !=
        cudaSuccess)
        return LC_ERR_CUDA;
    lc_detail::count_launch(1);
    return cuda_status();
}

// batch decode: units [0, units) of the batch's chunk records (or of a selection sel/sel_out;
// nunits: optional device count)
const void* batch_kernel(bool k64, bool sparse) {
    if (k64) return sparse ? (const void*)lc_decode_batch_kernel<true, true>
                           : (const void*)lc_decode_batch_kernel<true, false>;
    return sparse ? (const void*)lc_decode_batch_kernel<false, true>
                  : (const void*)lc_decode_batch_kernel<false, false>;
}

int32_t launch_batch_decode(const lc_batch* b, const uint32_t* sel, const uint64_t* sel_out,
                            const uint32_t* nunits, uint32_t units, void* d_out, uint32_t* work,
                            cudaStream_t st) {
    if (cudaMemsetAsync(work, 0, sizeof(uint32_t), st) != cudaSuccess) return LC_ERR_CUDA;
    BatchArgs a;
    a.work = work;
    a.small0 = sel ? units : (uint32_t)(b->n_chunks - b->n_small);
    a.sk0 = (const uint32_t*)b->d_small;
    a.sblk = a.sk0 ? a.sk0 + b->n_small + 1 : nullptr;
    a.small_keys = sel ? 0 : (uint32_t)b->small_keys;
    a.chunks = (const BatchChunk*)b->d_chunks;
    a.sel = sel;
    a.sel_out = sel_out;
    a.out = d_out;
    a.nunits = nunits;
    a.units = units;
    a.warp_bytes = warp_bytes_for(b->max_res_bits);
    const uint32_t smem = a.warp_bytes * kWarpsPerCta;
    const bool k64 = b->key_bits == 64;
    const void* fn = batch_kernel(k64, b->sparse);
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem);
    const uint32_t full = (uint32_t)(sms * (occ > 0 ? occ : 1));
    const uint32_t need = (units + kWarpsPerCta - 1) / kWarpsPerCta;
    const uint32_t grid = nunits ? full : (need + 1 < full ? need + 1 : full);
    if (!grid) return LC_OK;
    void* args[] = {&a};
    if (cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem, st) != cudaSuccess)
        return LC_ERR_CUDA;
    lc_detail::count_launch(1);
    return cuda_status();
}

// lc_decode_host pipeline resources: an H2D and a D2H copy stream plus one event per span and
// stage.  Pipes are pooled per device: a call takes a free pipe of its device (creating one
// when every pipe is busy enqueueing), so concurrent callers never share events and never hold
// a lock while they enqueue; pipes live until process exit.
constexpr uint32_t kMaxSpans = 64;
struct HostPipe {
    int dev = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t up[kMaxSpans] = {}, dec[kMaxSpans] = {}, done = nullptr;
};
std::mutex g_pipe_mu;
std::vector<HostPipe*> g_pipe_free;  // idle pipes of every device

void pipe_destroy(HostPipe* p) {
    if (p->h2d) cudaStreamDestroy(p->h2d);
    if (p->d2h) cudaStreamDestroy(p->d2h);
    if (p->done) cudaEventDestroy(p->done);
    for (uint32_t k = 0; k < kMaxSpans; ++k) {
        if (p->up[k]) cudaEventDestroy(p->up[k]);
        if (p->dec[k]) cudaEventDestroy(p->dec[k]);
    }
    delete p;
}

HostPipe* pipe_acquire() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pipe_mu);
        for (size_t k = 0; k < g_pipe_free.size(); ++k)
            if (g_pipe_free[k]->dev == dev) {
                HostPipe* p = g_pipe_free[k];
                g_pipe_free.erase(g_pipe_free.begin() + k);
                return p;
            }
    }
    HostPipe* p = new HostPipe;
    p->dev = dev;
    bool ok = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) == cudaSuccess;
    for (uint32_t k = 0; ok && k < kMaxSpans; ++k)
        ok = cudaEventCreateWithFlags(&p->up[k], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&p->dec[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {  // partially created: release what exists
        pipe_destroy(p);
        return nullptr;
    }
    return p;
}

void pipe_release(HostPipe* p) {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    g_pipe_free.push_back(p);
}

// host->device copy of `bytes` bytes
int32_t copy_up(void* d, const void* h, uint64_t bytes, cudaStream_t st) {
    if (!bytes) return LC_OK;
    return cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess ? LC_OK
                                                                                : LC_ERR_CUDA;
}

// The blob slices the decode of keys [i0, i1) reads (FORMAT F2 sections; exactly what
// lc_decode_kernel stages and prefetches for chunks [c0, c1)): hint[c0 .. c1], starts
// [s_lo, s_hi), params [p_lo, p_hi), words [w_lo, w_hi).  The bounds come from the hint
// values, so the hint slice is checked (non-decreasing, within [0, L - 1]) before use: a
// corrupt hint returns LC_ERR_FORMAT instead of sizing copies past the sections.
struct SpanSlices {
    uint64_t c0, c1, s_lo, s_hi, p_lo, p_hi, w_lo, w_hi;
};
int32_t span_slices(const lc_header& h, const uint8_t* blob, uint64_t i0, uint64_t i1,
                    SpanSlices* o) {
    const uint32_t* hint = (const uint32_t*)(blob + h.off_hint);
    const uint64_t H = h.n_hint - 1, L = h.n_seg, b = h.res_bits;
    o->c0 = i0 >> 10;
    o->c1 = (i1 + 1023) >> 10;  // <= H
    for (uint64_t c = o->c0; c <= o->c1; ++c)
        if (hint[c] >= L || (c > o->c0 && hint[c] < hint[c - 1])) return LC_ERR_FORMAT;
    const uint64_t j0 = hint[o->c0], j1 = hint[o->c1 < H ? o->c1 : H];
    const uint64_t r4 = (L + 1 + 3) & ~3ULL;  // starts entries inside the 256-byte-padded section
    o->s_lo = j0 & ~3ULL;
    o->s_hi = ((j1 + 2 + 3) & ~3ULL) < r4 ? ((j1 + 2 + 3) & ~3ULL) : r4;
    o->p_lo = j0 & ~3ULL;
    o->p_hi = j1 + 1;
    o->w_lo = b ? o->c0 * 32 * b : 0;
    o->w_hi = b ? (o->c1 * 32 * b + 4 < h.n_words ? o->c1 * 32 * b + 4 : h.n_words) : 0;
    return LC_OK;
}

// shard buffer layout: hint | starts | params | words slices, each 256-byte aligned
struct ShardLayout {
    uint64_t o_hint, o_starts, o_params, o_words, total;
};
ShardLayout shard_layout(const SpanSlices& sl) {
    auto r256_ = [](uint64_t x) { return (x + 255) & ~255ULL; };
    ShardLayout y;
    y.o_hint = 0;
    y.o_starts = r256_(4 * (sl.c1 - sl.c0 + 1));
    y.o_params = y.o_starts + r256_(4 * (sl.s_hi - sl.s_lo));
    y.o_words = y.o_params + r256_(16 * (sl.p_hi - sl.p_lo));
    y.total = y.o_words + r256_(4 * (sl.w_hi - sl.w_lo));
    return y;
}

// header + span checks shared by lc_shard_bytes / lc_shard_upload
int32_t shard_plan(const void* h_blob, uint64_t blob_bytes, uint64_t i0, uint64_t i1,
                   lc_header* h, SpanSlices* sl) {
    if (!h_blob) return LC_ERR_ARG;
    if (blob_bytes < sizeof(lc_header)) return LC_ERR_FORMAT;
    std::memcpy(h, h_blob, sizeof *h);
    int32_t st = lc_detail::check_header(h, blob_bytes);
    if (st) return st;
    if ((i0 & 1023) || i0 >= i1 || i1 > h->n) return LC_ERR_ARG;
    return span_slices(*h, (const uint8_t*)h_blob, i0, i1, sl);
}

// queries per thread of the access-layout kernel (LC_ACC_Q = 1 | 2 | 4 overrides, for A/B)
int acc_queries_per_thread() {
    static const int q = [] {
        const char* e = std::getenv("LC_ACC_Q");
        const int x = e ? std::atoi(e) : 0;
        return x == 1 || x == 2 || x == 4 ? x : 1;
    }();
    return q;
}

// f(K64, MODE, Q) with compile-time constants
template <typename F>
void dispatch_acc(bool k64, int mode, int qp, F&& f) {
    auto with_k = [&](auto K) {
        auto with_m = [&](auto M) {
            if (qp == 1) f(K, M, std::integral_constant<int, 1>{});
            else if (qp == 4) f(K, M, std::integral_constant<int, 4>{});
            else f(K, M, std::integral_constant<int, 2>{});
        };
        if (mode == kAccess) with_m(std::integral_constant<int, kAccess>{});
        else if (mode == kQuantileExact) with_m(std::integral_constant<int, kQuantileExact>{});
        else with_m(std::integral_constant<int, kQuantileApprox>{});
    };
    if (k64) with_k(std::true_type{});
    else with_k(std::false_type{});
}

int32_t launch_access(const lc_view* v, const uint64_t* d_in, uint64_t q, uint64_t qdiv, int mode,
                      void* d_out, uint32_t* d_err, cudaStream_t st) {
    AccessArgs a;
    a.sec = sections_of(v);
    a.idx = d_in;
    a.out = d_out;
    a.err = d_err;
    a.q = q;
    a.qdiv = qdiv;
    a.n = (uint32_t)v->h.n;
    a.b = v->h.res_bits;
    a.bias = bias_of(v);
    a.center = v->h.eps - a.bias;
    a.mask = mask_of(a.b);
    const uint64_t per = 256 * access_per_thread(mode);
    const uint64_t grid = (q + per - 1) / per;
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    const unsigned g = (unsigned)grid;
    const bool k64 = v->h.key_bits == 64;
    if (v->d_acc) {  // access layout attached: no binary search, one record per query
        const int q_per = acc_queries_per_thread();
        const uint64_t per2 = 256ull * q_per;
        const uint64_t grid2 = (q + per2 - 1) / per2;
        if (grid2 > 0x7fffffffULL) return LC_ERR_ARG;
        dispatch_acc(k64, mode, q_per, [&](auto K, auto M, auto Q) {
            lc_access_dir_kernel<decltype(K)::value, decltype(M)::value, decltype(Q)::value>
                <<<(unsigned)grid2, 256, 0, st>>>(a);
        });
        lc_detail::count_launch(1);
        return cuda_status();
    }
    switch (mode) {
        case kAccess:
            if (k64) lc_access_kernel<true, kAccess><<<g, 256, 0, st>>>(a);
            else lc_access_kernel<false, kAccess><<<g, 256, 0, st>>>(a);
            break;
        case kQuantileExact:
            if (k64) lc_access_kernel<true, kQuantileExact><<<g, 256, 0, st>>>(a);
            else lc_access_kernel<false, kQuantileExact><<<g, 256, 0, st>>>(a);
            break;
        default:
            if (k64) lc_access_kernel<true, kQuantileApprox><<<g, 256, 0, st>>>(a);
            else lc_access_kernel<false, kQuantileApprox><<<g, 256, 0, st>>>(a);
    }
    lc_detail::count_launch(1);
    return cuda_status();
}

uint64_t r256(uint64_t x) { return (x + 255) & ~255ULL; }

// f(K64, FREE, IDX) with the three flags as compile-time constants (std::bool_constant)
template <typename F>
void dispatch3(bool k64, bool free, bool idx, F&& f) {
    using T = std::true_type;
    using N = std::false_type;
    if (k64) {
        if (free) idx ? f(T{}, T{}, T{}) : f(T{}, T{}, N{});
        else idx ? f(T{}, N{}, T{}) : f(T{}, N{}, N{});
    } else {
        if (free) idx ? f(N{}, T{}, T{}) : f(N{}, T{}, N{});
        else idx ? f(N{}, N{}, T{}) : f(N{}, N{}, N{});
    }
}
}  // namespace

extern "C" {

int32_t lc_decode_span(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out, lc_stream stream) {
    if (!v || !v->d_blob) return LC_ERR_ARG;
    if (i0 > i1 || i1 > v->h.n) return LC_ERR_ARG;
    if (i0 == i1) return LC_OK;  // an empty span (e.g. a shard past the end) is a no-op
    if (is_shard(v) && (i0 < v->span_lo || i1 > v->span_hi)) return LC_ERR_ARG;
    if (i0 & 1023) return LC_ERR_ARG;
    if (!d_out || ((uintptr_t)d_out & 15)) return LC_ERR_ARG;
    return launch_decode(v, i0, i1, d_out, (cudaStream_t)stream);
}

int32_t lc_decode(const lc_view* v, void* d_out, lc_stream stream) {
    if (!v) return LC_ERR_ARG;
    if (is_shard(v)) return lc_decode_span(v, v->span_lo, v->span_hi, d_out, stream);
    return lc_decode_span(v, 0, v->h.n, d_out, stream);
}

int32_t lc_access(const lc_view* v, const uint64_t* d_idx, uint64_t q, void* d_out,
                  uint32_t* d_err, lc_stream stream) {
    if (!v || !v->d_blob || is_shard(v)) return LC_ERR_ARG;
    if (q == 0) return LC_OK;
    if (!d_idx || !d_out) return LC_ERR_ARG;
    return launch_access(v, d_idx, q, 1, kAccess, d_out, d_err, (cudaStream_t)stream);
}

int32_t lc_range_decode(const lc_view* v, const uint64_t* d_start, uint64_t q, uint32_t len,
                        void* d_out, uint32_t* d_err, lc_stream stream) {
    if (!v || !v->d_blob || is_shard(v)) return LC_ERR_ARG;
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
    a.bias = bias_of(v);
    a.mask = mask_of(a.b);
    a.nwords = v->h.n_words;
    const uint64_t grid = (q + 255) / 256;  // 8 warps x 32 ranges per CTA
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    const bool k64 = v->h.key_bits == 64;
    cudaStream_t st = (cudaStream_t)stream;
    if (len <= 64 && v->d_acc) {  // access layout attached: no search, one contiguous gather
        const uint32_t smem = kRdWarps * rd_smem_per_warp();
        const uint64_t grid = (q + 32 * kRdWarps - 1) / (32 * kRdWarps);
        const void* fn = len == 64 ? (k64 ? (const void*)lc_range64_dir_kernel<true, true>
                                          : (const void*)lc_range64_dir_kernel<false, true>)
                                   : (k64 ? (const void*)lc_range64_dir_kernel<true, false>
                                          : (const void*)lc_range64_dir_kernel<false, false>);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, kRdCarveout);
        void* args[] = {&a};
        if (cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(32 * kRdWarps), args, smem, st) != cudaSuccess)
            return LC_ERR_CUDA;
        lc_detail::count_launch(1);
        return cuda_status();
    }
    if (len <= 64) {  // the config-5 shape (and shorter): cp.async ring kernel
        const uint32_t smem = 8 * r64_smem_per_warp(a.b);
        const void* fn = len == 64 ? (k64 ? (const void*)lc_range64_kernel<true, true>
                                          : (const void*)lc_range64_kernel<false, true>)
                                   : (k64 ? (const void*)lc_range64_kernel<true, false>
                                          : (const void*)lc_range64_kernel<false, false>);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        void* args[] = {&a};
        if (cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(256), args, smem, st) != cudaSuccess)
            return LC_ERR_CUDA;
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
    if (!v || !v->d_blob || is_shard(v)) return LC_ERR_ARG;
    if (q == 0 || q > 0xffffffffULL) return LC_ERR_ARG;  // N k < 2^64 for k <= q
    if (m == 0) return LC_OK;
    if (!d_k || !d_out) return LC_ERR_ARG;
    return launch_access(v, d_k, m, q, exact ? kQuantileExact : kQuantileApprox, d_out, d_err,
                         (cudaStream_t)stream);
}

int32_t lc_next_geq(const lc_view* v, const uint64_t* d_x, uint64_t m, uint64_t* d_out_idx,
                    void* d_out_key, lc_stream stream) {
    if (!v || !v->d_blob || is_shard(v)) return LC_ERR_ARG;
    if (m == 0) return LC_OK;
    if (!d_x || (!d_out_idx && !d_out_key)) return LC_ERR_ARG;
    SuccArgs a;
    a.sec = sections_of(v);
    a.x = d_x;
    a.out_idx = d_out_idx;
    a.out_key = d_out_key;
    a.m = m;
    a.band = 2 * (uint64_t)v->h.eps;
    a.n = (uint32_t)v->h.n;
    a.L = (uint32_t)v->h.n_seg;
    a.b = v->h.res_bits;
    a.bias = bias_of(v);
    a.mask = mask_of(a.b);
    const uint64_t grid = (m + 256 * kSuccQ - 1) / (256 * kSuccQ);
    if (grid > 0x7fffffffULL) return LC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)grid;
    dispatch3(v->h.key_bits == 64, is_free(v), v->d_first != nullptr, [&](auto K, auto F, auto I) {
        lc_next_geq_kernel<decltype(K)::value, decltype(F)::value, decltype(I)::value>
            <<<g, 256, 0, st>>>(a);
    });
    lc_detail::count_launch(1);
    return cuda_status();
}

uint64_t lc_search_index_bytes(const lc_view* v) {
    if (!v) return 0;
    const uint64_t L = v->h.n_seg;
    return 8 * (idx_sample_off(L) + (L + kIdxStride - 1) / kIdxStride);
}

int32_t lc_search_index_build(lc_view* v, void* d_index, lc_stream stream) {
    if (!v || !v->d_blob || is_shard(v) || !d_index || ((uintptr_t)d_index & 127)) return LC_ERR_ARG;
    const Sections sec = sections_of(v);
    const uint32_t b = v->h.res_bits;
    const unsigned grid = (unsigned)((v->h.n_seg + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    if (is_free(v)) lc_first_kernel<true><<<grid, 256, 0, st>>>(sec, (uint64_t*)d_index, b, mask_of(b), bias_of(v));
    else lc_first_kernel<false><<<grid, 256, 0, st>>>(sec, (uint64_t*)d_index, b, mask_of(b), bias_of(v));
    lc_detail::count_launch(1);
    const int32_t rc = cuda_status();
    if (!rc) v->d_first = (const uint64_t*)d_index;
    return rc;
}

uint64_t lc_access_layout_bytes(const lc_view* v) {
    if (!v) return 0;
    const uint64_t H = v->h.n_hint - 1;
    return 256 * H + 16 * (2 * v->h.n_seg + ((v->h.n * v->h.res_bits) >> 7));
}

int32_t lc_access_layout_build(lc_view* v, void* d_layout, lc_stream stream) {
    if (!v || !v->d_blob || is_shard(v) || !d_layout || ((uintptr_t)d_layout & 127)) return LC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    lc_view t = *v;
    t.d_acc = d_layout;
    const Sections sec = sections_of(&t);
    const uint64_t H = v->h.n_hint - 1, L = v->h.n_seg;
    if (cudaMemsetAsync(d_layout, 0, 256 * H, st) != cudaSuccess) return LC_ERR_CUDA;
    if (L > 1) lc_acc_bits_kernel<<<(unsigned)((L - 1 + 255) / 256), 256, 0, st>>>(sec, (uint2*)sec.dir);
    lc_acc_dir_kernel<<<(unsigned)((H + 7) / 8), 256, 0, st>>>(sec, (uint2*)sec.dir, (uint32_t)H);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (L + 7) / 8;  // one warp per segment, 8 warps per CTA
    const unsigned grid = (unsigned)(want < (uint64_t)sms * 16 ? want : (uint64_t)sms * 16);
    lc_acc_build_kernel<<<grid, 256, 0, st>>>(sec, (ulonglong2*)sec.acc, v->h.res_bits);
    lc_detail::count_launch(L > 1 ? 3 : 2);
    const int32_t rc = cuda_status();
    if (!rc) v->d_acc = d_layout;
    return rc;
}

uint64_t lc_intersect_scratch_bytes(const lc_view* a) {
    if (!a) return 0;
    const uint64_t na = a->h.n, kw = a->h.key_bits / 8;
    const uint64_t nblk = (na + 255) / 256;
    return r256(na * kw) + r256(4 * ((na + 31) / 32)) + r256(4 * (nblk + 1));
}

int32_t lc_intersect(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                     void* d_out, uint64_t* d_count, lc_stream stream) {
    if (!a || !b || !a->d_blob || !b->d_blob || !d_scratch || !d_out || !d_count) return LC_ERR_ARG;
    if (is_shard(a) || is_shard(b)) return LC_ERR_ARG;
    if (a->h.key_bits != b->h.key_bits) return LC_ERR_ARG;
    if (scratch_bytes < lc_intersect_scratch_bytes(a) || ((uintptr_t)d_scratch & 255)) return LC_ERR_ARG;
    // symmetric: decode the shorter list and search the longer one (the scratch and output sized
    // for a also hold the shorter list and the intersection)
    if (b->h.n < a->h.n) std::swap(a, b);
    const uint64_t na = a->h.n, kw = a->h.key_bits / 8;
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
    g.bias = bias_of(b);
    g.band = 2 * (uint64_t)b->h.eps;
    g.mask = mask_of(g.b);
    g.nblk = (uint32_t)((na + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    int32_t rc = launch_decode(a, 0, na, sc, st);
    if (rc) return rc;
    const unsigned fgrid = (g.nblk + kIsectQ - 1) / kIsectQ;
    dispatch3(kw == 8, is_free(b), b->d_first != nullptr, [&](auto K, auto F, auto I) {
        lc_isect_flag_kernel<decltype(K)::value, decltype(F)::value, decltype(I)::value>
            <<<fgrid, 256, 0, st>>>(g);
    });
    lc_isect_scan_kernel<<<1, 1024, 0, st>>>(g);
    if (kw == 8) lc_isect_write_kernel<true><<<g.nblk, 256, 0, st>>>(g);
    else lc_isect_write_kernel<false><<<g.nblk, 256, 0, st>>>(g);
    lc_detail::count_launch(3);
    return cuda_status();
}

uint64_t lc_union_scratch_bytes(const lc_view* a, const lc_view* b) {
    if (!a || !b) return 0;
    const uint64_t na = a->h.n, nb = b->h.n, kw = a->h.key_bits / 8;
    const uint64_t ns = na < nb ? na : nb, nl = na < nb ? nb : na;
    const uint64_t nblk = (ns + 255) / 256;
    // short keys, rank, flags, counts, rho, coff
    return r256(ns * kw) + r256(4 * ns) + r256(4 * ((ns + 31) / 32)) + r256(4 * (nblk + 1)) +
           r256(4 * ns) + r256(4 * ((nl + 1023) / 1024 + 1));
}

int32_t lc_union(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                 void* d_out, uint64_t* d_count, lc_stream stream) {
    if (!a || !b || !a->d_blob || !b->d_blob || !d_scratch || !d_out || !d_count) return LC_ERR_ARG;
    if (is_shard(a) || is_shard(b)) return LC_ERR_ARG;
    if (a->h.key_bits != b->h.key_bits) return LC_ERR_ARG;
    if (scratch_bytes < lc_union_scratch_bytes(a, b) || ((uintptr_t)d_scratch & 255)) return LC_ERR_ARG;
    if ((uintptr_t)d_out % (a->h.key_bits / 8)) return LC_ERR_ARG;
    // union = long ∪ (short \ long): only the shorter list is decoded, searched and compacted
    const lc_view* lg = a->h.n >= b->h.n ? a : b;
    const lc_view* sh = a->h.n >= b->h.n ? b : a;
    const uint64_t nl = lg->h.n, ns = sh->h.n, kw = a->h.key_bits / 8;
    cudaStream_t st = (cudaStream_t)stream;
    const bool k64 = kw == 8;
    uint8_t* p = (uint8_t*)d_scratch;
    uint8_t* sS = p;
    uint32_t* rank = (uint32_t*)(p += r256(ns * kw));
    uint32_t* flags = (uint32_t*)(p += r256(4 * ns));
    const uint64_t nblk = (ns + 255) / 256;
    uint32_t* counts = (uint32_t*)(p += r256(4 * ((ns + 31) / 32)));
    uint32_t* rho = (uint32_t*)(p += r256(4 * (nblk + 1)));
    uint32_t* coff = (uint32_t*)(p += r256(4 * ns));
    IsectArgs g{};
    g.sb = sections_of(lg);
    g.a_keys = sS;
    g.flags = flags;
    g.counts = counts;
    g.out = d_out;
    g.d_count = d_count;  // |C| after the scan, then nl + |C|
    g.na = (uint32_t)ns;
    g.nb = (uint32_t)nl;
    g.Lb = (uint32_t)lg->h.n_seg;
    g.b = lg->h.res_bits;
    g.bias = bias_of(lg);
    g.band = 2 * (uint64_t)lg->h.eps;
    g.mask = mask_of(g.b);
    g.nblk = (uint32_t)nblk;
    int32_t rc = launch_decode(sh, 0, ns, sS, st);
    if (rc) return rc;
    const unsigned fgrid = (g.nblk + kIsectQ - 1) / kIsectQ;
    dispatch3(k64, is_free(lg), lg->d_first != nullptr, [&](auto K, auto F, auto I) {
        lc_union_rank_kernel<decltype(K)::value, decltype(F)::value, decltype(I)::value>
            <<<fgrid, 256, 0, st>>>(g, rank);
    });
    lc_isect_scan_kernel<<<1, 1024, 0, st>>>(g);
    if (k64) lc_union_place_kernel<true><<<g.nblk, 256, 0, st>>>(g, rank, rho);
    else lc_union_place_kernel<false><<<g.nblk, 256, 0, st>>>(g, rank, rho);
    const uint32_t H = (uint32_t)((nl + 1023) / 1024);
    lc_union_coff_kernel<<<(H + 1 + 255) / 256, 256, 0, st>>>(rho, counts + g.nblk, H, coff, nl,
                                                                d_count);
    lc_detail::count_launch(4);
    if ((rc = cuda_status())) return rc;
    return launch_decode(lg, 0, nl, d_out, st, rho, coff);
}

int32_t lc_shard_bytes(const void* h_blob, uint64_t blob_bytes, uint64_t i0, uint64_t i1,
                       uint64_t* shard_bytes) {
    if (!shard_bytes) return LC_ERR_ARG;
    lc_header h;
    SpanSlices sl;
    const int32_t st = shard_plan(h_blob, blob_bytes, i0, i1, &h, &sl);
    if (st) return st;
    *shard_bytes = shard_layout(sl).total;
    return LC_OK;
}

int32_t lc_shard_upload(const void* h_blob, uint64_t blob_bytes, uint64_t i0, uint64_t i1,
                        void* d_shard, uint64_t shard_bytes, lc_view* v, lc_stream stream) {
    if (!v || !d_shard || ((uintptr_t)d_shard & 255)) return LC_ERR_ARG;
    lc_header h;
    SpanSlices sl;
    int32_t st = shard_plan(h_blob, blob_bytes, i0, i1, &h, &sl);
    if (st) return st;
    const ShardLayout y = shard_layout(sl);
    if (shard_bytes < y.total) return LC_ERR_ARG;
    const uint8_t* B = (const uint8_t*)h_blob;
    uint8_t* D = (uint8_t*)d_shard;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = copy_up(D + y.o_hint, B + h.off_hint + 4 * sl.c0, 4 * (sl.c1 - sl.c0 + 1), s)) ||
        (st = copy_up(D + y.o_starts, B + h.off_starts + 4 * sl.s_lo, 4 * (sl.s_hi - sl.s_lo), s)) ||
        (st = copy_up(D + y.o_params, B + h.off_params + 16 * sl.p_lo, 16 * (sl.p_hi - sl.p_lo), s)) ||
        (st = copy_up(D + y.o_words, B + h.off_words + 4 * sl.w_lo, 4 * (sl.w_hi - sl.w_lo), s)))
        return st;
    v->h = h;
    v->d_blob = d_shard;
    v->d_first = nullptr;
    v->span_lo = i0;
    v->span_hi = i1;
    // section base addresses as if the whole sections were present (wrapping 64-bit address
    // arithmetic; the kernels only dereference indices inside the uploaded slices)
    const uint64_t d = (uint64_t)(uintptr_t)d_shard;
    v->sec_base[0] = d + y.o_starts - 4 * sl.s_lo;
    v->sec_base[1] = d + y.o_params - 16 * sl.p_lo;
    v->sec_base[2] = d + y.o_hint - 4 * sl.c0;
    v->sec_base[3] = d + y.o_words - 4 * sl.w_lo;
    return cuda_status();
}

// ---------------------------------------------------------------------------- batches
namespace {
int32_t batch_scan(const void* h_blobs, uint64_t h_bytes, const uint64_t* blob_off, uint32_t m,
                   uint64_t* n_chunks, uint32_t* key_bits, uint64_t* n_small = nullptr,
                   uint64_t* small_keys = nullptr) {
    if (!h_blobs || !blob_off || !m || !n_chunks) return LC_ERR_ARG;
    uint64_t c = 0, ns = 0, sk = 0;
    for (uint32_t k = 0; k < m; ++k) {
        if ((blob_off[k] & 255) || blob_off[k] + sizeof(lc_header) > h_bytes) return LC_ERR_ARG;
        lc_header h;
        std::memcpy(&h, (const uint8_t*)h_blobs + blob_off[k], sizeof h);
        const int32_t st = lc_detail::check_header(&h, h_bytes - blob_off[k]);
        if (st) return st;
        if (k == 0) *key_bits = h.key_bits;
        else if (h.key_bits != *key_bits) return LC_ERR_ARG;
        c += h.n_hint - 1;
        const uint64_t tail = h.n & 1023;
        if (tail && tail <= kSmallUnit) {
            ++ns;
            sk += tail;
        }
    }
    *n_chunks = c;
    if (n_small) *n_small = ns;
    if (small_keys) *small_keys = sk;
    return LC_OK;
}
}  // namespace

int32_t lc_batch_dir_bytes(const void* h_blobs, uint64_t h_bytes, const uint64_t* blob_off,
                           uint32_t m, uint64_t* dir_bytes) {
    if (!dir_bytes) return LC_ERR_ARG;
    uint64_t nc = 0, ns = 0, sk = 0;
    uint32_t kb = 0;
    const int32_t st = batch_scan(h_blobs, h_bytes, blob_off, m, &nc, &kb, &ns, &sk);
    if (st) return st;
    *dir_bytes = sizeof(BatchList) * (uint64_t)m + sizeof(BatchChunk) * nc + 4 * (ns + 1) +
                 4 * ((sk + 31) / 32);
    return LC_OK;
}

int32_t lc_batch_init(lc_batch* b, const void* h_blobs, uint64_t h_bytes, const uint64_t* blob_off,
                      uint32_t m, const void* d_blobs, const uint64_t* out_off, void* d_dir,
                      uint64_t dir_bytes, lc_stream stream) {
    if (!b || !d_blobs || ((uintptr_t)d_blobs & 255) || !d_dir || ((uintptr_t)d_dir & 15))
        return LC_ERR_ARG;
    uint64_t nc = 0, nsm = 0, skeys = 0;
    uint32_t kb = 0;
    int32_t st = batch_scan(h_blobs, h_bytes, blob_off, m, &nc, &kb, &nsm, &skeys);
    if (st) return st;
    if (nc >= (1ULL << 32) || skeys >= (1ULL << 32)) return LC_ERR_TOO_LARGE;
    const uint64_t o_small = sizeof(BatchList) * (uint64_t)m + sizeof(BatchChunk) * nc;
    const uint64_t need = o_small + 4 * (nsm + 1) + 4 * ((skeys + 31) / 32);
    if (dir_bytes < need) return LC_ERR_ARG;
    std::vector<uint8_t> host(need);
    BatchList* lists = (BatchList*)host.data();
    BatchChunk* chunks = (BatchChunk*)(host.data() + sizeof(BatchList) * (uint64_t)m);
    // chunk records: units of more than kSmallUnit keys first (one warp each), then the small
    // ones (their keys flattened, one thread per key); a list's chunk0 is its first record
    const uint64_t nsmall = nsm;
    uint32_t* sk0 = (uint32_t*)(host.data() + o_small);        // small chunk -> first flat key
    uint32_t* sblk = sk0 + nsm + 1;                             // 32 flat keys -> small chunk
    uint64_t flat = 0;
    uint64_t c = 0, cs = nc - nsmall, pos = 0, segs = 0, payload = 0;
    uint32_t maxb = 0;
    for (uint32_t k = 0; k < m; ++k) {
        const uint8_t* B = (const uint8_t*)h_blobs + blob_off[k];
        lc_header h;
        std::memcpy(&h, B, sizeof h);
        const uint64_t H = h.n_hint - 1, L = h.n_seg;
        const uint32_t* hint = (const uint32_t*)(B + h.off_hint);
        for (uint64_t q = 0; q <= H; ++q)  // chunk records copy the hint pairs: check them
            if (hint[q] >= L || (q && hint[q] < hint[q - 1])) return LC_ERR_FORMAT;
        const uint64_t out = out_off ? out_off[k] : pos;
        const uint32_t bias = bias_of_header(h);
        BatchList& e = lists[k];
        e.blob = (uint64_t)(uintptr_t)d_blobs + blob_off[k];
        e.out = out;
        e.n = (uint32_t)h.n;
        e.L = (uint32_t)L;
        e.off_params = (uint32_t)h.off_params;
        e.off_hint = (uint32_t)h.off_hint;
        e.off_words = (uint32_t)h.off_words;
        e.chunk0 = (uint32_t)c;
        e.b = h.res_bits;
        e.bias = bias;
        e.eps = h.eps;
        e.flags = h.flags;
        e.pad[1] = 0;
        const uint64_t tail = h.n & 1023;
        e.pad[0] = tail && tail <= kSmallUnit ? (uint32_t)cs : 0xffffffffu;  // small record
        if (h.off_words >= (1ULL << 32)) return LC_ERR_TOO_LARGE;
        for (uint64_t q = 0; q < H; ++q) {
            const uint64_t nkq = h.n - (q << 10) < 1024 ? h.n - (q << 10) : 1024;
            if (nkq <= kSmallUnit) {  // flattened small keys [flat, flat + nkq)
                const uint64_t u = cs - (nc - nsmall);
                sk0[u] = (uint32_t)flat;
                for (uint64_t f = (flat + 31) & ~31ULL; f < flat + nkq; f += 32) sblk[f >> 5] = (uint32_t)u;
                flat += nkq;
            }
            BatchChunk& r = chunks[nkq <= kSmallUnit ? cs++ : c++];
            r.blob = e.blob;
            r.out = out + (q << 10);
            r.off_params = e.off_params;
            r.off_words = e.off_words;
            r.j0 = hint[q];
            r.jlast = hint[q + 1];
            r.key0 = (uint32_t)(q << 10);
            r.nk_b = (uint32_t)nkq | ((uint32_t)h.res_bits << 16);
            r.bias = bias;
            r.list = k;
        }
        pos += h.n;
        segs += L;
        maxb = h.res_bits > maxb ? h.res_bits : maxb;
        // what a decode reads: header, starts, params, hint, words (no alignment padding)
        payload += sizeof(lc_header) + 4 * (L + 1) + 16 * L + 4 * h.n_hint +
                   4 * ((h.n * h.res_bits + 31) / 32);
    }
    sk0[nsmall] = (uint32_t)flat;
    if (cudaMemcpyAsync(d_dir, host.data(), need, cudaMemcpyHostToDevice, (cudaStream_t)stream) !=
        cudaSuccess)
        return LC_ERR_CUDA;
    b->m = m;
    b->key_bits = kb;
    b->max_res_bits = maxb;
    b->sparse = segs * 64 < pos;
    b->n_total = pos;
    b->n_chunks = nc;
    b->n_small = nsmall;
    b->small_keys = skeys;
    b->payload_bytes = payload;
    b->d_lists = d_dir;
    b->d_chunks = (const uint8_t*)d_dir + sizeof(BatchList) * (uint64_t)m;
    b->d_small = (const uint8_t*)d_dir + o_small;
    return LC_OK;
}

namespace {
// Scratch layout of a batched AND / OR (lc_batchops.cuh) from the plan's totals.
struct SetopLayout {
    uint64_t nwords, nblk;
    uint64_t o_sl, o_soff, o_loff, o_cap, o_uoff, o_sel, o_selout, o_blks, o_blkl, o_keys,
        o_flags, o_mw, o_counts, o_rank, o_misc, total;
};
SetopLayout setop_layout(const lc_setop_plan& q, uint32_t key_bits) {
    const uint64_t P = q.n_pairs, S = q.short_keys, Lt = q.long_keys, U = q.units;
    SetopLayout y;
    y.nwords = (S + 31) / 32 + 1;
    y.nblk = (S + 255) / 256;
    y.o_sl = 0;
    y.o_soff = r256(8ULL * P);
    y.o_loff = y.o_soff + r256(8 * (P + 1));
    y.o_cap = y.o_loff + r256(8 * (P + 1));
    y.o_uoff = y.o_cap + r256(8 * (P + 1));
    y.o_sel = y.o_uoff + r256(8 * (P + 1));
    y.o_selout = y.o_sel + r256(4 * U);
    y.o_blks = y.o_selout + r256(8 * U);
    y.o_blkl = y.o_blks + r256(4 * ((S + 1023) / 1024 + 1));
    y.o_keys = y.o_blkl + r256(4 * ((Lt + 1023) / 1024 + 1));
    y.o_flags = y.o_keys + r256((key_bits / 8) * (S + Lt));
    y.o_mw = y.o_flags + r256(4 * y.nwords);
    y.o_counts = y.o_mw + r256(4 * y.nwords);
    y.o_rank = y.o_counts + r256(4 * (y.nblk + 1));
    y.o_misc = y.o_rank + (q.op == LC_SETOP_OR ? r256(4 * S) : 0);  // total, work, err
    y.total = y.o_misc + 256;
    return y;
}

int32_t setop_batch(const lc_batch* bt, const lc_setop_plan* q, const uint32_t* d_pairs, bool OR,
                    void* d_scratch, uint64_t scratch_bytes, void* d_out, uint64_t* d_out_off,
                    uint64_t* d_counts, cudaStream_t st) {
    if (!bt || !q || !bt->d_lists || !d_scratch || ((uintptr_t)d_scratch & 255) || !d_out ||
        !d_out_off || !d_counts || (q->op == LC_SETOP_OR) != OR || (q->n_pairs && !d_pairs))
        return LC_ERR_ARG;
    const uint32_t P = q->n_pairs;
    if (!P) return LC_OK;
    const SetopLayout y = setop_layout(*q, bt->key_bits);
    if (scratch_bytes < y.total) return LC_ERR_ARG;
    uint8_t* D = (uint8_t*)d_scratch;
    uint64_t* misc = (uint64_t*)(D + y.o_misc);  // [0] scan total, [1] work counter, [2] error
    if (cudaMemsetAsync(D + y.o_flags, 0, 4 * y.nwords, st) != cudaSuccess ||
        cudaMemsetAsync(misc + 2, 0, 8, st) != cudaSuccess)
        return LC_ERR_CUDA;
    // ---- plan on the device: short / long sides, offsets, chunk records to decode
    PlanArgs pa;
    pa.lists = (const BatchList*)bt->d_lists;
    pa.pairs = d_pairs;
    pa.sl = (uint32_t*)(D + y.o_sl);
    pa.s_off = (uint64_t*)(D + y.o_soff);
    pa.l_off = (uint64_t*)(D + y.o_loff);
    pa.cap_off = (uint64_t*)(D + y.o_cap);
    pa.u_off = (uint64_t*)(D + y.o_uoff);
    pa.sel = (uint32_t*)(D + y.o_sel);
    pa.sel_out = (uint64_t*)(D + y.o_selout);
    pa.err = (uint32_t*)(misc + 2);
    pa.blk_s = (uint32_t*)(D + y.o_blks);
    pa.blk_l = (uint32_t*)(D + y.o_blkl);
    pa.U = q->units;
    pa.S = q->short_keys;
    pa.P = P;
    pa.m = bt->m;
    pa.n_chunks = (uint32_t)bt->n_chunks;
    pa.OR = OR;
    const unsigned gp = (P + 255) / 256;
    lc_bplan_kernel<<<gp, 256, 0, st>>>(pa);
    lc_bscan_kernel<<<1, 1024, 0, st>>>(pa);
    lc_bexpand_kernel<<<gp, 256, 0, st>>>(pa);
    lc_detail::count_launch(3);
    int32_t rc = launch_batch_decode(bt, pa.sel, pa.sel_out, nullptr, (uint32_t)q->units,
                                     D + y.o_keys, (uint32_t*)(misc + 1), st);
    if (rc) return rc;
    const bool k64 = bt->key_bits == 64;
    SetopArgs a;
    a.lists = pa.lists;
    a.sl = pa.sl;
    a.s_off = pa.s_off;
    a.l_off = pa.l_off;
    a.cap_off = pa.cap_off;
    a.keys_s = D + y.o_keys;
    a.keys_l = D + y.o_keys + (bt->key_bits / 8) * q->short_keys;
    a.flags = (uint32_t*)(D + y.o_flags);
    a.mw = (uint32_t*)(D + y.o_mw);
    a.counts = (uint32_t*)(D + y.o_counts);
    a.rank = (uint32_t*)(D + y.o_rank);
    a.total = misc;
    a.out = d_out;
    a.d_out_off = d_out_off;
    a.d_counts = d_counts;
    a.blk_s = pa.blk_s;
    a.blk_l = pa.blk_l;
    a.S = q->short_keys;
    a.Lt = q->long_keys;
    a.P = P;
    a.nblk = (uint32_t)y.nblk;
    a.nwords = (uint32_t)y.nwords;
    const unsigned gs = (unsigned)y.nblk;
    if (k64) OR ? lc_bprobe_kernel<true, true><<<gs, 256, 0, st>>>(a) : lc_bprobe_kernel<true, false><<<gs, 256, 0, st>>>(a);
    else OR ? lc_bprobe_kernel<false, true><<<gs, 256, 0, st>>>(a) : lc_bprobe_kernel<false, false><<<gs, 256, 0, st>>>(a);
    IsectArgs sa{};
    sa.counts = a.counts;
    sa.nblk = a.nblk;
    sa.d_count = a.total;
    lc_isect_scan_kernel<<<1, 1024, 0, st>>>(sa);
    lc_bmw_kernel<<<(unsigned)((y.nwords + 255) / 256), 256, 0, st>>>(a);
    if (k64) OR ? lc_bwrite_s_kernel<true, true><<<gs, 256, 0, st>>>(a) : lc_bwrite_s_kernel<true, false><<<gs, 256, 0, st>>>(a);
    else OR ? lc_bwrite_s_kernel<false, true><<<gs, 256, 0, st>>>(a) : lc_bwrite_s_kernel<false, false><<<gs, 256, 0, st>>>(a);
    uint32_t nl = 5;
    if (OR && q->long_keys) {
        const unsigned gl = (unsigned)((q->long_keys + 8 * kWlKeys - 1) / (8 * kWlKeys));
        if (k64) lc_bwrite_l_kernel<true><<<gl, 256, 0, st>>>(a);
        else lc_bwrite_l_kernel<false><<<gl, 256, 0, st>>>(a);
        ++nl;
    }
    const unsigned gq = (unsigned)((P + 1 + 255) / 256);
    if (OR) lc_bpairs_kernel<true><<<gq, 256, 0, st>>>(a);
    else lc_bpairs_kernel<false><<<gq, 256, 0, st>>>(a);
    lc_detail::count_launch(nl);
    return cuda_status();
}
}  // namespace

int32_t lc_setop_batch_plan(const lc_batch* b, const uint64_t* h_n, const uint32_t* h_pairs,
                            uint32_t n_pairs, int32_t op, lc_setop_plan* plan) {
    if (!b || !h_n || !plan || (!h_pairs && n_pairs) || (op != LC_SETOP_AND && op != LC_SETOP_OR))
        return LC_ERR_ARG;
    const bool OR = op == LC_SETOP_OR;
    uint64_t S = 0, Lt = 0, U = 0;
    for (uint32_t p = 0; p < n_pairs; ++p) {
        const uint32_t x = h_pairs[2 * p], y = h_pairs[2 * p + 1];
        if (x >= b->m || y >= b->m) return LC_ERR_ARG;
        const uint64_t ns = h_n[x] <= h_n[y] ? h_n[x] : h_n[y], nl = h_n[x] <= h_n[y] ? h_n[y] : h_n[x];
        S += ns;
        U += (ns + 1023) >> 10;
        if (OR) {
            Lt += nl;
            U += (nl + 1023) >> 10;
        }
    }
    if (S >= (1ULL << 32) || U >= (1ULL << 32)) return LC_ERR_TOO_LARGE;
    plan->n_pairs = n_pairs;
    plan->op = op;
    plan->short_keys = S;
    plan->long_keys = Lt;
    plan->units = U;
    plan->scratch_bytes = setop_layout(*plan, b->key_bits).total;
    plan->out_keys = S + Lt;
    return LC_OK;
}

int32_t lc_intersect_batch(const lc_batch* b, const lc_setop_plan* plan, const uint32_t* d_pairs,
                           void* d_scratch, uint64_t scratch_bytes, void* d_out,
                           uint64_t* d_out_off, uint64_t* d_counts, lc_stream stream) {
    return setop_batch(b, plan, d_pairs, false, d_scratch, scratch_bytes, d_out, d_out_off,
                       d_counts, (cudaStream_t)stream);
}

int32_t lc_union_batch(const lc_batch* b, const lc_setop_plan* plan, const uint32_t* d_pairs,
                       void* d_scratch, uint64_t scratch_bytes, void* d_out, uint64_t* d_out_off,
                       uint64_t* d_counts, lc_stream stream) {
    return setop_batch(b, plan, d_pairs, true, d_scratch, scratch_bytes, d_out, d_out_off,
                       d_counts, (cudaStream_t)stream);
}

int32_t lc_decode_batch(const lc_batch* b, void* d_out, uint32_t* d_work, lc_stream stream) {
    if (!b || !b->d_chunks || !d_out || ((uintptr_t)d_out % (b->key_bits / 8)) || !d_work ||
        ((uintptr_t)d_work & 3))
        return LC_ERR_ARG;
    if (!b->n_chunks) return LC_OK;
    return launch_batch_decode(b, nullptr, nullptr, nullptr, (uint32_t)b->n_chunks, d_out, d_work,
                               (cudaStream_t)stream);
}

int32_t lc_decode_host(const void* h_blob, uint64_t blob_bytes, void* d_blob, void* d_out,
                       void* h_out, lc_stream stream) {
    if (!h_blob || !d_blob || !d_out || !h_out) return LC_ERR_ARG;
    if (blob_bytes < sizeof(lc_header)) return LC_ERR_FORMAT;
    lc_view v;
    int32_t st = lc_view_init(&v, h_blob, d_blob, blob_bytes);
    if (st) return st;
    const lc_header& h = v.h;
    const uint8_t* B = (const uint8_t*)h_blob;
    const uint64_t n = h.n, w = h.key_bits / 8;
    // spans of >= 4 Mi keys (multiples of 1024), at most kMaxSpans (a ramped 1/4, 1/2, ... span
    // schedule measured 0.35 ms slower on config 2: the gap to the PCIe floor is the two
    // directions sharing the link, not pipeline fill)
    uint64_t per = (n + kMaxSpans - 1) / kMaxSpans;
    if (per < (4u << 20)) per = 4u << 20;
    per = (per + 1023) & ~1023ULL;
    // every span's slices first: a corrupt hint fails before anything is enqueued
    SpanSlices sl[kMaxSpans];
    uint32_t ns = 0;
    for (uint64_t i0 = 0; i0 < n; i0 += per, ++ns)
        if ((st = span_slices(h, B, i0, i0 + per < n ? i0 + per : n, &sl[ns]))) return st;
    HostPipe* p = pipe_acquire();
    if (!p) return LC_ERR_CUDA;
    cudaStream_t s = (cudaStream_t)stream;
    // order the pipeline after whatever the caller queued on its stream
    cudaEventRecord(p->done, s);
    cudaStreamWaitEvent(p->h2d, p->done, 0);
    cudaStreamWaitEvent(p->d2h, p->done, 0);
    uint8_t* D = (uint8_t*)d_blob;
    for (uint32_t k = 0; k < ns && !st; ++k) {
        const uint64_t i0 = k * per, i1 = i0 + per < n ? i0 + per : n;
        const SpanSlices& q = sl[k];
        // exactly the slices the span's kernel stages, at their offsets in the device blob
        if ((st = copy_up(D + h.off_hint + 4 * q.c0, B + h.off_hint + 4 * q.c0,
                          4 * (q.c1 - q.c0 + 1), p->h2d)) ||
            (st = copy_up(D + h.off_starts + 4 * q.s_lo, B + h.off_starts + 4 * q.s_lo,
                          4 * (q.s_hi - q.s_lo), p->h2d)) ||
            (st = copy_up(D + h.off_params + 16 * q.p_lo, B + h.off_params + 16 * q.p_lo,
                          16 * (q.p_hi - q.p_lo), p->h2d)) ||
            (st = copy_up(D + h.off_words + 4 * q.w_lo, B + h.off_words + 4 * q.w_lo,
                          4 * (q.w_hi - q.w_lo), p->h2d)))
            break;
        cudaEventRecord(p->up[k], p->h2d);
        cudaStreamWaitEvent(s, p->up[k], 0);
        if ((st = launch_decode(&v, i0, i1, (uint8_t*)d_out + i0 * w, s))) break;
        cudaEventRecord(p->dec[k], s);
        cudaStreamWaitEvent(p->d2h, p->dec[k], 0);
        if (cudaMemcpyAsync((uint8_t*)h_out + i0 * w, (uint8_t*)d_out + i0 * w, (i1 - i0) * w,
                            cudaMemcpyDeviceToHost, p->d2h) != cudaSuccess)
            st = LC_ERR_CUDA;
    }
    // join the copy streams back into the caller's stream (also after an error, so the pipe
    // is idle before it is reused)
    cudaEventRecord(p->done, p->d2h);
    cudaStreamWaitEvent(s, p->done, 0);
    cudaEventRecord(p->done, p->h2d);
    cudaStreamWaitEvent(s, p->done, 0);
    pipe_release(p);
    return st ? st : cuda_status();
}

#ifdef LC_DEBUG_BOUNDS
// bounds-checked builds only: violations counted since the previous call (and reset), summed
// over the translation units; g_where = source line / index / limit of the last one seen
static uint32_t g_where[3];
uint32_t lc_debug_violations(void) {
    using namespace lc_detail;
    uint32_t (*const tus[])(uint32_t*) = {debug_violations_0_0, debug_violations_0_1,
                                          debug_violations_1_0, debug_violations_1_1,
                                          debug_violations_2_0, debug_violations_2_1};
    uint32_t v = debug_take(g_where);
    for (auto f : tus) v += f(g_where);
    return v;
}
void lc_debug_where(uint32_t* out3) { std::memcpy(out3, g_where, sizeof g_where); }
#endif

}  // extern "C"
