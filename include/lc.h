/*
 * lc.h -- C ABI of the B200-native learned-compression decoder (arxiv 2412.10770).
 *
 * The method (Def. 2 / Eq. 1, §II-A): a sorted key list K is stored as an
 * eps-PLA f (segments (s_j, alpha_j, beta_j)) plus residuals Delta[i] = K[i] - floor(f(i)) in
 * ceil(log2(2 eps + 1)) bits; decompression is K[i] = floor(f(i)) + Delta[i] (
 * Fig. 2 decoding stage).  The byte format "LCG1" is frozen in FORMAT.md.
 *
 * Conventions for every entry point
 *  - Return value: int32_t status, LC_OK (0) or a negative LC_ERR_* code; never aborts.
 *  - Pointers prefixed d_ are DEVICE pointers owned by the caller (e.g. torch CUDA tensors);
 *    the library never allocates, frees or synchronizes device memory in the device calls.
 *  - Device calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *    Host-detectable argument problems are returned immediately; per-query index problems
 *    are reported on the device through *d_err (see lc_access).
 *  - The library is stateless: any number of concurrent calls on distinct streams may read
 *    the same blob.
 */
#ifndef LC_H_
#define LC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (names follow SPEC.md:113,164,174,184,465 error kinds). */
enum {
    LC_OK = 0,
    LC_ERR_ARG = -1,       /* null/misaligned pointer, bad size, eps > 2^31-1, key_bits != 32|64 */
    LC_ERR_EMPTY = -2,     /* n == 0 (EmptyInput) */
    LC_ERR_UNSORTED = -3,  /* keys not strictly increasing, duplicates included (UnsortedInput) */
    LC_ERR_TOO_LARGE = -4, /* n >= 2^32, or a key >= 2^32 with key_bits == 32 */
    LC_ERR_FORMAT = -5,    /* bad magic/version/offsets, truncated or non-monotone blob */
    LC_ERR_ALLOC = -6,     /* host allocation failed */
    LC_ERR_CUDA = -7       /* a CUDA launch or copy failed (cudaGetLastError) */
};

/* FORMAT F1: the first 128 bytes of every blob, little-endian. */
typedef struct lc_header {
    char magic[4];        /* "LCG1" */
    uint16_t version;     /* 1 */
    uint8_t key_bits;     /* 32 | 64 */
    uint8_t res_bits;     /* b = ceil(log2(2 eps + 1)) */
    uint32_t eps;         /* error bound of the eps-PLA */
    uint32_t hint_log2;   /* 10: one segment hint every 1024 keys */
    uint64_t n;           /* N keys */
    uint64_t n_seg;       /* L segments */
    uint64_t n_hint;      /* H + 1, H = ceil(N / 1024) */
    uint64_t n_words;     /* W residual words */
    uint64_t off_starts, off_params, off_hint, off_words, total_bytes;
    uint32_t flags;       /* 0, or LC_FLAG_FREE_INTERCEPT (FORMAT F7) */
    uint8_t reserved[36];
} lc_header;

/* Header flag (FORMAT F7): segments use a free integer intercept (O'Rourke's rule)
 * instead of the F2 anchor; params hold base = beta - eps and the decode bias is 0. */
#define LC_FLAG_FREE_INTERCEPT 1u

/* Encoder option of lc_encode_ex (not stored in blobs): the fewest segments on the format's
 * integer lattice — the "optimal ... minimize the number of required line segments" of
 * with the segment form of the other flags (F4 anchored, or F7 with
 * LC_FLAG_FREE_INTERCEPT).  The greedy rules are maximal per segment but not always minimal in
 * count on the lattice (L26); this option runs the greedy fit from every start and a
 * shortest-cover DP (O(n * segment length) time, O(n) memory).  Decoding is unchanged. */
#define LC_FLAG_MIN_SEGMENTS 2u

/* A blob resident in device memory: a host copy of its header plus the device pointer.
 * d_blob must be 256-byte aligned (torch / cudaMalloc allocations are). */
typedef struct lc_view {
    lc_header h;
    const void* d_blob;
    /* Optional successor-search index (lc_search_index_build): d_first[j] = K[s_j], the first
     * key of segment j, as uint64, in caller-owned device memory.  NULL (lc_view_init's
     * default): lc_next_geq / lc_intersect / lc_union search the params section directly. */
    const uint64_t* d_first;
    /* Optional access layout (lc_access_layout_build), NULL by default (lc_view_init).  When
     * attached, lc_access and lc_quantile locate a key's segment through its directory (no
     * binary search) and read the segment parameters and the residual field from one record
     * instead of two sections. */
    const void* d_acc;
    /* Shard views only (lc_shard_upload; both 0 for a whole-blob view): the view holds the
     * slices of keys [span_lo, span_hi) and nothing else.  Only lc_decode (which then decodes
     * the shard) and lc_decode_span (spans inside the shard) accept a shard view; every other
     * device call returns LC_ERR_ARG for it. */
    uint64_t span_lo, span_hi;
    /* Shard views: device addresses of starts[0], params[0], hint[0], words[0] as if the whole
     * sections were present (only the shard's slices are backed by memory, at d_blob).  Not
     * meant to be dereferenced by callers; zero for whole-blob views. */
    uint64_t sec_base[4];
} lc_view;

/* A CUDA stream (binary-compatible with cudaStream_t / CUstream). */
typedef struct CUstream_st* lc_stream;

/* ----------------------------------------------------------------------------- host side */

/* Build an LCG1 blob from n sorted keys (FORMAT F4 greedy anchored cone, the eps-PLA of Def. 2
 * PAPER.md:171-181; residual packing PAPER.md:184-186).  NOT on the hot path.
 *   keys:      host array of n keys, uint32_t if key_bits == 32 else uint64_t
 *   eps:       error bound, 0 <= eps <= 2^31 - 1
 *   *blob:     receives a host buffer of *blob_bytes bytes owned by the caller; release it
 *              with lc_free.
 * Errors: LC_ERR_EMPTY (n == 0), LC_ERR_UNSORTED, LC_ERR_TOO_LARGE, LC_ERR_ARG, LC_ERR_ALLOC. */
int32_t lc_encode(const void* keys, uint64_t n, uint32_t key_bits, uint32_t eps, void** blob,
                  uint64_t* blob_bytes);

/* lc_encode with format flags: flags = LC_FLAG_FREE_INTERCEPT selects the FORMAT F7 encoder
 * (greedy maximal extension over all integer lines, the O'Rourke rule of PAPER.md:188 on the
 * format's lattice: fewer segments, same decode kernels), which needs eps <= 2^30 - 1;
 * LC_FLAG_MIN_SEGMENTS (combinable) the fewest-segments segmentation.  flags = 0 is lc_encode.  Output ownership and errors as lc_encode; unknown flag bits or
 * eps out of range give LC_ERR_ARG. */
int32_t lc_encode_ex(const void* keys, uint64_t n, uint32_t key_bits, uint32_t eps,
                     uint32_t flags, void** blob, uint64_t* blob_bytes);

/* Release a blob returned by lc_encode / lc_encode_ex (NULL is a no-op).  The compressed
 * representation K^c of Def. 1 is owned by the caller until released. */
void lc_free(void* blob);

/* Full validation of a HOST copy of a blob (header, offsets, monotone starts, slope guard,
 * hint array, residual range, zero padding): the invariants that make Dec(K^c) well defined —
 * segments covering [0, N) in order (Eq. 1), every residual within
 * [-eps, eps] (Def. 2) so each field fits ceil(log2(2 eps + 1)) bits
 * (PAPER.md:186), decoded keys strictly increasing (Def. 1's sorted K).
 * LC_OK or LC_ERR_FORMAT / LC_ERR_ARG.  The device calls trust the header checks of
 * lc_view_init plus the hint checks of lc_decode_host / lc_shard_*; validate blobs from
 * untrusted sources before uploading them. */
int32_t lc_validate(const void* blob, uint64_t blob_bytes);

/* Fill *v from the blob's 128-byte header (a host copy) and the device pointer of the same blob
 * (blob_bytes bytes): the handle every device call takes for K^c resident in HBM (the decode
 * side of Fig. 2).  Checks the header fields only (FORMAT F1: magic, version,
 * b = ceil(log2(2 eps + 1)) per PAPER.md:186, section offsets recomputed from N, L, b) and
 * d_blob alignment; LC_ERR_FORMAT / LC_ERR_ARG.  Leaves the optional index, access layout and
 * shard fields empty. */
int32_t lc_view_init(lc_view* v, const void* host_header128, const void* d_blob,
                     uint64_t blob_bytes);

/* ---------------------------------------------------------------------------- device side */

/* Full decompression Dec(K^c) (Def. 1): d_out[i] = K[i] for i in [0, n), each
 * key_bits/8 bytes (d_out 16-byte aligned).  One kernel launch, asynchronous on stream. */
int32_t lc_decode(const lc_view* v, void* d_out, lc_stream stream);

/* Decode the key span [i0, i1) into d_out[0 .. i1-i0): the shard of a multi-GPU decode
 * (the paper's §IV-E ① "reduce the data dependencies ... to maximize
 * parallelism").  i0 must be a multiple of 1024 (unless i0 == i1: an empty span
 * is a no-op); i1 <= n, and for a shard view [i0, i1) inside [span_lo, span_hi).  LC_ERR_ARG
 * otherwise. */
int32_t lc_decode_span(const lc_view* v, uint64_t i0, uint64_t i1, void* d_out,
                       lc_stream stream);

/* ---------------------------------------------------------------- shards (multi-GPU decode)
 * A shard of keys [i0, i1) is what one GPU needs to decode that span and nothing more
 * (SURVEY §8(e)): the hint slice hint[i0/1024 .. ceil(i1/1024)], the segments the span touches
 * (starts and params from hint[i0/1024] to hint[ceil(i1/1024)], the straddling segment
 * duplicated across neighbouring shards) and the residual words [i0 b / 32, i1 b / 32 + 1),
 * each slice 256-byte aligned in one device buffer.  i0 must be a multiple of 1024 and
 * i0 < i1 <= n. */

/* Device bytes of the shard [i0, i1) of the host blob h_blob (header and hint slice read).
 * LC_ERR_FORMAT for a bad header or a hint slice that is not non-decreasing within [0, L-1]
 * (the slice bounds come from it), LC_ERR_ARG for a bad span. */
int32_t lc_shard_bytes(const void* h_blob, uint64_t blob_bytes, uint64_t i0, uint64_t i1,
                       uint64_t* shard_bytes);

/* Copy the shard [i0, i1) of the host blob h_blob (pinned memory for true asynchrony) into the
 * caller's device buffer d_shard (>= lc_shard_bytes, 256-byte aligned) asynchronously on
 * `stream`, and fill *v as a shard view of it (span_lo = i0, span_hi = i1).  lc_decode(v, d_out)
 * then writes keys [i0, i1) to d_out[0 .. i1 - i0).  h_blob must stay valid until the copies
 * complete.  Errors as lc_shard_bytes, plus LC_ERR_ARG (null pointers, buffer too small or
 * misaligned) and LC_ERR_CUDA. */
int32_t lc_shard_upload(const void* h_blob, uint64_t blob_bytes, uint64_t i0, uint64_t i1,
                        void* d_shard, uint64_t shard_bytes, lc_view* v, lc_stream stream);

/* Batched random access Dec(K^c)[i] ("f(j) + Delta[j]"; Table I caption
 * PAPER.md:309, binary search for the segment).  d_idx: q uint64 indices (device);
 * d_out: q keys of key_bits/8 bytes.  An index >= n yields 0 in its slot and sets bit 0 of
 * *d_err (atomicOr) when d_err is not NULL.  q == 0 is a no-op. */
int32_t lc_access(const lc_view* v, const uint64_t* d_idx, uint64_t q, void* d_out,
                  uint32_t* d_err, lc_stream stream);

/* Range decode: d_out[r*len + k] = K[d_start[r] + k] for r < q, k < len — Dec(K^c)[i]
 * over len consecutive indices, the blocked decode inside and across segments
 * (K[i] = floor(f(i)) + Delta[i]; BASELINE config 5: 10^7 ranges of 64 keys).
 * A range with start + len > n yields zeros and sets bit 0 of *d_err.  1 <= len <= 2^20;
 * q == 0 is a no-op.  Ranges of up to 64 keys run a staged kernel (a shared-memory ring of the
 * ranges' slices); with an access layout attached (lc_access_layout_build) they are decoded
 * through it (same results). */
int32_t lc_range_decode(const lc_view* v, const uint64_t* d_start, uint64_t q, uint32_t len,
                        void* d_out, uint32_t* d_err, lc_stream stream);

/* Quantiles (§III-C, Table I): d_out[t] = the k_t-th q-quantile of the
 * list, K[min(floor(N * k_t / q), N - 1)], for t < m (d_k: m uint64 ranks, 0 <= k_t <= q).
 *   exact != 0: the exact key, f(i) + Delta[i] (one segment search + residual per quantile);
 *   exact == 0: the segments-only approximation floor(f(i)) with no residual read; its error
 *               is at most eps (approximate query processing); it saturates
 *               at 2^key_bits - 1 when the prediction overshoots the key width.
 * 1 <= q <= 2^32 - 1 (LC_ERR_ARG otherwise).  A rank k_t > q yields 0 and sets bit 0 of *d_err.
 * m == 0 is a no-op. */
int32_t lc_quantile(const lc_view* v, const uint64_t* d_k, uint64_t m, uint64_t q, int32_t exact,
                    void* d_out, uint32_t* d_err, lc_stream stream);

/* Successor search (NEXT-2; segments as skip pointers, Fig. 4b): for t < m,
 * d_out_idx[t] = min{i : K[i] >= x_t} (n if none) and d_out_key[t] = that key (0 if none).
 * d_x: m uint64 probe keys (for a 32-bit list a probe >= 2^32 is past every key).  Either
 * output pointer may be NULL (not both).  m == 0 is a no-op.  Binary search over the
 * segments' first keys K[s_j] — the bases for anchored blobs (FORMAT F2), base + u(s_j) for F7
 * blobs (decoded only when the probe lies in the band [base_j, base_j + 2 eps)), or the search
 * index when one is attached (lc_search_index_build) — then inside one segment, decoding only
 * the probed keys. */
int32_t lc_next_geq(const lc_view* v, const uint64_t* d_x, uint64_t m, uint64_t* d_out_idx,
                    void* d_out_key, lc_stream stream);

/* Device bytes of v's successor-search index: the n_seg first keys (uint64, padded to a 256-byte
 * multiple) followed by a sample of every 16th of them: about 8.5 bytes per segment. */
uint64_t lc_search_index_bytes(const lc_view* v);

/* Build v's successor-search index into d_index (>= lc_search_index_bytes(v) bytes, 128-byte
 * aligned, caller-owned, kept alive while v is used) asynchronously on `stream`, and attach it
 * (v->d_first = d_index).  The index is the auxiliary segment-localisation structure of
 * PAPER.md:286 (§III-B) for key-space search (Fig. 4b): the segments' first
 * keys in one dense array plus a sample of every 16th (one per 128-byte line), so a successor
 * search binary-searches the small sample (kept in L2 with evict_last) and then one line of
 * the first keys, instead of ~23 levels of 16-byte params records; F7 blobs no longer decode
 * K[s_j] during the search.  Results of lc_next_geq / lc_intersect / lc_union are identical
 * with and without it.  Errors: LC_ERR_ARG (null or misaligned d_index). */
int32_t lc_search_index_build(lc_view* v, void* d_index, lc_stream stream);

/* Device bytes of v's access layout: 256 H + 16 (2 L + floor(N b / 128)) bytes,
 * H = ceil(N / 1024). */
uint64_t lc_access_layout_bytes(const lc_view* v);

/* Build v's access layout into d_layout (>= lc_access_layout_bytes(v) bytes, 128-byte aligned,
 * caller-owned, kept alive while v is used) asynchronously on `stream`, and attach it
 * (v->d_acc = d_layout).  An auxiliary structure aligned with the memory hierarchy
 * (§IV-E ②) for random access f(j) + Delta[j] and quantiles
 * (PAPER.md:296-315), in two parts:
 *   directory: for every 32 keys (word w of 1024-key block h) 8 bytes {bits, entry}: bit t of
 *     bits is set iff key 1024 h + 32 w + t starts a segment (block position 0 excluded: hint[h]
 *     names the segment holding key 1024 h), entry = rank | dist << 11 with rank = the bits set
 *     in words < w of the block and dist = 32 w - (start of the segment holding key
 *     1024 h + 32 w), 2^21 - 1 when larger.  Key i's segment is then
 *     j = hint[h] + rank + popc(bits at or below i) and its start follows from the highest such
 *     bit or from dist, with no binary search (Table I's O(log) search, becomes
 *     one L2 round trip);
 *   records (from byte 256 H): record j, at 16-byte unit 2 j + floor(s_j b / 128), holds segment
 *     j's {base, slope_fx} (16 B) followed by the 16-byte units floor(s_j b / 128) ..
 *     floor(s_{j+1} b / 128) of the residual words (a copy), so params and the residual field
 *     come from one record (usually one DRAM line) instead of two sections.
 * lc_range_decode with len <= 64 uses it too: the bitmaps shifted to a range's first key are the
 * segment-boundary masks of its keys, and the records of consecutive segments are contiguous,
 * so a range is one gather of <= 31 units plus its first segment's params (no search).
 * The blob (FORMAT F1-F7) is unchanged; results of lc_access / lc_quantile / lc_range_decode are
 * identical with and without the layout.  Errors: LC_ERR_ARG (null or misaligned d_layout,
 * shard view). */
int32_t lc_access_layout_build(lc_view* v, void* d_layout, lc_stream stream);

/* Device scratch bytes lc_intersect needs for list a (its decoded keys, a match bitmap and
 * per-CTA offsets). */
uint64_t lc_intersect_scratch_bytes(const lc_view* a);

/* Intersection of two compressed lists, the AND query of inverted-index processing
 * (§III-A): d_out receives the sorted keys present in both lists and
 * *d_count (device uint64) their number.  a is decoded into d_scratch (>=
 * lc_intersect_scratch_bytes(a) bytes, 256-byte aligned) and each of its keys is searched in b
 * with next_geq, so segments of b that hold none of a's keys are never read.  When b is the
 * shorter list the roles are swapped internally (the scratch and d_out sized for a suffice).
 * d_out capacity: a->h.n keys.  Both lists must have the same key_bits. */
int32_t lc_intersect(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                     void* d_out, uint64_t* d_count, lc_stream stream);

/* Device scratch bytes lc_union needs for lists a and b. */
uint64_t lc_union_scratch_bytes(const lc_view* a, const lc_view* b);

/* Union of two compressed lists, the OR query of inverted-index processing:
 * d_out receives the sorted keys present in either list (each once) and *d_count (device
 * uint64) their number.  Only the shorter list s is decoded (into d_scratch, >=
 * lc_union_scratch_bytes(a, b) bytes, 256-byte aligned); each of its keys is searched in the
 * longer list l with next_geq (segments as skip pointers), the keys absent from l are written
 * to their final slots, and l is decoded once straight into d_out with every key shifted by
 * the number of inserted keys below it (no decoded copy of l, no merge pass).  d_out capacity:
 * a->h.n + b->h.n keys, aligned to the key width.  Same key_bits required.  Either argument
 * order gives the same result. */
int32_t lc_union(const lc_view* a, const lc_view* b, void* d_scratch, uint64_t scratch_bytes,
                 void* d_out, uint64_t* d_count, lc_stream stream);

/* ------------------------------------------------------------- batches (many short lists)
 * An inverted index is many posting lists (§III-A); decoding them one call
 * each is launch-bound (a 1e6-key list decodes in ~10 us).  A batch groups m blobs that live in
 * one device buffer (each 256-byte aligned) and decodes all of them in ONE launch: the work
 * units are the 1024-key chunks of all lists (a short list is one partial chunk), described by
 * a host-built directory in device memory.  All lists of a batch share key_bits; eps, and so
 * the residual width b, may differ per list. */
typedef struct lc_batch {
    uint32_t m;             /* lists */
    uint32_t key_bits;      /* common key width (32 | 64) */
    uint32_t max_res_bits;  /* widest residual field of the batch */
    uint32_t sparse;        /* fewer than one segment per 64 keys overall (decode variant) */
    uint64_t n_total;       /* keys over all lists */
    uint64_t n_chunks;      /* 1024-key chunks over all lists (a list's last one may be partial) */
    uint64_t n_small;       /* of which partial chunks of <= 64 keys (records stored last) */
    uint64_t small_keys;    /* keys in those small chunks */
    uint64_t payload_bytes; /* bytes of the lists' headers and sections, without the 256-byte
                               alignment padding: what a decode reads */
    const void* d_lists;    /* device directory: m list records (64 B each) ... */
    const void* d_chunks;   /* ... then n_chunks chunk records (48 B each) ... */
    const void* d_small;    /* ... then the small chunks' key prefix (n_small + 1 uint32) and the
                               small chunk of every 32nd small key (ceil(small_keys / 32)) */
} lc_batch;

/* Directory bytes of the batch of m blobs at host byte offsets blob_off[k] of h_blobs (each a
 * full LCG1 blob; headers checked).  LC_ERR_FORMAT for a bad header, LC_ERR_ARG for m == 0,
 * mixed key widths or an unaligned offset. */
int32_t lc_batch_dir_bytes(const void* h_blobs, uint64_t h_bytes, const uint64_t* blob_off,
                           uint32_t m, uint64_t* dir_bytes);

/* Fill *b and write the batch directory into d_dir (>= lc_batch_dir_bytes, 16-byte aligned)
 * asynchronously on `stream` (from a library-internal host staging copy: h_* may be released on
 * return).  h_blobs holds the m blobs at blob_off[k]; d_blobs is the device copy of the same
 * bytes (same offsets, 256-byte aligned base).  out_off[k] is the element offset of list k's
 * keys in the batch output, or NULL for packed lists in order (prefix sums of n).  Every
 * list's hint section is checked (non-decreasing, within [0, L - 1]) since chunk records copy
 * it: LC_ERR_FORMAT otherwise. */
int32_t lc_batch_init(lc_batch* b, const void* h_blobs, uint64_t h_bytes, const uint64_t* blob_off,
                      uint32_t m, const void* d_blobs, const uint64_t* out_off, void* d_dir,
                      uint64_t dir_bytes, lc_stream stream);

/* Decode every list of the batch in one launch: list k's keys to d_out[out_off[k] ..
 * out_off[k] + n_k) (elements of key_bits / 8 bytes).  Dec(K^c) per list (Def. 1).
 * d_work: a caller-owned 4-byte device counter (the launch's work queue), zeroed on `stream`
 * by the call; concurrent calls need distinct counters. */
int32_t lc_decode_batch(const lc_batch* b, void* d_out, uint32_t* d_work, lc_stream stream);

/* Batched AND / OR queries (inverted-index processing, §III-A, Fig. 4):
 * pair p = (pairs[2 p], pairs[2 p + 1]) names two lists of the batch.  All pairs run in a fixed
 * number of launches whatever their number, planned on the device (no host pass over the
 * batch, no upload).  The shorter list s_p of each pair is decoded; for AND each of its keys is
 * searched in the compressed longer list l_p (next_geq: segments as skip pointers), for OR both
 * are decoded and every key is placed in its union slot by ranks.
 *
 * lc_setop_batch_plan sizes one query batch on the host (O(pairs)): h_n[k] is list k's key
 * count (m entries, as given to lc_batch_init), h_pairs the 2 P list indices.  The device calls
 * then take the same pairs in device memory (d_pairs); other pairs give unspecified results but
 * never write outside d_scratch / d_out (a pair index >= m is clamped to m - 1).
 * Results: pair p's keys at d_out[d_out_off[p] .. d_out_off[p] + d_counts[p]) (device arrays of
 * P + 1 and P uint64; AND results are packed, OR results sit at capacity offsets
 * sum_{q < p} (n_s + n_l)).  d_scratch: >= plan->scratch_bytes (256-byte aligned); d_out:
 * >= plan->out_keys keys.  Errors: LC_ERR_ARG (bad pair index on the host, buffers too small,
 * a plan of the other operation), LC_ERR_TOO_LARGE (>= 2^32 short keys). */
enum { LC_SETOP_AND = 0, LC_SETOP_OR = 1 };
typedef struct lc_setop_plan {
    uint32_t n_pairs;
    int32_t op;              /* LC_SETOP_AND | LC_SETOP_OR */
    uint64_t short_keys;     /* sum over pairs of the shorter list's keys */
    uint64_t long_keys;      /* OR: sum of the longer lists' keys (0 for AND) */
    uint64_t units;          /* 1024-key chunk records decoded */
    uint64_t scratch_bytes;  /* device scratch the call needs */
    uint64_t out_keys;       /* output capacity in keys */
} lc_setop_plan;
int32_t lc_setop_batch_plan(const lc_batch* b, const uint64_t* h_n, const uint32_t* h_pairs,
                            uint32_t n_pairs, int32_t op, lc_setop_plan* plan);
int32_t lc_intersect_batch(const lc_batch* b, const lc_setop_plan* plan, const uint32_t* d_pairs,
                           void* d_scratch, uint64_t scratch_bytes, void* d_out,
                           uint64_t* d_out_off, uint64_t* d_counts, lc_stream stream);
int32_t lc_union_batch(const lc_batch* b, const lc_setop_plan* plan, const uint32_t* d_pairs,
                       void* d_scratch, uint64_t scratch_bytes, void* d_out, uint64_t* d_out_off,
                       uint64_t* d_counts, lc_stream stream);

/* End-to-end decode from HOST memory to HOST memory on one stream: copies the blob
 * (h_blob, blob_bytes; pinned memory for true asynchrony) into the caller's device buffer
 * d_blob (>= blob_bytes, 256-byte aligned), decodes into the caller's device buffer d_out
 * (>= n*key_bits/8 bytes) and copies the keys to h_out.  Work is split into spans so that
 * the device->host copy of one span overlaps the decode of the next.  Asynchronous: the
 * caller synchronizes the stream before reading h_out. */
int32_t lc_decode_host(const void* h_blob, uint64_t blob_bytes, void* d_blob, void* d_out,
                       void* h_out, lc_stream stream);

/* Human-readable name of a status code (static string): the error kinds of the method's
 * interfaces (EmptyInput, UnsortedInput, CorruptPayload, IndexOutOfRange, ... SPEC.md:113,
 * 164, 174, 184, 465; the paper's Def. 1 input is a sorted list). */
const char* lc_status_str(int32_t status);

/* Number of device kernels launched by this library in this process so far (monotone,
 * thread-safe counter; bench.py reports its delta over the timed region as gpu_launches, the
 * evidence that the measured throughput of the decode path of PAPER.md:94-95 ran in these
 * kernels). */
uint64_t lc_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LC_H_ */
