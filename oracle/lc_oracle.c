/*
 * oracle/lc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the learned-compression format
 * "LCG1" (FORMAT.md) for arxiv 2412.10770.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The product
 * (paper_2412_10770_b200/) shares no code, header, table or constant generator with it.
 *
 * Citations are PAPER.md lines (section / equation) or FORMAT.md clauses (F1-F6), which
 * restate SURVEY.md §8(c).
 *
 * Pins (tests/test_oracle_*.py): round trip Dec(Enc(K)) = K (Def. 1), residual bound
 * |K[i] - floor(f(i))| <= eps recomputed with exact rationals (Def. 2, Eq. 1), width table
 * (PAPER.md:94,186), greedy maximality by brute force at reduced precision (F4), arithmetic
 * progression closed forms, overflow-guard cases, ratio from byte counts (Def. 1), and a
 * Python big-int transliteration for tiny inputs.  Nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* status codes: same numeric meaning as the product's lc.h (restated, not shared) */
#define OR_OK 0
#define OR_ERR_ARG -1
#define OR_ERR_EMPTY -2
#define OR_ERR_UNSORTED -3
#define OR_ERR_TOO_LARGE -4
#define OR_ERR_FORMAT -5
#define OR_ERR_ALLOC -6

#define OR_HEADER_BYTES 128u
#define OR_ALIGN 256u
#define OR_HINT_LOG2 10u

/* ---------------------------------------------------------------------------------------
 * Residual width  b = ceil(log2(2*eps+1))   (§II-A; Fig. 2)
 * Written as the smallest b with 2^b >= 2*eps+1 (so eps = 0 gives b = 0, FORMAT L9).
 */
uint32_t oracle_width(uint64_t eps) {
    uint32_t b = 0;
    u128 need = (u128)2 * eps + 1;
    while (((u128)1 << b) < need) b++;
    return b;
}

/* ---------------------------------------------------------------------------------------
 * Greedy anchored integer cone (FORMAT F4-F6), the eps-PLA fit of Def. 2
 * in the north star's integer fixed point:  f(i) = base_j + slope_j * (i - s_j) / 2^F,
 * floor(f(i)) = base_j + floor(slope_j * (i - s_j) / 2^F).
 *
 * F (=32 in the format) and gmax (=2^63-1 in the format: slope * d_max <= gmax) are
 * parameters only so that tests can brute-force the greedy at reduced precision (P4).
 *
 *   force_break (nullable, n bytes): force_break[e] != 0 forces a new segment to start at e
 *   slope_mode: 0 = lo + floor((hi-lo)/2) (F5), 1 = lo, 2 = hi      (P9 adversarial blobs)
 *
 * Writes L segments into starts[0..L), base[0..L), slope[0..L) (caller sizes them n) and
 * returns L, or a negative status.
 */
/* One F4 segment anchored at s over keys [s, n): the end e of the greedy extension and its
 * slope (F5 or the P9 slope_mode).  Keys must be sorted (checked by the callers). */
static uint64_t or_fit_f4(const uint64_t* K, uint64_t n, uint64_t s, uint64_t eps, uint32_t F,
                          uint64_t gmax, const uint8_t* force_break, int slope_mode,
                          uint64_t* slope) {
    uint64_t b0 = K[s];
    u128 lo = 0, hi = gmax;
    uint64_t e = s + 1;
    while (e < n) {
        if (force_break && force_break[e]) break;
        u128 d = e - s;
        u128 D = (u128)(K[e] - b0); /* exact, D >= 1 */
        /* l = ceil((D - eps) * 2^F / d), clipped at 0 when D <= eps */
        u128 l = 0;
        if (D > eps) {
            u128 num = (D - eps) << F;
            l = num / d + (num % d != 0);
        }
        /* h = floor(((D + eps + 1) * 2^F - 1) / d), then the overflow guard gmax / d */
        u128 h = ((((D + eps + 1) << F) - 1) / d);
        u128 g = (u128)gmax / d;
        if (g < h) h = g;
        u128 nlo = lo > l ? lo : l;
        u128 nhi = hi < h ? hi : h;
        if (nlo > nhi) break; /* F6: break at the first infeasible index */
        lo = nlo;
        hi = nhi;
        e++;
    }
    if (e - s == 1) *slope = 0;
    else if (slope_mode == 1) *slope = (uint64_t)lo;
    else if (slope_mode == 2) *slope = (uint64_t)hi;
    else *slope = (uint64_t)(lo + (hi - lo) / 2);
    return e;
}

int64_t oracle_segment_ex(const uint64_t* K, uint64_t n, uint64_t eps, uint32_t F,
                          uint64_t gmax, const uint8_t* force_break, int slope_mode,
                          uint64_t* starts, uint64_t* base, uint64_t* slope) {
    if (n == 0) return OR_ERR_EMPTY;
    if (F > 32) return OR_ERR_ARG;
    for (uint64_t i = 1; i < n; i++)
        if (K[i] <= K[i - 1]) return OR_ERR_UNSORTED;
    uint64_t L = 0;
    uint64_t s = 0;
    while (s < n) {
        uint64_t sl;
        uint64_t e = or_fit_f4(K, n, s, eps, F, gmax, force_break, slope_mode, &sl);
        starts[L] = s;
        base[L] = K[s];
        slope[L] = sl;
        L++;
        s = e;
    }
    return (int64_t)L;
}

int64_t oracle_segment(const uint64_t* K, uint64_t n, uint64_t eps, uint32_t F, uint64_t gmax,
                       uint64_t* starts, uint64_t* base, uint64_t* slope) {
    return oracle_segment_ex(K, n, eps, F, gmax, 0, 0, starts, base, slope);
}

/* ---------------------------------------------------------------------------------------
 * FORMAT F7: greedy maximal extension over integer lines with a free intercept (O'Rourke's
 * rule, on the format's lattice).  Written as the definition: every admissible
 * intercept beta = K[s] + delta, delta in [max(-eps, eps - K[s]), eps], keeps its own exact
 * slope interval (the F4 cone computed from beta instead of K[s]); a segment grows while any
 * intercept still has a non-empty interval.  O(segment length * (2 eps + 1)) -- slow on
 * purpose.  The chosen intercept is the feasible delta with the least |delta| (the negative
 * one on a tie), its slope the middle of its interval (F5); base = beta - eps (F7).
 * F / gmax as in oracle_segment_ex (reduced precision for the brute-force pins).
 * Scratch (5 arrays of 2 eps + 1) is the caller's.
 */
typedef __int128 or_i128;
typedef struct {
    or_i128 *lo, *hi, *nlo, *nhi;
    uint8_t* alive;
} or_free_scratch;

static int or_free_alloc(or_free_scratch* w, uint64_t eps) {
    const uint64_t m = 2 * eps + 1;
    w->lo = malloc(m * sizeof(or_i128));
    w->hi = malloc(m * sizeof(or_i128));
    w->nlo = malloc(m * sizeof(or_i128));
    w->nhi = malloc(m * sizeof(or_i128));
    w->alive = malloc(m);
    return w->lo && w->hi && w->nlo && w->nhi && w->alive;
}

static void or_free_release(or_free_scratch* w) {
    free(w->lo); free(w->hi); free(w->nlo); free(w->nhi); free(w->alive);
}

/* one F7 segment from s over keys [s, n): its end, base (= beta - eps) and slope */
static uint64_t or_fit_free(const uint64_t* K, uint64_t n, uint64_t s, uint64_t eps, uint32_t F,
                            uint64_t gmax, or_free_scratch* w, uint64_t* base, uint64_t* slope) {
    typedef or_i128 i128;
    const uint64_t m = 2 * eps + 1; /* delta = t - eps, t in [0, m) */
    i128 *lo = w->lo, *hi = w->hi, *nlo = w->nlo, *nhi = w->nhi;
    uint8_t* alive = w->alive;
    /* admissible intercepts: K[s] + delta - eps >= 0 */
    const i128 dmin = K[s] >= 2 * eps ? -(i128)eps : (i128)eps - (i128)K[s];
    for (uint64_t t = 0; t < m; t++) {
        alive[t] = ((i128)t - (i128)eps) >= dmin;
        lo[t] = 0;
        hi[t] = gmax;
    }
    uint64_t e = s + 1;
    while (e < n) {
        const i128 d = (i128)(e - s);
        int any = 0;
        for (uint64_t t = 0; t < m; t++) {
            if (!alive[t]) continue;
            const i128 delta = (i128)t - (i128)eps;
            const i128 Dp = (i128)(K[e] - K[s]) - delta; /* K[e] - beta */
            /* S*d >= (Dp - eps) 2^F  and  S*d <= (Dp + eps + 1) 2^F - 1  and  S*d <= gmax */
            i128 l = 0;
            if (Dp > (i128)eps) {
                const i128 num = (Dp - (i128)eps) << F;
                l = num / d + (num % d != 0);
            }
            i128 h = ((((Dp + (i128)eps + 1) << F) - 1) / d); /* Dp + eps + 1 >= 2 */
            if ((i128)gmax / d < h) h = (i128)gmax / d;
            nlo[t] = lo[t] > l ? lo[t] : l;
            nhi[t] = hi[t] < h ? hi[t] : h;
            if (nlo[t] <= nhi[t]) any = 1;
        }
        if (!any) break; /* F6/F7: the first infeasible index ends the segment */
        for (uint64_t t = 0; t < m; t++) {
            if (!alive[t]) continue;
            if (nlo[t] > nhi[t]) { alive[t] = 0; continue; }
            lo[t] = nlo[t];
            hi[t] = nhi[t];
        }
        e++;
    }
    /* least |delta|, negative first */
    uint64_t pick = m;
    for (uint64_t k = 0; k <= eps && pick == m; k++) {
        if (alive[eps - k]) pick = eps - k;
        else if (alive[eps + k]) pick = eps + k;
    }
    const i128 delta = (i128)pick - (i128)eps;
    *base = (uint64_t)((i128)K[s] + delta - (i128)eps);
    *slope = e - s == 1 ? 0 : (uint64_t)(lo[pick] + (hi[pick] - lo[pick]) / 2);
    return e;
}

int64_t oracle_segment_free(const uint64_t* K, uint64_t n, uint64_t eps, uint32_t F,
                            uint64_t gmax, uint64_t* starts, uint64_t* base, uint64_t* slope) {
    if (n == 0) return OR_ERR_EMPTY;
    if (F > 32 || eps > 0x3fffffffULL) return OR_ERR_ARG;
    for (uint64_t i = 1; i < n; i++)
        if (K[i] <= K[i - 1]) return OR_ERR_UNSORTED;
    or_free_scratch w;
    if (!or_free_alloc(&w, eps)) {
        or_free_release(&w);
        return OR_ERR_ALLOC;
    }
    uint64_t L = 0, s = 0;
    while (s < n) {
        uint64_t b, sl;
        const uint64_t e = or_fit_free(K, n, s, eps, F, gmax, &w, &b, &sl);
        starts[L] = s;
        base[L] = b;
        slope[L] = sl;
        L++;
        s = e;
    }
    or_free_release(&w);
    return (int64_t)L;
}

/* ---------------------------------------------------------------------------------------
 * Fewest segments (NEXT-3: "optimal online eps-PLA ... to minimize the number of required line
 * segments") on the format's integer lattice, where the greedy rules above are
 * maximal per segment but not always minimal in count (reading L26: a suffix of a feasible
 * integer segment need not be feasible).  Written as the definition: a segment [s, e) is
 * feasible iff e <= emax(s), the end of the greedy fit from s (a prefix of a feasible segment is
 * feasible with the same line), so the fewest segments covering [s, n) are
 *   f(n) = 0,  f(s) = 1 + min { f(e) : s < e <= emax(s) },
 * taking the LARGEST minimising e (deterministic tie-break, the product's too); every chosen
 * [s, e) is then refitted on exactly its keys with the same rule (F4 anchor / F7 free intercept,
 * F5 middle slope).  Plain O(n * segment length) loops; free != 0 selects F7.
 */
int64_t oracle_segment_min(const uint64_t* K, uint64_t n, uint64_t eps, int free_icpt,
                           uint32_t F, uint64_t gmax, uint64_t* starts, uint64_t* base,
                           uint64_t* slope) {
    if (n == 0) return OR_ERR_EMPTY;
    if (F > 32 || (free_icpt && eps > 0x3fffffffULL)) return OR_ERR_ARG;
    for (uint64_t i = 1; i < n; i++)
        if (K[i] <= K[i - 1]) return OR_ERR_UNSORTED;
    uint64_t* emax = malloc(n * 8);
    uint64_t* f = malloc((n + 1) * 8);
    uint64_t* nxt = malloc(n * 8);
    or_free_scratch w = {0, 0, 0, 0, 0};
    if (!emax || !f || !nxt || (free_icpt && !or_free_alloc(&w, eps))) {
        free(emax); free(f); free(nxt); or_free_release(&w);
        return OR_ERR_ALLOC;
    }
    for (uint64_t s = 0; s < n; s++) {
        uint64_t b, sl;
        emax[s] = free_icpt ? or_fit_free(K, n, s, eps, F, gmax, &w, &b, &sl)
                            : or_fit_f4(K, n, s, eps, F, gmax, 0, 0, &sl);
    }
    f[n] = 0;
    for (uint64_t s = n; s-- > 0;) {
        uint64_t best = UINT64_MAX, arg = s + 1;
        for (uint64_t e = s + 1; e <= emax[s]; e++)
            if (f[e] <= best) { best = f[e]; arg = e; } /* <=: the largest e among the minima */
        f[s] = best + 1;
        nxt[s] = arg;
    }
    uint64_t L = 0;
    for (uint64_t s = 0; s < n; s = nxt[s]) {
        const uint64_t e = nxt[s];
        uint64_t b = K[s], sl;
        if (free_icpt) or_fit_free(K, e, s, eps, F, gmax, &w, &b, &sl);
        else or_fit_f4(K, e, s, eps, F, gmax, 0, 0, &sl);
        starts[L] = s;
        base[L] = b;
        slope[L] = sl;
        L++;
    }
    free(emax); free(f); free(nxt); or_free_release(&w);
    return (int64_t)L;
}

/* --------------------------------------------------------------------------- blob layout */

static uint64_t rd64(const uint8_t* p) {
    uint64_t v = 0;
    for (int k = 7; k >= 0; k--) v = (v << 8) | p[k];
    return v;
}
static uint32_t rd32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static void wr64(uint8_t* p, uint64_t v) {
    for (int k = 0; k < 8; k++) p[k] = (uint8_t)(v >> (8 * k));
}
static void wr32(uint8_t* p, uint32_t v) {
    for (int k = 0; k < 4; k++) p[k] = (uint8_t)(v >> (8 * k));
}
static uint64_t up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

typedef struct {
    uint32_t key_bits, b, eps, hint_log2, flags;
    uint64_t n, L, n_hint, W, o_starts, o_params, o_hint, o_words, total;
} or_hdr;

/* FORMAT F1/F2 layout: header, then starts u32[L+1], params {u64 base, i64 slope}[L],
 * hint u32[H+1], words u32[W], each at the next 256-byte-aligned offset. */
static void or_layout(or_hdr* h) {
    uint64_t H = (h->n + 1023) / 1024;
    h->n_hint = H + 1;
    h->W = up((h->n * h->b + 31) / 32 + 1, 4);
    h->o_starts = OR_ALIGN;
    h->o_params = up(h->o_starts + 4 * (h->L + 1), OR_ALIGN);
    h->o_hint = up(h->o_params + 16 * h->L, OR_ALIGN);
    h->o_words = up(h->o_hint + 4 * h->n_hint, OR_ALIGN);
    h->total = h->o_words + 4 * h->W;
}

/* bit p of the LSB-first residual stream in little-endian u32 words (FORMAT F3) */
static uint32_t bit_at(const uint8_t* words, uint64_t p) {
    return (rd32(words + 4 * (p >> 5)) >> (p & 31)) & 1u;
}

/* FORMAT F3: u = sum_{t<b} bit(i*b+t) * 2^t */
static uint64_t field_at(const uint8_t* words, uint64_t i, uint32_t b) {
    uint64_t u = 0;
    for (uint32_t t = 0; t < b; t++) u |= (uint64_t)bit_at(words, i * b + t) << t;
    return u;
}

/* decode bias c of FORMAT F3: eps for anchored blobs, 0 for free-intercept blobs (F7) */
static uint64_t bias_of(const or_hdr* h) { return (h->flags & 1u) ? 0 : h->eps; }

/* base + floor(slope * d / 2^32) (Eq. 1 in fixed point, F3); floor(f(i)) for anchored blobs,
 * floor(f(i)) - eps for free-intercept blobs (F7 stores base = beta - eps) */
static uint64_t predict(uint64_t base, uint64_t slope, uint64_t d) {
    return base + (uint64_t)(((u128)slope * d) >> 32);
}

/*
 * Build an LCG1 blob (FORMAT F1-F6).  keys: n keys as u64 (key_bits 32 or 64).
 * force_break / slope_mode as in oracle_segment_ex (NULL / 0 give the normative encoder).
 * *blob is malloc'ed; free with oracle_free.
 */
static int32_t or_encode(const uint64_t* K, uint64_t n, uint32_t key_bits, uint64_t eps,
                         uint32_t flags, const uint8_t* force_break, int slope_mode,
                         uint8_t** blob, uint64_t* blob_bytes) {
    if (!blob || !blob_bytes) return OR_ERR_ARG;
    if (n == 0) return OR_ERR_EMPTY;
    if (!K) return OR_ERR_ARG;
    if (key_bits != 32 && key_bits != 64) return OR_ERR_ARG;
    if (eps > ((flags & 1u) ? 0x3fffffffULL : 0x7fffffffULL)) return OR_ERR_ARG;
    if (n >= (1ULL << 32)) return OR_ERR_TOO_LARGE;
    for (uint64_t i = 1; i < n; i++)
        if (K[i] <= K[i - 1]) return OR_ERR_UNSORTED;
    if (key_bits == 32 && K[n - 1] > 0xffffffffULL) return OR_ERR_TOO_LARGE;

    uint64_t* st = malloc(n * 8), *ba = malloc(n * 8), *sl = malloc(n * 8);
    if (!st || !ba || !sl) { free(st); free(ba); free(sl); return OR_ERR_ALLOC; }
    int64_t L = (flags & 2u)   /* fewest segments (encoder option, not stored in the header) */
                    ? oracle_segment_min(K, n, eps, (int)(flags & 1u), 32, 0x7fffffffffffffffULL,
                                         st, ba, sl)
                : (flags & 1u)
                    ? oracle_segment_free(K, n, eps, 32, 0x7fffffffffffffffULL, st, ba, sl)
                    : oracle_segment_ex(K, n, eps, 32, 0x7fffffffffffffffULL, force_break,
                                        slope_mode, st, ba, sl);
    flags &= 1u; /* the header records the format (F7 bit) only */
    if (L < 0) { free(st); free(ba); free(sl); return (int32_t)L; }

    or_hdr h;
    memset(&h, 0, sizeof h);
    h.key_bits = key_bits;
    h.b = oracle_width(eps);
    h.eps = (uint32_t)eps;
    h.hint_log2 = OR_HINT_LOG2;
    h.flags = flags;
    h.n = n;
    h.L = (uint64_t)L;
    or_layout(&h);
    uint8_t* B = calloc(1, h.total);
    if (!B) { free(st); free(ba); free(sl); return OR_ERR_ALLOC; }

    /* F1 header */
    memcpy(B, "LCG1", 4);
    B[4] = 1; B[5] = 0; /* version 1 */
    B[6] = (uint8_t)key_bits;
    B[7] = (uint8_t)h.b;
    wr32(B + 8, h.eps);
    wr32(B + 12, h.hint_log2);
    wr64(B + 16, h.n);
    wr64(B + 24, h.L);
    wr64(B + 32, h.n_hint);
    wr64(B + 40, h.W);
    wr64(B + 48, h.o_starts);
    wr64(B + 56, h.o_params);
    wr64(B + 64, h.o_hint);
    wr64(B + 72, h.o_words);
    wr64(B + 80, h.total);
    wr32(B + 88, h.flags);

    /* F2 starts (with starts[L] = N) and params */
    for (uint64_t j = 0; j < h.L; j++) {
        wr32(B + h.o_starts + 4 * j, (uint32_t)st[j]);
        wr64(B + h.o_params + 16 * j, ba[j]);
        wr64(B + h.o_params + 16 * j + 8, sl[j]);
    }
    wr32(B + h.o_starts + 4 * h.L, (uint32_t)n);

    /* F2 hint: hint[h] = max{j : starts[j] <= 1024 h} for h < H, hint[H] = L - 1 */
    uint64_t H = h.n_hint - 1;
    for (uint64_t q = 0, j = 0; q < H; q++) {
        while (j + 1 < h.L && st[j + 1] <= 1024 * q) j++;
        wr32(B + h.o_hint + 4 * q, (uint32_t)j);
    }
    wr32(B + h.o_hint + 4 * H, (uint32_t)(h.L - 1));

    /* residuals u_i = K[i] - floor(f(i)) + eps in [0, 2 eps], packed LSB-first (F2, F3):
     * K[i] - (base + floor(slope d / 2^32)) + c with the decode bias c (F3, F7) */
    uint64_t j = 0;
    for (uint64_t i = 0; i < n; i++) {
        while (j + 1 < h.L && st[j + 1] <= i) j++;
        uint64_t u = K[i] - predict(ba[j], sl[j], i - st[j]) + bias_of(&h);
        for (uint32_t t = 0; t < h.b; t++) {
            if ((u >> t) & 1) {
                uint64_t p = i * h.b + t;
                B[h.o_words + 4 * (p >> 5) + ((p & 31) >> 3)] |= (uint8_t)(1u << (p & 7));
            }
        }
    }
    free(st); free(ba); free(sl);
    *blob = B;
    *blob_bytes = h.total;
    return OR_OK;
}

int32_t oracle_encode_ex(const uint64_t* K, uint64_t n, uint32_t key_bits, uint64_t eps,
                         const uint8_t* force_break, int slope_mode, uint8_t** blob,
                         uint64_t* blob_bytes) {
    return or_encode(K, n, key_bits, eps, 0, force_break, slope_mode, blob, blob_bytes);
}

int32_t oracle_encode(const uint64_t* K, uint64_t n, uint32_t key_bits, uint64_t eps,
                      uint8_t** blob, uint64_t* blob_bytes) {
    return or_encode(K, n, key_bits, eps, 0, 0, 0, blob, blob_bytes);
}

/* FORMAT F7 blob (flags = 1): free-intercept segments from oracle_segment_free */
int32_t oracle_encode_free(const uint64_t* K, uint64_t n, uint32_t key_bits, uint64_t eps,
                           uint8_t** blob, uint64_t* blob_bytes) {
    return or_encode(K, n, key_bits, eps, 1, 0, 0, blob, blob_bytes);
}

/* fewest segments (oracle_segment_min): free != 0 for F7 blobs */
int32_t oracle_encode_min(const uint64_t* K, uint64_t n, uint32_t key_bits, uint64_t eps,
                          int32_t free_icpt, uint8_t** blob, uint64_t* blob_bytes) {
    return or_encode(K, n, key_bits, eps, 2u | (free_icpt ? 1u : 0u), 0, 0, blob, blob_bytes);
}

void oracle_free(void* p) { free(p); }

/* ------------------------------------------------------------------------------ decoding */

static int or_read_hdr(const uint8_t* B, uint64_t bytes, or_hdr* h) {
    if (!B || bytes < OR_HEADER_BYTES) return OR_ERR_FORMAT;
    if (memcmp(B, "LCG1", 4) != 0) return OR_ERR_FORMAT;
    if (B[4] != 1 || B[5] != 0) return OR_ERR_FORMAT;
    h->key_bits = B[6];
    h->b = B[7];
    h->eps = rd32(B + 8);
    h->hint_log2 = rd32(B + 12);
    h->n = rd64(B + 16);
    h->L = rd64(B + 24);
    uint64_t n_hint = rd64(B + 32), W = rd64(B + 40);
    uint64_t o1 = rd64(B + 48), o2 = rd64(B + 56), o3 = rd64(B + 64), o4 = rd64(B + 72);
    uint64_t tot = rd64(B + 80);
    if (h->key_bits != 32 && h->key_bits != 64) return OR_ERR_FORMAT;
    if (h->eps > 0x7fffffffu || h->b != oracle_width(h->eps)) return OR_ERR_FORMAT;
    if (h->hint_log2 != OR_HINT_LOG2) return OR_ERR_FORMAT;
    if (h->n == 0 || h->n >= (1ULL << 32) || h->L == 0 || h->L > h->n) return OR_ERR_FORMAT;
    h->flags = rd32(B + 88);
    if (h->flags > 1u) return OR_ERR_FORMAT;
    if ((h->flags & 1u) && h->eps > 0x3fffffffu) return OR_ERR_FORMAT; /* F7 */
    for (int k = 92; k < 128; k++)
        if (B[k] != 0) return OR_ERR_FORMAT;
    or_layout(h);
    if (n_hint != h->n_hint || W != h->W || o1 != h->o_starts || o2 != h->o_params ||
        o3 != h->o_hint || o4 != h->o_words || tot != h->total)
        return OR_ERR_FORMAT;
    if (bytes < h->total) return OR_ERR_FORMAT; /* truncated */
    return OR_OK;
}

/* j = max{t : starts[t] <= i}: plain binary search over the starts section (F3) */
static uint64_t seg_of(const uint8_t* B, const or_hdr* h, uint64_t i) {
    uint64_t lo = 0, hi = h->L; /* starts[lo] <= i < starts[hi] */
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (rd32(B + h->o_starts + 4 * mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

/* FORMAT F3 for one index: key = (base_j + floor(slope_j d / 2^32) + u - c) mod 2^64,
 * truncated to key_bits (c = eps, or 0 for F7 blobs). */
static uint64_t key_at(const uint8_t* B, const or_hdr* h, uint64_t i, uint64_t j) {
    uint64_t s = rd32(B + h->o_starts + 4 * j);
    uint64_t base = rd64(B + h->o_params + 16 * j);
    uint64_t slope = rd64(B + h->o_params + 16 * j + 8);
    uint64_t u = field_at(B + h->o_words, i, h->b);
    uint64_t k = predict(base, slope, i - s) + u - bias_of(h);
    if (h->key_bits == 32) k &= 0xffffffffULL;
    return k;
}

static void put_key(void* out, uint32_t key_bits, uint64_t pos, uint64_t k) {
    if (key_bits == 32) ((uint32_t*)out)[pos] = (uint32_t)k;
    else ((uint64_t*)out)[pos] = k;
}

/* Full decode of keys [i0, i1) (Def. 1; Fig. 2 decoding stage PAPER.md:94-95):
 * out receives i1-i0 keys of key_bits/8 bytes each. */
int32_t oracle_decode_span(const uint8_t* B, uint64_t bytes, uint64_t i0, uint64_t i1, void* out) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    if (i0 > i1 || i1 > h.n) return OR_ERR_ARG;
    if (i0 == i1) return OR_OK;
    uint64_t j = seg_of(B, &h, i0);
    for (uint64_t i = i0; i < i1; i++) {
        while (j + 1 < h.L && rd32(B + h.o_starts + 4 * (j + 1)) <= i) j++;
        put_key(out, h.key_bits, i - i0, key_at(B, &h, i, j));
    }
    return OR_OK;
}

int32_t oracle_decode(const uint8_t* B, uint64_t bytes, void* out) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    return oracle_decode_span(B, bytes, 0, h.n, out);
}

/* The same decode split into 65536-key spans over OpenMP threads (timing the CPU baseline on
 * all host cores); each span is oracle_decode_span unchanged. Returns threads used. */
int32_t oracle_decode_mt(const uint8_t* B, uint64_t bytes, void* out, int32_t* threads_used) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    uint64_t chunks = (h.n + 65535) / 65536;
    int32_t bad = 0, nt = 1;
#pragma omp parallel
    {
#pragma omp single
        {
#ifdef _OPENMP
            nt = omp_get_num_threads();
#endif
        }
#pragma omp for schedule(dynamic, 4)
        for (int64_t c = 0; c < (int64_t)chunks; c++) {
            uint64_t a = (uint64_t)c * 65536, e = a + 65536 < h.n ? a + 65536 : h.n;
            uint8_t* o = (uint8_t*)out + a * (h.key_bits / 8);
            if (oracle_decode_span(B, bytes, a, e, o)) bad = 1;
        }
    }
    if (threads_used) *threads_used = nt;
    return bad ? OR_ERR_FORMAT : OR_OK;
}

/* Random access Dec(K^c)[i] ("f(j) + Delta[j]"; Table I caption PAPER.md:309,
 * binary search for the segment).  Out-of-range i: out = 0 and *err |= 1. */
int32_t oracle_access(const uint8_t* B, uint64_t bytes, const uint64_t* idx, uint64_t q,
                      void* out, uint32_t* err) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    uint32_t e = 0;
#pragma omp parallel for schedule(static) reduction(| : e)
    for (int64_t t = 0; t < (int64_t)q; t++) {
        uint64_t i = idx[t];
        if (i >= h.n) {
            put_key(out, h.key_bits, (uint64_t)t, 0);
            e |= 1u;
            continue;
        }
        put_key(out, h.key_bits, (uint64_t)t, key_at(B, &h, i, seg_of(B, &h, i)));
    }
    if (err) *err |= e;
    return OR_OK;
}

/* Segments-only prediction floor(f(i)) = base_j + floor(slope_j (i - s_j) / 2^32) (Eq. 1;
 * omitting the residuals gives approximate answers with error <= eps),
 * saturated at the key width's maximum (reading L24).  Out-of-range i: out = 0 and
 * *err |= 1. */
int32_t oracle_predict(const uint8_t* B, uint64_t bytes, const uint64_t* idx, uint64_t q,
                       void* out, uint32_t* err) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    uint32_t e = 0;
    for (uint64_t t = 0; t < q; t++) {
        uint64_t i = idx[t];
        if (i >= h.n) {
            put_key(out, h.key_bits, t, 0);
            e |= 1u;
            continue;
        }
        uint64_t j = seg_of(B, &h, i);
        uint64_t s = rd32(B + h.o_starts + 4 * j);
        uint64_t slope = rd64(B + h.o_params + 16 * j + 8);
        /* floor(f(i)) = base + floor(slope d / 2^32) + (eps - c): F7 bases sit eps below beta */
        u128 f = (u128)rd64(B + h.o_params + 16 * j) + (((u128)slope * (i - s)) >> 32) +
                 (h.eps - bias_of(&h));
        u128 top = h.key_bits == 32 ? (u128)0xffffffffULL : (u128)0xffffffffffffffffULL;
        put_key(out, h.key_bits, t, (uint64_t)(f > top ? top : f)); /* saturate (DESIGN L24) */
    }
    if (err) *err |= e;
    return OR_OK;
}

/* Range decode: out[len*r + k] = K[start_r + k], k < len.  start_r + len > n: the range's
 * slots are 0 and *err |= 1. */
int32_t oracle_range(const uint8_t* B, uint64_t bytes, const uint64_t* start, uint64_t q,
                     uint32_t len, void* out, uint32_t* err) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    uint32_t e = 0;
#pragma omp parallel for schedule(static) reduction(| : e)
    for (int64_t r = 0; r < (int64_t)q; r++) {
        uint64_t s0 = start[r];
        if (s0 > h.n || len > h.n - s0) {
            for (uint32_t k = 0; k < len; k++) put_key(out, h.key_bits, (uint64_t)r * len + k, 0);
            e |= 1u;
            continue;
        }
        uint64_t j = len ? seg_of(B, &h, s0) : 0;
        for (uint32_t k = 0; k < len; k++) {
            uint64_t i = s0 + k;
            while (j + 1 < h.L && rd32(B + h.o_starts + 4 * (j + 1)) <= i) j++;
            put_key(out, h.key_bits, (uint64_t)r * len + k, key_at(B, &h, i, j));
        }
    }
    if (err) *err |= e;
    return OR_OK;
}

/* Full validation of a host blob (FORMAT F1/F2 invariants; SPEC.md:464 idea of checking
 * magic, version, monotone starts).  Also checks residual fields <= 2 eps and zero padding. */
int32_t oracle_validate(const uint8_t* B, uint64_t bytes) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    /* zero filler between sections and after the header */
    uint64_t ends[4] = {h.o_starts + 4 * (h.L + 1), h.o_params + 16 * h.L,
                        h.o_hint + 4 * h.n_hint, h.total};
    uint64_t begins[4] = {h.o_starts, h.o_params, h.o_hint, h.o_words};
    for (uint64_t p = OR_HEADER_BYTES; p < h.o_starts; p++)
        if (B[p]) return OR_ERR_FORMAT;
    for (int s = 0; s < 3; s++)
        for (uint64_t p = ends[s]; p < begins[s + 1]; p++)
            if (B[p]) return OR_ERR_FORMAT;
    /* starts: 0 = s_0 < s_1 < ... < s_L = N */
    if (rd32(B + h.o_starts) != 0) return OR_ERR_FORMAT;
    if (rd32(B + h.o_starts + 4 * h.L) != h.n) return OR_ERR_FORMAT;
    for (uint64_t j = 0; j < h.L; j++)
        if (rd32(B + h.o_starts + 4 * (j + 1)) <= rd32(B + h.o_starts + 4 * j)) return OR_ERR_FORMAT;
    /* params: 0 <= slope, slope * (len - 1) <= 2^63 - 1 */
    for (uint64_t j = 0; j < h.L; j++) {
        uint64_t slope = rd64(B + h.o_params + 16 * j + 8);
        uint64_t len = rd32(B + h.o_starts + 4 * (j + 1)) - rd32(B + h.o_starts + 4 * j);
        if (slope >> 63) return OR_ERR_FORMAT;
        if ((u128)slope * (len - 1) > (u128)0x7fffffffffffffffULL) return OR_ERR_FORMAT;
    }
    /* hint */
    uint64_t H = h.n_hint - 1;
    for (uint64_t q = 0; q < H; q++)
        if (rd32(B + h.o_hint + 4 * q) != seg_of(B, &h, 1024 * q)) return OR_ERR_FORMAT;
    if (rd32(B + h.o_hint + 4 * H) != h.L - 1) return OR_ERR_FORMAT;
    /* residual fields in [0, 2 eps]; stream bits past n*b are zero */
    for (uint64_t i = 0; i < h.n; i++)
        if (field_at(B + h.o_words, i, h.b) > 2ULL * h.eps) return OR_ERR_FORMAT;
    /* anchor (F2, anchored blobs only): the field at every segment start is eps */
    if (!(h.flags & 1u))
        for (uint64_t j = 0; j < h.L; j++)
            if (field_at(B + h.o_words, rd32(B + h.o_starts + 4 * j), h.b) != h.eps)
                return OR_ERR_FORMAT;
    for (uint64_t p = h.n * h.b; p < 32 * h.W; p++)
        if (bit_at(B + h.o_words, p)) return OR_ERR_FORMAT;
    /* decoded keys strictly increasing and within key_bits (corruption detector) */
    uint64_t prev = 0, j = 0;
    for (uint64_t i = 0; i < h.n; i++) {
        while (j + 1 < h.L && rd32(B + h.o_starts + 4 * (j + 1)) <= i) j++;
        uint64_t s = rd32(B + h.o_starts + 4 * j);
        uint64_t base = rd64(B + h.o_params + 16 * j);
        uint64_t slope = rd64(B + h.o_params + 16 * j + 8);
        u128 full = (u128)base + (((u128)slope * (i - s)) >> 32) +
                    field_at(B + h.o_words, i, h.b);
        if (full < bias_of(&h)) return OR_ERR_FORMAT;
        full -= bias_of(&h);
        if (full > (h.key_bits == 32 ? (u128)0xffffffffULL : (u128)0xffffffffffffffffULL))
            return OR_ERR_FORMAT;
        if (i > 0 && (uint64_t)full <= prev) return OR_ERR_FORMAT;
        prev = (uint64_t)full;
    }
    return OR_OK;
}

/* header fields for the Python side: out[0..14] = key_bits, b, eps, hint_log2, n, L,
 * n_hint, W, o_starts, o_params, o_hint, o_words, total, flags */
int32_t oracle_header(const uint8_t* B, uint64_t bytes, uint64_t* out) {
    or_hdr h;
    int32_t st = or_read_hdr(B, bytes, &h);
    if (st) return st;
    uint64_t v[14] = {h.key_bits, h.b, h.eps, h.hint_log2, h.n, h.L, h.n_hint, h.W,
                      h.o_starts, h.o_params, h.o_hint, h.o_words, h.total, h.flags};
    memcpy(out, v, sizeof v);
    return OR_OK;
}
