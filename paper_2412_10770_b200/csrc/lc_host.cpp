// lc_host.cpp -- host side of the C ABI (include/lc.h): encoders, validator, view setup.
//
// Two encoders: the greedy anchored integer cone of FORMAT F4-F6 (the eps-PLA of Def. 2,
// PAPER.md:171-181, fitted greedily per the north star) and the free-intercept O'Rourke rule of
// FORMAT F7 on the format's integer lattice; residual packing per
// PAPER.md:184-186.  It is written independently of
// oracle/ (which tests compare byte for byte) and optimised for throughput: the
// cone is tested with 64x64->128 multiplications and divides only when a bound tightens.
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lc.h"
#include "lc_internal.h"

static_assert(sizeof(lc_header) == 128, "FORMAT F1: 128-byte header");
static_assert(offsetof(lc_header, flags) == 88, "FORMAT F1: flags at offset 88");

namespace {

using u128 = unsigned __int128;
constexpr uint64_t kSlopeMax = 0x7fffffffffffffffULL;  // guard G = 2^63 - 1 (FORMAT F2)
constexpr uint32_t kEpsMaxFree = 0x3fffffffu;           // FORMAT F7: eps <= 2^30 - 1

// floor(x / d) for a quotient known to be < 2^64
inline uint64_t div_q64(u128 x, uint64_t d) {
#if defined(__x86_64__)
    uint64_t q, r;
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    __asm__("divq %4" : "=a"(q), "=d"(r) : "a"(lo), "d"(hi), "rm"(d));
    return q;
#else
    return (uint64_t)(x / d);
#endif
}

inline uint64_t rup(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Layout {
    uint64_t H, n_hint, W, o_starts, o_params, o_hint, o_words, total;
};

Layout layout_of(uint64_t n, uint64_t L, uint32_t b) {
    Layout y;
    y.H = (n + 1023) >> 10;
    y.n_hint = y.H + 1;
    y.W = rup((n * b + 31) / 32 + 1, 4);
    y.o_starts = 256;
    y.o_params = rup(y.o_starts + 4 * (L + 1), 256);
    y.o_hint = rup(y.o_params + 16 * L, 256);
    y.o_words = rup(y.o_hint + 4 * y.n_hint, 256);
    y.total = y.o_words + 4 * y.W;
    return y;
}

template <typename K>
int32_t check_sorted(const K* k, uint64_t n) {
    for (uint64_t i = 1; i < n; ++i)
        if (k[i] <= k[i - 1]) return LC_ERR_UNSORTED;
    return LC_OK;
}

// One greedy segment anchored at s (FORMAT F4): returns its end e and slope (F5).
template <typename K>
inline uint64_t fit_segment(const K* k, uint64_t n, uint64_t s, uint64_t eps, uint64_t* slope) {
    const uint64_t base = k[s];
    uint64_t lo = 0, hi = kSlopeMax;  // current cone [lo, hi] of slope * 2^32
    uint64_t e = s + 1;
    for (; e < n; ++e) {
        const uint64_t d = e - s;
        const uint64_t D = (uint64_t)k[e] - base;
        const u128 lod = (u128)lo * d, hid = (u128)hi * d;
        const u128 X = ((((u128)D + eps + 1) << 32) - 1);  // slope <= floor(X / d)
        if (lod > X || lod > (u128)kSlopeMax) break;       // lo above the upper bound or guard
        uint64_t nlo = lo, nhi = hi;
        if (D > eps) {
            const u128 Y = (u128)(D - eps) << 32;          // slope >= ceil(Y / d)
            if (Y > hid) break;                            // lower bound above hi
            if (Y > lod) nlo = div_q64(Y + d - 1, d);
        }
        if (X < hid) nhi = div_q64(X, d);
        if ((u128)kSlopeMax < hid) {
            const uint64_t g = kSlopeMax / d;
            if (g < nhi) nhi = g;
        }
        if (nlo > nhi) break;  // F6
        lo = nlo;
        hi = nhi;
    }
    *slope = (e - s == 1) ? 0 : lo + (hi - lo) / 2;
    return e;
}

// ------------------------------------------------------------------ FORMAT F7 (free intercept)
// Segment [s, e) with intercept beta = K[s] + delta and slope S (x 2^-32) must satisfy, per key
// i (d = i - s, D = K[i] - K[s]):  S d >= (D - eps - delta) 2^32  and  S d <= (D + eps + 1 -
// delta) 2^32 - 1, plus 0 <= S <= G / d_max.  For fixed delta this is the F4 cone; as functions
// of delta the bounds are lines  lo_i(delta) = (Lo_i - delta) 2^32 / d_i  (Lo_i = D - eps) and
// up_i(delta) = ((Up_i - delta) 2^32 - 1) / d_i  (Up_i = D + eps + 1).  Keys arrive with d
// increasing, so every new line is flatter than all earlier ones: the max of the lower lines and
// the min of the upper lines are convex-hull-trick envelopes with pushes at one end, and the new
// key's constraints cut the real-feasible delta set by a ray (new lower line vs old upper
// envelope: a left ray; old lower envelope vs new upper line, and the guard: right rays).
// A witness (delta, S) is tested in O(1) per key; only when it fails are the exact integer ends
// of the feasible delta interval re-derived by binary search and a new witness placed in its
// middle.  All comparisons are exact in 128-bit integers (|values| < 2^99).
using i128 = __int128;

// floor(a / d) for d > 0, clamped to kSlopeMax + 1 (every caller clamps to <= kSlopeMax);
// one divq when the quotient fits 64 bits instead of a 128-bit library division
inline i128 fdiv(i128 a, int64_t d) {
    if (a < 0) return -(i128)(((unsigned __int128)(-a) + (uint64_t)d - 1) / (uint64_t)d);
    const unsigned __int128 ua = (unsigned __int128)a;
    if ((uint64_t)(ua >> 64) >= (uint64_t)d) return (i128)kSlopeMax + 1;
    return (i128)div_q64(ua, (uint64_t)d);
}
inline i128 cdiv0(i128 a, int64_t d) {  // max(0, ceil(a / d)), d > 0, same clamp
    return a <= 0 ? 0 : fdiv(a + d - 1, d);
}

struct Line {
    int64_t c;   // Lo_i (lower band) or Up_i (upper band)
    int64_t d;   // i - s >= 1
};

class FreeFit {
public:
    explicit FreeFit(uint64_t eps) : eps_((int64_t)eps) {
        lo_.reserve(64);
        up_.reserve(64);
    }

    // fits the segment starting at s; returns e, writes base (= beta - eps) and slope
    template <typename K>
    uint64_t fit(const K* k, uint64_t n, uint64_t s, uint64_t* base, uint64_t* slope) {
        const uint64_t ks = (uint64_t)k[s];
        dlo_ = ks >= 2 * (uint64_t)eps_ ? -eps_ : eps_ - (int64_t)ks;  // beta - eps >= 0
        p_ = dlo_;
        q_ = eps_;
        lo_.clear();
        up_.clear();
        wd_ = clamp0();
        cl_ = 0;
        ch_ = kSlopeMax;
        gd_ = kSlopeMax;
        const uint64_t dmax_key = (uint64_t)0x7fffffff + 2 * (uint64_t)eps_;
        uint64_t e = s + 1;
        for (; e < n; ++e) {
            const int64_t d = (int64_t)(e - s);
            const uint64_t D = (uint64_t)k[e] - ks;
            if (D > dmax_key) break;  // floor(S d / 2^32) <= 2^31 - 1 under the guard
            const Line lo{(int64_t)D - eps_, d}, up{(int64_t)D + eps_ + 1, d};
            const uint64_t gd = kSlopeMax / (uint64_t)d;
            if (!cone_step(lo, up, gd) && !refit(lo, up, gd)) break;
            push_lo(lo);
            push_up(up);
            gd_ = gd;
        }
        int64_t dc;
        uint64_t sc = 0;
        if (e - s == 1) {
            dc = clamp0();
        } else {
            choose(&dc, &sc);
        }
        *base = (uint64_t)((int64_t)(ks - (uint64_t)eps_) + dc);  // K[s] + delta - eps >= 0
        *slope = sc;
        return e;
    }

private:
    int64_t eps_, dlo_ = 0, p_ = 0, q_ = 0, wd_ = 0;
    uint64_t cl_ = 0, ch_ = 0, gd_ = 0;  // slope interval [cl_, ch_] of the witness intercept
    std::vector<Line> lo_, up_;

    int64_t clamp0() const { return dlo_ > 0 ? dlo_ : 0; }

    // (c - delta) 2^32 for the lower band, (c - delta) 2^32 - 1 for the upper band
    static i128 lnum(const Line& l, int64_t x) { return ((i128)(l.c - x)) << 32; }
    static i128 unum(const Line& l, int64_t x) { return (((i128)(l.c - x)) << 32) - 1; }

    // envelope positions: lo_ back = flattest = rightmost region; up_ back = flattest = leftmost
    static bool lo_ge(const Line& a, const Line& b, int64_t x) {  // lo_a(x) >= lo_b(x)
        return (i128)(a.c - x) * b.d >= (i128)(b.c - x) * a.d;
    }
    static bool up_le(const Line& a, const Line& b, int64_t x) {  // up_a(x) <= up_b(x)
        return unum(a, x) * b.d <= unum(b, x) * a.d;
    }
    // crossing abscissa of lines a (steeper, d_a < d_b) and b: (c_a d_b - c_b d_a)/(d_b - d_a)
    // (the upper band's crossings share a -2^-32 shift, which cancels in comparisons)
    static bool cross_le(const Line& a, const Line& b, const Line& c, const Line& e) {
        // x(a, b) <= x(c, e)
        const i128 n1 = (i128)a.c * b.d - (i128)b.c * a.d, d1 = b.d - a.d;
        const i128 n2 = (i128)c.c * e.d - (i128)e.c * c.d, d2 = e.d - c.d;
        return n1 * d2 <= n2 * d1;
    }
    void push_lo(const Line& l) {
        while (lo_.size() >= 2) {
            const Line& t = lo_.back();
            const Line& t1 = lo_[lo_.size() - 2];
            if (cross_le(t, l, t1, t)) lo_.pop_back();  // x(t, new) <= x(t1, t): t never maximal
            else break;
        }
        lo_.push_back(l);
    }
    void push_up(const Line& l) {
        while (up_.size() >= 2) {
            const Line& t = up_.back();
            const Line& t1 = up_[up_.size() - 2];
            if (cross_le(t1, t, t, l)) up_.pop_back();  // x(t, new) >= x(t1, t): t never minimal
            else break;
        }
        up_.push_back(l);
    }
    const Line& lo_at(int64_t x) const {  // active line of max_i lo_i at x (lo_ non-empty)
        size_t a = 0, b = lo_.size() - 1;
        while (a < b) {
            const size_t m = (a + b) >> 1;
            if (lo_ge(lo_[m], lo_[m + 1], x)) b = m;
            else a = m + 1;
        }
        return lo_[a];
    }
    const Line& up_at(int64_t x) const {  // active line of min_i up_i at x (up_ non-empty)
        size_t a = 0, b = up_.size() - 1;
        while (a < b) {
            const size_t m = (a + b) >> 1;
            if (up_le(up_[m], up_[m + 1], x)) b = m;
            else a = m + 1;
        }
        return up_[a];
    }
    // lo_a(x) <= up_b(x) and lo_a(x) <= gd (real comparisons)
    static bool lo_le_up(const Line& a, const Line& b, int64_t x) {
        return lnum(a, x) * b.d <= unum(b, x) * a.d;
    }
    static bool lo_le_g(const Line& a, uint64_t gd_num, int64_t gd_den, int64_t x) {
        // lo_a(x) <= G / gd_den  <=>  lnum * gd_den <= G * d_a
        return lnum(a, x) * gd_den <= (i128)gd_num * a.d;
    }

    // the F4 cone at the witness intercept wd_, advanced by one key (divides only when a bound
    // tightens); false when it empties -- then refit() moves the intercept
    bool cone_step(const Line& lo, const Line& up, uint64_t gd) {
        const int64_t d = lo.d;
        const i128 lod = (i128)cl_ * d, hid = (i128)ch_ * d;
        const i128 X = unum(up, wd_), Y = lnum(lo, wd_);  // S d <= X, S d >= Y
        if (lod > X || Y > hid || cl_ > gd) return false;
        uint64_t nlo = cl_, nhi = ch_;
        if (Y > lod) nlo = (uint64_t)cdiv0(Y, d);
        if (X < hid) nhi = (uint64_t)fdiv(X, d);
        if (gd < nhi) nhi = gd;
        if (nlo > nhi) return false;
        cl_ = nlo;
        ch_ = nhi;
        return true;
    }

    // membership tests for the state extended by (lo, up) with guard G / d
    bool old_ok(int64_t x) const {
        return lo_.empty() || up_.empty() || lo_le_up(lo_at(x), up_at(x), x);
    }
    bool ray_a(const Line& lo, int64_t x) const { return up_.empty() || lo_le_up(lo, up_at(x), x); }
    bool ray_bc(const Line& lo, const Line& up, int64_t x) const {
        if (!lo_le_g(lo, kSlopeMax, lo.d, x)) return false;
        if (lo_.empty()) return true;
        const Line& a = lo_at(x);
        return lo_le_up(a, up, x) && lo_le_g(a, kSlopeMax, lo.d, x);
    }
    // real-feasibility of x for the state extended by (lo, up): one lookup per envelope
    struct Eval {
        bool a, bc, old;
        const Line *la, *ua;  // active envelope lines at x (nullptr if the envelope is empty)
    };
    Eval eval(const Line& lo, const Line& up, int64_t x) const {
        Eval r{true, lo_le_g(lo, kSlopeMax, lo.d, x), true, nullptr, nullptr};
        if (!lo_.empty()) r.la = &lo_at(x);
        if (!up_.empty()) {
            r.ua = &up_at(x);
            r.a = lo_le_up(lo, *r.ua, x);
            if (r.la) r.old = lo_le_up(*r.la, *r.ua, x);
        }
        if (r.la && r.bc) r.bc = lo_le_up(*r.la, up, x) && lo_le_g(*r.la, kSlopeMax, lo.d, x);
        return r;
    }
    bool real_ok(const Line& lo, const Line& up, int64_t x) const {
        const Eval r = eval(lo, up, x);
        return r.a && r.bc && r.old;
    }
    // integer slope interval at x for the extended state; false if empty.  la / ua: the active
    // envelope lines at x when the caller has them (nullptr: look them up)
    bool int_range(const Line* lo, const Line* up, uint64_t gd, int64_t x, uint64_t* slo,
                   uint64_t* shi, const Line* la = nullptr, const Line* ua = nullptr) const {
        i128 l = 0, h = (i128)gd;
        if (!lo_.empty()) {
            const Line& a = la ? *la : lo_at(x);
            const i128 c = cdiv0(lnum(a, x), a.d);  // clamped values only feed the l > h test
            if (c > l) l = c;
        }
        if (lo) {
            const i128 c = cdiv0(lnum(*lo, x), lo->d);
            if (c > l) l = c;
        }
        if (l > h) return false;
        if (up) {
            const i128 f = fdiv(unum(*up, x), up->d);
            if (f < h) h = f;
        }
        if (!up_.empty() && l <= h) {
            const Line& b = ua ? *ua : up_at(x);
            const i128 f = fdiv(unum(b, x), b.d);
            if (f < h) h = f;
        }
        if (l > h) return false;
        *slo = (uint64_t)l;
        *shi = (uint64_t)h;
        return true;
    }
    template <typename P>
    static int64_t first_true(int64_t a, int64_t b, P pred) {  // F..F T..T on [a, b]; b+1 if none
        int64_t lo = a, hi = b + 1;
        while (lo < hi) {
            const int64_t m = lo + ((hi - lo) >> 1);
            if (pred(m)) hi = m;
            else lo = m + 1;
        }
        return lo;
    }
    template <typename P>
    static int64_t last_true(int64_t a, int64_t b, P pred) {  // T..T F..F on [a, b]; a-1 if none
        int64_t lo = a - 1, hi = b;
        while (lo < hi) {
            const int64_t m = hi - ((hi - lo) >> 1);
            if (pred(m)) lo = m;
            else hi = m - 1;
        }
        return lo;
    }

    // the witness fails on the new key: re-derive the exact feasible interval and a new witness
    bool refit(const Line& lo, const Line& up, uint64_t gd) {
        const int64_t w = wd_;
        const Eval ew = eval(lo, up, w);
        const bool a = ew.a, bc = ew.bc;
        auto ok = [&](int64_t x) { return real_ok(lo, up, x); };
        int64_t p, q;
        if (!a && !bc) return false;
        if (a && bc) {  // w stays real-feasible
            uint64_t sl, sh;
            if (int_range(&lo, &up, gd, w, &sl, &sh, ew.la, ew.ua)) {  // defensive: the cone
                cl_ = sl;                                              // step already said no
                ch_ = sh;
                return true;
            }
            p = ok(p_) ? p_ : first_true(p_ + 1, w, ok);  // both ends by bisection around w
            q = ok(q_) ? q_ : last_true(w, q_ - 1, ok);
        } else if (!a) {  // the new lower line cut the right side off: a left ray below w
            q = last_true(p_, w - 1, [&](int64_t x) { return ray_a(lo, x); });
            if (q < p_ || !ok(q)) return false;
            p = first_true(p_, q, ok);
        } else {  // the new upper line or the guard cut the left side off
            p = first_true(w + 1, q_, [&](int64_t x) { return ray_bc(lo, up, x); });
            if (p > q_ || !ok(p)) return false;
            q = last_true(p, q_, ok);
        }
        // an integer slope at some integer delta in [p, q], searched from the middle outward
        const int64_t mid = p + ((q - p) >> 1);
        for (int64_t k = 0; mid - k >= p || mid + k <= q; ++k) {
            for (int sgn = 0; sgn < 2; ++sgn) {
                const int64_t x = sgn ? mid + k : mid - k;
                if (x < p || x > q || (sgn && k == 0)) continue;
                uint64_t sl, sh;
                if (int_range(&lo, &up, gd, x, &sl, &sh)) {
                    p_ = p;
                    q_ = q;
                    wd_ = x;
                    cl_ = sl;
                    ch_ = sh;
                    return true;
                }
            }
        }
        return false;
    }

    // F7 choice for the committed state: least |delta| (negative first), middle slope.  The
    // witness w is feasible; the real-feasible set I is an interval containing it.  If I holds
    // 0 the scan runs |delta| = 0, 1, ... (both signs, exact integer test) and stops by |w|;
    // otherwise the end of I nearest 0 is bisected and the scan walks away from 0 from there.
    void choose(int64_t* dc, uint64_t* sc) {
        const int64_t w = wd_;
        const int64_t dlast = lo_.back().d;
        auto ok = [&](int64_t x) {
            if (!old_ok(x)) return false;
            return lo_le_g(lo_at(x), kSlopeMax, dlast, x);
        };
        auto hit = [&](int64_t x) {
            uint64_t sl, sh;
            if (!int_range(nullptr, nullptr, gd_, x, &sl, &sh)) return false;
            *dc = x;
            *sc = sl + (sh - sl) / 2;
            return true;
        };
        const int64_t z = w >= 0 ? (p_ > 0 ? p_ : 0) : (q_ < 0 ? q_ : 0);
        if (z == 0 && ok(0)) {
            for (int64_t k = 0; k <= (w >= 0 ? w : -w); ++k) {
                if (-k >= p_ && hit(-k)) return;
                if (k > 0 && k <= q_ && hit(k)) return;
            }
        } else if (w >= 0) {  // I lies right of 0: scan up from its left end
            for (int64_t x = ok(z) ? z : first_true(z + 1, w, ok); x <= w; ++x)
                if (hit(x)) return;
        } else {  // I lies left of 0: scan down from its right end
            for (int64_t x = ok(z) ? z : last_true(w, z - 1, ok); x >= w; --x)
                if (hit(x)) return;
        }
        *dc = w;  // not reached: the witness is feasible
        *sc = cl_ + (ch_ - cl_) / 2;
    }
};

template <typename K>
int32_t encode_t(const K* keys, uint64_t n, uint32_t key_bits, uint32_t eps, uint32_t flags,
                 void** out_blob, uint64_t* out_bytes) {
    int32_t st = check_sorted(keys, n);
    if (st) return st;
    if (key_bits == 32 && (uint64_t)keys[n - 1] > 0xffffffffULL) return LC_ERR_TOO_LARGE;
    std::vector<uint32_t> starts;
    std::vector<uint64_t> params;  // interleaved base, slope
    starts.reserve(n / 8 + 16);
    params.reserve(n / 4 + 32);
    const bool free_base = flags & LC_FLAG_FREE_INTERCEPT;
    FreeFit ff(eps);
    if (flags & LC_FLAG_MIN_SEGMENTS) {
        // Fewest segments on the lattice (NEXT-3): [s, e) is feasible iff
        // e <= emax(s), the greedy end from s (a prefix keeps its line), so
        // f(s) = 1 + min{f(e) : s < e <= emax(s)}, f(n) = 0, the largest minimising e on a
        // tie; each chosen [s, e) is refitted on exactly its keys.  O(n * segment length).
        std::vector<uint32_t> f(n + 1), nxt(n);
        std::vector<uint32_t> emax(n);
        for (uint64_t s = 0; s < n; ++s) {
            uint64_t slope, base;
            emax[s] = (uint32_t)(free_base ? ff.fit(keys, n, s, &base, &slope)
                                           : fit_segment(keys, n, s, eps, &slope));
        }
        f[n] = 0;
        for (uint64_t s = n; s-- > 0;) {
            uint32_t best = 0xffffffffu, arg = (uint32_t)s + 1;
            for (uint64_t e = s + 1; e <= emax[s]; ++e)
                if (f[e] <= best) {
                    best = f[e];
                    arg = (uint32_t)e;
                }
            f[s] = best + 1;
            nxt[s] = arg;
        }
        for (uint64_t s = 0; s < n; s = nxt[s]) {
            const uint64_t e = nxt[s];
            uint64_t slope, base = (uint64_t)keys[s];
            if (free_base) ff.fit(keys, e, s, &base, &slope);
            else fit_segment(keys, e, s, eps, &slope);
            starts.push_back((uint32_t)s);
            params.push_back(base);
            params.push_back(slope);
        }
        flags &= ~(uint32_t)LC_FLAG_MIN_SEGMENTS;  // an encoder option, not a format flag
    } else {
        for (uint64_t s = 0; s < n;) {
            uint64_t slope, base = (uint64_t)keys[s];
            const uint64_t e = free_base ? ff.fit(keys, n, s, &base, &slope)
                                         : fit_segment(keys, n, s, eps, &slope);
            starts.push_back((uint32_t)s);
            params.push_back(base);
            params.push_back(slope);
            s = e;
        }
    }
    const uint64_t bias = free_base ? 0 : eps;  // FORMAT F3 decode bias c
    const uint64_t L = starts.size();
    const uint32_t b = lc_detail::res_bits(eps);
    const Layout y = layout_of(n, L, b);
    uint8_t* blob = (uint8_t*)std::calloc(1, y.total);
    if (!blob) return LC_ERR_ALLOC;

    lc_header h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "LCG1", 4);
    h.version = 1;
    h.key_bits = (uint8_t)key_bits;
    h.res_bits = (uint8_t)b;
    h.eps = eps;
    h.hint_log2 = 10;
    h.flags = flags;
    h.n = n;
    h.n_seg = L;
    h.n_hint = y.n_hint;
    h.n_words = y.W;
    h.off_starts = y.o_starts;
    h.off_params = y.o_params;
    h.off_hint = y.o_hint;
    h.off_words = y.o_words;
    h.total_bytes = y.total;
    std::memcpy(blob, &h, sizeof h);

    uint32_t* S = (uint32_t*)(blob + y.o_starts);
    std::memcpy(S, starts.data(), 4 * L);
    S[L] = (uint32_t)n;
    std::memcpy(blob + y.o_params, params.data(), 16 * L);

    // hint[q] = segment holding key 1024 q; hint[H] = L - 1
    uint32_t* Hn = (uint32_t*)(blob + y.o_hint);
    for (uint64_t q = 0, j = 0; q < y.H; ++q) {
        const uint64_t key = q << 10;
        while (j + 1 < L && S[j + 1] <= key) ++j;
        Hn[q] = (uint32_t)j;
    }
    Hn[y.H] = (uint32_t)(L - 1);

    // residual fields u = K[i] - floor(f(i)) + eps = K[i] - base - floor(slope d / 2^32) + c,
    // LSB-first into 32-bit words
    if (b) {
        uint32_t* Wd = (uint32_t*)(blob + y.o_words);
        uint64_t acc = 0;
        uint32_t nbits = 0;
        uint64_t w = 0;
        for (uint64_t j = 0; j < L; ++j) {
            const uint64_t s = S[j], e = S[j + 1];
            const uint64_t base = params[2 * j], slope = params[2 * j + 1];
            uint64_t run = 0;  // slope * d, < 2^63 by the guard
            for (uint64_t i = s; i < e; ++i, run += slope) {
                const uint64_t u = (uint64_t)keys[i] - base - (run >> 32) + bias;
                acc |= u << nbits;
                nbits += b;
                if (nbits >= 32) {
                    Wd[w++] = (uint32_t)acc;
                    acc >>= 32;
                    nbits -= 32;
                }
            }
        }
        if (nbits) Wd[w++] = (uint32_t)acc;
    }
    *out_blob = blob;
    *out_bytes = y.total;
    return LC_OK;
}

std::atomic<uint64_t> g_launches{0};

}  // namespace

namespace lc_detail {

uint32_t res_bits(uint64_t eps) {
    uint32_t b = 0;
    while ((1ULL << b) < 2 * eps + 1) ++b;  // eps <= 2^31 - 1 so 2 eps + 1 < 2^32
    return b;
}

int32_t check_header(const lc_header* h, uint64_t blob_bytes) {
    if (std::memcmp(h->magic, "LCG1", 4) != 0 || h->version != 1) return LC_ERR_FORMAT;
    if (h->key_bits != 32 && h->key_bits != 64) return LC_ERR_FORMAT;
    if (h->eps > 0x7fffffffu || h->res_bits != res_bits(h->eps)) return LC_ERR_FORMAT;
    if (h->hint_log2 != 10) return LC_ERR_FORMAT;
    if (h->n == 0 || h->n >= (1ULL << 32) || h->n_seg == 0 || h->n_seg > h->n)
        return LC_ERR_FORMAT;
    if (h->flags & ~(uint32_t)LC_FLAG_FREE_INTERCEPT) return LC_ERR_FORMAT;
    if ((h->flags & LC_FLAG_FREE_INTERCEPT) && h->eps > kEpsMaxFree) return LC_ERR_FORMAT;
    for (int i = 0; i < 36; ++i)
        if (h->reserved[i]) return LC_ERR_FORMAT;
    const Layout y = layout_of(h->n, h->n_seg, h->res_bits);
    if (h->n_hint != y.n_hint || h->n_words != y.W || h->off_starts != y.o_starts ||
        h->off_params != y.o_params || h->off_hint != y.o_hint || h->off_words != y.o_words ||
        h->total_bytes != y.total)
        return LC_ERR_FORMAT;
    if (blob_bytes < y.total) return LC_ERR_FORMAT;
    return LC_OK;
}

void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace lc_detail

extern "C" {

int32_t lc_encode_ex(const void* keys, uint64_t n, uint32_t key_bits, uint32_t eps,
                     uint32_t flags, void** blob, uint64_t* blob_bytes) {
    if (!blob || !blob_bytes) return LC_ERR_ARG;
    if (key_bits != 32 && key_bits != 64) return LC_ERR_ARG;
    if (flags & ~(uint32_t)(LC_FLAG_FREE_INTERCEPT | LC_FLAG_MIN_SEGMENTS)) return LC_ERR_ARG;
    if (eps > ((flags & LC_FLAG_FREE_INTERCEPT) ? kEpsMaxFree : 0x7fffffffu)) return LC_ERR_ARG;
    if (n == 0) return LC_ERR_EMPTY;
    if (!keys) return LC_ERR_ARG;
    if (n >= (1ULL << 32)) return LC_ERR_TOO_LARGE;
    if (key_bits == 32)
        return encode_t((const uint32_t*)keys, n, key_bits, eps, flags, blob, blob_bytes);
    return encode_t((const uint64_t*)keys, n, key_bits, eps, flags, blob, blob_bytes);
}

int32_t lc_encode(const void* keys, uint64_t n, uint32_t key_bits, uint32_t eps, void** blob,
                  uint64_t* blob_bytes) {
    return lc_encode_ex(keys, n, key_bits, eps, 0, blob, blob_bytes);
}

void lc_free(void* blob) { std::free(blob); }

int32_t lc_validate(const void* blob, uint64_t blob_bytes) {
    if (!blob || blob_bytes < sizeof(lc_header)) return blob ? LC_ERR_FORMAT : LC_ERR_ARG;
    lc_header h;
    std::memcpy(&h, blob, sizeof h);
    int32_t st = lc_detail::check_header(&h, blob_bytes);
    if (st) return st;
    const uint8_t* B = (const uint8_t*)blob;
    const uint64_t n = h.n, L = h.n_seg, b = h.res_bits, eps = h.eps;
    const bool free_base = h.flags & LC_FLAG_FREE_INTERCEPT;
    const uint64_t bias = free_base ? 0 : eps;  // FORMAT F3 decode bias c
    // zero filler between header/sections
    const uint64_t sec_beg[4] = {h.off_starts, h.off_params, h.off_hint, h.off_words};
    const uint64_t sec_end[4] = {h.off_starts + 4 * (L + 1), h.off_params + 16 * L,
                                 h.off_hint + 4 * h.n_hint, h.total_bytes};
    for (uint64_t p = sizeof(lc_header); p < sec_beg[0]; ++p)
        if (B[p]) return LC_ERR_FORMAT;
    for (int s = 0; s < 3; ++s)
        for (uint64_t p = sec_end[s]; p < sec_beg[s + 1]; ++p)
            if (B[p]) return LC_ERR_FORMAT;
    const uint32_t* S = (const uint32_t*)(B + h.off_starts);
    const uint64_t* P = (const uint64_t*)(B + h.off_params);
    const uint32_t* Hn = (const uint32_t*)(B + h.off_hint);
    const uint32_t* Wd = (const uint32_t*)(B + h.off_words);
    if (S[0] != 0 || S[L] != n) return LC_ERR_FORMAT;
    for (uint64_t j = 0; j < L; ++j) {
        if (S[j + 1] <= S[j]) return LC_ERR_FORMAT;
        const uint64_t slope = P[2 * j + 1];
        if (slope > kSlopeMax) return LC_ERR_FORMAT;
        if ((u128)slope * (S[j + 1] - 1 - S[j]) > (u128)kSlopeMax) return LC_ERR_FORMAT;
    }
    for (uint64_t q = 0, j = 0; q < h.n_hint - 1; ++q) {
        while (j + 1 < L && S[j + 1] <= (q << 10)) ++j;
        if (Hn[q] != j) return LC_ERR_FORMAT;
    }
    if (Hn[h.n_hint - 1] != L - 1) return LC_ERR_FORMAT;
    // residual fields <= 2 eps, decoded keys strictly increasing and within key_bits,
    // stream bits past n*b zero
    const uint64_t kmax = h.key_bits == 32 ? 0xffffffffULL : ~0ULL;
    uint64_t prev = 0;
    for (uint64_t j = 0; j < L; ++j) {
        const uint64_t base = P[2 * j], slope = P[2 * j + 1];
        uint64_t run = 0;
        for (uint64_t i = S[j]; i < S[j + 1]; ++i, run += slope) {
            uint64_t u = 0;
            if (b) {
                const uint64_t p = i * b;
                const uint64_t two = (uint64_t)Wd[p >> 5] | ((uint64_t)Wd[(p >> 5) + 1] << 32);
                u = (two >> (p & 31)) & ((1ULL << b) - 1);
            }
            if (u > 2 * eps) return LC_ERR_FORMAT;
            if (!free_base && i == S[j] && u != eps) return LC_ERR_FORMAT;  // F2 anchor
            const u128 full = (u128)base + (run >> 32) + u;
            if (full < bias || full - bias > kmax) return LC_ERR_FORMAT;
            const uint64_t key = (uint64_t)(full - bias);
            if (i > 0 && key <= prev) return LC_ERR_FORMAT;
            prev = key;
        }
    }
    const uint64_t used = n * b;
    for (uint64_t w = used >> 5; w < h.n_words; ++w) {
        uint32_t v = Wd[w];
        if (w == (used >> 5)) v &= (used & 31) ? ~((1u << (used & 31)) - 1) : ~0u;
        if (v) return LC_ERR_FORMAT;
    }
    return LC_OK;
}

int32_t lc_view_init(lc_view* v, const void* host_header128, const void* d_blob,
                     uint64_t blob_bytes) {
    if (!v || !host_header128 || !d_blob) return LC_ERR_ARG;
    if ((uintptr_t)d_blob % 256) return LC_ERR_ARG;
    lc_header h;
    std::memcpy(&h, host_header128, sizeof h);
    int32_t st = lc_detail::check_header(&h, blob_bytes);
    if (st) return st;
    v->h = h;
    v->d_blob = d_blob;
    v->d_first = nullptr;
    v->d_acc = nullptr;
    v->span_lo = v->span_hi = 0;
    std::memset(v->sec_base, 0, sizeof v->sec_base);
    return LC_OK;
}

const char* lc_status_str(int32_t s) {
    switch (s) {
        case LC_OK: return "LC_OK";
        case LC_ERR_ARG: return "LC_ERR_ARG";
        case LC_ERR_EMPTY: return "LC_ERR_EMPTY";
        case LC_ERR_UNSORTED: return "LC_ERR_UNSORTED";
        case LC_ERR_TOO_LARGE: return "LC_ERR_TOO_LARGE";
        case LC_ERR_FORMAT: return "LC_ERR_FORMAT";
        case LC_ERR_ALLOC: return "LC_ERR_ALLOC";
        case LC_ERR_CUDA: return "LC_ERR_CUDA";
        default: return "LC_ERR_UNKNOWN";
    }
}

uint64_t lc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
