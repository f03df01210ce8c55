// bplb_core.h -- integer core shared by the CUDA kernels and the host side of
// libbplb.so (and compiled into the host-only arithmetic test
// tests/core_arith_test.cpp).  Everything here is exact integer arithmetic.
//
// Reference semantics (all citations /root/reference/pkg/src/binpack/...):
//   kinds / order ............ bounds.py:48-67
//   lambda ranges ............ bounds.py:219-273 (MT upper end ceil(c/2), VB2 cap)
//   per-lambda sums .......... bounds.py:373-460 (_sweep_*), 293-323 (_batch_matrix)
//   ceil-div / f(c) <= 0 ..... bounds.py:284-290, 500-501
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BPLB_HD __host__ __device__ __forceinline__
#else
#define BPLB_HD static inline
#endif

enum {
    K_MT = 0, K_RAD2 = 1, K_FS1 = 2, K_CCM1 = 3, K_VB2 = 4, K_BJ1 = 5, K_COUNT = 6
};

// Parameter domain of each kind, uncapped (bounds.py:219-273).
BPLB_HD void bplb_domain(int kind, int64_t c, int64_t* lo, int64_t* hi) {
    switch (kind) {
    case K_MT: *lo = 0; *hi = (c == 1) ? 0 : (c + 1) / 2; break;  // _mt_hi, :219-225
    case K_RAD2: *lo = c / 4 + 1; *hi = c / 3; break;
    case K_FS1: *lo = 1; *hi = 100; break;
    case K_CCM1: *lo = 1; *hi = c / 2; break;
    case K_VB2: *lo = 2; *hi = c; break;
    default: *lo = 1; *hi = c; break;
    }
}

// VB2 upper end with the accumulator cap floor((2^64-1)/(r*max_w)) applied
// when the instance is non-empty (bounds.py:38-40, 268-272).  Within the
// envelope r < 2^25 and max_w <= 2^30, so r*max_w fits in 64 bits.
BPLB_HD int64_t bplb_vb2_hi(int64_t c, int64_t r, int64_t maxw) {
    if (r <= 0) return c;
    unsigned long long prod = (unsigned long long)r * (unsigned long long)maxw;
    unsigned long long cap = 0xFFFFFFFFFFFFFFFFull / prod;
    return cap < (unsigned long long)c ? (int64_t)cap : c;
}

// Exact division n / d for n < 2^31, 1 <= d < 2^31 by a multiply-high:
//   l = ceil(log2 d), k = 31 + l, m = ceil(2^k / d) < 2^32,
//   floor(n/d) = (n*m) >> k = umulhi(2n, m) >> l.
// Proof: e = m*d - 2^k is in [0, d); n*e < 2^31 * 2^l = 2^k, so the error
// term n*e/(d*2^k) < 1/d cannot carry the quotient past the next integer.
// Exhaustively checked on small d and randomly on the full range by
// tests/core_arith_test.cpp.
struct Div31 {
    uint32_t m;
    uint32_t l;
};

BPLB_HD Div31 bplb_div31(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < (unsigned long long)d) ++l;
    unsigned long long num = 1ull << (31 + l);
    Div31 r;
    r.m = (uint32_t)((num + d - 1) / d);
    r.l = l;
    return r;
}

BPLB_HD uint32_t bplb_udiv31(uint32_t n, Div31 dv) {
#if defined(__CUDA_ARCH__)
    return __umulhi(n << 1, dv.m) >> dv.l;
#else
    return (uint32_t)((((unsigned long long)(n << 1)) * dv.m) >> 32) >> dv.l;
#endif
}

// (a * b - delta) mod c for a, b < 2^31, c < 2^31, delta in {0,1}: Barrett
// reduction with cinv = floor(2^64 / c) (exact result after <= 2 corrections).
BPLB_HD unsigned long long bplb_cinv(uint32_t c) {
    return c == 1 ? 0xFFFFFFFFFFFFFFFFull : (0xFFFFFFFFFFFFFFFFull / c);
}

BPLB_HD uint32_t bplb_mulmod(uint32_t a, uint32_t b, uint32_t delta, uint32_t c,
                             unsigned long long cinv) {
    unsigned long long x = (unsigned long long)a * b;
    if (x == 0 && delta) return c - 1;  // (0 - 1) mod c
    x -= delta;
#if defined(__CUDA_ARCH__)
    unsigned long long q = __umul64hi(x, cinv);
#else
    unsigned long long q = (unsigned long long)(((unsigned __int128)x * cinv) >> 64);
#endif
    unsigned long long r = x - q * c;
    while (r >= c) r -= c;
    return (uint32_t)r;
}

BPLB_HD uint64_t bplb_ceil_div(uint64_t s, uint64_t f) { return (s + f - 1) / f; }

// ---------------------------------------------------------------------------
// Per-node statistics (everything the per-lambda formulas need besides the
// lookup structure).  "small" = 2w < c, "eq" = 2w == c, "big" = 2w > c
// (includes w == c, counted again in n_full).  mirrored = {c - w : c/2 < w < c}.
// ---------------------------------------------------------------------------
struct NodeStats {
    int32_t r, maxw;
    int32_t n_small, n_eq, n_big, n_full;
    int64_t W;         // sum of weights
    int64_t Vs, Vm;    // sum of smalls, sum of mirrored values
    int64_t dq, dr;    // (Vs - Vm) = c*dq + dr   (VB2 closed form)
    uint64_t cinv;     // floor((2^64 - 1) / c): division-free floor(x / c)
};

BPLB_HD void bplb_stats_finish(NodeStats* st, int64_t c) {
    int64_t dv = st->Vs - st->Vm;
    st->dq = dv / c;
    st->dr = dv - st->dq * c;
    st->cinv = 0xFFFFFFFFFFFFFFFFull / (uint64_t)c;
}

// VB2 per-lambda transformed sum from D(lambda) = sum over VB2 items of the
// modular state s:
//   small w:    s = (w*lambda - 1) mod c
//   mirrored w: s = (w*lambda) mod c  (= c-1 - ((c-w)*lambda - 1) mod c)
// B_s - B_m = lambda*dq + (lambda*dr - (n_s - n_m) - (D - n_m(c-1))) / c  (exact)
// S = 2(B_s - B_m) + (n_eq + 2 n_big)(lambda - 1)            (bounds.py:433-438)
BPLB_HD int64_t bplb_vb2_sum(const NodeStats& st, int64_t c, int64_t lam, uint64_t D) {
    int64_t n_m = st.n_big - st.n_full;
    int64_t dn = (int64_t)st.n_small - n_m;
    int64_t dR = (int64_t)D - n_m * (c - 1);
    int64_t num = lam * st.dr - dn - dR;  // exact multiple of c
#if defined(__CUDA_ARCH__)
    // 32-bit divide when it fits (always for small c): 64-bit division is emulated
    const int64_t q = (num == (int64_t)(int32_t)num && c <= 0x7FFFFFFF) ? (int64_t)((int32_t)num / (int32_t)c)
                                                                        : num / c;
    int64_t dB = lam * st.dq + q;
#else
    int64_t dB = lam * st.dq + num / c;
#endif
    return 2 * dB + ((int64_t)st.n_eq + 2 * (int64_t)st.n_big) * (lam - 1);
}

// FS1 zero-remainder term Z(lambda) = sum of w with c | w(lambda+1).  Those
// are exactly the multiples of m = c / gcd(c, lambda+1), so with cumulative
// tables Z = sum_j W(j m) - W(j m - 1) over j <= max_w / m (<= 101 terms).
BPLB_HD int64_t bplb_gcd(int64_t a, int64_t b) {
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}
template <class L>
BPLB_HD int64_t bplb_fs1_zero(const L& lk, int64_t c, int64_t maxw, int64_t lam) {
    const int64_t m = c / bplb_gcd(c, lam + 1);
    int64_t z = 0;
    for (int64_t v = m; v <= maxw; v += m) {
        int64_t n1, w1, n0, w0;
        lk.both(v, &n1, &w1);
        lk.both(v - 1, &n0, &w0);
        z += w1 - w0;
    }
    return z;
}

// FS1 per-lambda transformed sum from P = sum of (w(lambda+1) mod c) and
// Z = sum of w over items with zero remainder:
//   f(w) = c*floor(w(lambda+1)/c) - [rem == 0]*w    (bounds.py:173-178, 305-307)
//   S = (lambda+1)*W - P - Z ;  F = c*lambda.
BPLB_HD int64_t bplb_fs1_sum(const NodeStats& st, int64_t lam, uint64_t P, uint64_t Z) {
    return (lam + 1) * st.W - (int64_t)P - (int64_t)Z;
}

// Transformed capacities f(c, lambda) per kind (bounds.py:284, 376, 387,
// 407, 438, 460).
BPLB_HD int64_t bplb_fc(int kind, int64_t c, int64_t lam) {
    switch (kind) {
    case K_MT: case K_RAD2: return c;
    case K_FS1: return c * lam;
    case K_CCM1: return 2 * (c / lam);
    case K_VB2: return 2 * (lam - 1);
    default: { int64_t cm = c % lam; return (c / lam) * (lam - cm); }
    }
}

// One transformed item f_k(w) for 1 <= w <= c, lambda in the kind's domain:
// the scalar transforms _mt/_rad2/_fs1/_ccm1/_vb2/_bj1 (bounds.py:155-206),
// used to tabulate f over (lambda, w) once per capacity (batched small-c
// path).  piece(v) = max(0, ceil(v*lambda/c) - 1) as in _vb2.
BPLB_HD int64_t bplb_vb2_piece(int64_t v, int64_t c, int64_t lam) {
    const int64_t q = (v * lam + c - 1) / c - 1;
    return q > 0 ? q : 0;
}
BPLB_HD int64_t bplb_cell(int kind, int64_t w, int64_t c, int64_t lam) {
    switch (kind) {
    case K_MT:  // bounds.py:155-160
        return c - lam < w ? c : (w < lam ? 0 : w);
    case K_RAD2: {  // bounds.py:163-170; lambda > c/4 makes the recursion depth <= 1
        const bool mirror = w >= 2 * lam;
        const int64_t x = mirror ? c - w : w;
        int64_t f;
        if (x < lam) f = 0;
        else if (x <= c - 2 * lam) f = c / 3;
        else f = c / 2;
        return mirror ? c - f : f;
    }
    case K_FS1: {  // bounds.py:173-178
        const int64_t num = w * (lam + 1), q = num / c;
        return num - q * c == 0 ? w * lam : q * c;
    }
    case K_CCM1:  // bounds.py:181-186
        if (2 * w > c) return 2 * (c / lam - (c - w) / lam);
        if (2 * w == c) return c / lam;
        return 2 * (w / lam);
    case K_VB2:  // bounds.py:189-197
        if (2 * w > c) return 2 * bplb_vb2_piece(c, c, lam) - 2 * bplb_vb2_piece(c - w, c, lam);
        if (2 * w == c) return bplb_vb2_piece(c, c, lam);
        return 2 * bplb_vb2_piece(w, c, lam);
    default: {  // K_BJ1, bounds.py:200-206
        const int64_t cm = c % lam, base = (w / lam) * (lam - cm), wm = w % lam;
        return wm <= cm ? base : base + wm - cm;
    }
    }
}

#if defined(__CUDACC__)
// 64-bit ceil-division kept out of line: it is rare (S >= 2^32) and large.
__device__ __noinline__ static uint64_t bplb_ceil_div64_slow(uint64_t s, uint64_t f) {
    return (s + f - 1) / f;
}
#endif

BPLB_HD int64_t bplb_bound(int64_t S, int64_t F) {
    if (F <= 0) return 0;
#if defined(__CUDA_ARCH__)
    if ((((uint64_t)S | (uint64_t)F) >> 32) == 0) {
        const uint32_t s = (uint32_t)S, f = (uint32_t)F;
        return (int64_t)(s / f + (s % f != 0));
    }
    return (int64_t)bplb_ceil_div64_slow((uint64_t)S, (uint64_t)F);
#else
    return (int64_t)bplb_ceil_div((uint64_t)S, (uint64_t)F);
#endif
}

// ---------------------------------------------------------------------------
// Lookup-based per-lambda sums (the reference's analytic sweeps,
// bounds.py:373-460).  L provides n_le(x) = #{w <= x} and w_le(x) = sum of
// those weights for any int64 x (clamped to [-1, c]).
// ---------------------------------------------------------------------------
template <class L>
BPLB_HD int64_t bplb_mt_sum(const L& lk, int64_t c, int64_t r, int64_t lam) {
    // _sweep_mt, bounds.py:373-376
    int64_t n1, w1, n0, w0;
    lk.both(c - lam, &n1, &w1);
    lk.both(lam - 1, &n0, &w0);
    return c * (r - n1) + w1 - w0;
}

template <class L>
BPLB_HD int64_t bplb_rad2_sum(const L& lk, int64_t c, int64_t r, int64_t lam) {
    // _sweep_rad2, bounds.py:379-387
    int64_t third = c / 3, half = c / 2;
    int64_t a = lk.n_le(lam - 1), b = lk.n_le(c - 2 * lam);
    int64_t d = lk.n_le(2 * lam - 1), e = lk.n_le(c - lam);
    return (b - a) * third + (d - b) * half + (e - d) * (c - third) + (r - e) * c;
}

// Harmonic parts, split over t so a warp can share one lambda (t0 = first t,
// dt = stride).  CCM1: returns sum over t in [1, hs/lam] of
//   (n_small - N(t*lam - 1)) - (N(c - t*lam) - (r - n_big))      (bounds.py:390-407)
template <class L>
BPLB_HD int64_t bplb_ccm1_part(const L& lk, const NodeStats& st, int64_t c, int64_t lam,
                               int64_t t0, int64_t dt) {
    const int64_t hs = (c - 1) / 2, tmax = hs / lam;
    const int64_t base = (int64_t)st.n_small + (int64_t)st.r - (int64_t)st.n_big;
    int64_t acc = 0;
#pragma unroll 4
    for (int64_t t = t0; t <= tmax; t += dt)
        acc += base - lk.n_le(t * lam - 1) - lk.n_le(c - t * lam);
    return acc;
}
BPLB_HD int64_t bplb_ccm1_from_part(const NodeStats& st, int64_t c, int64_t lam, int64_t part) {
    const int64_t cq = c / lam;
    return 2 * part + (int64_t)st.n_eq * cq + 2 * (int64_t)st.n_big * cq;
}
template <class L>
BPLB_HD int64_t bplb_ccm1_sum(const L& lk, const NodeStats& st, int64_t c, int64_t lam) {
    return bplb_ccm1_from_part(st, c, lam, bplb_ccm1_part(lk, st, c, lam, 1, 1));
}

// BJ1 (bounds.py:441-460): bucket t holds weights in [t*lam, (t+1)*lam - 1].
//   rem_sum   += W(hi_t) - W(lo_t) - lo_t (N(hi_t) - N(lo_t)),  lo_t = t*lam + cm
//   floor_sum += r - N(hi_t)  for t < tmax   (= r - N((t+1)*lam - 1))
template <class L>
BPLB_HD void bplb_bj1_part(const L& lk, const NodeStats& st, int64_t c, int64_t lam, int64_t t0,
                           int64_t dt, int64_t* floor_part, int64_t* rem_part) {
    const int64_t r = st.r, cm = c % lam, tmax = st.maxw / lam;
    int64_t fl = 0, rem = 0;
#pragma unroll 4
    for (int64_t t = t0; t <= tmax; t += dt) {
        const int64_t lo_v = lam * t + cm, hi_v = lam * (t + 1) - 1;
        int64_t nl, wl, nh, wh;
        lk.both(lo_v, &nl, &wl);
        lk.both(hi_v, &nh, &wh);
        rem += (wh - wl) - lo_v * (nh - nl);
        if (t < tmax) fl += r - nh;
    }
    *floor_part = fl;
    *rem_part = rem;
}
BPLB_HD int64_t bplb_bj1_from_parts(int64_t c, int64_t lam, int64_t fl, int64_t rem) {
    return (lam - c % lam) * fl + rem;
}
template <class L>
BPLB_HD int64_t bplb_bj1_sum(const L& lk, const NodeStats& st, int64_t c, int64_t lam) {
    int64_t fl, rem;
    bplb_bj1_part(lk, st, c, lam, 0, 1, &fl, &rem);
    return bplb_bj1_from_parts(c, lam, fl, rem);
}
