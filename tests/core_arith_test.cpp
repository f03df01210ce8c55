// Host-side check of the integer core shared with the CUDA kernels
// (paper_2402_14821_b200/csrc/bplb_core.h).  Compiled and run by
// tests/test_core_arith.py on CPU (no GPU needed).
//
// It checks, against brute-force scalar transforms (bounds.py:155-206):
//   - the magic-number division and the Barrett mulmod,
//   - every per-lambda closed form the kernels use: the lookup sweeps
//     (sorted-array and table lookups), the VB2 / FS1 modular walks
//     (emulated step by step exactly as the warp does), the CCM1/BJ1 dense
//     division sums, and the split (warp-cooperative) harmonic parts.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include "../paper_2402_14821_b200/csrc/bplb_core.h"

typedef __int128 i128;
static i128 fdiv(i128 a, i128 b) { i128 q = a / b; if ((a % b) && ((a < 0) != (b < 0))) --q; return q; }

static i128 f_value(int kind, i128 w, i128 c, i128 lam) {
    switch (kind) {
    case K_MT: return (c - lam < w) ? c : (w < lam ? 0 : w);
    case K_RAD2: {
        auto base = [&](i128 v) -> i128 { return v < lam ? 0 : (v <= c - 2 * lam ? fdiv(c, 3) : fdiv(c, 2)); };
        return w >= 2 * lam ? c - base(c - w) : base(w);
    }
    case K_FS1: { i128 num = w * (lam + 1); return (num % c == 0) ? w * lam : fdiv(num, c) * c; }
    case K_CCM1:
        if (2 * w > c) return 2 * (fdiv(c, lam) - fdiv(c - w, lam));
        if (2 * w == c) return fdiv(c, lam);
        return 2 * fdiv(w, lam);
    case K_VB2: {
        auto piece = [&](i128 v) -> i128 { i128 x = -fdiv(-(v * lam), c) - 1; return x > 0 ? x : 0; };
        if (2 * w > c) return 2 * piece(c) - 2 * piece(c - w);
        if (2 * w == c) return piece(c);
        return 2 * piece(w);
    }
    default: {
        i128 cm = c % lam, q = fdiv(w, lam), wm = w - q * lam, base = q * (lam - cm);
        return wm <= cm ? base : base + wm - cm;
    }
    }
}
static int64_t brute_S(int kind, const std::vector<int>& w, int64_t c, int64_t lam) {
    i128 s = 0;
    for (int x : w) s += f_value(kind, x, c, lam);
    return (int64_t)s;
}

struct LkSortedH {
    std::vector<int> sw;
    std::vector<long long> pre;
    int64_t n_le(int64_t x) const { return std::upper_bound(sw.begin(), sw.end(), x, [](int64_t a, int b) { return a < b; }) - sw.begin(); }
    void both(int64_t x, int64_t* n, int64_t* w) const { *n = n_le(x); *w = pre[*n]; }
};
struct LkTableH {
    std::vector<long long> cnt, wle;
    int64_t c;
    int64_t idx(int64_t x) const { return (x < -1 ? -1 : (x > c ? c : x)) + 1; }
    int64_t n_le(int64_t x) const { return cnt[idx(x)]; }
    void both(int64_t x, int64_t* n, int64_t* w) const { *n = cnt[idx(x)]; *w = wle[idx(x)]; }
};

static NodeStats stats_of(const std::vector<int>& w, int64_t c) {
    NodeStats st{};
    st.r = (int)w.size();
    for (int x : w) {
        st.maxw = std::max(st.maxw, x);
        st.W += x;
        if (2 * (int64_t)x < c) { st.n_small++; st.Vs += x; }
        else if (2 * (int64_t)x == c) st.n_eq++;
        else { st.n_big++; st.Vm += c - x; if (x == c) st.n_full++; }
    }
    bplb_stats_finish(&st, c);
    return st;
}

static int fails = 0;
#define CHECK(cond, ...) do { if (!(cond)) { if (fails < 20) { printf("FAIL %s:%d ", __FILE__, __LINE__); printf(__VA_ARGS__); printf("\n"); } ++fails; } } while (0)

int main(int argc, char** argv) {
    std::mt19937_64 rng(12345);
    // ---- Div31 ----
    for (uint32_t d = 1; d <= 3000; ++d) {
        Div31 dv = bplb_div31(d);
        for (uint32_t q = 0; q < 50; ++q) for (int e = -1; e <= 1; ++e) {
            int64_t n = (int64_t)q * d + e; if (n < 0) continue;
            CHECK(bplb_udiv31((uint32_t)n, dv) == (uint32_t)(n / d), "div31 n=%lld d=%u", (long long)n, d);
        }
        for (int t = 0; t < 200; ++t) {
            uint32_t n = (uint32_t)(rng() & 0x7FFFFFFF);
            CHECK(bplb_udiv31(n, dv) == n / d, "div31 n=%u d=%u", n, d);
        }
    }
    for (int t = 0; t < 2000000; ++t) {
        uint32_t d = (uint32_t)(rng() % 0x7FFFFFFF) + 1;
        if (t & 1) d = (uint32_t)(rng() % 4000000) + 1;
        uint32_t n = (uint32_t)(rng() & 0x7FFFFFFF);
        if (t % 3 == 0) n = (uint32_t)std::min<uint64_t>(0x7FFFFFFFull, (uint64_t)(n / d) * d - 1 + (rng() % 3));
        CHECK(bplb_udiv31(n, bplb_div31(d)) == n / d, "div31 big n=%u d=%u", n, d);
    }
    for (uint32_t d : {1u, 2u, 3u, 0x40000000u, 0x7FFFFFFFu, 0x7FFFFFFEu}) {
        for (uint32_t n : {0u, 1u, 0x7FFFFFFFu, 0x7FFFFFFEu, 0x40000000u}) {
            CHECK(bplb_udiv31(n, bplb_div31(d)) == n / d, "div31 edge n=%u d=%u", n, d);
        }
    }
    // ---- mulmod ----
    for (int t = 0; t < 2000000; ++t) {
        uint32_t c = (uint32_t)(rng() % ((1u << 30))) + 1;
        if (t & 1) c = (uint32_t)(rng() % 2000) + 1;
        uint32_t a = (uint32_t)(rng() % (1u << 31)), b = (uint32_t)(rng() % (1u << 31));
        uint32_t dl = (uint32_t)(rng() & 1);
        unsigned long long x = (unsigned long long)a * b;
        uint32_t want = (x == 0 && dl) ? c - 1 : (uint32_t)((x - dl) % c);
        CHECK(bplb_mulmod(a, b, dl, c, bplb_cinv(c)) == want, "mulmod a=%u b=%u c=%u", a, b, c);
    }
    // ---- per-lambda closed forms vs brute force ----
    int n_inst = argc > 1 ? atoi(argv[1]) : 3000;
    for (int it = 0; it < n_inst; ++it) {
        int64_t c;
        int r;
        int mode = it % 4;
        if (mode == 0) { c = 1 + rng() % 130; r = rng() % 14; }
        else if (mode == 1) { c = 1 + rng() % 2000; r = rng() % 60; }
        else if (mode == 2) { c = 1 + rng() % 200000; r = rng() % 40; }
        else { c = 2 * (1 + rng() % 500); r = rng() % 40; }  // even c: 2w == c items
        std::vector<int> w(r);
        for (auto& x : w) {
            x = (int)(1 + rng() % c);
            if (rng() % 8 == 0) x = (int)c;
            if (c % 2 == 0 && rng() % 8 == 0) x = (int)(c / 2);
        }
        NodeStats st = stats_of(w, c);
        LkSortedH ls;
        ls.sw = w;
        std::sort(ls.sw.begin(), ls.sw.end());
        ls.pre.assign(r + 1, 0);
        for (int i = 0; i < r; ++i) ls.pre[i + 1] = ls.pre[i] + ls.sw[i];
        LkTableH lt;
        lt.c = c;
        lt.cnt.assign(c + 2, 0);
        lt.wle.assign(c + 2, 0);
        for (int x : w) { lt.cnt[x + 1]++; lt.wle[x + 1] += x; }
        for (int64_t i = 1; i < c + 2; ++i) { lt.cnt[i] += lt.cnt[i - 1]; lt.wle[i] += lt.wle[i - 1]; }
        // VB2 items in kernel order (sorted smalls, then sorted big < c)
        std::vector<uint32_t> vb2;
        for (int x : ls.sw) if (2 * (int64_t)x != c && x < c) vb2.push_back((uint32_t)x);
        for (int kind = 0; kind < K_COUNT; ++kind) {
            int64_t lo, hi;
            bplb_domain(kind, c, &lo, &hi);
            if (kind == K_VB2) hi = bplb_vb2_hi(c, r, st.maxw);
            if (hi < lo) continue;
            // sample lambdas: all for small ranges, else random + ends
            std::vector<int64_t> lams;
            if (hi - lo < 400) for (int64_t l = lo; l <= hi; ++l) lams.push_back(l);
            else {
                for (int64_t l = lo; l < lo + 40; ++l) lams.push_back(l);
                for (int64_t l = hi - 40; l <= hi; ++l) lams.push_back(l);
                for (int s = 0; s < 100; ++s) lams.push_back(lo + (int64_t)(rng() % (hi - lo + 1)));
            }
            // modular walks: emulate from lam0 = lams[0] stepping by 1
            const uint32_t c32 = (uint32_t)c;
            const unsigned long long cinv = bplb_cinv(c32);
            for (int64_t lam : lams) {
                int64_t want = brute_S(kind, w, c, lam);
                int64_t got_s = 0, got_t = 0;
                switch (kind) {
                case K_MT: got_s = bplb_mt_sum(ls, c, r, lam); got_t = bplb_mt_sum(lt, c, r, lam); break;
                case K_RAD2: got_s = bplb_rad2_sum(ls, c, r, lam); got_t = bplb_rad2_sum(lt, c, r, lam); break;
                case K_CCM1: {
                    got_s = bplb_ccm1_sum(ls, st, c, lam);
                    int64_t part = 0;
                    for (int l = 0; l < 32; ++l) part += bplb_ccm1_part(lt, st, c, lam, 1 + l, 32);
                    got_t = bplb_ccm1_from_part(st, c, lam, part);
                    // dense division form
                    Div31 dv = bplb_div31((uint32_t)lam);
                    int64_t A = 0;
                    for (int x : ls.sw) {
                        if (2 * (int64_t)x < c) A += bplb_udiv31((uint32_t)x, dv);
                        else if (2 * (int64_t)x > c) A -= bplb_udiv31((uint32_t)(c - x), dv);
                    }
                    int64_t cq = c / lam;
                    int64_t dense = 2 * A + (int64_t)st.n_eq * cq + 2 * (int64_t)st.n_big * cq;
                    CHECK(dense == want, "ccm1 dense c=%lld lam=%lld", (long long)c, (long long)lam);
                    break;
                }
                case K_BJ1: {
                    got_s = bplb_bj1_sum(ls, st, c, lam);
                    int64_t fl = 0, rem = 0;
                    for (int l = 0; l < 32; ++l) { int64_t a, b; bplb_bj1_part(lt, st, c, lam, l, 32, &a, &b); fl += a; rem += b; }
                    got_t = bplb_bj1_from_parts(c, lam, fl, rem);
                    Div31 dv = bplb_div31((uint32_t)lam);
                    uint32_t cm = (uint32_t)(c % lam);
                    int64_t qs = 0, es = 0;
                    for (int x : w) {
                        uint32_t q = bplb_udiv31((uint32_t)x, dv), wm = (uint32_t)x - q * (uint32_t)lam;
                        qs += q;
                        es += wm > cm ? wm - cm : 0;
                    }
                    CHECK((lam - (int64_t)cm) * qs + es == want, "bj1 dense c=%lld lam=%lld", (long long)c, (long long)lam);
                    break;
                }
                case K_FS1: case K_VB2: {
                    // emulate the warp walk: init at lam - 3 (if in range) and step
                    int64_t l0 = std::max(lo, lam - 3);
                    std::vector<uint32_t> items = kind == K_VB2 ? vb2 : std::vector<uint32_t>(w.begin(), w.end());
                    std::vector<uint32_t> s(items.size());
                    for (size_t i = 0; i < items.size(); ++i) {
                        uint32_t x = items[i];
                        s[i] = kind == K_FS1 ? bplb_mulmod(x, (uint32_t)(l0 + 1), 0, c32, cinv)
                                             : bplb_mulmod(x, (uint32_t)l0, (2 * (uint64_t)x < (uint64_t)c) ? 1u : 0u, c32, cinv);
                    }
                    for (int64_t l = l0; l < lam; ++l)
                        for (size_t i = 0; i < items.size(); ++i) {
                            uint32_t a = s[i] + items[i], b = s[i] + items[i] - c32;
                            s[i] = std::min(a, b);
                        }
                    unsigned long long D = 0, Z = 0;
                    for (size_t i = 0; i < items.size(); ++i) { D += s[i]; if (s[i] == 0) Z += items[i]; }
                    if (kind == K_VB2) {
                        got_s = got_t = bplb_vb2_sum(st, c, lam, D);
                    } else {
                        // the kernels take Z from the lookup tables (multiples of c/gcd)
                        CHECK((unsigned long long)bplb_fs1_zero(ls, c, st.maxw, lam) == Z, "fs1 zero sorted");
                        CHECK((unsigned long long)bplb_fs1_zero(lt, c, st.maxw, lam) == Z, "fs1 zero table");
                        got_s = bplb_fs1_sum(st, lam, D, (uint64_t)bplb_fs1_zero(ls, c, st.maxw, lam));
                        got_t = bplb_fs1_sum(st, lam, D, (uint64_t)bplb_fs1_zero(lt, c, st.maxw, lam));
                    }
                    break;
                }
                }
                CHECK(got_s == want, "kind=%d sorted c=%lld r=%d lam=%lld got=%lld want=%lld", kind, (long long)c, r,
                      (long long)lam, (long long)got_s, (long long)want);
                CHECK(got_t == want, "kind=%d table c=%lld r=%d lam=%lld got=%lld want=%lld", kind, (long long)c, r,
                      (long long)lam, (long long)got_t, (long long)want);
                int64_t F = bplb_fc(kind, c, lam);
                CHECK(F == (int64_t)f_value(kind, c, c, lam), "fc kind=%d c=%lld lam=%lld", kind, (long long)c, (long long)lam);
            }
        }
    }
    // VB2 cap binding example (test_bounds.py:166-172 scaled into the envelope)
    CHECK(bplb_vb2_hi((int64_t)1 << 30, 1 << 24, (1 << 30) - 1) < ((int64_t)1 << 30), "vb2 cap should bind");
    printf(fails ? "FAILED %d checks\n" : "OK\n", fails);
    return fails ? 1 : 0;
}
