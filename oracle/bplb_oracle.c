/*
 * bplb_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's lower-bound engine
 * (/root/reference/pkg/src/binpack/bounds.py and parallel.py), used as the
 * CPU checker for the CUDA path and as the CPU baseline ("port") in bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path
 * (paper_2402_14821_b200/) never links or calls anything in this directory.
 *
 * Parity is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/binpack and
 * records dff_bound_batch / lower_bound_seq / lower_bound_par outputs).
 *
 * Every function cites the reference file:line it restates.  The structure
 * follows the reference deliberately (histogram "cumulatives" + analytic
 * sweeps for c <= 2^22, the dense _batch_matrix form otherwise and for FS1,
 * dense quotient sums for VB2) so that the CPU baseline measures the
 * reference's algorithm, not a GPU-style reformulation.
 *
 * Integer widths: all sums are int64 exactly as in the reference's numpy
 * path (bounds.py:463-501); scalar transforms use __int128 where the
 * reference relies on Python's unbounded ints (bounds.py:155-206).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef __int128 i128;

enum { OR_MT = 0, OR_RAD2 = 1, OR_FS1 = 2, OR_CCM1 = 3, OR_VB2 = 4, OR_BJ1 = 5 };

static int g_threads = 1;

void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int or_get_max_threads(void) { long n = sysconf(_SC_NPROCESSORS_ONLN); return n < 1 ? 1 : (int)n; }

/* Minimal dynamic parallel-for over [0, n) in chunks (pthreads; the image has
 * no OpenMP runtime).  fn(ctx, begin, end) processes one chunk. */
typedef void (*range_fn)(void *ctx, int64_t b, int64_t e);
typedef struct { range_fn fn; void *ctx; int64_t n, chunk; int64_t next; } pf_t;
static void *pf_worker(void *arg) {
    pf_t *p = (pf_t *)arg;
    for (;;) {
        int64_t b = __atomic_fetch_add(&p->next, p->chunk, __ATOMIC_RELAXED);
        if (b >= p->n) break;
        int64_t e = b + p->chunk < p->n ? b + p->chunk : p->n;
        p->fn(p->ctx, b, e);
    }
    return NULL;
}
static void par_for(int threads, int64_t n, int64_t chunk, range_fn fn, void *ctx) {
    if (n <= 0) return;
    if (threads <= 1 || n <= chunk) { fn(ctx, 0, n); return; }
    pf_t p = {fn, ctx, n, chunk, 0};
    int nt = threads;
    if ((int64_t)nt > (n + chunk - 1) / chunk) nt = (int)((n + chunk - 1) / chunk);
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nt);
    for (int i = 1; i < nt; i++) pthread_create(&tid[i], NULL, pf_worker, &p);
    pf_worker(&p);
    for (int i = 1; i < nt; i++) pthread_join(tid[i], NULL);
    free(tid);
}

static int64_t floordiv(int64_t a, int64_t b) { /* Python // for b > 0 */
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}
static i128 floordiv128(i128 a, i128 b) {
    i128 q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

/* ---- scalar transforms: bounds.py:155-206 ------------------------------ */
static i128 f_mt(i128 w, i128 c, i128 lam) { /* bounds.py:155-160 */
    if (c - lam < w) return c;
    if (w < lam) return 0;
    return w;
}
static i128 f_rad2(i128 w, i128 c, i128 lam) { /* bounds.py:163-170 */
    if (w >= 2 * lam) return c - f_rad2(c - w, c, lam);
    if (w < lam) return 0;
    if (w <= c - 2 * lam) return floordiv128(c, 3);
    return floordiv128(c, 2);
}
static i128 f_fs1(i128 w, i128 c, i128 lam) { /* bounds.py:173-178 */
    i128 num = w * (lam + 1);
    i128 q = floordiv128(num, c), rem = num - q * c;
    if (rem == 0) return w * lam;
    return q * c;
}
static i128 f_ccm1(i128 w, i128 c, i128 lam) { /* bounds.py:181-186 */
    if (2 * w > c) return 2 * (floordiv128(c, lam) - floordiv128(c - w, lam));
    if (2 * w == c) return floordiv128(c, lam);
    return 2 * floordiv128(w, lam);
}
static i128 vb2_piece(i128 v, i128 c, i128 lam) { /* bounds.py:190-191 */
    i128 x = -floordiv128(-(v * lam), c) - 1;
    return x > 0 ? x : 0;
}
static i128 f_vb2(i128 w, i128 c, i128 lam) { /* bounds.py:189-197 */
    if (2 * w > c) return 2 * vb2_piece(c, c, lam) - 2 * vb2_piece(c - w, c, lam);
    if (2 * w == c) return vb2_piece(c, c, lam);
    return 2 * vb2_piece(w, c, lam);
}
static i128 f_bj1(i128 w, i128 c, i128 lam) { /* bounds.py:200-206 */
    i128 cm = c - floordiv128(c, lam) * lam;
    i128 q = floordiv128(w, lam);
    i128 base = q * (lam - cm);
    i128 wm = w - q * lam;
    if (wm <= cm) return base;
    return base + wm - cm;
}
static i128 f_value(int kind, i128 w, i128 c, i128 lam) {
    switch (kind) {
    case OR_MT: return f_mt(w, c, lam);
    case OR_RAD2: return f_rad2(w, c, lam);
    case OR_FS1: return f_fs1(w, c, lam);
    case OR_CCM1: return f_ccm1(w, c, lam);
    case OR_VB2: return f_vb2(w, c, lam);
    default: return f_bj1(w, c, lam);
    }
}

/* dff_value without the domain assertion (bounds.py:242-250). */
int64_t or_dff_value(int kind, int64_t w, int64_t c, int64_t lam) {
    return (int64_t)f_value(kind, w, c, lam);
}

/* ---- lambda_range: bounds.py:219-273 ------------------------------------ */
void or_lambda_range(int kind, int64_t c, int64_t r, int64_t maxw, int has_red,
                     int64_t *lo, int64_t *hi) {
    switch (kind) {
    case OR_MT: *lo = 0; *hi = (c == 1) ? 0 : (c + 1) / 2; return; /* _mt_hi :219-225 */
    case OR_RAD2: *lo = c / 4 + 1; *hi = c / 3; return;
    case OR_FS1: *lo = 1; *hi = 100; return;
    case OR_CCM1: *lo = 1; *hi = c / 2; return;
    case OR_VB2: {                                                  /* :268-272 */
        *lo = 2; *hi = c;
        if (has_red && r > 0) {
            unsigned __int128 prod = (unsigned __int128)r * (unsigned __int128)maxw;
            unsigned __int128 cap = ((unsigned __int128)UINT64_MAX) / prod;
            if (cap < (unsigned __int128)*hi) *hi = (int64_t)cap;
        }
        return;
    }
    default: *lo = 1; *hi = c; return;
    }
}

/* ---- dff_bound (scalar, exact): bounds.py:276-290 ----------------------- */
int64_t or_dff_bound(int kind, const int64_t *w, int64_t r, int64_t c, int64_t lam) {
    i128 fc = f_value(kind, c, c, lam);
    if (fc <= 0) return 0;
    i128 total = 0;
    for (int64_t i = 0; i < r; i++) total += f_value(kind, w[i], c, lam);
    return (int64_t)(-floordiv128(-total, fc));
}

/* ---- _batch_matrix column sums: bounds.py:293-323 (dense r x L form) ----- */
typedef struct { int kind; const int64_t *w; int64_t r, c, lo, maxw; int64_t *sums, *fc; const void *cu;
                 const int64_t *smalls, *mirrored; int64_t ns, nm, n_eq, n_big; int64_t *out; } sweep_ctx;
/* One cell of _batch_matrix in numpy int64 semantics (bounds.py:293-323);
 * every operand is non-negative, so C division equals numpy's floor division. */
static int64_t bm_value(int kind, int64_t w, int64_t c, int64_t lam) {
    switch (kind) {
    case OR_MT: return w > c - lam ? c : (w < lam ? 0 : w);
    case OR_RAD2: {
        int64_t third = c / 3, half = c / 2;
        int64_t v = w >= 2 * lam ? c - w : w;
        int64_t base = v < lam ? 0 : (v <= c - 2 * lam ? third : half);
        return w >= 2 * lam ? c - base : base;
    }
    case OR_FS1: {
        int64_t num = w * (lam + 1);
        return num % c == 0 ? w * lam : (num / c) * c;
    }
    case OR_CCM1: {
        int64_t cq = c / lam;
        if (2 * w > c) return 2 * (cq - (c - w) / lam);
        return 2 * w == c ? cq : 2 * (w / lam);
    }
    case OR_VB2: {
        int64_t pc = lam - 1 > 0 ? lam - 1 : 0;
        if (2 * w > c) {
            int64_t pv = ((c - w) * lam + c - 1) / c - 1;
            return 2 * pc - 2 * (pv > 0 ? pv : 0);
        }
        if (2 * w == c) return pc;
        int64_t pv = (w * lam + c - 1) / c - 1;
        return 2 * (pv > 0 ? pv : 0);
    }
    default: {
        int64_t cm = c % lam, base = (w / lam) * (lam - cm), wm = w % lam;
        return wm <= cm ? base : base + wm - cm;
    }
    }
}

static void bm_range(void *p, int64_t b, int64_t e) {
    sweep_ctx *x = (sweep_ctx *)p;
    for (int64_t j = b; j < e; j++) {
        int64_t lam = x->lo + j;
        int64_t s = 0;
        for (int64_t i = 0; i < x->r; i++) s += bm_value(x->kind, x->w[i], x->c, lam);
        x->sums[j] = s;
        x->fc[j] = bm_value(x->kind, x->c, x->c, lam);
    }
}
static void batch_matrix_sums(int kind, const int64_t *w, int64_t r, int64_t c,
                              int64_t lo, int64_t L, int64_t *sums, int64_t *fc) {
    sweep_ctx x = {kind, w, r, c, lo, 0, sums, fc, NULL, NULL, NULL, 0, 0, 0, 0, NULL};
    par_for(g_threads, L, 16, bm_range, &x);
}

/* ---- _Cumulatives: bounds.py:331-348 ------------------------------------- */
typedef struct {
    int64_t c, r;
    int64_t *count; /* count[x+1] = #{w <= x}, x in [-1, c] */
    int64_t *wsum;  /* wsum[x+1]  = sum{w : w <= x} */
} cum_t;

static void cum_init(cum_t *cu, const int64_t *w, int64_t r, int64_t c) {
    cu->c = c; cu->r = r;
    cu->count = (int64_t *)calloc((size_t)(c + 2), sizeof(int64_t));
    cu->wsum = (int64_t *)calloc((size_t)(c + 2), sizeof(int64_t));
    for (int64_t i = 0; i < r; i++) { cu->count[w[i] + 1] += 1; cu->wsum[w[i] + 1] += w[i]; }
    for (int64_t x = 1; x < c + 2; x++) { cu->count[x] += cu->count[x - 1]; cu->wsum[x] += cu->wsum[x - 1]; }
}
static void cum_free(cum_t *cu) { free(cu->count); free(cu->wsum); }
static int64_t clampv(int64_t v, int64_t c) { return v < -1 ? -1 : (v > c ? c : v); }
static int64_t n_le(const cum_t *cu, int64_t v) { return cu->count[clampv(v, cu->c) + 1]; } /* :344-345 */
static int64_t w_le(const cum_t *cu, int64_t v) { return cu->wsum[clampv(v, cu->c) + 1]; }  /* :347-348 */

/* _floor_div_sums: bounds.py:361-370  (sum over w <= hi_value of floor(w/lam)) */
static int64_t floor_div_sum(const cum_t *cu, int64_t lam, int64_t hi_value, int64_t n_le_hi) {
    int64_t tmax = hi_value / lam, s = 0;
    for (int64_t t = 1; t <= tmax; t++) s += n_le_hi - n_le(cu, lam * t - 1);
    return s;
}

/* _sweep_mt: bounds.py:373-376 */
static void sweep_mt(const cum_t *cu, int64_t lam, int64_t *s, int64_t *f) {
    int64_t c = cu->c;
    *s = c * (cu->r - n_le(cu, c - lam)) + w_le(cu, c - lam) - w_le(cu, lam - 1);
    *f = c;
}
/* _sweep_rad2: bounds.py:379-387 */
static void sweep_rad2(const cum_t *cu, int64_t lam, int64_t *s, int64_t *f) {
    int64_t c = cu->c, third = c / 3, half = c / 2;
    int64_t n2 = n_le(cu, c - 2 * lam) - n_le(cu, lam - 1);
    int64_t n3 = n_le(cu, 2 * lam - 1) - n_le(cu, c - 2 * lam);
    int64_t n4 = n_le(cu, c - lam) - n_le(cu, 2 * lam - 1);
    int64_t n5 = cu->r - n_le(cu, c - lam);
    *s = n2 * third + n3 * half + n4 * (c - third) + n5 * c;
    *f = c;
}
/* _sweep_ccm1: bounds.py:390-407 */
static void sweep_ccm1(const cum_t *cu, int64_t lam, int64_t *s, int64_t *f) {
    int64_t c = cu->c, below_half = (c - 1) / 2;
    int64_t n_small = n_le(cu, below_half);
    int64_t n_eq = n_le(cu, c / 2) - n_small;
    int64_t n_big = cu->r - n_le(cu, c / 2);
    int64_t cq = c / lam;
    int64_t t_small = floor_div_sum(cu, lam, below_half, n_small);
    int64_t tmax = below_half / lam, t_big = 0;
    for (int64_t t = 1; t <= tmax; t++) t_big += n_le(cu, c - lam * t) - (cu->r - n_big);
    *s = 2 * t_small + n_eq * cq + 2 * n_big * cq - 2 * t_big;
    *f = 2 * cq;
}
/* _sweep_bj1: bounds.py:441-460 */
static void sweep_bj1(const cum_t *cu, int64_t lam, int64_t max_weight, int64_t *s, int64_t *f) {
    int64_t c = cu->c, cm = c % lam, cq = c / lam;
    int64_t floor_sum = floor_div_sum(cu, lam, max_weight, cu->r);
    int64_t tmax = max_weight / lam + 1, rem_sum = 0;
    for (int64_t t = 0; t < tmax; t++) {
        int64_t lo_v = lam * t + cm, hi_v = lam * (t + 1) - 1;
        int64_t nin = n_le(cu, hi_v) - n_le(cu, lo_v);
        int64_t win = w_le(cu, hi_v) - w_le(cu, lo_v);
        rem_sum += win - lo_v * nin;
    }
    *s = (lam - cm) * floor_sum + rem_sum;
    *f = cq * (lam - cm);
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static void vb2_range(void *p, int64_t b, int64_t e) {
    sweep_ctx *x = (sweep_ctx *)p;
    for (int64_t j = b; j < e; j++) {
        int64_t lam = x->lo + j, qs = 0, qm = 0;
        /* quotient_sum: ((col * row - 1) // c).sum()  (bounds.py:419-429) */
        for (int64_t i = 0; i < x->ns; i++) qs += floordiv(x->smalls[i] * lam - 1, x->c);
        for (int64_t i = 0; i < x->nm; i++) qm += floordiv(x->mirrored[i] * lam - 1, x->c);
        x->sums[j] = 2 * qs + (x->n_eq + 2 * x->n_big) * (lam - 1) - 2 * qm;
        x->fc[j] = 2 * (lam - 1);
    }
}

/* _sweep_vb2: bounds.py:410-438 (dense quotient sums over smalls / mirrored) */
static void sweep_vb2(const int64_t *w, int64_t r, int64_t c, int64_t lo, int64_t L,
                      int64_t *sums, int64_t *fc) {
    int64_t *smalls = (int64_t *)malloc(sizeof(int64_t) * (size_t)(r + 1));
    int64_t *mirrored = (int64_t *)malloc(sizeof(int64_t) * (size_t)(r + 1));
    int64_t ns = 0, nm = 0, n_eq = 0, n_big = 0;
    for (int64_t i = 0; i < r; i++) {
        if (2 * w[i] < c) smalls[ns++] = w[i];
        if (2 * w[i] > c && w[i] < c) mirrored[nm++] = c - w[i];
        if (2 * w[i] == c) n_eq++;
        if (2 * w[i] > c) n_big++;
    }
    qsort(smalls, (size_t)ns, sizeof(int64_t), cmp_i64);
    qsort(mirrored, (size_t)nm, sizeof(int64_t), cmp_i64);
    sweep_ctx x = {OR_VB2, w, r, c, lo, 0, sums, fc, NULL, smalls, mirrored, ns, nm, n_eq, n_big, NULL};
    par_for(g_threads, L, 16, vb2_range, &x);
    free(smalls); free(mirrored);
}

#define OR_VEC_MAX_C (1LL << 31)      /* bounds.py:44 */
#define OR_VEC_MAX_R (1LL << 20)      /* bounds.py:45 */
#define OR_ANALYTIC_MAX_C (1LL << 22) /* bounds.py:328 */

static void scalar_range(void *p, int64_t b, int64_t e) {
    sweep_ctx *x = (sweep_ctx *)p;
    for (int64_t j = b; j < e; j++) x->out[j] = or_dff_bound(x->kind, x->w, x->r, x->c, x->lo + j);
}
static void analytic_range(void *p, int64_t b, int64_t e) {
    sweep_ctx *x = (sweep_ctx *)p;
    const cum_t *cu = (const cum_t *)x->cu;
    for (int64_t j = b; j < e; j++) {
        int64_t lam = x->lo + j;
        if (x->kind == OR_MT) sweep_mt(cu, lam, &x->sums[j], &x->fc[j]);
        else if (x->kind == OR_RAD2) sweep_rad2(cu, lam, &x->sums[j], &x->fc[j]);
        else if (x->kind == OR_CCM1) sweep_ccm1(cu, lam, &x->sums[j], &x->fc[j]);
        else sweep_bj1(cu, lam, x->maxw, &x->sums[j], &x->fc[j]);
    }
}

/* dff_bound_batch: bounds.py:463-501.  out has hi-lo+1 entries. */
void or_dff_bound_batch(int kind, const int64_t *w, int64_t r, int64_t c,
                        int64_t lo, int64_t hi, int64_t *out) {
    if (hi < lo) return;
    int64_t L = hi - lo + 1;
    if (c > OR_VEC_MAX_C || r > OR_VEC_MAX_R) { /* :473-476 scalar fallback */
        sweep_ctx x = {kind, w, r, c, lo, 0, NULL, NULL, NULL, NULL, NULL, 0, 0, 0, 0, out};
        par_for(g_threads, L, 16, scalar_range, &x);
        return;
    }
    if (r == 0) { memset(out, 0, sizeof(int64_t) * (size_t)L); return; } /* :478-479 */
    int64_t *sums = (int64_t *)malloc(sizeof(int64_t) * (size_t)L);
    int64_t *fc = (int64_t *)malloc(sizeof(int64_t) * (size_t)L);
    int done = 0;
    if (c <= OR_ANALYTIC_MAX_C && kind != OR_FS1) {
        if (kind == OR_VB2) {
            sweep_vb2(w, r, c, lo, L, sums, fc);
        } else {
            cum_t cu;
            cum_init(&cu, w, r, c);
            int64_t maxw = 0;
            for (int64_t i = 0; i < r; i++) if (w[i] > maxw) maxw = w[i];
            sweep_ctx x = {kind, w, r, c, lo, maxw, sums, fc, &cu, NULL, NULL, 0, 0, 0, 0, NULL};
            par_for(g_threads, L, 64, analytic_range, &x);
            cum_free(&cu);
        }
        done = 1;
    }
    if (!done) batch_matrix_sums(kind, w, r, c, lo, L, sums, fc); /* :495-499 */
    for (int64_t j = 0; j < L; j++) {                            /* :500-501 */
        int64_t safe = fc[j] > 1 ? fc[j] : 1;
        out[j] = fc[j] > 0 ? floordiv(sums[j] + safe - 1, safe) : 0;
    }
    free(sums); free(fc);
}

/* Best value (and lowest arg lambda) of one kind's full range; helper for
 * lower_bound_seq.  Returns 0 for an empty range (bounds.py:514-520). */
static int64_t kind_best(int kind, const int64_t *w, int64_t r, int64_t c, int64_t maxw,
                         int64_t *nlam, int64_t *arg) {
    int64_t lo, hi;
    or_lambda_range(kind, c, r, maxw, 1, &lo, &hi);
    *nlam = hi >= lo ? hi - lo + 1 : 0;
    *arg = lo;
    if (hi < lo) return 0;
    int64_t *vals = (int64_t *)malloc(sizeof(int64_t) * (size_t)(*nlam));
    or_dff_bound_batch(kind, w, r, c, lo, hi, vals);
    int64_t best = vals[0];
    *arg = lo;
    for (int64_t j = 1; j < *nlam; j++) if (vals[j] > best) { best = vals[j]; *arg = lo + j; }
    free(vals);
    return best;
}

/*
 * lower_bound_seq: bounds.py:504-527.  kinds[0..nkinds) in evaluation order.
 * Outputs: per_dff[i] for the i-th processed kind (*n_done of them), lb,
 * exceeded, evals.  arg_out (optional) receives the lowest arg-max lambda.
 */
void or_lower_bound_seq(const int64_t *w, int64_t r, int64_t c, int64_t k,
                        const int32_t *kinds, int32_t nkinds,
                        int64_t *per_dff, int64_t *arg_out, int32_t *n_done,
                        int64_t *lb, int32_t *exceeded, int64_t *evals) {
    int64_t maxw = 0;
    for (int64_t i = 0; i < r; i++) if (w[i] > maxw) maxw = w[i];
    *lb = 0; *evals = 0; *exceeded = 0; *n_done = 0;
    for (int32_t i = 0; i < nkinds; i++) {
        int64_t nlam, arg;
        int64_t best = kind_best(kinds[i], w, r, c, maxw, &nlam, &arg);
        *evals += nlam;
        per_dff[i] = best;
        if (arg_out) arg_out[i] = arg;
        *n_done = i + 1;
        if (best > *lb) *lb = best;
        if (*lb > k) { *exceeded = 1; return; }
    }
    *exceeded = *lb > k;
}

/*
 * Batched CPU baseline: lower_bound_seq over every node of a CSR batch
 * (one node per OpenMP task; numpy inside each node is single-threaded in
 * the reference, so nodes are the natural unit of host parallelism).
 */
typedef struct { const int64_t *w, *offsets; int64_t c, k; const int32_t *kinds; int32_t nkinds;
                 int64_t *lb_out; uint8_t *exceeded_out; int64_t *best_out; } batch_ctx;
static void batch_range(void *p, int64_t b, int64_t e) {
    batch_ctx *x = (batch_ctx *)p;
    for (int64_t n = b; n < e; n++) {
        int64_t per[6] = {0, 0, 0, 0, 0, 0};
        int32_t nd, ex;
        int64_t lb, ev;
        or_lower_bound_seq(x->w + x->offsets[n], x->offsets[n + 1] - x->offsets[n], x->c, x->k,
                           x->kinds, x->nkinds, per, NULL, &nd, &lb, &ex, &ev);
        x->lb_out[n] = lb;
        x->exceeded_out[n] = (uint8_t)ex;
        if (x->best_out)
            for (int i = 0; i < x->nkinds; i++) x->best_out[n * x->nkinds + i] = i < nd ? per[i] : -1;
    }
}
void or_check_batch(const int64_t *w, const int64_t *offsets, int64_t n_nodes, int64_t c,
                    int64_t k, const int32_t *kinds, int32_t nkinds,
                    int64_t *lb_out, uint8_t *exceeded_out, int64_t *best_out /* n*nkinds or NULL */) {
    int saved = g_threads;
    g_threads = 1; /* per-node work is serial; parallelise over nodes (g_threads is
                      only read by the per-node sweeps, which now run single-threaded) */
    batch_ctx x = {w, offsets, c, k, kinds, nkinds, lb_out, exceeded_out, best_out};
    par_for(saved, n_nodes, 1, batch_range, &x);
    g_threads = saved;
}

/* ---- knapsack reasoning per bin ---------------------------
 * Restates /root/reference/pkg/src/binpack/propagator.py:98-224 with the
 * reference's own structure: a bitset over loads 0..c (Python int there,
 * uint64 words here), _add_weights (:98-102: bits |= bits << w, cut at c),
 * reachable_sums (:105-110), _window (:123-126), _use_avoid (:144-149),
 * _exclusion_sums (:170-187, the same divide and conquer) and _knapsack_bin
 * (:190-224).  Output conventions as bplb_knapsack_bins (include/bplb.h):
 * returns 0 ok / 1 Wipeout "no reachable load"; action per open item 0 keep,
 * 1 remove, 2 commit, 3 Wipeout; flags 0x100 reach only, 0x200 filter on the
 * input interval without the committed-load skip (knapsack_item_filter). */
typedef struct { int64_t nw; int64_t c; } kb_t;

static void kb_add(const kb_t *k, uint64_t *bits, int64_t w) { /* :98-102, one weight */
    const int64_t ws = w >> 6, bs = w & 63;
    for (int64_t i = k->nw - 1; i >= ws; --i) {
        uint64_t v = bits[i - ws] << bs;
        if (bs && i - ws - 1 >= 0) v |= bits[i - ws - 1] >> (64 - bs);
        bits[i] |= v;
    }
    const int64_t top = (k->c + 1) & 63;
    if (top) bits[k->nw - 1] &= ((uint64_t)1 << top) - 1;
}

static int kb_any(const kb_t *k, const uint64_t *bits, int64_t lo, int64_t hi) { /* bits & _window(lo, hi) */
    if (hi < lo) return 0;
    if (lo < 0) lo = 0;
    if (hi > k->c) hi = k->c;
    for (int64_t v = lo; v <= hi; ) {
        const int64_t i = v >> 6, b = v & 63;
        uint64_t word = bits[i] >> b;
        const int64_t span = hi - v + 1;
        if (span < 64 - b) word &= ((uint64_t)1 << span) - 1;
        if (word) return 1;
        v += 64 - b;
    }
    return 0;
}

static void kb_excl(const kb_t *k, const int32_t *w, int64_t lo, int64_t hi, const uint64_t *excl,
                    uint64_t **out, int depth, uint64_t *scratch_base) { /* rec, :177-183 */
    if (hi - lo == 1) { memcpy(out[lo], excl, (size_t)k->nw * 8); return; }
    const int64_t mid = (lo + hi) / 2;
    uint64_t *t = scratch_base + (size_t)depth * k->nw;
    memcpy(t, excl, (size_t)k->nw * 8);
    for (int64_t i = mid; i < hi; ++i) kb_add(k, t, w[i]);
    kb_excl(k, w, lo, mid, t, out, depth + 1, scratch_base);
    memcpy(t, excl, (size_t)k->nw * 8);
    for (int64_t i = lo; i < mid; ++i) kb_add(k, t, w[i]);
    kb_excl(k, w, mid, hi, t, out, depth + 1, scratch_base);
}

int or_knapsack_bin(int64_t c, int64_t committed, int64_t lo, int64_t hi, const int32_t *w, int64_t m,
                    int32_t flags, int32_t *lo_out, int32_t *hi_out, uint8_t *action, uint64_t *reach_out) {
    kb_t k = {(c + 64) / 64, c};
    uint64_t *reach = (uint64_t *)calloc((size_t)k.nw, 8);
    if (committed <= c) reach[committed >> 6] = (uint64_t)1 << (committed & 63); /* base, :109 */
    uint64_t *base = (uint64_t *)malloc((size_t)k.nw * 8);
    memcpy(base, reach, (size_t)k.nw * 8);
    for (int64_t i = 0; i < m; ++i) kb_add(&k, reach, w[i]);               /* :110 / :202 */
    if (reach_out) memcpy(reach_out, reach, (size_t)k.nw * 8);
    int64_t first = -1, last = -1;                                           /* :203-209 */
    for (int64_t v = lo; v <= hi; ++v)
        if (reach[v >> 6] >> (v & 63) & 1) { if (first < 0) first = v; last = v; }
    free(reach);
    if (first < 0) {
        *lo_out = (int32_t)lo; *hi_out = (int32_t)hi;
        if (action && !(flags & 0x100)) for (int64_t i = 0; i < m; ++i) action[i] = 0;
        free(base);
        return 1;
    }
    *lo_out = (int32_t)first; *hi_out = (int32_t)last;
    if (!(flags & 0x200)) { lo = first; hi = last; }
    if ((flags & 0x100)) { free(base); return 0; }
    if ((!(flags & 0x200) && lo <= committed) || m == 0) {                  /* :213-218 */
        for (int64_t i = 0; i < m; ++i) action[i] = 0;
        free(base);
        return 0;
    }
    int depth = 1;
    for (int64_t t = m; t > 1; t = (t + 1) / 2) ++depth;
    uint64_t *excl_mem = (uint64_t *)malloc((size_t)m * k.nw * 8);
    uint64_t **excl = (uint64_t **)malloc((size_t)m * sizeof(uint64_t *));
    uint64_t *scratch = (uint64_t *)malloc((size_t)(depth + 1) * k.nw * 8);
    for (int64_t i = 0; i < m; ++i) excl[i] = excl_mem + (size_t)i * k.nw;
    kb_excl(&k, w, 0, m, base, excl, 0, scratch);                           /* :219 */
    for (int64_t i = 0; i < m; ++i) {                                        /* :220-224 / :144-149 */
        const int64_t wt = w[i];
        const int use = hi >= wt ? kb_any(&k, excl[i], lo - wt < 0 ? 0 : lo - wt, hi - wt) : 0;
        const int avoid = kb_any(&k, excl[i], lo, hi);
        action[i] = (uint8_t)(use ? (avoid ? 0 : 2) : (avoid ? 1 : 3));
    }
    free(scratch); free(excl); free(excl_mem); free(base);
    return 0;
}

typedef struct {
    int64_t c; const int64_t *cl, *lo, *hi, *off; const int32_t *w; int32_t flags;
    int32_t *st, *lo_out, *hi_out; uint8_t *act;
} kbb_t;
static void kbb_range(void *p, int64_t b, int64_t e) {
    kbb_t *q = (kbb_t *)p;
    for (int64_t i = b; i < e; ++i)
        q->st[i] = or_knapsack_bin(q->c, q->cl[i], q->lo[i], q->hi[i], q->w + q->off[i], q->off[i + 1] - q->off[i],
                                   q->flags, q->lo_out + i, q->hi_out + i, q->act ? q->act + q->off[i] : NULL, NULL);
}
/* many independent bins (the batched form the GPU runs), g_threads threads */
void or_knapsack_bins(int64_t c, int64_t n, const int64_t *cl, const int64_t *lo, const int64_t *hi,
                      const int32_t *w, const int64_t *off, int32_t flags, int32_t *st, int32_t *lo_out,
                      int32_t *hi_out, uint8_t *act) {
    kbb_t q = {c, cl, lo, hi, off, w, flags, st, lo_out, hi_out, act};
    par_for(g_threads, n, 16, kbb_range, &q);
}
