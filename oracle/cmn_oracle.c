/*
 * cmn_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * synchronous data-parallel update step of ChainerMN (arXiv 1908.00213, §6).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1908_00213_b200/csrc); neither side includes or links the other.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off guarantees the only fused multiply-adds are the explicit
 * fmaf() calls written below.
 *
 * What it computes (readings listed in DESIGN.md §3):
 *   1. layout     off_0 = 0, off_{t+1} = align(off_t + n_t), L = off_T
 *                 (parameters are "collected easily by traversing" the model,
 *                  PAPER.md:184 §3.2; packing order = registration order)
 *   2. pack       b_i[off_t + k] = cast(g_{i,t}[k]); pads = 0
 *                 cast = identity (fp32) or IEEE fp32->fp16 round-to-nearest-even
 *                 ("half-precision floats for communication", App. A.1)
 *   3. all-reduce r[j] = tree(b_0[j], ..., b_{N-1}[j]), fp32 additions
 *                 ("obtain and distribute the sum of gradients", §6.1.2)
 *   4. fp16 only  r[j] <- fp16_RNE(r[j]) (payload stays half precision)
 *   5. average    a = r / N, one IEEE fp32 division (correctly rounded)
 *                 ("calculates the average of gradients by dividing the sum by the
 *                  number of replicas", §6.1.2; reading R3)
 *   6. update     v' = fmaf(mu, v, a); w' = fmaf(-lr, v', w)   (momentum SGD,
 *                 the optimizer multi_node_optimizer wraps, §6.3;
 *                 form v = mu v + g, w -= lr v from SPEC.md:462)
 *   7. exact      abar[j] = (sum_i g_i[j]) / N in fp64, m[j] = (1/N) sum_i |g_i[j]|
 *                 (the tolerance gate's reference, no rounding order involved)
 *
 * Every function is elementwise and single-threaded.  No blocking, fusion or
 * reordering beyond the definition above.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_FP32 0
#define ORC_FP16 1

/* ------------------------------------------------------------------ bits */

static uint32_t f32_bits(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static float bits_f32(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

/* IEEE-754 binary32 -> binary16, round to nearest, ties to even.
 * Reading c.2 #4: no flush-to-zero, |x| >= 65520 -> +-inf,
 * NaN -> quiet NaN of the same sign. */
uint16_t orc_f32_to_f16(float x)
{
    uint32_t u = f32_bits(x);
    uint32_t sign = (u >> 16) & 0x8000u;
    uint32_t a = u & 0x7fffffffu;

    if (a > 0x7f800000u)                 /* NaN */
        return (uint16_t)(sign | 0x7e00u);
    if (a >= 0x477ff000u)                /* >= 65520 (incl. inf): overflow to inf */
        return (uint16_t)(sign | 0x7c00u);
    if (a >= 0x38800000u) {              /* >= 2^-14: normal half */
        uint32_t e = (a >> 23) - 112u;   /* rebias 127 -> 15 */
        uint32_t mant = a & 0x7fffffu;
        uint32_t h = (e << 10) | (mant >> 13);
        uint32_t rem = mant & 0x1fffu;
        if (rem > 0x1000u || (rem == 0x1000u && (h & 1u)))
            h += 1u;                     /* a carry into the exponent is correct */
        return (uint16_t)(sign | h);
    }
    if (a <= 0x33000000u)                /* <= 2^-25: rounds to (signed) zero */
        return (uint16_t)sign;
    {                                    /* half subnormal: units of 2^-24 */
        uint32_t e = a >> 23;            /* 102 .. 112 */
        uint32_t mant = (a & 0x7fffffu) | 0x800000u;
        uint32_t s = 126u - e;           /* value = mant * 2^(e-150) = (mant >> s) * 2^-24 */
        uint32_t q = mant >> s;
        uint32_t rem = mant & ((1u << s) - 1u);
        uint32_t half = 1u << (s - 1u);
        if (rem > half || (rem == half && (q & 1u)))
            q += 1u;
        return (uint16_t)(sign | q);
    }
}

/* binary16 -> binary32 (exact). */
float orc_f16_to_f32(uint16_t h)
{
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t e = ((uint32_t)h >> 10) & 0x1fu;
    uint32_t m = (uint32_t)h & 0x3ffu;
    if (e == 0x1fu)                                  /* inf / NaN */
        return bits_f32(sign | 0x7f800000u | (m << 13));
    if (e == 0) {                                    /* zero / subnormal: m * 2^-24 */
        float v = (float)m * 0x1p-24f;               /* exact: m < 2^10 */
        return sign ? -v : v;
    }
    return bits_f32(sign | ((e + 112u) << 23) | (m << 13));
}

/* ---------------------------------------------------------------- layout */

/* Step 1.  off has T+1 entries; returns L = off[T] (or -1 on bad input). */
int64_t orc_layout(int T, const int64_t *n, int64_t align, int64_t *off)
{
    if (T < 0 || align <= 0) return -1;
    off[0] = 0;
    for (int t = 0; t < T; ++t) {
        if (n[t] < 0) return -1;
        int64_t end = off[t] + n[t];
        off[t + 1] = (end + align - 1) / align * align;
    }
    return off[T];
}

/* ------------------------------------------------------------------ pack */

/* Step 2.  b has L elements of the comm dtype (float or uint16 fp16 bits). */
void orc_pack(int T, const int64_t *n, const int64_t *off, int64_t L,
              const float *const *g, int dtype, void *b)
{
    if (dtype == ORC_FP32) {
        float *bf = (float *)b;
        for (int64_t j = 0; j < L; ++j) bf[j] = 0.0f;
        for (int t = 0; t < T; ++t)
            for (int64_t k = 0; k < n[t]; ++k)
                bf[off[t] + k] = g[t][k];
    } else {
        uint16_t *bh = (uint16_t *)b;
        for (int64_t j = 0; j < L; ++j) bh[j] = 0;
        for (int t = 0; t < T; ++t)
            for (int64_t k = 0; k < n[t]; ++k)
                bh[off[t] + k] = orc_f32_to_f16(g[t][k]);
    }
}

/* Inverse mapping (tests: unpack(pack(x)) == x). */
void orc_unpack_f32(int T, const int64_t *n, const int64_t *off,
                    const float *b, float *const *out)
{
    for (int t = 0; t < T; ++t)
        for (int64_t k = 0; k < n[t]; ++k)
            out[t][k] = b[off[t] + k];
}

/* ---------------------------------------------------------------- reduce */

/* Pairwise tree over x[lo..hi] (inclusive); the low half holds ceil(n/2)
 * elements.  For N = 8: ((x0+x1)+(x2+x3))+((x4+x5)+(x6+x7)).
 * Reading c.2 #2: the paper delegates the order to NCCL/MPI
 * (PAPER.md:480-486); a fixed order is required for bitwise-identical
 * replicas ("deterministic behaviour"). */
float orc_tree_sum(const float *x, int lo, int hi)
{
    if (lo == hi) return x[lo];
    int n = hi - lo + 1;
    int m = lo + (n + 1) / 2 - 1;        /* last index of the low half */
    float a = orc_tree_sum(x, lo, m);
    float c = orc_tree_sum(x, m + 1, hi);
    return a + c;
}

/* Steps 3-4.  b[i] is worker i's packed buffer (comm dtype); r (comm dtype)
 * receives the reduced buffer that every worker ends up holding. */
int orc_reduce_tree(int N, int64_t L, const void *const *b, int dtype, void *r)
{
    float *x = (float *)malloc(sizeof(float) * (size_t)(N > 0 ? N : 1));
    if (!x || N < 1) { free(x); return -1; }
    for (int64_t j = 0; j < L; ++j) {
        for (int i = 0; i < N; ++i)
            x[i] = dtype == ORC_FP32 ? ((const float *)b[i])[j]
                                     : orc_f16_to_f32(((const uint16_t *)b[i])[j]);
        float s = orc_tree_sum(x, 0, N - 1);
        if (dtype == ORC_FP32) ((float *)r)[j] = s;
        else ((uint16_t *)r)[j] = orc_f32_to_f16(s);
    }
    free(x);
    return 0;
}

/* ---------------------------------------------------------------- update */

/* Steps 5-6.  r is the reduced buffer (comm dtype), w/v per tensor (fp32,
 * in place).  a_out (optional, may be NULL or hold NULL entries) receives
 * the averaged gradient a. */
void orc_update_momentum_sgd(int T, const int64_t *n, const int64_t *off,
                             const void *r, int dtype, int N, float lr, float mu,
                             float *const *w, float *const *v, float *const *a_out)
{
    float n_rep = (float)N;              /* "dividing the sum by the number of replicas" */
    for (int t = 0; t < T; ++t) {
        for (int64_t k = 0; k < n[t]; ++k) {
            int64_t j = off[t] + k;
            float rj = dtype == ORC_FP32 ? ((const float *)r)[j]
                                         : orc_f16_to_f32(((const uint16_t *)r)[j]);
            float a = rj / n_rep;
            float vn = fmaf(mu, v[t][k], a);
            float wn = fmaf(-lr, vn, w[t][k]);
            v[t][k] = vn;
            w[t][k] = wn;
            if (a_out && a_out[t]) a_out[t][k] = a;
        }
    }
}

/* Fused Adam update (NEXT-1; the optimizer the paper's own example wraps,
 * PAPER.md:529 Fig. 4).  Standard bias-corrected Adam (Kingma & Ba) with the
 * per-step constants computed in fp32 from the step count t >= 1:
 *   m' = beta1*m + (1-beta1)*a        v' = beta2*v + (1-beta2)*a*a
 *   w' = w - alpha_t * m' / (sqrt(v') + eps),
 *   alpha_t = alpha * sqrt(1-beta2^t) / (1-beta1^t)
 * Each line is evaluated as written: fp32 mult/add (no contraction), sqrtf,
 * one division. */
void orc_update_adam(int T, const int64_t *n, const int64_t *off,
                     const void *r, int dtype, int N, float alpha, float beta1,
                     float beta2, float eps, int step,
                     float *const *w, float *const *m, float *const *v)
{
    float n_rep = (float)N;
    double b1t = pow((double)beta1, (double)step);
    double b2t = pow((double)beta2, (double)step);
    float alpha_t = (float)((double)alpha * sqrt(1.0 - b2t) / (1.0 - b1t));
    float c1 = 1.0f - beta1, c2 = 1.0f - beta2;
    for (int t = 0; t < T; ++t) {
        for (int64_t k = 0; k < n[t]; ++k) {
            int64_t j = off[t] + k;
            float rj = dtype == ORC_FP32 ? ((const float *)r)[j]
                                         : orc_f16_to_f32(((const uint16_t *)r)[j]);
            float a = rj / n_rep;
            float mn = beta1 * m[t][k] + c1 * a;
            float vn = beta2 * v[t][k] + c2 * (a * a);
            float den = sqrtf(vn) + eps;
            float wn = w[t][k] - alpha_t * (mn / den);
            m[t][k] = mn;
            v[t][k] = vn;
            w[t][k] = wn;
        }
    }
}

/* ----------------------------------------------------------------- exact */

/* Step 7.  g32[i] is worker i's packed fp32 buffer (before any cast).
 * avg[j] = (sum_i g_i[j]) / N and mag[j] = (sum_i |g_i[j]|) / N in fp64. */
void orc_exact_avg(int N, int64_t L, const float *const *g32, double *avg, double *mag)
{
    for (int64_t j = 0; j < L; ++j) {
        double s = 0.0, sa = 0.0;
        for (int i = 0; i < N; ++i) {
            s += (double)g32[i][j];
            sa += fabs((double)g32[i][j]);
        }
        avg[j] = s / (double)N;
        if (mag) mag[j] = sa / (double)N;
    }
}

/* ------------------------------------------------------------ whole step */

/* One full synchronous data-parallel step (steps 2-6) for N simulated
 * workers.  g[i*T + t] is worker i's gradient of tensor t.  Scratch is
 * allocated here; returns 0 on success. */
int orc_step(int N, int T, const int64_t *n, const int64_t *off, int64_t L,
             const float *const *g, int dtype, float lr, float mu,
             float *const *w, float *const *v, float *const *a_out, void *r_out)
{
    size_t es = dtype == ORC_FP32 ? 4 : 2;
    void **b = (void **)calloc((size_t)N, sizeof(void *));
    void *r = r_out ? r_out : malloc(es * (size_t)(L > 0 ? L : 1));
    int rc = 0;
    if (!b || !r) { rc = -1; goto done; }
    for (int i = 0; i < N; ++i) {
        b[i] = malloc(es * (size_t)(L > 0 ? L : 1));
        if (!b[i]) { rc = -1; goto done; }
        orc_pack(T, n, off, L, g + (size_t)i * T, dtype, b[i]);
    }
    rc = orc_reduce_tree(N, L, (const void *const *)b, dtype, r);
    if (rc == 0)
        orc_update_momentum_sgd(T, n, off, r, dtype, N, lr, mu, w, v, a_out);
done:
    if (b) for (int i = 0; i < N; ++i) free(b[i]);
    free(b);
    if (!r_out) free(r);
    return rc;
}

/* ------------------------------------------------------- array helpers */

void orc_f32_to_f16_array(const float *x, uint16_t *h, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) h[i] = orc_f32_to_f16(x[i]);
}

void orc_f16_to_f32_array(const uint16_t *h, float *x, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) x[i] = orc_f16_to_f32(h[i]);
}
