/* ASan + UBSan driver for the plain-C oracle (SURVEY §5 sanitizers; test
 * infrastructure).  Built together with oracle/cmn_oracle.c under
 * -fsanitize=address,undefined -fno-sanitize-recover=all and run by
 * tests/test_oracle_sanitizers.py: every oracle entry point on ragged,
 * empty and padded layouts, both payload dtypes, N = 1..8, multi-step
 * momentum and Adam.  Any out-of-bounds access, leak, signed overflow,
 * misaligned access or bad shift aborts with a nonzero exit. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

uint16_t orc_f32_to_f16(float x);
float orc_f16_to_f32(uint16_t h);
int64_t orc_layout(int T, const int64_t *n, int64_t align, int64_t *off);
void orc_pack(int T, const int64_t *n, const int64_t *off, int64_t L, const float *const *g, int dtype,
              void *b);
void orc_unpack_f32(int T, const int64_t *n, const int64_t *off, const float *b, float *const *out);
float orc_tree_sum(const float *x, int lo, int hi);
int orc_reduce_tree(int N, int64_t L, const void *const *b, int dtype, void *r);
void orc_update_momentum_sgd(int T, const int64_t *n, const int64_t *off, const void *r, int dtype, int N,
                             float lr, float mu, float *const *w, float *const *v, float *const *a_out);
void orc_update_adam(int T, const int64_t *n, const int64_t *off, const void *r, int dtype, int N,
                     float alpha, float beta1, float beta2, float eps, int step, float *const *w,
                     float *const *m, float *const *v);
void orc_exact_avg(int N, int64_t L, const float *const *g32, double *avg, double *mag);
int orc_step(int N, int T, const int64_t *n, const int64_t *off, int64_t L, const float *const *g,
             int dtype, float lr, float mu, float *const *w, float *const *v, float *const *a_out,
             void *r_out);
void orc_f32_to_f16_array(const float *x, uint16_t *h, int64_t n);
void orc_f16_to_f32_array(const uint16_t *h, float *x, int64_t n);

static uint64_t s_state = 190800213u;
static uint32_t rnd(void) {           /* splitmix64 */
    uint64_t z = (s_state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return (uint32_t)((z ^ (z >> 31)) >> 32);
}
static float rndf(void) { return ((float)(rnd() >> 8) - 8388608.0f) * 0x1p-23f; }

static int run_case(int T, const int64_t *n, int N, int dtype, int steps) {
    int64_t *off = malloc(sizeof(int64_t) * (size_t)(T + 1));
    int64_t L = orc_layout(T, n, 64, off);
    if (L < 0) { free(off); return 1; }
    float **g = calloc((size_t)N * (size_t)T, sizeof(float *));
    float **w = calloc((size_t)T, sizeof(float *)), **v = calloc((size_t)T, sizeof(float *));
    float **m = calloc((size_t)T, sizeof(float *)), **a = calloc((size_t)T, sizeof(float *));
    for (int t = 0; t < T; ++t) {
        size_t cnt = (size_t)(n[t] > 0 ? n[t] : 1);
        w[t] = malloc(cnt * 4); v[t] = calloc(cnt, 4); m[t] = calloc(cnt, 4); a[t] = malloc(cnt * 4);
        for (int64_t k = 0; k < n[t]; ++k) w[t][k] = rndf();
        for (int i = 0; i < N; ++i) {
            g[(size_t)i * T + t] = malloc(cnt * 4);
            for (int64_t k = 0; k < n[t]; ++k) g[(size_t)i * T + t][k] = rndf() * 0x1p-6f;
        }
    }
    size_t es = dtype == 0 ? 4 : 2;
    void **b = calloc((size_t)N, sizeof(void *));
    float **g32 = calloc((size_t)N, sizeof(float *));
    for (int i = 0; i < N; ++i) {
        b[i] = malloc(es * (size_t)(L > 0 ? L : 1));
        g32[i] = malloc(4 * (size_t)(L > 0 ? L : 1));
        orc_pack(T, n, off, L, (const float *const *)(g + (size_t)i * T), dtype, b[i]);
        orc_pack(T, n, off, L, (const float *const *)(g + (size_t)i * T), 0, g32[i]);
    }
    void *r = malloc(es * (size_t)(L > 0 ? L : 1));
    int rc = orc_reduce_tree(N, L, (const void *const *)b, dtype, r);
    double *avg = malloc(8 * (size_t)(L > 0 ? L : 1)), *mag = malloc(8 * (size_t)(L > 0 ? L : 1));
    orc_exact_avg(N, L, (const float *const *)g32, avg, mag);
    for (int s = 0; s < steps && rc == 0; ++s) {
        orc_update_momentum_sgd(T, n, off, r, dtype, N, 0.1f, 0.9f, w, v, a);
        orc_update_adam(T, n, off, r, dtype, N, 1e-3f, 0.9f, 0.999f, 1e-8f, s + 1, w, m, v);
        rc = orc_step(N, T, n, off, L, (const float *const *)g, dtype, 0.05f, 0.5f, w, v, a, NULL);
    }
    if (dtype == 0 && rc == 0) {
        float **u = calloc((size_t)T, sizeof(float *));
        for (int t = 0; t < T; ++t) u[t] = malloc(4 * (size_t)(n[t] > 0 ? n[t] : 1));
        orc_unpack_f32(T, n, off, (const float *)b[0], u);
        for (int t = 0; t < T && rc == 0; ++t)
            if (n[t] > 0 && memcmp(u[t], g[t], 4 * (size_t)n[t]) != 0) rc = 2;
        for (int t = 0; t < T; ++t) free(u[t]);
        free(u);
    }
    for (int i = 0; i < N; ++i) { free(b[i]); free(g32[i]); }
    for (size_t i = 0; i < (size_t)N * (size_t)T; ++i) free(g[i]);
    for (int t = 0; t < T; ++t) { free(w[t]); free(v[t]); free(m[t]); free(a[t]); }
    free(b); free(g32); free(g); free(w); free(v); free(m); free(a); free(r); free(avg); free(mag); free(off);
    return rc;
}

int main(void) {
    static const int64_t ragged[] = {1, 3, 4097, 0, 65, 7, 12289, 64, 0};
    static const int64_t mlp[] = {78400, 100, 10000, 100, 1000, 10};
    static const int64_t empty[] = {0, 0, 0};
    int fails = 0;
    for (int N = 1; N <= 8; ++N)
        for (int dt = 0; dt < 2; ++dt) {
            fails += run_case(9, ragged, N, dt, 2) != 0;
            fails += run_case(3, empty, N, dt, 1) != 0;
        }
    fails += run_case(6, mlp, 3, 0, 2) != 0;
    fails += run_case(6, mlp, 8, 1, 1) != 0;
    /* the conversions on a strided sweep of all bit patterns, specials included */
    for (uint64_t u = 0; u < (1ull << 32); u += 65537u) {
        float x;
        uint32_t b32 = (uint32_t)u;
        memcpy(&x, &b32, 4);
        uint16_t h = orc_f32_to_f16(x);
        (void)orc_f16_to_f32(h);
    }
    float xs[5] = {0.0f, -0.0f, INFINITY, NAN, 65520.0f};
    uint16_t hs[5];
    orc_f32_to_f16_array(xs, hs, 5);
    orc_f16_to_f32_array(hs, xs, 5);
    float one = 1.0f;
    (void)orc_tree_sum(&one, 0, 0);
    printf("oracle sanitize: %d failing cases\n", fails);
    return fails != 0;
}
