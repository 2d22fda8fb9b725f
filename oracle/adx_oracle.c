/*
 * adx_oracle.c -- CPU fp64 restatement of the AsyncDiff reference hot path.
 * TEST INFRASTRUCTURE ONLY (see adx_oracle.h).  Parity pinned by the
 * reference's goldens: tests/test_oracle_golden.py.
 *
 * Matrices are stored column-major, like the reference's Eigen::MatrixXd
 * (proj/include/asyncdiff/diffusion.hpp:10-11), and GEMV is evaluated as an
 * ordered column sweep y += W(:,k) u_k for k = 0..K-1, so every output
 * element is a left-to-right sum over k.
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -fopenmp).
 */
#define _GNU_SOURCE
#include "adx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAX_STAGES 256
#define OR_MAX_LINKS 256

static __thread char g_err[1024];
static int g_threads = 1;

const char* or_last_error(void) { return g_err; }
void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ===================================================================== RNG
 * std::mt19937_64 (published MT19937-64 parameters) + the reference's
 * explicit uniform/normal/below algorithms, proj/include/asyncdiff/rng.hpp. */
#define MT_NN 312
#define MT_MM 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void or_rng_seed(or_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_NN; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_NN;
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t or_rng_next_u64(or_rng* r) {
    static const uint64_t mag01[2] = {0ULL, MT_A};
    uint64_t x;
    if (r->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        for (; i < MT_NN - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[x & 1ULL];
        r->mti = 0;
    }
    x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:19-21 */
double or_rng_uniform(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }

static double uniform_lohi(or_rng* r, double lo, double hi) { return lo + (hi - lo) * or_rng_uniform(r); }

/* rng.hpp:26-40: Box-Muller, cos first, sin cached */
double or_rng_normal(or_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = or_rng_uniform(r);
    double u2 = or_rng_uniform(r);
    while (u1 <= 0.0) u1 = or_rng_uniform(r);
    double rr = sqrt(-2.0 * log(u1));
    double a = 2.0 * M_PI * u2;
    r->spare = rr * sin(a);
    r->have_spare = 1;
    return rr * cos(a);
}

/* rng.hpp:43-46 */
uint64_t or_rng_below(or_rng* r, uint64_t n) { return (uint64_t)(or_rng_uniform(r) * (double)n); }

/* rng.hpp:55-60 splitmix64 */
uint64_t or_mix_seed(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void or_random_normals(uint64_t seed, int n, double* out) {
    or_rng r;
    or_rng_seed(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = or_rng_normal(&r);
}

/* Bulk draws for the UNet-family oracle (oracle/unet_model.py, test
 * infrastructure): n consecutive float32 values (float)(lo + (hi-lo)*uniform())
 * or (float)normal() from one Rng state -- the same stream a C++ caller gets
 * from static_cast<float>(rng.uniform(lo, hi)) / static_cast<float>(rng.normal()). */
long long or_rng_sizeof(void) { return (long long)sizeof(or_rng); }

void or_rng_fill_uniform_f32(or_rng* r, long long n, double lo, double hi, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = (float)uniform_lohi(r, lo, hi);
}

void or_rng_fill_normal_f32(or_rng* r, long long n, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = (float)or_rng_normal(r);
}

/* ================================================================ schedule
 * proj/src/diffusion.cpp:39-77 */
int or_build_schedule(int T, double beta_start, double beta_end, int kind, double* betas,
                      double* alphas, double* alpha_bars) {
    if (T < 1) return fail(OR_INVALID_ARGUMENT, "build_schedule: T must be >= 1, got %d", T);
    if (!(beta_start > 0.0) || !(beta_start <= beta_end) || !(beta_end < 1.0))
        return fail(OR_INVALID_ARGUMENT,
                    "build_schedule: need 0 < beta_start <= beta_end < 1, got beta_start=%f "
                    "beta_end=%f",
                    beta_start, beta_end);
    if (T == 1) {
        betas[0] = beta_start;
    } else {
        for (int t = 1; t <= T; ++t) {
            double frac = (double)(t - 1) / (double)(T - 1);
            if (kind == OR_LINEAR) {
                betas[t - 1] = beta_start + frac * (beta_end - beta_start);
            } else {
                double r = sqrt(beta_start) + frac * (sqrt(beta_end) - sqrt(beta_start));
                betas[t - 1] = r * r;
            }
        }
    }
    alpha_bars[0] = 1.0;
    for (int t = 1; t <= T; ++t) {
        alphas[t - 1] = 1.0 - betas[t - 1];
        alpha_bars[t] = alpha_bars[t - 1] * alphas[t - 1];
    }
    return OR_OK;
}

/* proj/src/diffusion.cpp:79-93 */
int or_forward_diffuse(const double* x0, const double* noise, int d, int t,
                       const double* alpha_bars, int T, double* out) {
    if (t < 1 || t > T)
        return fail(OR_OUT_OF_RANGE, "forward_diffuse: t=%d outside [1, %d]", t, T);
    double abar = alpha_bars[t];
    double a = sqrt(abar), b = sqrt(1.0 - abar);
    for (int i = 0; i < d; ++i) out[i] = a * x0[i] + b * noise[i];
    return OR_OK;
}

/* proj/src/diffusion.cpp:95-116: predict_x0 then re-noise with the same eps */
int or_ddim_step(const double* x, const double* eps, int d, int t, const double* alpha_bars,
                 int T, double* out) {
    if (t < 1 || t > T)
        return fail(OR_OUT_OF_RANGE, "predict_x0: t=%d outside [1, %d]", t, T);
    for (int i = 0; i < d; ++i)
        if (!isfinite(eps[i]))
            return fail(OR_DOMAIN, "predict_x0: non-finite eps at t=%d", t);
    double abar_t = alpha_bars[t];
    double abar_prev = alpha_bars[t - 1];
    double s1 = sqrt(1.0 - abar_t), s2 = sqrt(abar_t);
    double s3 = sqrt(abar_prev), s4 = sqrt(1.0 - abar_prev);
    for (int i = 0; i < d; ++i) {
        double x0 = (x[i] - s1 * eps[i]) / s2;
        out[i] = s3 * x0 + s4 * eps[i];
    }
    return OR_OK;
}

/* ================================================================== model */
typedef struct {
    int in, h, out;
    double *w1, *b1, *tin, *w2, *b2; /* column-major */
    long long macs;
} or_stage;

struct or_model {
    int L, E, d;
    int widths[OR_MAX_STAGES + 1];
    int n_links;
    int links[OR_MAX_LINKS][2]; /* sorted (producer, consumer) */
    double* proj;               /* E x E column-major */
    or_stage st[OR_MAX_STAGES];
};

static int cmp_link(const void* a, const void* b) {
    const int* x = (const int*)a;
    const int* y = (const int*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/* proj/src/denoiser.cpp:75-122 make_denoiser_shell */
int or_model_shell(int L, const int* widths, const int* links, int n_links, int E,
                   or_model** out) {
    if (L < 2) return fail(OR_INVALID_ARGUMENT, "make_denoiser_shell: L must be >= 2, got %d", L);
    if (L > OR_MAX_STAGES || n_links > OR_MAX_LINKS)
        return fail(OR_INVALID_ARGUMENT, "make_denoiser_shell: model too large for oracle");
    for (int i = 0; i <= L; ++i)
        if (widths[i] < 1)
            return fail(OR_INVALID_ARGUMENT, "make_denoiser_shell: widths must be positive");
    if (widths[0] != widths[L])
        return fail(OR_INVALID_ARGUMENT,
                    "make_denoiser_shell: widths[0] (data dim) must equal widths[L] (eps dim)");
    if (E < 2 || E % 2 != 0)
        return fail(OR_INVALID_ARGUMENT,
                    "make_denoiser_shell: time_embed_dim must be even and >= 2");
    for (int k = 0; k < n_links; ++k) {
        int p = links[2 * k], c = links[2 * k + 1];
        if (p < 1 || c > L || p >= c)
            return fail(OR_INVALID_ARGUMENT, "make_denoiser_shell: bad skip link (%d, %d)", p, c);
    }
    or_model* m = (or_model*)calloc(1, sizeof(or_model));
    m->L = L;
    m->E = E;
    m->d = widths[0];
    memcpy(m->widths, widths, sizeof(int) * (size_t)(L + 1));
    m->n_links = n_links;
    memcpy(m->links, links, sizeof(int) * 2 * (size_t)n_links);
    qsort(m->links, (size_t)n_links, sizeof(m->links[0]), cmp_link);
    m->proj = (double*)calloc((size_t)E * E, sizeof(double));
    for (int i = 1; i <= L; ++i) {
        or_stage* s = &m->st[i - 1];
        int in = (i == 1) ? widths[0] + E : widths[i - 1];
        for (int k = 0; k < m->n_links; ++k)
            if (m->links[k][1] == i) in += widths[m->links[k][0]];
        s->in = in;
        s->h = widths[i];
        s->out = widths[i];
        s->w1 = (double*)calloc((size_t)s->h * in, sizeof(double));
        s->b1 = (double*)calloc((size_t)s->h, sizeof(double));
        s->tin = (double*)calloc((size_t)s->h * E, sizeof(double));
        s->w2 = (double*)calloc((size_t)s->out * s->h, sizeof(double));
        s->b2 = (double*)calloc((size_t)s->out, sizeof(double));
        s->macs = (long long)s->h * in + (long long)s->h * E + (long long)s->out * s->h;
    }
    *out = m;
    return OR_OK;
}

/* denoiser.cpp:21-27: row-major fill order (i outer, j inner) */
static void xavier(or_rng* r, double* m, int rows, int cols, double scale) {
    double a = sqrt(6.0 / (double)(rows + cols));
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) m[(size_t)j * rows + i] = scale * uniform_lohi(r, -a, a);
}

/* denoiser.cpp:124-142 build_toy_denoiser */
int or_model_build_toy(int L, const int* widths, int skip_spec, uint64_t seed, int E,
                       or_model** out) {
    int links[OR_MAX_LINKS * 2];
    int n = 0;
    if (skip_spec == OR_SKIP_UNET_MIRROR)
        for (int i = 1; i < L + 1 - i; ++i) {
            links[2 * n] = i;
            links[2 * n + 1] = L + 1 - i;
            ++n;
        }
    int rc = or_model_shell(L, widths, links, n, E, out);
    if (rc) return rc;
    or_model* m = *out;
    or_rng r;
    or_rng_seed(&r, seed);
    xavier(&r, m->proj, E, E, 1.0);
    for (int i = 0; i < L; ++i) {
        or_stage* s = &m->st[i];
        xavier(&r, s->w1, s->h, s->in, 1.0);
        /* 0.5 * xavier(h, E): scale applied after the draw, exact */
        xavier(&r, s->tin, s->h, E, 0.5);
        xavier(&r, s->w2, s->out, s->h, 1.0);
    }
    return OR_OK;
}

void or_model_free(or_model* m) {
    if (!m) return;
    free(m->proj);
    for (int i = 0; i < m->L; ++i) {
        free(m->st[i].w1);
        free(m->st[i].b1);
        free(m->st[i].tin);
        free(m->st[i].w2);
        free(m->st[i].b2);
    }
    free(m);
}

int or_model_num_stages(const or_model* m) { return m->L; }
int or_model_num_links(const or_model* m) { return m->n_links; }
void or_model_links(const or_model* m, int* out_pairs) {
    memcpy(out_pairs, m->links, sizeof(int) * 2 * (size_t)m->n_links);
}
long long or_model_stage_macs(const or_model* m, int stage) { return m->st[stage - 1].macs; }
void or_model_set_stage_macs(or_model* m, int stage, long long macs) { m->st[stage - 1].macs = macs; }

double* or_model_tensor(or_model* m, int stage, int which, int* rows, int* cols) {
    if (which == OR_T_PROJ) {
        *rows = m->E;
        *cols = m->E;
        return m->proj;
    }
    or_stage* s = &m->st[stage - 1];
    switch (which) {
        case OR_T_W1: *rows = s->h; *cols = s->in; return s->w1;
        case OR_T_B1: *rows = s->h; *cols = 1; return s->b1;
        case OR_T_TIN: *rows = s->h; *cols = m->E; return s->tin;
        case OR_T_W2: *rows = s->out; *cols = s->h; return s->w2;
        case OR_T_B2: *rows = s->out; *cols = 1; return s->b2;
    }
    return NULL;
}

/* y = W x, W rows x cols column-major: ordered column sweep (left-to-right sum
 * per output element).  Row blocks are independent, so the OpenMP split does
 * not change any result bit. */
static void gemv(const double* W, int rows, int cols, const double* x, double* y) {
    int nt = g_threads;
    if (nt <= 1 || (long long)rows * cols < (1LL << 20)) {
        for (int i = 0; i < rows; ++i) y[i] = 0.0;
        for (int k = 0; k < cols; ++k) {
            const double* c = W + (size_t)k * rows;
            double xk = x[k];
            for (int i = 0; i < rows; ++i) y[i] += c[i] * xk;
        }
        return;
    }
#pragma omp parallel num_threads(nt)
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num(), nth = omp_get_num_threads();
#else
        int tid = 0, nth = 1;
#endif
        int chunk = (rows + nth - 1) / nth;
        chunk = (chunk + 7) & ~7;
        int r0 = tid * chunk, r1 = r0 + chunk < rows ? r0 + chunk : rows;
        if (r0 < r1) {
            for (int i = r0; i < r1; ++i) y[i] = 0.0;
            for (int k = 0; k < cols; ++k) {
                const double* c = W + (size_t)k * rows;
                double xk = x[k];
                for (int i = r0; i < r1; ++i) y[i] += c[i] * xk;
            }
        }
    }
}

/* denoiser.cpp:31-41 */
int or_sinusoid(int t, int dim, double* s) {
    int half = dim / 2;
    for (int k = 0; k < half; ++k) {
        double freq = exp(-log(10000.0) * (double)k / (double)half);
        s[k] = cos(t * freq);
        s[half + k] = sin(t * freq);
    }
    return OR_OK;
}

/* denoiser.hpp:24: e_t = proj * sinusoid(t) */
static void embed(const or_model* m, int t, double* e) {
    double s[512];
    or_sinusoid(t, m->E, s);
    gemv(m->proj, m->E, m->E, s, e);
}

/* --------------------------------------------------------------- skip maps */
typedef struct {
    double* val[OR_MAX_LINKS]; /* NULL = absent; owned */
} skipmap;

static void skipmap_clear(skipmap* s, int n) {
    for (int k = 0; k < n; ++k) {
        free(s->val[k]);
        s->val[k] = NULL;
    }
}

static double* dupv(const double* v, int n) {
    double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    memcpy(r, v, sizeof(double) * (size_t)n);
    return r;
}

static void skipmap_copy(skipmap* dst, const skipmap* src, const or_model* m) {
    for (int k = 0; k < m->n_links; ++k) {
        free(dst->val[k]);
        dst->val[k] = src->val[k] ? dupv(src->val[k], m->widths[m->links[k][0]]) : NULL;
    }
}

/* denoiser.cpp:150-192 run_stage_range.  `cur` (length cur_n) is consumed
 * (freed); returns the last stage output (malloc'd). */
static int run_stage_range(const or_model* m, int first, int last, double* cur, int cur_n,
                           const double* e_t, skipmap* skips, double** out) {
    for (int i = first; i <= last; ++i) {
        const or_stage* s = &m->st[i - 1];
        /* links_into(i), ascending producer (links are sorted) */
        int extra = 0;
        for (int k = 0; k < m->n_links; ++k) {
            if (m->links[k][1] != i) continue;
            if (!skips->val[k]) {
                free(cur);
                return fail(OR_RUNTIME, "eval: missing skip feature for link (%d -> %d)",
                            m->links[k][0], i);
            }
            extra += m->widths[m->links[k][0]];
        }
        int un = cur_n + extra;
        double* u = cur;
        if (extra) {
            u = (double*)malloc(sizeof(double) * (size_t)un);
            memcpy(u, cur, sizeof(double) * (size_t)cur_n);
            int at = cur_n;
            for (int k = 0; k < m->n_links; ++k) {
                if (m->links[k][1] != i) continue;
                int w = m->widths[m->links[k][0]];
                memcpy(u + at, skips->val[k], sizeof(double) * (size_t)w);
                at += w;
            }
            free(cur);
        }
        if (un != s->in) {
            free(u);
            return fail(OR_RUNTIME, "eval: stage %d input width %d != expected %d", i, un, s->in);
        }
        double* z = (double*)malloc(sizeof(double) * (size_t)s->h);
        double* te = (double*)malloc(sizeof(double) * (size_t)s->h);
        gemv(s->w1, s->h, s->in, u, z);
        gemv(s->tin, s->h, m->E, e_t, te);
        /* z = (W1 u + b1) + Tin e_t ; h = lrelu_0.1(z)   (denoiser.cpp:14-16, 182-183) */
        for (int j = 0; j < s->h; ++j) {
            double v = (z[j] + s->b1[j]) + te[j];
            z[j] = v > 0.0 ? v : 0.1 * v;
        }
        double* y = (double*)malloc(sizeof(double) * (size_t)s->out);
        gemv(s->w2, s->out, s->h, z, y);
        for (int j = 0; j < s->out; ++j) y[j] += s->b2[j];
        free(u);
        free(z);
        free(te);
        for (int j = 0; j < s->out; ++j)
            if (!isfinite(y[j])) {
                free(y);
                return fail(OR_DOMAIN, "eval: non-finite activation at stage %d", i);
            }
        for (int k = 0; k < m->n_links; ++k)
            if (m->links[k][0] == i) {
                free(skips->val[k]);
                skips->val[k] = dupv(y, s->out);
            }
        cur = y;
        cur_n = s->out;
    }
    *out = cur;
    return OR_OK;
}

/* one stage of run_stage_range (denoiser.cpp:182-187) on an explicit concat
 * input u (length in); the multi-rank gloo test drives segments with it. */
int or_stage_forward(const or_model* m, int stage, const double* u, int un, int t_embed, double* y_out) {
    const or_stage* s = &m->st[stage - 1];
    if (un != s->in) return fail(OR_RUNTIME, "eval: stage %d input width %d != expected %d", stage, un, s->in);
    double e[512];
    embed(m, t_embed, e);
    double* z = (double*)malloc(sizeof(double) * (size_t)s->h);
    double* te = (double*)malloc(sizeof(double) * (size_t)s->h);
    gemv(s->w1, s->h, s->in, u, z);
    gemv(s->tin, s->h, m->E, e, te);
    for (int j = 0; j < s->h; ++j) {
        double v = (z[j] + s->b1[j]) + te[j];
        z[j] = v > 0.0 ? v : 0.1 * v;
    }
    gemv(s->w2, s->out, s->h, z, y_out);
    for (int j = 0; j < s->out; ++j) y_out[j] += s->b2[j];
    free(z);
    free(te);
    return OR_OK;
}

void or_embed(const or_model* m, int t, double* out) { embed(m, t, out); }

/* denoiser.cpp:222-233 */
int or_eval_full(const or_model* m, const double* x, int t_embed, double* eps_out) {
    double e[512];
    embed(m, t_embed, e);
    double* in = (double*)malloc(sizeof(double) * (size_t)(m->d + m->E));
    memcpy(in, x, sizeof(double) * (size_t)m->d);
    memcpy(in + m->d, e, sizeof(double) * (size_t)m->E);
    skipmap sk;
    memset(&sk, 0, sizeof sk);
    double* y = NULL;
    int rc = run_stage_range(m, 1, m->L, in, m->d + m->E, e, &sk, &y);
    skipmap_clear(&sk, m->n_links);
    if (rc) return rc;
    memcpy(eps_out, y, sizeof(double) * (size_t)m->d);
    free(y);
    return OR_OK;
}

/* ============================================================== partition
 * proj/src/partition.cpp:95-125 min_max_split: exact DP, strict '<' so ties
 * go to the smallest cut j. */
static void min_max_split(const long long* costs, int n, int parts, int* cuts) {
    long long* prefix = (long long*)calloc((size_t)n + 1, sizeof(long long));
    for (int i = 0; i < n; ++i) prefix[i + 1] = prefix[i] + costs[i];
    const long long kInf = 0x7fffffffffffffffLL / 4;
    long long* best = (long long*)malloc(sizeof(long long) * (size_t)(parts + 1) * (n + 1));
    int* choice = (int*)malloc(sizeof(int) * (size_t)(parts + 1) * (n + 1));
#define B(p, i) best[(size_t)(p) * (n + 1) + (i)]
#define C(p, i) choice[(size_t)(p) * (n + 1) + (i)]
    for (int p = 0; p <= parts; ++p)
        for (int i = 0; i <= n; ++i) {
            B(p, i) = kInf;
            C(p, i) = -1;
        }
    B(0, 0) = 0;
    for (int p = 1; p <= parts; ++p)
        for (int i = p; i <= n - (parts - p); ++i)
            for (int j = p - 1; j < i; ++j) {
                long long rs = prefix[i] - prefix[j];
                long long v = B(p - 1, j) > rs ? B(p - 1, j) : rs;
                if (v < B(p, i)) {
                    B(p, i) = v;
                    C(p, i) = j;
                }
            }
    cuts[parts] = n;
    for (int p = parts; p >= 1; --p) cuts[p - 1] = C(p, cuts[p]);
#undef B
#undef C
    free(prefix);
    free(best);
    free(choice);
}

/* proj/src/partition.cpp:133-198 */
int or_partition_balanced(const long long* costs, int L, int N, int strategy, int* stage_segment,
                          long long* seg_macs) {
    int* cuts = (int*)malloc(sizeof(int) * (size_t)(N + 2));
    if (strategy == OR_SEQUENTIAL_BALANCED) {
        if (N < 1 || N > L) {
            free(cuts);
            return fail(OR_INVALID_ARGUMENT, "partition_balanced: N=%d infeasible for L=%d", N, L);
        }
        min_max_split(costs, L, N, cuts);
        for (int seg = 0; seg < N; ++seg) {
            seg_macs[seg] = 0;
            for (int s = cuts[seg] + 1; s <= cuts[seg + 1]; ++s) {
                stage_segment[s - 1] = seg + 1;
                seg_macs[seg] += costs[s - 1];
            }
        }
        free(cuts);
        return OR_OK;
    }
    if (N < 1 || N > L - 1) {
        free(cuts);
        return fail(OR_INVALID_ARGUMENT,
                    "partition_balanced: first-last-grouped N=%d infeasible for L=%d (need N <= "
                    "L-1)",
                    N, L);
    }
    if (N == 1) {
        seg_macs[0] = 0;
        for (int s = 1; s <= L; ++s) {
            stage_segment[s - 1] = 1;
            seg_macs[0] += costs[s - 1];
        }
        free(cuts);
        return OR_OK;
    }
    stage_segment[0] = 1;
    stage_segment[L - 1] = 1;
    seg_macs[0] = costs[0] + costs[L - 1];
    min_max_split(costs + 1, L - 2, N - 1, cuts);
    for (int seg = 0; seg < N - 1; ++seg) {
        seg_macs[seg + 1] = 0;
        for (int i = cuts[seg]; i < cuts[seg + 1]; ++i) {
            stage_segment[i + 1] = seg + 2;
            seg_macs[seg + 1] += costs[i + 1];
        }
    }
    free(cuts);
    return OR_OK;
}

/* =================================================================== plan
 * proj/src/plan.cpp:17-97 plan_async, emitted in the flat layout. */
typedef struct {
    int* buf;
    int len, cap, overflow;
} ibuf;

static void put(ibuf* b, int v) {
    if (b->len < b->cap)
        b->buf[b->len] = v;
    else
        b->overflow = 1;
    b->len++;
}

static void put_eval(ibuf* b, int seg, int dev, int embed_t, int kind, int pseg, int pround,
                     int emits) {
    put(b, seg);
    put(b, dev);
    put(b, embed_t);
    put(b, kind);
    put(b, pseg);
    put(b, pround);
    put(b, emits);
}

int or_plan_async_flat(int T, int w, int N, int S, int time_shift, int* out, int cap,
                       int* out_len) {
    if (T < 1) return fail(OR_INVALID_ARGUMENT, "plan_async: T must be >= 1");
    if (w < 1 || w > T)
        return fail(OR_INVALID_ARGUMENT, "plan_async: w=%d outside [1, T=%d]", w, T);
    if (N < 1) return fail(OR_INVALID_ARGUMENT, "plan_async: N must be >= 1");
    if (S != 1 && S != 2) return fail(OR_INVALID_ARGUMENT, "plan_async: S must be 1 or 2, got %d", S);
    if (S == 2 && N < 2) return fail(OR_INVALID_ARGUMENT, "plan_async: S=2 requires N >= 2");
    ibuf b = {out, 0, cap, 0};
    int n_rounds = (S == 1) ? T - w : (T - w + 1) / 2;
    put(&b, T);
    put(&b, w);
    put(&b, N);
    put(&b, S);
    put(&b, N + S - 1);
    put(&b, time_shift ? 1 : 0);
    put(&b, n_rounds);
    for (int t = T; t > T - w; --t) put(&b, t);
#define EMB(tt) (time_shift ? ((tt) + 1 < T ? (tt) + 1 : T) : (tt))
    int t = T - w, r = 0;
    while (t >= 1) {
        int prev = (r == 0) ? -1 : r - 1;
        int last = (t - ((S == 2 && t >= 2) ? 2 : 1)) < 1;
        put(&b, r);
        put(&b, last ? 0 : 1);
        if (S == 2 && t >= 2) {
            put(&b, 2);
            put(&b, t);
            put(&b, t - 1);
            put(&b, N + 1);
            for (int n = 1; n < N; ++n)
                put_eval(&b, n, n - 1, EMB(t - 1), n == 1 ? 0 : 1, n == 1 ? 0 : n - 1,
                         n == 1 ? -1 : prev, -1);
            put_eval(&b, N, N - 1, EMB(t), 1, N - 1, prev, t);
            put_eval(&b, N, N, EMB(t - 1), 1, N - 1, prev, t - 1);
            t -= 2;
        } else {
            put(&b, 1);
            put(&b, t);
            put(&b, N);
            for (int n = 1; n <= N; ++n)
                put_eval(&b, n, n - 1, EMB(t), n == 1 ? 0 : 1, n == 1 ? 0 : n - 1,
                         n == 1 ? -1 : prev, n == N ? t : -1);
            t -= 1;
        }
        ++r;
    }
#undef EMB
    *out_len = b.len;
    if (b.overflow) return fail(OR_INVALID_ARGUMENT, "plan_async_flat: buffer too small (%d)", b.len);
    return OR_OK;
}

/* flat plan parsing */
typedef struct {
    int seg, dev, embed_t, kind, pseg, pround, emits;
} p_eval;
typedef struct {
    int index, broadcast, n_sampler, sampler[2], n_evals;
    p_eval ev[OR_MAX_STAGES + 1];
} p_round;
typedef struct {
    int T, w, N, S, D, shift, n_rounds;
    const int* warmup;
    p_round* rounds;
} p_plan;

static int parse_plan(const int* f, p_plan* p) {
    p->T = f[0];
    p->w = f[1];
    p->N = f[2];
    p->S = f[3];
    p->D = f[4];
    p->shift = f[5];
    p->n_rounds = f[6];
    p->warmup = f + 7;
    const int* q = f + 7 + p->w;
    p->rounds = (p_round*)calloc((size_t)(p->n_rounds > 0 ? p->n_rounds : 1), sizeof(p_round));
    for (int r = 0; r < p->n_rounds; ++r) {
        p_round* R = &p->rounds[r];
        R->index = *q++;
        R->broadcast = *q++;
        R->n_sampler = *q++;
        if (R->n_sampler < 0 || R->n_sampler > 2) return fail(OR_INVALID_ARGUMENT, "bad plan");
        for (int i = 0; i < R->n_sampler; ++i) R->sampler[i] = *q++;
        R->n_evals = *q++;
        if (R->n_evals < 0 || R->n_evals > OR_MAX_STAGES) return fail(OR_INVALID_ARGUMENT, "bad plan");
        for (int e = 0; e < R->n_evals; ++e) {
            p_eval* E = &R->ev[e];
            E->seg = *q++;
            E->dev = *q++;
            E->embed_t = *q++;
            E->kind = *q++;
            E->pseg = *q++;
            E->pround = *q++;
            E->emits = *q++;
        }
    }
    return OR_OK;
}

/* =============================================================== executor */
typedef struct {
    int used, seg, round;
    double* boundary;
    int bn;
    skipmap skips; /* crossing links produced by seg */
} bundle;

typedef struct {
    bundle* e;
    int cap;
} bstore;

/* executor.cpp:28-33 */
static int store_put(bstore* s, int seg, int round, bundle* b, const or_model* m) {
    for (int i = 0; i < s->cap; ++i)
        if (s->e[i].used && s->e[i].seg == seg && s->e[i].round == round) {
            free(b->boundary);
            skipmap_clear(&b->skips, m->n_links);
            return fail(OR_LOGIC, "BundleStore: entry (%d, %d) already written", seg, round);
        }
    for (int i = 0; i < s->cap; ++i)
        if (!s->e[i].used) {
            s->e[i] = *b;
            s->e[i].used = 1;
            s->e[i].seg = seg;
            s->e[i].round = round;
            return OR_OK;
        }
    int old = s->cap;
    s->cap = s->cap ? 2 * s->cap : 16;
    s->e = (bundle*)realloc(s->e, sizeof(bundle) * (size_t)s->cap);
    memset(s->e + old, 0, sizeof(bundle) * (size_t)(s->cap - old));
    s->e[old] = *b;
    s->e[old].used = 1;
    s->e[old].seg = seg;
    s->e[old].round = round;
    return OR_OK;
}

static const bundle* store_find(const bstore* s, int seg, int round) {
    for (int i = 0; i < s->cap; ++i)
        if (s->e[i].used && s->e[i].seg == seg && s->e[i].round == round) return &s->e[i];
    return NULL;
}

/* executor.cpp:41-51 */
static const bundle* store_newest(const bstore* s, int seg) {
    const bundle* best = NULL;
    int br = -2;
    for (int i = 0; i < s->cap; ++i)
        if (s->e[i].used && s->e[i].seg == seg && s->e[i].round > br) {
            best = &s->e[i];
            br = s->e[i].round;
        }
    return best;
}

/* executor.cpp:53-62: keep the warm-up tail and the last two rounds */
static void store_prune(bstore* s, int current_round, const or_model* m) {
    for (int i = 0; i < s->cap; ++i)
        if (s->e[i].used && s->e[i].round != -1 && s->e[i].round < current_round - 2) {
            free(s->e[i].boundary);
            skipmap_clear(&s->e[i].skips, m->n_links);
            s->e[i].used = 0;
        }
}

static int store_size(const bstore* s) {
    int n = 0;
    for (int i = 0; i < s->cap; ++i) n += s->e[i].used;
    return n;
}

static void store_free(bstore* s, const or_model* m) {
    for (int i = 0; i < s->cap; ++i)
        if (s->e[i].used) {
            free(s->e[i].boundary);
            skipmap_clear(&s->e[i].skips, m->n_links);
        }
    free(s->e);
}

typedef struct {
    const or_model* m;
    const int* stage_segment;
    int N;
    int first[OR_MAX_STAGES + 1], last[OR_MAX_STAGES + 1]; /* per segment, 1-based */
} part_view;

static int make_part_view(const or_model* m, const int* stage_segment, int N, part_view* pv) {
    pv->m = m;
    pv->stage_segment = stage_segment;
    pv->N = N;
    int expect_seg = 1;
    for (int n = 1; n <= N; ++n) pv->first[n] = pv->last[n] = 0;
    for (int s = 1; s <= m->L; ++s) {
        int g = stage_segment[s - 1];
        if (g < 1 || g > N) return fail(OR_INVALID_ARGUMENT, "Partition: stage %d unassigned", s);
        if (g != expect_seg) {
            if (g == expect_seg + 1 && pv->last[expect_seg] == s - 1)
                expect_seg = g;
            else
                return fail(OR_INVALID_ARGUMENT, "run: partition must be a contiguous cascade");
        }
        if (!pv->first[g]) pv->first[g] = s;
        pv->last[g] = s;
    }
    if (expect_seg != N) return fail(OR_INVALID_ARGUMENT, "run: partition segment count != plan.N");
    return OR_OK;
}

/* eval_segment + finish_segment, denoiser.cpp:194-267.  For seg == 1 `in` is
 * the latent x; otherwise the producer's bundle.  On return either *eps (seg
 * N) or *out_b (seg < N) is filled. */
static int eval_segment(const part_view* pv, int seg, const double* x, const bundle* in,
                        const skipmap* skips_in, int t_embed, double** eps, bundle* out_b) {
    const or_model* m = pv->m;
    double e[512];
    embed(m, t_embed, e);
    skipmap sk;
    memset(&sk, 0, sizeof sk);
    skipmap_copy(&sk, skips_in, m);
    double* cur;
    int cur_n;
    if (seg == 1) {
        if (!x) return fail(OR_INVALID_ARGUMENT, "eval_segment: segment 1 requires a Latent input");
        cur_n = m->d + m->E;
        cur = (double*)malloc(sizeof(double) * (size_t)cur_n);
        memcpy(cur, x, sizeof(double) * (size_t)m->d);
        memcpy(cur + m->d, e, sizeof(double) * (size_t)m->E);
    } else {
        if (!in)
            return fail(OR_INVALID_ARGUMENT,
                        "eval_segment: segment %d requires a HiddenBundle input, not a Latent", seg);
        if (in->seg != seg - 1)
            return fail(OR_INVALID_ARGUMENT,
                        "eval_segment: segment %d needs a bundle from segment %d, got one from "
                        "segment %d",
                        seg, seg - 1, in->seg);
        cur_n = in->bn;
        cur = dupv(in->boundary, cur_n);
    }
    double* y = NULL;
    int rc = run_stage_range(m, pv->first[seg], pv->last[seg], cur, cur_n, e, &sk, &y);
    if (rc) {
        skipmap_clear(&sk, m->n_links);
        return rc;
    }
    if (seg == pv->N) {
        *eps = y;
        skipmap_clear(&sk, m->n_links);
        return OR_OK;
    }
    memset(out_b, 0, sizeof *out_b);
    out_b->seg = seg;
    out_b->boundary = y;
    out_b->bn = m->widths[pv->last[seg]];
    for (int k = 0; k < m->n_links; ++k) {
        int p = m->links[k][0], c = m->links[k][1];
        if (sk.val[k] && p >= pv->first[seg] && p <= pv->last[seg] && c > pv->last[seg]) {
            out_b->skips.val[k] = sk.val[k];
            sk.val[k] = NULL;
        }
    }
    skipmap_clear(&sk, m->n_links);
    return OR_OK;
}

/* executor.cpp:111-119 */
static void collect_skips(const bstore* s, const part_view* pv, skipmap* out) {
    const or_model* m = pv->m;
    for (int seg = 1; seg < pv->N; ++seg) {
        const bundle* b = store_newest(s, seg);
        if (!b) continue;
        for (int k = 0; k < m->n_links; ++k)
            if (b->skips.val[k]) {
                free(out->val[k]);
                out->val[k] = dupv(b->skips.val[k], m->widths[m->links[k][0]]);
            }
    }
}

typedef struct {
    const part_view* pv;
    const bstore* store;
    const skipmap* skips;
    const double* latent;
    int round;
} round_ctx;

typedef struct {
    int has_bundle, has_eps, emits, rc;
    bundle b;
    double* eps;
    char err[512];
} outcome;

/* executor.cpp:121-156 */
static int execute_eval(const p_eval* ev, const round_ctx* ctx, outcome* o) {
    memset(o, 0, sizeof *o);
    int rc;
    double* eps = NULL;
    if (ev->kind == 0) {
        if (ev->seg != 1)
            return fail(OR_INVALID_ARGUMENT,
                        "eval_segment: segment %d requires a HiddenBundle input, not a Latent",
                        ev->seg);
        rc = eval_segment(ctx->pv, ev->seg, ctx->latent, NULL, ctx->skips, ev->embed_t, &eps, &o->b);
    } else {
        if (ev->pround >= ctx->round)
            return fail(OR_LOGIC, "executor: round %d reads a bundle from round %d", ctx->round,
                        ev->pround);
        const bundle* b = store_find(ctx->store, ev->pseg, ev->pround);
        if (!b)
            return fail(OR_LOGIC,
                        "executor: unresolvable cached ref (segment %d, round %d) in round %d",
                        ev->pseg, ev->pround, ctx->round);
        if (ev->seg == 1)
            return fail(OR_INVALID_ARGUMENT, "eval_segment: segment 1 requires a Latent input");
        rc = eval_segment(ctx->pv, ev->seg, NULL, b, ctx->skips, ev->embed_t, &eps, &o->b);
    }
    if (rc) return rc;
    if (ev->seg == ctx->pv->N) {
        if (ev->emits < 0) {
            free(eps);
            return fail(OR_LOGIC, "executor: final segment produced eps without a target");
        }
        o->has_eps = 1;
        o->eps = eps;
        o->emits = ev->emits;
    } else {
        o->has_bundle = 1;
    }
    return OR_OK;
}

/* executor.cpp:168-202 warm-up cascade (fresh skip map), then ddim. */
static int warmup(const part_view* pv, const p_plan* P, const double* alpha_bars, double* x,
                  bstore* store, double* traj_latents, double* traj_eps, int* step) {
    const or_model* m = pv->m;
    int d = m->d;
    for (int wi = 0; wi < P->w; ++wi) {
        int t = P->warmup[wi];
        skipmap sk;
        memset(&sk, 0, sizeof sk);
        bundle carry;
        memset(&carry, 0, sizeof carry);
        bundle* keep = (bundle*)calloc((size_t)pv->N, sizeof(bundle));
        double* eps = NULL;
        int rc = OR_OK;
        for (int seg = 1; seg <= pv->N && !rc; ++seg) {
            bundle nb;
            rc = eval_segment(pv, seg, seg == 1 ? x : NULL, seg == 1 ? NULL : &carry, &sk, t, &eps,
                              &nb);
            if (rc) break;
            if (seg < pv->N) {
                for (int k = 0; k < m->n_links; ++k)
                    if (nb.skips.val[k]) {
                        free(sk.val[k]);
                        sk.val[k] = dupv(nb.skips.val[k], m->widths[m->links[k][0]]);
                    }
                keep[seg - 1] = nb;
                carry = nb;
            }
        }
        skipmap_clear(&sk, m->n_links);
        if (!rc && wi + 1 == P->w) {
            for (int seg = 1; seg < pv->N && !rc; ++seg) {
                rc = store_put(store, seg, -1, &keep[seg - 1], m);
                keep[seg - 1].boundary = NULL;
                memset(&keep[seg - 1].skips, 0, sizeof(skipmap));
            }
        }
        for (int seg = 1; seg < pv->N; ++seg) {
            free(keep[seg - 1].boundary);
            skipmap_clear(&keep[seg - 1].skips, m->n_links);
        }
        free(keep);
        if (rc) {
            free(eps);
            return rc;
        }
        rc = or_ddim_step(x, eps, d, t, alpha_bars, P->T, x);
        if (traj_eps) memcpy(traj_eps + (size_t)(*step) * d, eps, sizeof(double) * (size_t)d);
        free(eps);
        if (rc) return rc;
        ++*step;
        if (traj_latents) memcpy(traj_latents + (size_t)(*step) * d, x, sizeof(double) * (size_t)d);
    }
    return OR_OK;
}

/* executor.cpp:224-241 + commit/prune (:316-318) */
static int finish_round(const part_view* pv, const p_plan* P, const p_round* R, outcome* outs,
                        int n_out, const double* alpha_bars, double* x, bstore* store,
                        double* traj_latents, double* traj_eps, int* step) {
    const or_model* m = pv->m;
    int d = m->d;
    int rc = OR_OK;
    for (int i = 0; i < R->n_sampler && !rc; ++i) {
        int t = R->sampler[i];
        const double* eps = NULL;
        for (int k = 0; k < n_out; ++k)
            if (outs[k].has_eps && outs[k].emits == t) eps = outs[k].eps;
        if (!eps) {
            rc = fail(OR_LOGIC, "executor: no eps available for sampler step t=%d", t);
            break;
        }
        int xt = P->T - *step;
        if (xt != t) {
            rc = fail(OR_LOGIC, "executor: sampler expected latent at t=%d, have t=%d", t, xt);
            break;
        }
        rc = or_ddim_step(x, eps, d, t, alpha_bars, P->T, x);
        if (rc) break;
        if (traj_eps) memcpy(traj_eps + (size_t)(*step) * d, eps, sizeof(double) * (size_t)d);
        ++*step;
        if (traj_latents) memcpy(traj_latents + (size_t)(*step) * d, x, sizeof(double) * (size_t)d);
    }
    /* commit in produced_by order (executor.cpp:574-577) */
    for (int seg = 1; seg < pv->N; ++seg)
        for (int k = 0; k < n_out; ++k)
            if (outs[k].has_bundle && outs[k].b.seg == seg) {
                if (!rc) rc = store_put(store, seg, R->index, &outs[k].b, m);
                else {
                    free(outs[k].b.boundary);
                    skipmap_clear(&outs[k].b.skips, m->n_links);
                }
                outs[k].has_bundle = 0;
            }
    for (int k = 0; k < n_out; ++k) {
        if (outs[k].has_eps) free(outs[k].eps);
        if (outs[k].has_bundle) {
            free(outs[k].b.boundary);
            skipmap_clear(&outs[k].b.skips, m->n_links);
        }
    }
    if (!rc) store_prune(store, R->index + 1, m);
    return rc;
}

static int check_plan_shape(const p_plan* P, const part_view* pv, int T) {
    if (P->N != pv->N) return fail(OR_INVALID_ARGUMENT, "run: partition segment count != plan.N");
    if (P->T != T) return fail(OR_INVALID_ARGUMENT, "run: plan T != schedule T");
    return OR_OK;
}

int or_run_serial(const or_model* m, const int* stage_segment, int N, const int* plan_flat,
                  const double* alpha_bars, int T, const double* x_T, double* traj_latents,
                  double* traj_eps, int* store_entries, int* broadcast_count) {
    part_view pv;
    int rc = make_part_view(m, stage_segment, N, &pv);
    if (rc) return rc;
    p_plan P;
    rc = parse_plan(plan_flat, &P);
    if (!rc) rc = check_plan_shape(&P, &pv, T);
    if (rc) {
        free(P.rounds);
        return rc;
    }
    int d = m->d, step = 0;
    double* x = dupv(x_T, d);
    if (traj_latents) memcpy(traj_latents, x_T, sizeof(double) * (size_t)d);
    bstore store = {NULL, 0};
    rc = warmup(&pv, &P, alpha_bars, x, &store, traj_latents, traj_eps, &step);
    int bc = 0;
    for (int r = 0; r < P.n_rounds && !rc; ++r) {
        const p_round* R = &P.rounds[r];
        skipmap snap;
        memset(&snap, 0, sizeof snap);
        collect_skips(&store, &pv, &snap);
        round_ctx ctx = {&pv, &store, &snap, x, R->index};
        outcome* outs = (outcome*)calloc((size_t)R->n_evals, sizeof(outcome));
        for (int e = 0; e < R->n_evals && !rc; ++e) rc = execute_eval(&R->ev[e], &ctx, &outs[e]);
        skipmap_clear(&snap, m->n_links);
        if (!rc)
            rc = finish_round(&pv, &P, R, outs, R->n_evals, alpha_bars, x, &store, traj_latents,
                              traj_eps, &step);
        free(outs);
        if (store_entries) store_entries[r] = store_size(&store);
        ++bc;
    }
    if (broadcast_count) *broadcast_count = bc;
    store_free(&store, m);
    free(x);
    free(P.rounds);
    return rc;
}

/* ---- parallel runtime: D worker threads per round, barrier, sorted commit
 * (executor.cpp:338-601).  Each worker evaluates the round's evals mapped to
 * its device against the immutable round-start snapshot. */
typedef struct {
    const p_round* R;
    const round_ctx* ctx;
    int device;
    outcome* out; /* per-eval slots */
    int rc;
    char err[1024];
} worker_arg;

static void* worker_main(void* p) {
    worker_arg* a = (worker_arg*)p;
    a->rc = OR_OK;
    for (int e = 0; e < a->R->n_evals; ++e) {
        if (a->R->ev[e].dev != a->device) continue;
        a->rc = execute_eval(&a->R->ev[e], a->ctx, &a->out[e]);
        if (a->rc) {
            snprintf(a->err, sizeof a->err, "%s", g_err);
            break;
        }
    }
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int or_run_parallel(const or_model* m, const int* stage_segment, int N, const int* plan_flat,
                    const double* alpha_bars, int T, const double* x_T, double* traj_latents,
                    double* traj_eps, double* wall_s) {
    part_view pv;
    int rc = make_part_view(m, stage_segment, N, &pv);
    if (rc) return rc;
    p_plan P;
    rc = parse_plan(plan_flat, &P);
    if (!rc) rc = check_plan_shape(&P, &pv, T);
    if (rc) {
        free(P.rounds);
        return rc;
    }
    /* GEMV inside a worker stays single-threaded, like the reference's Eigen GEMV */
    int saved_threads = g_threads;
    g_threads = 1;
    double t0 = now_s();
    int d = m->d, step = 0;
    double* x = dupv(x_T, d);
    if (traj_latents) memcpy(traj_latents, x_T, sizeof(double) * (size_t)d);
    bstore store = {NULL, 0};
    rc = warmup(&pv, &P, alpha_bars, x, &store, traj_latents, traj_eps, &step);
    pthread_t* th = (pthread_t*)calloc((size_t)P.D, sizeof(pthread_t));
    worker_arg* args = (worker_arg*)calloc((size_t)P.D, sizeof(worker_arg));
    for (int r = 0; r < P.n_rounds && !rc; ++r) {
        const p_round* R = &P.rounds[r];
        skipmap snap;
        memset(&snap, 0, sizeof snap);
        collect_skips(&store, &pv, &snap);
        round_ctx ctx = {&pv, &store, &snap, x, R->index};
        outcome* outs = (outcome*)calloc((size_t)R->n_evals, sizeof(outcome));
        for (int dv = 0; dv < P.D; ++dv) {
            args[dv].R = R;
            args[dv].ctx = &ctx;
            args[dv].device = dv;
            args[dv].out = outs;
            pthread_create(&th[dv], NULL, worker_main, &args[dv]);
        }
        for (int dv = 0; dv < P.D; ++dv) pthread_join(th[dv], NULL);
        for (int dv = 0; dv < P.D && !rc; ++dv)
            if (args[dv].rc) rc = fail(OR_RUNTIME, "run_parallel: device %d failed: %s", dv, args[dv].err);
        skipmap_clear(&snap, m->n_links);
        if (!rc)
            rc = finish_round(&pv, &P, R, outs, R->n_evals, alpha_bars, x, &store, traj_latents,
                              traj_eps, &step);
        free(outs);
    }
    if (wall_s) *wall_s = now_s() - t0;
    g_threads = saved_threads;
    free(th);
    free(args);
    store_free(&store, m);
    free(x);
    free(P.rounds);
    return rc;
}

/* proj/src/diffusion.cpp:118-142 */
int or_sequential_denoise(const or_model* m, const double* alpha_bars, int T, const double* x_T,
                          double* traj_latents, double* traj_eps) {
    int d = m->d;
    double* x = dupv(x_T, d);
    double* eps = (double*)malloc(sizeof(double) * (size_t)d);
    if (traj_latents) memcpy(traj_latents, x_T, sizeof(double) * (size_t)d);
    int rc = OR_OK;
    for (int t = T, step = 0; t >= 1; --t, ++step) {
        rc = or_eval_full(m, x, t, eps);
        if (rc) {
            char inner[1024];
            snprintf(inner, sizeof inner, "%s", g_err);
            rc = fail(OR_RUNTIME, "sequential_denoise: eps_fn failed at t=%d: %s", t, inner);
            break;
        }
        rc = or_ddim_step(x, eps, d, t, alpha_bars, T, x);
        if (rc) break;
        if (traj_eps) memcpy(traj_eps + (size_t)step * d, eps, sizeof(double) * (size_t)d);
        if (traj_latents) memcpy(traj_latents + (size_t)(step + 1) * d, x, sizeof(double) * (size_t)d);
    }
    free(x);
    free(eps);
    return rc;
}

/* proj/src/metrics.cpp:9-30 */
int or_compare_trajectories(const double* a, const double* b, int n, int d, double* per_step_mse,
                            double* final_mse, double* final_max_abs) {
    double last = 0.0;
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            double df = a[(size_t)i * d + k] - b[(size_t)i * d + k];
            s += df * df;
        }
        last = s / (double)d;
        if (per_step_mse) per_step_mse[i] = last;
    }
    if (final_mse) *final_mse = last;
    double mx = 0.0;
    for (int k = 0; k < d; ++k) {
        double df = fabs(a[(size_t)(n - 1) * d + k] - b[(size_t)(n - 1) * d + k]);
        if (df > mx) mx = df;
    }
    if (final_max_abs) *final_max_abs = mx;
    return OR_OK;
}
