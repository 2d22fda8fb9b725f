/*
 * adx_oracle.h -- CPU fp64 restatement of the AsyncDiff reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2406_06911_b200/ links or
 * calls this library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it, and only as the checker or
 * as the timed CPU baseline.
 *
 * Route B of SURVEY.md §8c: the reference (/root/reference/proj) cannot be
 * compiled here -- it needs Eigen3 (proj/CMakeLists.txt:12), a vendor/ tree
 * with doctest/json/CLI11 that is absent (proj/CMakeLists.txt:10) and a
 * missing tests/acceptance.cpp (proj/tests/CMakeLists.txt:22) -- so this is a
 * clean-room restatement of its published algorithm in plain C.  Each
 * function cites the reference file:line it follows.  Parity is PINNED by the
 * reference's own golden vectors: see
 * tests/test_oracle_golden.py.
 *
 * Third-party arithmetic: the reference's GEMV is Eigen's (unpinned >= 3.3);
 * Eigen's summation order is internal, so this oracle (left-to-right sums) is
 * not bit-identical to an Eigen build.  The reference's goldens carry a
 * relative tolerance of 1e-9, which covers that.
 */
#ifndef ADX_ORACLE_H
#define ADX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's exception classes */
enum {
    OR_OK = 0,
    OR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    OR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    OR_DOMAIN = 3,           /* std::domain_error */
    OR_RUNTIME = 4,          /* std::runtime_error */
    OR_LOGIC = 5             /* std::logic_error */
};

const char* or_last_error(void);
void or_set_threads(int n); /* row-parallel GEMV (OpenMP) for test speed; 1 = scalar */

/* ---- RNG: proj/include/asyncdiff/rng.hpp:12-60 ---- */
typedef struct {
    uint64_t mt[312];
    int mti;
    double spare;
    int have_spare;
} or_rng;

void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_uniform(or_rng* r);
double or_rng_normal(or_rng* r);
uint64_t or_rng_below(or_rng* r, uint64_t n);
uint64_t or_mix_seed(uint64_t a, uint64_t b);
/* convenience: n normals from Rng(seed) (test_util.hpp random_vec) */
void or_random_normals(uint64_t seed, int n, double* out);

/* bulk float32 draws for the UNet-family oracle (oracle/unet_model.py) */
long long or_rng_sizeof(void);
void or_rng_fill_uniform_f32(or_rng* r, long long n, double lo, double hi, float* out);
void or_rng_fill_normal_f32(or_rng* r, long long n, float* out);

/* ---- schedule + sampler: proj/src/diffusion.cpp:39-142 ---- */
enum { OR_LINEAR = 0, OR_SCALED_LINEAR = 1 };
int or_build_schedule(int T, double beta_start, double beta_end, int kind,
                      double* betas, double* alphas, double* alpha_bars);
int or_ddim_step(const double* x, const double* eps, int d, int t,
                 const double* alpha_bars, int T, double* out);
int or_forward_diffuse(const double* x0, const double* noise, int d, int t,
                       const double* alpha_bars, int T, double* out);

/* ---- denoiser: proj/src/denoiser.cpp:14-267 ---- */
typedef struct or_model or_model;
enum { OR_SKIP_NONE = 0, OR_SKIP_UNET_MIRROR = 1 };
/* tensor ids for or_model_tensor */
enum { OR_T_PROJ = 0, OR_T_W1 = 1, OR_T_B1 = 2, OR_T_TIN = 3, OR_T_W2 = 4, OR_T_B2 = 5 };

int or_model_build_toy(int L, const int* widths, int skip_spec, uint64_t seed, int E,
                       or_model** out);
int or_model_shell(int L, const int* widths, const int* links, int n_links, int E,
                   or_model** out);
void or_model_free(or_model* m);
int or_model_num_stages(const or_model* m);
int or_model_num_links(const or_model* m);
void or_model_links(const or_model* m, int* out_pairs);
long long or_model_stage_macs(const or_model* m, int stage);
void or_model_set_stage_macs(or_model* m, int stage, long long macs);
/* row-major view: element (i,j) at [i*cols+j]; stage ignored for PROJ */
double* or_model_tensor(or_model* m, int stage, int which, int* rows, int* cols);

int or_sinusoid(int t, int dim, double* out);
int or_eval_full(const or_model* m, const double* x, int t_embed, double* eps_out);
int or_stage_forward(const or_model* m, int stage, const double* u, int un, int t_embed, double* y_out);
void or_embed(const or_model* m, int t, double* out);

/* ---- partition: proj/src/partition.cpp:95-208 ---- */
enum { OR_SEQUENTIAL_BALANCED = 0, OR_FIRST_LAST_GROUPED = 1 };
/* stage_segment[s-1] = 1-based segment of stage s; seg_macs[N] */
int or_partition_balanced(const long long* costs, int L, int N, int strategy,
                          int* stage_segment, long long* seg_macs);

/* ---- plan: proj/src/plan.cpp:17-97 ----
 * flat layout (ints):
 *   [T, w, N, S, D, time_shift, n_rounds, warmup[w]...,
 *    per round: index, broadcast, n_sampler, sampler[n_sampler]..., n_evals,
 *               per eval: segment, device, embed_t, input_kind(0=latent,1=cached),
 *                         producer_segment, producer_round, emits_eps_for(-1=none)]
 */
int or_plan_async_flat(int T, int w, int N, int S, int time_shift, int* out, int cap,
                       int* out_len);

/* ---- executor: proj/src/executor.cpp:28-331 (serial), 338-601 (parallel) ----
 * partition given as stage_segment (contiguous cascade required).
 * traj_latents: (T+1)*d, traj_eps: T*d (either may be NULL).
 * store_entries: n_rounds ints (may be NULL).  Returns broadcast count via out. */
int or_run_serial(const or_model* m, const int* stage_segment, int N, const int* plan_flat,
                  const double* alpha_bars, int T, const double* x_T,
                  double* traj_latents, double* traj_eps, int* store_entries,
                  int* broadcast_count);
/* D worker threads (pthreads), barrier + sorted commit per round; bit-identical
 * to or_run_serial.  wall_s (may be NULL) = x_T -> x_0 wall time. */
int or_run_parallel(const or_model* m, const int* stage_segment, int N, const int* plan_flat,
                    const double* alpha_bars, int T, const double* x_T,
                    double* traj_latents, double* traj_eps, double* wall_s);
/* sequential_denoise(eval_full): proj/src/diffusion.cpp:118-142 */
int or_sequential_denoise(const or_model* m, const double* alpha_bars, int T,
                          const double* x_T, double* traj_latents, double* traj_eps);

/* compare_trajectories: proj/src/metrics.cpp:9-30 */
int or_compare_trajectories(const double* a, const double* b, int steps_plus_one, int d,
                            double* per_step_mse, double* final_mse, double* final_max_abs);

#ifdef __cplusplus
}
#endif
#endif
