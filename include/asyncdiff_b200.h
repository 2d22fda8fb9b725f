/*
 * asyncdiff_b200.h -- C ABI of the B200-native AsyncDiff async denoising
 * engine (libasyncdiff_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ pipeline API
 * (the headers under /root/reference/proj/include/asyncdiff/).  Every entry point cites
 * the reference declaration it replaces.  Plain pointers and sizes only; no
 * torch or CUDA types cross this boundary.  Errors: every function returns an
 * adx_status; the message of the last failure on the calling thread is
 * adx_last_error().  Status codes map 1:1 onto the reference's exception
 * classes (std::invalid_argument, out_of_range, domain_error, runtime_error,
 * logic_error) so a C++ facade can rethrow the same type with the same text
 * (see include/asyncdiff_b200.hpp).
 *
 * Matrices crossing the boundary are row-major fp64 (element (i,j) at
 * [i*cols + j]); latents/eps are fp64 vectors, like the reference's
 * Eigen::VectorXd (proj/include/asyncdiff/diffusion.hpp:10-11).
 */
#ifndef ASYNCDIFF_B200_H
#define ASYNCDIFF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef enum {
    ADX_OK = 0,
    ADX_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    ADX_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range    */
    ADX_ERR_DOMAIN = 3,           /* std::domain_error    */
    ADX_ERR_RUNTIME = 4,          /* std::runtime_error   */
    ADX_ERR_LOGIC = 5,            /* std::logic_error     */
    ADX_ERR_CUDA = 6              /* CUDA / NCCL failure (runtime_error class) */
} adx_status;

const char* adx_last_error(void);
int adx_version(void);          /* 100 * major + minor */
int adx_device_count(void);     /* visible CUDA devices (0 without a GPU) */

/* precision of the device arithmetic */
typedef enum {
    ADX_F64 = 0,  /* fp64 weights + activations: golden parity mode            */
    ADX_F32 = 1,  /* fp32 weights + activations: north_star rel-L2 <= 1e-3 mode */
    ADX_BF16 = 2  /* bf16 weights, fp32 activations/accumulation                */
} adx_precision;

/* -------------------------------------------------------------- schedule
 * build_schedule: proj/include/asyncdiff/diffusion.hpp:36-37,
 *                 proj/src/diffusion.cpp:39-77.  kind 0=linear 1=scaled-linear.
 * betas/alphas: T doubles, alpha_bars: T+1 doubles (caller-owned). */
/* n standard normals from Rng(seed) (mt19937_64 + the reference's normal(), rng.hpp; the
 * draw of x_T in draw_x_T, experiment.cpp:131-136, with the seed already mixed) */
int adx_random_normals(uint64_t seed, long long n, double* out);
int adx_build_schedule(int T, double beta_start, double beta_end, int kind, double* betas,
                       double* alphas, double* alpha_bars);

/* ddim_step on the GPU (device `ordinal`): proj/include/asyncdiff/diffusion.hpp:50-51,
 * proj/src/diffusion.cpp:95-116.  alpha_bars has T+1 entries.  Non-finite eps ->
 * ADX_ERR_DOMAIN "predict_x0: non-finite eps at t=..", t outside [1,T] ->
 * ADX_ERR_OUT_OF_RANGE. */
int adx_ddim_step(int ordinal, int precision, const double* x, const double* eps, int d, int t,
                  const double* alpha_bars, int T, double* out);

/* ------------------------------------------------------------------ model
 * LayeredDenoiser: proj/include/asyncdiff/denoiser.hpp:29-72. */
typedef struct adx_model adx_model;
enum { ADX_SKIP_NONE = 0, ADX_SKIP_UNET_MIRROR = 1 };
enum { ADX_T_PROJ = 0, ADX_T_W1 = 1, ADX_T_B1 = 2, ADX_T_TIN = 3, ADX_T_W2 = 4, ADX_T_B2 = 5 };

/* build_toy_denoiser: denoiser.hpp:68-70, denoiser.cpp:124-142 (xavier init from Rng(seed)).
 * widths has n_widths entries (must be L+1). */
int adx_model_build_toy(int L, const int* widths, int n_widths, int skip_spec, uint64_t seed,
                        int time_embed_dim, adx_model** out);
/* make_denoiser_shell: denoiser.hpp:73-76, denoiser.cpp:75-122 (zero weights). */
int adx_model_shell(int L, const int* widths, int n_widths, const int* link_pairs, int n_links,
                    int time_embed_dim, adx_model** out);
void adx_model_destroy(adx_model* m);
int adx_model_info(const adx_model* m, int* L, int* time_embed_dim, int* n_links);
int adx_model_widths(const adx_model* m, int* out /* L+1 */);
int adx_model_links(const adx_model* m, int* out_pairs /* 2*n_links */);
/* Stage::in_width/hidden_width/out_width/cost_macs (denoiser.hpp:29-43) */
int adx_model_stage_shape(const adx_model* m, int stage, int* in, int* hidden, int* out,
                          long long* cost_macs);
int adx_model_set_stage_macs(adx_model* m, int stage, long long cost_macs);
/* host fp64 row-major tensor, mutable in place (stage ignored for PROJ).
 * Engines created afterwards see the edits. */
int adx_model_tensor(adx_model* m, int stage, int which, double** data, int* rows, int* cols);
/* TimeEmbedding::sinusoid (denoiser.cpp:31-41) */
int adx_sinusoid(int t, int dim, double* out);

/* -------------------------------------------------------------- partition
 * Partition: proj/include/asyncdiff/partition.hpp:19-44. */
typedef struct adx_partition adx_partition;
enum { ADX_SEQUENTIAL_BALANCED = 0, ADX_FIRST_LAST_GROUPED = 1 };

/* partition_balanced: partition.hpp:39-40, partition.cpp:95-198 */
int adx_partition_balanced(const adx_model* m, int N, int strategy, adx_partition** out);
/* extension: the same min-max DP (partition.cpp:95-125 semantics, ties to the smallest
 * cut) over measured per-stage costs (e.g. adx_engine_stage_times, in any unit) */
int adx_partition_by_cost(const adx_model* m, int N, const double* stage_cost, adx_partition** out);
/* explicit partition (tests' uniform_partition, plan_test.cpp:14-22):
 * seg_sizes[n_segments], stages[sum(seg_sizes)] 1-based, devices/macs per segment */
int adx_partition_create(int n_segments, const int* seg_sizes, const int* stages,
                         const int* devices, const long long* macs, int strategy,
                         adx_partition** out);
void adx_partition_destroy(adx_partition* p);
int adx_partition_num_segments(const adx_partition* p);
int adx_partition_strategy(const adx_partition* p);
int adx_partition_segment(const adx_partition* p, int seg, int* stages, int cap, int* n_stages,
                          long long* macs, int* device);
int adx_partition_contiguous(const adx_partition* p);                       /* partition.hpp:29 */
int adx_partition_segment_of_stage(const adx_partition* p, int stage, int* seg); /* :27 */
int adx_partition_validate(const adx_partition* p, const adx_model* m);     /* :33 */
/* crossing_links: partition.hpp:43-44, partition.cpp:200-208 */
int adx_crossing_links(const adx_model* m, const adx_partition* p, int* out_pairs, int cap,
                       int* n_links);

/* ------------------------------------------------------------------- plan
 * ExecutionPlan: proj/include/asyncdiff/plan.hpp:12-53.
 * Flat layout (ints), shared with the oracle:
 *   [T, w, N, S, D, time_shift, n_rounds, warmup[w]...,
 *    per round: index, broadcast, n_sampler, sampler[n_sampler]..., n_evals,
 *               per eval: segment, device, embed_t, input_kind (0 latent, 1 cached),
 *                         producer_segment, producer_round, emits_eps_for (-1 none)] */
typedef struct adx_plan adx_plan;
/* plan_async: plan.hpp:53, plan.cpp:17-97 */
int adx_plan_async(int T, int w, int N, int S, int time_shift, adx_plan** out);
int adx_plan_from_flat(const int* flat, int len, adx_plan** out);
int adx_plan_to_flat(const adx_plan* p, int* out, int cap, int* len);
void adx_plan_destroy(adx_plan* p);
/* validate_plan: plan.hpp:56, plan.cpp:99-200.  Violations joined by '\n'. */
int adx_plan_validate(const adx_plan* p, char* buf, int cap, int* n_violations);

/* PlanCounts: plan.hpp:58-66; plan_counts: plan.cpp:202-232 */
typedef struct {
    int broadcasts_paper_convention;
    int broadcasts_strictly_needed;
    int device_count;
    long long max_device_macs;
    long long sequential_total_macs;
} adx_plan_counts_t;
int adx_plan_counts(const adx_plan* p, const adx_partition* part, adx_plan_counts_t* out,
                    long long* evals_per_segment /* N or NULL */,
                    long long* per_device_macs /* D or NULL */);
/* shift_embeddings: plan.hpp:69, plan.cpp:234-244 */
int adx_shift_embeddings(const int* timesteps, int n, int w, int* out);
/* render_plan: plan.hpp:72, plan.cpp:246-286 */
int adx_render_plan(const adx_plan* p, char* buf, int cap, int* len);

/* ----------------------------------------------------------------- engine
 * Device-resident denoiser: weights uploaded once per CUDA device, lazily,
 * in the engine's precision.  `ordinals` lists the CUDA devices virtual
 * device v maps to (v % n_ordinals): several virtual devices may share one
 * GPU (they then run on separate streams of that GPU). */
typedef struct adx_engine adx_engine;
int adx_engine_create(const adx_model* m, int precision, const int* ordinals, int n_ordinals,
                      adx_engine** out);
void adx_engine_destroy(adx_engine* e);
/* bytes of weights resident per ordinal (for the roofline) */
int adx_engine_weight_bytes(const adx_engine* e, int ordinal_index, long long* bytes);

/* Mean device time of one full-model pass (the 2L stage GEMV launches, one CUDA
 * graph, CUDA events on its stream) over `iters` back-to-back passes, plus the
 * algorithmic weight bytes one pass streams: the HBM roofline of the GEMV. */
int adx_engine_time_eval(adx_engine* e, int t_embed, int iters, double* ms_per_pass,
                         long long* bytes_per_pass, int* launches_per_pass);
/* device ms of every stage evaluated on its own (each stage captured into its own
 * CUDA graph and replayed): stage_ms[L], the measured per-component costs that feed
 * the cost model (costsim.hpp:13-19 segment_cost_s) */
int adx_engine_stage_times(adx_engine* e, int t_embed, int iters, double* stage_ms);

/* Microbenchmark of the stage GEMV kernel: a dependent chain of `chain` square
 * n x n GEMVs (distinct weights), one CUDA graph, `iters` launches; device ms
 * per GEMV.  pdl=1 enables programmatic dependent launch between them. */
int adx_bench_gemv(int ordinal, int precision, int n, int chain, int iters, int pdl,
                   double* ms_per_gemv);

/* One eager full-model pass with CUDA events around every tensor-core launch:
 * out9 = {launches, ms, algorithmic FLOPs} for conv3x3, GEMM, attention. */
int adx_engine_profile_pass(adx_engine* e, int t_embed, double* out9);
/* the per-launch records of the last adx_engine_profile_pass: 4 doubles per launch
 * (kind 0 conv3x3 / 1 GEMM / 2 attention / 3 GroupNorm / 4 LayerNorm, algorithmic FLOPs,
 * compulsory HBM bytes, device ms); *n = the record count (at most `cap` are written) */
int adx_profile_records(double* out, int cap, int* n);

/* eval_full: denoiser.hpp:79, denoiser.cpp:222-233 (on ordinals[0]) */
int adx_eval_full(adx_engine* e, const double* x, int t_embed, double* eps_out);

/* eval_segment: denoiser.hpp:91-95, denoiser.cpp:235-267.
 * input_is_latent=1: `input` is the latent x (d values), produced_by ignored.
 * input_is_latent=0: `input` is a HiddenBundle boundary from segment produced_by.
 * skips_in: n_skips links (pairs) with their features concatenated in
 * skip_vals (each feature has width widths[producer]).
 * Output: if seg == N, eps in out (d values), *out_is_eps=1.  Otherwise the
 * bundle boundary in out and the crossing links produced by the segment in
 * out_links/out_vals (caller capacity cap_links / cap_vals). */
int adx_eval_segment(adx_engine* e, const adx_partition* p, int seg, const double* input,
                     int input_len, int input_is_latent, int produced_by, const int* skip_links,
                     const double* skip_vals, int n_skips, int t_embed, double* out, int out_cap,
                     int* out_len, int* out_is_eps, int* out_links, double* out_vals,
                     int cap_links, int cap_vals, int* n_out_links);

/* RunOptions: executor.hpp:44-49 (+ InstrumentedDenoiser delays, executor.hpp:53-59) */
typedef struct {
    double round_timeout_s;        /* default 30 */
    uint64_t jitter_seed;          /* executor.cpp:445-449: device d's stream starts with a GPU */
    double max_jitter_s;           /* sleep of Rng(mix_seed(jitter_seed, d)).uniform() * max_jitter_s */
    const double* segment_delay_s; /* NULL or n_delays (must equal N) per-segment GPU sleeps */
    int n_delays;
    int use_graph;                 /* 1: capture the whole run in one CUDA graph (default) */
    int instrument;                /* 1: per-round / per-eval CUDA-event timing into RunStats */
} adx_run_options;
void adx_run_options_default(adx_run_options* o);

/* RunStats: executor.hpp:30-42.  Arrays are caller-provided (may be NULL):
 * round_wall_s/round_comm_s/store_entries_per_round: n_rounds entries;
 * device_busy_s/device_evals: D entries. */
typedef struct {
    int broadcast_count;
    int n_rounds;
    double warmup_wall_s;
    double total_wall_s;
    double* round_wall_s;
    double* round_comm_s;
    double* device_busy_s;
    long long* device_evals;
    int* store_entries_per_round;
} adx_run_stats;

/* A session is one compiled run: (plan, partition, placement) with its
 * device buffers, streams and (optionally) one CUDA graph spanning every
 * device.  mode: 0 = run_serial (all evals on virtual device 0, plan order),
 * 1 = run_parallel (virtual device v = plan device v), 2 = sequential_denoise
 * (T full-model evals, plan/partition ignored except for T).  workers must
 * equal plan.D in mode 1 (executor.cpp:509-511). */
enum { ADX_MODE_SERIAL = 0, ADX_MODE_PARALLEL = 1, ADX_MODE_SEQUENTIAL = 2 };
typedef struct adx_session adx_session;
int adx_session_create(adx_engine* e, const adx_plan* plan, const adx_partition* part,
                       const double* alpha_bars, int T, int mode, int workers,
                       const adx_run_options* opts, adx_session** out);
void adx_session_destroy(adx_session* s);
/* Host in / host out, blocking: x_T (d) -> latents ((T+1)*d), eps (T*d).
 * Either output may be NULL. */
int adx_session_run(adx_session* s, const double* x_T, double* traj_latents, double* traj_eps,
                    adx_run_stats* stats);
/* Device-resident timing path: x_T already uploaded by adx_session_upload;
 * runs `iters` times back to back and returns the mean device time per run
 * (CUDA events on the session's launch stream). */
int adx_session_upload(adx_session* s, const double* x_T);
int adx_session_time(adx_session* s, int iters, double* ms_per_run);
/* kernels launched per run (the graph's kernel nodes) */
int adx_session_kernel_count(const adx_session* s, int* n);
/* algorithmic weight bytes streamed per run (every eval streams its segment's
 * W1/W2 once) -- the numerator of the HBM roofline */
int adx_session_weight_bytes(const adx_session* s, long long* bytes);
/* trajectory of the last run (device -> host, fp64) */
int adx_session_download(adx_session* s, double* traj_latents, double* traj_eps);

/* One-shot wrappers mirroring the reference signatures (session create/run/destroy). */
/* run_serial: executor.hpp:63-75, executor.cpp:248-331 */
int adx_run_serial(adx_engine* e, const adx_plan* plan, const adx_partition* part,
                   const double* x_T, const double* alpha_bars, int T,
                   const adx_run_options* opts, double* traj_latents, double* traj_eps,
                   adx_run_stats* stats);
/* run_parallel: executor.hpp:79-93, executor.cpp:501-601 */
int adx_run_parallel(adx_engine* e, const adx_plan* plan, const adx_partition* part,
                     const double* x_T, const double* alpha_bars, int T, int workers,
                     const adx_run_options* opts, double* traj_latents, double* traj_eps,
                     adx_run_stats* stats);
/* sequential_denoise(eval_full): diffusion.hpp:66-67, diffusion.cpp:118-142 */
int adx_sequential_denoise(adx_engine* e, const double* x_T, const double* alpha_bars, int T,
                           double* traj_latents, double* traj_eps);

/* ------------------------------------------------- one process per GPU
 * The same async loop with rank v of a torchrun job evaluating the plan's
 * device-v evals on its own GPU (run_parallel's worker d, executor.cpp:444-496)
 * and exchanging stage outputs / eps over NCCL p2p, one NCCL group per
 * exchange point.  adx_rank_program exports the rank's op list (12 ints per
 * op: kind, seg, t, wslot, rslot, step, eps_step, point, peer, stage, slot,
 * elems; kinds 0 eval, 1 group, 2 send, 3 recv, 4 end, 5 ddim) -- the CPU
 * gloo test replays it with the oracle to check the exchange schedule. */
typedef struct adx_rank_session adx_rank_session;
int adx_rank_program(const adx_plan* plan, const adx_partition* part, const adx_model* m, int rank,
                     int* out, int cap, int* n_ops);
int adx_nccl_unique_id(char* out128);
/* collective over ranks 0..plan.D-1 (same nccl_id); engine = this rank's GPU */
int adx_rank_session_create(adx_engine* e, const adx_plan* plan, const adx_partition* part,
                            const double* alpha_bars, int T, int rank, const char* nccl_id,
                            const adx_run_options* opts, adx_rank_session** out);
void adx_rank_session_destroy(adx_rank_session* s);
/* collective; x_T / outputs are used on rank 0 only */
int adx_rank_session_run(adx_rank_session* s, const double* x_T, double* traj_latents,
                         double* traj_eps);
int adx_rank_session_time(adx_rank_session* s, int iters, double* ms_per_run);
int adx_rank_session_kernel_count(const adx_rank_session* s, int* n);

/* ------------------------------------------------------ UNet-shaped family
 * A LayeredDenoiser whose stages are UNet blocks (conv_in, resnet[+spatial
 * transformer], stride-2 down, nearest-2x up, mid, out) with the reference's
 * mirror skip links as channel-concat skips.  The returned
 * adx_model works with every partition / plan / engine / run entry point above
 * (engine precision ADX_F32: bf16 tensor-core stages, fp32 latent and eps). */
typedef struct {
    int H, W, c_lat;
    int n_levels;
    int ch[8];
    int attn[8];          /* SpatialTransformer depth per level (0: none; SD-2.1 1, SDXL 0/2/10) */
    int n_res, head_dim, ctx_len, ctx_dim, temb_dim, groups, mid_attn;
    uint64_t seed;
    int cfg;              /* classifier-free guidance: batch-2 stages, eps_u + scale (eps_c - eps_u) */
    float cfg_scale;
    int frames;           /* video: frames per sample (latent / eps = frames x H x W x c_lat); >= 1 */
    int motion;           /* temporal-attention motion module after every resnet (frames >= 2) */
} adx_unet_spec;
int adx_model_build_unet(const adx_unet_spec* spec, adx_model** out);
/* kind (0 conv_in, 1 res, 2 down, 3 up, 4 out, 5 mid res), cin, cskip, cout, H, W, attn */
int adx_unet_stage_info(const adx_model* m, int stage, int* info7);
/* stage parameters (stage 0 = shared time-embedding MLP) for the builder-written oracle */
int adx_unet_stage_params(const adx_model* m, int stage, char* names, int names_cap, int* shapes,
                          int* n_params, float* data, long long data_cap, long long* n_data);
int adx_unet_context(const adx_model* m, float* out /* batch x ctx_len x ctx_dim; CFG: [uncond, cond] */);

/* --------------------------------- tcgen05 kernels of the UNet-shaped family
 * (no reference function: builder-written oracle, SURVEY §8a extension list).
 * A/B/X/Wt are bf16 bit patterns (uint16), outputs fp32.  iters > 0 also times
 * `iters` back-to-back launches (CUDA events). */
/* C[M x N] = act(A[M x K] . B[N x K]^T + bias); K % 64 == 0; bn in {0,32,64,80,96,128,160,192,256};
 * act 0 none, 1 SiLU, 2 GEGLU over 256-row tiles of [128 hidden | 128 gate] rows (C is M x N/2) */
int adx_tc_gemm(int ordinal, int M, int N, int K, const uint16_t* A, const uint16_t* B,
                const float* bias, int act, float* C, int bn, int iters, double* ms_per_iter);
/* stride-2 conv3x3 (pad 1), NHWC bf16: out [batch][H/2][W/2][Cout] from X [batch][H][W][Cin] (H, W
 * even); the A boxes are read with TMA element strides of 2 (no discarded output rows) */
int adx_tc_conv3x3_s2_bf16(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X,
                           const uint16_t* Wt, const float* bias, uint16_t* out, int bn, int splits, int iters,
                           double* ms_per_iter);
/* C [M x N] bf16 = [A1 | A2] . B^T + bias with A1 [M x K1], A2 [M x K2] read in place (the
 * UNet skip concatenation; K1, K2 multiples of 64); bn / splits force the tile plan */
int adx_tc_gemm_cat_bf16(int ordinal, int M, int N, int K1, int K2, const uint16_t* A1, const uint16_t* A2,
                         const uint16_t* B, const float* bias, uint16_t* out, int bn, int splits);
/* the bf16 mode's LayerNorm-folded GEMM (kernel test): y = rstd_m (H . W1'^T - mean_m colsum1) +
 * bias1 with the row statistics of H [M x C] (bf16) reduced inside the GEMM, W1' [N x C] =
 * W1 diag(gamma) and bias1 = b + W1 beta folded by the caller (geglu: N = 2H rows tile-
 * interleaved, y [M x H]); bn forces the N tile (0: the launcher's plan) */
int adx_tc_ln_fold_supported(void);
/* the fused GEGLU epilogue's weight-row group G: N tile t = hidden rows [G t, G t + G), then their
 * gate rows H + the same (callers of adx_tc_gemm with act 2 interleave W and bias this way) */
int adx_tc_geglu_group(void);
/* per-CTA %globaltimer stamps (16 per CTA) of the last stream-K attention launch; zeros unless
 * built with -DADX_SK_TIMELINE (diagnostics) */
int adx_sk_timeline(unsigned long long* out, int n_ctas); /* 1 when built with -DADX_TC_STATW=2 (else the fold is rejected) */
int adx_tc_ln_fold_bf16(int ordinal, int M, int C, int N, const uint16_t* H, const uint16_t* W1, const float* bias1,
                        const float* colsum1, int geglu, float eps, uint16_t* y_out, int bn, int iters,
                        double* ms_per_iter);
/* fused multi-head attention (64-wide heads, scale 1/8): out[L x C] bf16 from Q [L x C],
 * K [Lk x C] and V [Lk x ldv] (row-major, ldv >= C, multiple of 8) */
int adx_tc_attention(int ordinal, int L, int Lk, int C, const uint16_t* Q, const uint16_t* K,
                     const uint16_t* V, int ldv, uint16_t* out, int iters, double* ms_per_iter);
/* the ADX_F32 mode's fused attention: fp32 Q [batch][L][C], K and V [batch][Lk][C] split on
 * the device into bf16 hi / lo planes, S and O as three split products each on the tensor
 * cores (fp32 accumulation), fp32 softmax; out [batch][L][C] fp32 */
int adx_tc_attention_f32(int ordinal, int batch, int L, int Lk, int C, const float* Q, const float* K,
                         const float* V, float* out, int iters, double* ms_per_iter);
/* video motion-module temporal attention: for every (pixel, 64-wide head) the frames
 * attend to each other; qkv frame-major [frames][HW][3C] bf16 (q | k | v), out
 * [frames][HW][C] bf16; 2 <= frames <= 32 */
int adx_temporal_attention(int ordinal, int frames, int HW, int C, const uint16_t* qkv, uint16_t* out, int iters,
                           double* ms_per_iter);
/* conv3x3 / stride 1 / pad 1, NHWC: X [batch][H][W][Cin], Wt [Cout][9*Cin] ((r*3+s)*Cin+ci) */
int adx_tc_conv3x3(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X,
                   const uint16_t* Wt, const float* bias, float* out, int iters, double* ms_per_iter);
/* tile-plan override for tuning (tools_tc_tune.py): every following GEMM / conv
 * launch in this process uses N tile `bn` and split-K factor `splits` (0, 0:
 * back to the measured plan table, then the model) */
int adx_tc_plan_override(int bn, int splits);
/* bf16-output epilogue (the UNet pass's: TMA-store staging, bf16 residual with row stride ldr,
 * output row stride ldo >= N, columns past N untouched); bn / splits force a tile plan */
int adx_tc_gemm_bf16(int ordinal, int M, int N, int K, const uint16_t* A, const uint16_t* B, const float* bias,
                     const uint16_t* residual, int ldr, uint16_t* out, int ldo, int bn, int splits, int iters,
                     double* ms_per_iter);
int adx_tc_conv3x3_bf16(int ordinal, int batch, int H, int W, int Cin, int Cout, const uint16_t* X,
                        const uint16_t* Wt, const float* bias, const uint16_t* residual, uint16_t* out, int bn,
                        int splits, int iters, double* ms_per_iter);
/* GroupNorm(+SiLU) of bf16 NHWC images over a channel concat [x0 (c0) | x1 (c1)] (x1 NULL when
 * c1 == 0): the UNet pass's norm kernels (cooperative one-launch path for one image, stats +
 * apply for batches); iters > 0 also times it (graph of `iters` launches) */
int adx_group_norm_bf16(int ordinal, int batch, int HW, int c0, int c1, int groups, const uint16_t* x0,
                        const uint16_t* x1, const float* gamma, const float* beta, float eps, int act,
                        uint16_t* out, int iters, double* ms_per_iter);
int adx_gn_timeline(unsigned long long* out, int n);
/* per-CTA %globaltimer stamps (8 per CTA) of the last tc_gemm / conv launch: diagnostics of
 * -DADX_TC_TIMELINE builds (tools/tools_tc_timeline.py); zeros in the product build */
int adx_tc_timeline(unsigned long long* out, int n_ctas);

/* ------------------------------------------------------ §8(f) next rows */
/* save_checkpoint / load_checkpoint: proj/include/asyncdiff/serialize.hpp:35-36,
 * serialize.cpp:226-308 (<base>.json metadata + <base>.bin row-major LE fp64) */
int adx_model_save_checkpoint(const adx_model* m, const char* base);
int adx_model_load_checkpoint(const char* base, adx_model** out);
/* plan_to_json / plan_from_json: serialize.hpp:29-30, serialize.cpp:109-159 */
int adx_plan_to_json(const adx_plan* p, char* buf, int cap, int* len);
int adx_plan_from_json(const char* text, adx_plan** out);

/* LatencyReport / CostComparison: costsim.hpp:13-50 */
typedef struct {
    double sequential_total_s, async_total_s, warmup_s, comm_total_s, speedup, comm_ratio,
        approx_step_s, approx_total_s;
} adx_latency_report;
typedef struct {
    double predicted_total_s, measured_total_s, rel_error_total, predicted_comm_ratio,
        measured_comm_ratio, rel_error_comm_ratio, calibrated_comm_cost_s;
} adx_cost_comparison;
/* predict_async: costsim.cpp:18-50.  round_bytes == NULL: flat comm_cost_s per
 * broadcasting round (reference); else bytes-aware comm = comm_latency_s +
 * round_bytes[r] / (link_gbs GB/s) (the NVLink cost model). */
int adx_predict_async(const adx_plan* p, const double* seg_cost, int n_seg, double comm_cost_s,
                      double sampler_cost_s, double comm_latency_s, double link_gbs,
                      const long long* round_bytes, adx_latency_report* out,
                      double* round_compute_s, double* round_comm_s);
/* calibrate_and_compare: costsim.cpp:52-79 */
int adx_calibrate_and_compare(const adx_plan* p, const double* delays, int n,
                              const double* measured_round_comm_s, int n_rounds,
                              int broadcast_count, double measured_total_s,
                              adx_cost_comparison* out);
/* bytes crossing devices per round in the one-process-per-GPU program */
int adx_round_exchange_bytes(const adx_plan* p, const adx_partition* part, const adx_model* m,
                             int precision, long long* out /* n_rounds */);

/* compare_trajectories: metrics.hpp, metrics.cpp:9-30 (host arithmetic) */
int adx_compare_trajectories(const double* a, const double* b, int n_latents, int d,
                             double* per_step_mse, double* final_mse, double* final_max_abs);

#ifdef __cplusplus
}
#endif
#endif /* ASYNCDIFF_B200_H */
