// tc_gemm.cuh -- tcgen05 GEMM / implicit-GEMM conv3x3 (see tc_gemm.cu).
#pragma once

#include "host.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <functional>

namespace adx {

// fused epilogue: out = scale * (act(acc + bias[n] + chan_add[img][n]) + residual[m][n])
struct TcArgs {
    // filled by the launcher
    int M = 0, N = 0, k_blocks = 0;
    int H = 0, W = 0, box_w = 0, box_h = 0, cin = 0;
    int m_tiles = 0, n_tiles = 0, batch = 1;  // output tile grid (per image) and images
    // epilogue
    const float* bias = nullptr;          // [N]
    const float* chan_add = nullptr;      // [images][N] (e.g. time-embedding projection)
    int chan_add_shared = 0;              // 1: every image uses row 0 (CFG batch at one timestep)
    int chan_add_rows = 0;                // > 0: output row m uses chan_add row m / chan_add_rows
                                          //   (video: a per-frame add over frame-major GEMM rows)
    const __nv_bfloat16* residual = nullptr;
    const float* residual_f32 = nullptr;  // fp32 residual (ADX_F32 mode); at most one of the two
    long long ldr = 0;
    int act = 0;                          // 0 none, 1 SiLU (applied before the residual),
                                          // 2 GEGLU over tile-interleaved [hidden | gate] columns
                                          //   (GEMM only; output width N/2; see geglu_interleave_rows)
    float out_scale = 1.0f;
    __nv_bfloat16* out_bf16 = nullptr;    // exactly one of out_bf16 / out_f32
    float* out_f32 = nullptr;
    long long ldo = 0;
    int sub2 = 0;                         // conv: stride 2 (output H/2 x W/2; A read with TMA element strides)
    int n_store = 0;                      // store only the first n_store columns (0: all N)
    int splits = 1;                       // filled by the launcher: split-K factor (cluster size)
    int tma_store = 0;                    // filled by the launcher: bf16 output written per 32x16
                                          //   chunk from SMEM by the TMA (GEMM, S = 1, BN <= 192)
    int tma_res = 0;                      // filled by the launcher: the bf16 residual arrives by TMA in
                                          //   the TMA-store staging blocks (with tma_store)
    int k_split = 0;                      // filled by tc_gemm_cat: A = [A1 | A2] along K, A2 from column k_split
    int n_fast = 0;                       // filled by the launcher: persistent tile order n-fastest
                                          //   (A tiles reused while L2-hot when A is the big operand)
    // LayerNorm fold (GEMM, unsplit, K = the LayerNorm width): A is the RAW LayerNorm input h and
    // the weights carry the gain (W' = W diag(gamma)).  Two statistics warps read every A tile
    // from the SMEM ring as the MMAs consume it and reduce each row's sum and (shifted) sum of
    // squares -> (mean, rstd) per row; the epilogue computes rstd (acc - mean colsum(W')_n) +
    // bias'_n with bias' = bias + W beta (host-folded).  No producer involvement, no extra pass.
    const float* ln_colsum = nullptr;     // [N], indexed like bias; non-null enables the fold
    float ln_eps = 1e-5f;
};

// per-CTA %globaltimer stamps of the last launch (ADX_TC_TIMELINE builds; zeros otherwise)
void tc_timeline(unsigned long long* out, int n_ctas);
// force (bn, splits) for every following launch (tuning); (0, 0) restores the plan table / model
void tc_plan_override(int bn, int splits);
// ADX_TC_TRACE=1: print every launch's shape / plan (and, when profiling, its isolated time)
bool tc_trace();

// In-run kernel profiling (eager passes only): when enabled, every tensor-core launch is,
// after it completes, replayed in isolation from a small CUDA graph and timed with events;
// kind 0 conv3x3, 1 GEMM, 2 attention, with its algorithmic FLOPs; kinds 3 (GroupNorm) and 4
// (LayerNorm) with their algorithmic bytes are only traced (ADX_TC_TRACE=1).
void tc_profile_enable(bool on);
void tc_profile_measure(cudaStream_t st, int kind, double flops, const std::function<void(cudaStream_t)>& launch);
void tc_profile_measure(cudaStream_t st, int kind, double flops, double bytes,
                        const std::function<void(cudaStream_t)>& launch);
// the records of the last collected pass: (kind, flops, compulsory bytes, ms) x n; returns n
int tc_profile_records(double* out, int cap);
// per kind: {launches, total ms, total flops}; clears the records
void tc_profile_collect(double out[3][3]);

// D[M x N] = A[M x K] . B[N x K]^T (bf16 in, fp32 accumulate in TMEM); bn = 0 picks the tile width
// and the split-K factor jointly (tile_plan); small-M layers are split over K across a
// thread-block cluster and reduced deterministically over DSMEM
void tc_gemm(const void* A, const void* B, int M, int N, int K, TcArgs p, cudaStream_t st, int bn = 0);
// same with explicit row strides (elements; multiples of 8) -- e.g. one head's slice of a packed QKV
// C = [A1 | A2] . B^T with A1 [M x K1] and A2 [M x K2] (dense rows) read in place: the channel
// concatenation of a UNet skip never materialised (K1, K2 multiples of 64; no residual)
// whether this build has the LayerNorm-fold statistics warps (-DADX_TC_STATW=2)
bool tc_ln_fold_supported();
// the fused GEGLU epilogue's weight-row group: N tile t holds hidden rows [G t, G t + G) and then
// their gate rows H + the same (the host interleaves ff1's rows and bias this way)
int tc_geglu_group();
void tc_gemm_cat(const void* A1, int K1, const void* A2, int K2, const void* B, int M, int N, TcArgs p,
                 cudaStream_t st, int bn = 0);
void tc_gemm_strided(const void* A, long long lda, const void* B, long long ldb, int M, int N, int K, TcArgs p,
                     cudaStream_t st, int bn = 0);
// conv3x3 / stride 1 / pad 1 over NHWC bf16 X [batch][H][W][Cin], weights Wt [Cout][3*3*Cin]
void tc_conv3x3(const void* X, const void* Wt, int batch, int H, int W, int Cin, int Cout, TcArgs p,
                cudaStream_t st, int bn = 0);

}  // namespace adx
