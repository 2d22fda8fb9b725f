// unet_kernels.cuh -- bandwidth-bound UNet kernels (see unet_kernels.cu).
#pragma once

#include "host.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace adx {

// NHWC channel concat of up to two tensors (c1 = 0: single tensor); bf16 activations
// (ADX_BF16 mode) or fp32 activations (ADX_F32 mode)
template <typename T>
struct Cat2T {
    const T* p0 = nullptr;
    int c0 = 0;
    const T* p1 = nullptr;
    int c1 = 0;
};
using Cat2 = Cat2T<__nv_bfloat16>;
using Cat2F = Cat2T<float>;

void group_norm(const Cat2& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, __nv_bfloat16* out, float2* scratch, cudaStream_t st);
void group_norm(const Cat2F& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, float* out, float2* scratch, cudaStream_t st);
void layer_norm(const float* x, int tokens, int C, const float* gamma, const float* beta, float eps, float* out,
                cudaStream_t st);
// fp32 activations -> the split-bf16 operand of the ADX_F32 mode: every group of g
// consecutive columns becomes 3g bf16 columns, pattern 0 = [hi | hi | lo] (A side),
// pattern 1 = [hi | lo | hi] (B side), hi = bf16(x), lo = bf16(x - hi); then
// A'.B'^T = hi.hi + hi.lo + lo.hi (the lo.lo term is ~2^-16 relative)
void split3(const float* x, long long rows, int cols, long long ldx, int g, int pattern, __nv_bfloat16* out,
            cudaStream_t st);
// x (n contiguous fp32) -> hi = bf16(x), lo = bf16(x - hi), same layout (tc_attention_x planes)
void split2(const float* x, long long n, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t st);
// fp32 row softmax over the first `valid` columns written as the split-bf16 A operand
// [hi | hi | lo] (3 x padded per row; split3 pattern 0 with g = padded); S is not modified
void softmax_split_rows(const float* S, long long lds, int rows, int valid, int padded, __nv_bfloat16* out,
                        cudaStream_t st);
// fp32 row softmax over the first `valid` columns, in place, zeros in [valid, padded)
void softmax_rows_f32(float* S, long long lds, int rows, int valid, int padded, cudaStream_t st);
// VT[d][k] = V[k * ldv + d] (k < L; 0 for L <= k < Lpad), fp32, hd rows
void transpose_f32(const float* V, long long ldv, int L, int Lpad, int hd, float* VT, cudaStream_t st);
// video motion modules: self-attention across the frames of every (pixel, 64-wide head);
// qkv frame-major [frames][HW][3C] (q | k | v), out [frames][HW][C]; 2 <= frames <= 32
void temporal_attention(const __nv_bfloat16* qkv, int frames, int HW, int C, __nv_bfloat16* out, cudaStream_t st);
void temporal_attention(const float* qkv, int frames, int HW, int C, float* out, cudaStream_t st);
// classifier-free guidance: out[i] = e[i] + scale * (e[n + i] - e[i])  (e = [eps_u | eps_c])
void cfg_combine(const float* e, long long n, float scale, float* out, cudaStream_t st);
// latent (fp32 / fp64, HWC) -> fp32 NHWC with cpad channels
void pack_latent_f32(const void* x, bool f64, long long pixels, int c_lat, int cpad, float* out, cudaStream_t st);
// per-CTA %globaltimer stamps of the last gn_fused launch (ADX_GN_TIMELINE builds; zeros otherwise)
void gn_timeline(unsigned long long* out, int n);
// scratch for group_norm; must be zeroed once at allocation (holds a self-resetting ticket counter)
size_t group_norm_scratch_bytes(int batch, int HW, int groups, int C);
void layer_norm(const __nv_bfloat16* x, int tokens, int C, const float* gamma, const float* beta, float eps,
                __nv_bfloat16* out, cudaStream_t st);
void softmax_rows(const float* S, long long lds, int rows, int valid, __nv_bfloat16* P, long long ldp, int padded,
                  cudaStream_t st);
void geglu(const __nv_bfloat16* F, long long tokens, int H, __nv_bfloat16* out, cudaStream_t st);
void upsample2x(const __nv_bfloat16* x, int batch, int H, int W, int C, __nv_bfloat16* out, cudaStream_t st);
void concat_channels(const Cat2& x, long long pixels, __nv_bfloat16* out, cudaStream_t st);
void pack_latent(const void* x, bool f64, long long pixels, int c_lat, int cpad, __nv_bfloat16* out,
                 cudaStream_t st);
// VT[d][k] = V[k * ldv + d] per image of a stacked batch (V rows b * L.., VT [b][hd][Lpad])
void transpose_head(const __nv_bfloat16* V, long long ldv, int L, int Lpad, int hd, __nv_bfloat16* VT,
                    cudaStream_t st, int batch = 1);

}  // namespace adx
