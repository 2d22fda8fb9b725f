// unet_kernels.cuh -- bandwidth-bound UNet kernels (see unet_kernels.cu).
#pragma once

#include "host.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace adx {

// NHWC channel concat of up to two tensors (c1 = 0: single tensor)
struct Cat2 {
    const __nv_bfloat16* p0 = nullptr;
    int c0 = 0;
    const __nv_bfloat16* p1 = nullptr;
    int c1 = 0;
};

void group_norm(const Cat2& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, __nv_bfloat16* out, float2* scratch, cudaStream_t st);
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
void transpose_head(const __nv_bfloat16* V, long long ldv, int L, int Lpad, int hd, __nv_bfloat16* VT,
                    cudaStream_t st);

}  // namespace adx
