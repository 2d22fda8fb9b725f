// unet_kernels.cu -- bandwidth-bound kernels of the UNet-shaped denoiser family
// (NHWC bf16 activations, fp32 math): GroupNorm(+SiLU) over a channel concat,
// LayerNorm, row softmax, GEGLU, nearest 2x upsample, channel concat, latent
// pack / eps unpack, per-head transpose.  All reductions use a fixed order
// (deterministic, placement independent).
#include "unet_kernels.cuh"

#include <cuda_bf16.h>

#include <stdexcept>
#include <string>

namespace adx {

#define CKU(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float b2f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// channel c of pixel p of image n from a two-segment channel concat
__device__ __forceinline__ float cat_at(const Cat2& x, long long pix, int c) {
    return c < x.c0 ? b2f(x.p0[pix * x.c0 + c]) : b2f(x.p1[pix * x.c1 + (c - x.c0)]);
}

// GroupNorm pass 1: partial (sum, sumsq) per (image, chunk, group), fp32 over <= kChunkPix pixels
constexpr int kChunkPix = 256;
__global__ void gn_partials(Cat2 x, int HW, int groups, int chunks, float2* part) {
    const int n = blockIdx.z, ch = blockIdx.y, g = blockIdx.x;
    const int C = x.c0 + x.c1, cpg = C / groups;
    const int p0 = ch * kChunkPix, p1 = min(HW, p0 + kChunkPix);
    float s = 0.f, ss = 0.f;
    const int elems = (p1 - p0) * cpg;
    for (int e = threadIdx.x; e < elems; e += blockDim.x) {
        const int pp = p0 + e / cpg, c = g * cpg + e % cpg;
        const float v = cat_at(x, static_cast<long long>(n) * HW + pp, c);
        s += v;
        ss += v * v;
    }
    __shared__ float sh[2][32];
    s = warp_sum(s);
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = s;
        sh[1][threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f, b = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a += sh[0][w];
            b += sh[1][w];
        }
        part[(static_cast<long long>(n) * chunks + ch) * groups + g] = make_float2(a, b);
    }
}

// GroupNorm pass 2: every block merges the partials of its image in fp64
// (fixed order), then normalises its pixels: y = (x-mu)*rstd*gamma + beta (+SiLU)
__global__ void gn_apply(Cat2 x, int HW, int groups, int chunks, const float2* part, const float* gamma,
                         const float* beta, float eps, int act, bf16* out, int pix_per_block) {
    extern __shared__ float st[];  // [2*groups]: mean, rstd
    const int n = blockIdx.y;
    const int C = x.c0 + x.c1, cpg = C / groups;
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        double s = 0.0, ss = 0.0;
        for (int ch = 0; ch < chunks; ++ch) {
            const float2 v = part[(static_cast<long long>(n) * chunks + ch) * groups + g];
            s += v.x;
            ss += v.y;
        }
        const double cnt = static_cast<double>(HW) * cpg;
        const double mu = s / cnt;
        const double var = fmax(ss / cnt - mu * mu, 0.0);
        st[g] = static_cast<float>(mu);
        st[groups + g] = static_cast<float>(rsqrt(var + eps));
    }
    __syncthreads();
    const long long base = static_cast<long long>(blockIdx.x) * pix_per_block;
    const long long end = min(static_cast<long long>(HW), base + pix_per_block);
    for (long long e = threadIdx.x; e < (end - base) * C; e += blockDim.x) {
        const long long pp = base + e / C;
        const int c = static_cast<int>(e % C);
        const long long pix = static_cast<long long>(n) * HW + pp;
        const int g = c / cpg;
        float v = (cat_at(x, pix, c) - st[g]) * st[groups + g] * gamma[c] + beta[c];
        if (act) v = silu(v);
        out[pix * C + c] = __float2bfloat16(v);
    }
}

// LayerNorm over C per token, one warp per token
__global__ void layernorm_k(const bf16* x, int tokens, int C, const float* gamma, const float* beta, float eps,
                            bf16* out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= tokens) return;
    const bf16* r = x + static_cast<long long>(warp) * C;
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += b2f(r[c]);
    const float mu = warp_sum(s) / C;
    float ss = 0.f;
    for (int c = lane; c < C; c += 32) {
        const float d = b2f(r[c]) - mu;
        ss += d * d;
    }
    const float rstd = rsqrtf(warp_sum(ss) / C + eps);
    bf16* o = out + static_cast<long long>(warp) * C;
    for (int c = lane; c < C; c += 32) o[c] = __float2bfloat16((b2f(r[c]) - mu) * rstd * gamma[c] + beta[c]);
}

// softmax over the first `valid` columns of each fp32 row (already scaled);
// P bf16 with zeros in the padding columns [valid, ldp)
__global__ void softmax_rows(const float* S, long long lds, int valid, bf16* P, long long ldp, int padded) {
    const long long row = blockIdx.x;
    const float* r = S + row * lds;
    __shared__ float red[32];
    float mx = -INFINITY;
    for (int c = threadIdx.x; c < valid; c += blockDim.x) mx = fmaxf(mx, r[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float s = 0.f;
    for (int c = threadIdx.x; c < valid; c += blockDim.x) s += __expf(r[c] - mx);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        red[0] = t;
    }
    __syncthreads();
    const float inv = 1.0f / red[0];
    bf16* p = P + row * ldp;
    for (int c = threadIdx.x; c < padded; c += blockDim.x)
        p[c] = __float2bfloat16(c < valid ? __expf(r[c] - mx) * inv : 0.f);
}

// out[t][j] = F[t][j] * gelu(F[t][j + H])   (diffusers GEGLU: hidden * gelu(gate))
__global__ void geglu_k(const bf16* F, long long tokens, int H, bf16* out) {
    const long long n = tokens * H;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long t = i / H;
        const int j = static_cast<int>(i % H);
        const float a = b2f(F[t * 2 * H + j]), g = b2f(F[t * 2 * H + H + j]);
        out[i] = __float2bfloat16(a * gelu(g));
    }
}

__global__ void upsample2x_k(const bf16* x, int batch, int H, int W, int C, bf16* out) {
    const long long n = static_cast<long long>(batch) * 2 * H * 2 * W * C;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % C);
        long long p = i / C;
        const int w2 = static_cast<int>(p % (2 * W));
        p /= 2 * W;
        const int h2 = static_cast<int>(p % (2 * H));
        const long long b = p / (2 * H);
        out[i] = x[((b * H + h2 / 2) * W + w2 / 2) * C + c];
    }
}

__global__ void concat_k(Cat2 x, long long pixels, bf16* out) {
    const int C = x.c0 + x.c1;
    const long long n = pixels * C;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / C;
        const int c = static_cast<int>(i % C);
        out[i] = c < x.c0 ? x.p0[p * x.c0 + c] : x.p1[p * x.c1 + (c - x.c0)];
    }
}

// latent (fp32 or fp64, H*W*c_lat, HWC order) -> bf16 NHWC with cpad channels (zeros above c_lat)
template <typename T>
__global__ void pack_latent_k(const T* x, long long pixels, int c_lat, int cpad, bf16* out) {
    const long long n = pixels * cpad;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / cpad;
        const int c = static_cast<int>(i % cpad);
        out[i] = __float2bfloat16(c < c_lat ? static_cast<float>(x[p * c_lat + c]) : 0.f);
    }
}

// VT[d][k] = V[k * ldv + d] for k < L, 0 for L <= k < Lpad  (one head, head_dim rows)
__global__ void transpose_head_k(const bf16* V, long long ldv, int L, int Lpad, int hd, bf16* VT) {
    __shared__ bf16 tile[32][33];
    const int k0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, d = d0 + threadIdx.x;
        tile[i][threadIdx.x] = (k < L && d < hd) ? V[static_cast<long long>(k) * ldv + d] : __float2bfloat16(0.f);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int d = d0 + i, k = k0 + threadIdx.x;
        if (d < hd && k < Lpad) VT[static_cast<long long>(d) * Lpad + k] = tile[threadIdx.x][i];
    }
}

int grid_for(long long n, int threads = 256) {
    return static_cast<int>(std::min<long long>((n + threads - 1) / threads, 148LL * 16));
}

}  // namespace

void group_norm(const Cat2& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, __nv_bfloat16* out, float2* scratch, cudaStream_t st) {
    const int C = x.c0 + x.c1;
    if (C % groups) throw std::invalid_argument("group_norm: channels not divisible by groups");
    const int chunks = (HW + kChunkPix - 1) / kChunkPix;
    gn_partials<<<dim3(groups, chunks, batch), 256, 0, st>>>(x, HW, groups, chunks, scratch);
    CKU(cudaGetLastError());
    const int ppb = std::max(1, 8192 / C);
    gn_apply<<<dim3((HW + ppb - 1) / ppb, batch), 256, 2 * groups * sizeof(float), st>>>(
        x, HW, groups, chunks, scratch, gamma, beta, eps, silu_act, out, ppb);
    CKU(cudaGetLastError());
}

size_t group_norm_scratch_bytes(int batch, int HW, int groups) {
    return static_cast<size_t>(batch) * ((HW + kChunkPix - 1) / kChunkPix) * groups * sizeof(float2);
}

void layer_norm(const __nv_bfloat16* x, int tokens, int C, const float* gamma, const float* beta, float eps,
                __nv_bfloat16* out, cudaStream_t st) {
    layernorm_k<<<(tokens + 7) / 8, 256, 0, st>>>(x, tokens, C, gamma, beta, eps, out);
    CKU(cudaGetLastError());
}

void softmax_rows(const float* S, long long lds, int rows, int valid, __nv_bfloat16* P, long long ldp, int padded,
                  cudaStream_t st) {
    softmax_rows<<<rows, 256, 0, st>>>(S, lds, valid, P, ldp, padded);
    CKU(cudaGetLastError());
}

void geglu(const __nv_bfloat16* F, long long tokens, int H, __nv_bfloat16* out, cudaStream_t st) {
    geglu_k<<<grid_for(tokens * H), 256, 0, st>>>(F, tokens, H, out);
    CKU(cudaGetLastError());
}

void upsample2x(const __nv_bfloat16* x, int batch, int H, int W, int C, __nv_bfloat16* out, cudaStream_t st) {
    upsample2x_k<<<grid_for(4LL * batch * H * W * C), 256, 0, st>>>(x, batch, H, W, C, out);
    CKU(cudaGetLastError());
}

void concat_channels(const Cat2& x, long long pixels, __nv_bfloat16* out, cudaStream_t st) {
    concat_k<<<grid_for(pixels * (x.c0 + x.c1)), 256, 0, st>>>(x, pixels, out);
    CKU(cudaGetLastError());
}

void pack_latent(const void* x, bool f64, long long pixels, int c_lat, int cpad, __nv_bfloat16* out,
                 cudaStream_t st) {
    if (f64)
        pack_latent_k<double><<<grid_for(pixels * cpad), 256, 0, st>>>(static_cast<const double*>(x), pixels, c_lat,
                                                                      cpad, out);
    else
        pack_latent_k<float><<<grid_for(pixels * cpad), 256, 0, st>>>(static_cast<const float*>(x), pixels, c_lat,
                                                                     cpad, out);
    CKU(cudaGetLastError());
}

void transpose_head(const __nv_bfloat16* V, long long ldv, int L, int Lpad, int hd, __nv_bfloat16* VT,
                    cudaStream_t st) {
    transpose_head_k<<<dim3((Lpad + 31) / 32, (hd + 31) / 32), dim3(32, 8), 0, st>>>(V, ldv, L, Lpad, hd, VT);
    CKU(cudaGetLastError());
}

}  // namespace adx
