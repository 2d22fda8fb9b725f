// unet_kernels.cu -- bandwidth-bound kernels of the UNet-shaped denoiser family
// (NHWC bf16 activations, fp32 math): GroupNorm(+SiLU) over a channel concat,
// LayerNorm, row softmax, GEGLU, nearest 2x upsample, channel concat, latent
// pack / eps unpack, per-head transpose.  All reductions use a fixed order
// (deterministic, placement independent).
#include "unet_kernels.cuh"

#include "pdl.cuh"
#include "tc_gemm.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <utility>
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

// x * sigmoid(x) with the MUFU reciprocal: an IEEE division here was a branchy ~15-instruction
// sequence per element (the GroupNorm apply phase's bottleneck); 1 / (1 + e^-x) -> 0 as x -> -inf
__device__ __forceinline__ float silu(float x) { return x * __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&b);
    }
    return u;
}

// 8 consecutive elements of an activation tensor: one 16-byte vector (bf16) or two (fp32)
template <typename T>
struct Vec8;
template <>
struct Vec8<bf16> {
    using raw = uint4;
    __device__ static raw load(const bf16* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
    __device__ static void unpack(const raw& u, float* f) { unpack8(u, f); }
    __device__ static raw pack(const float* f) { return pack8(f); }
    __device__ static void store(bf16* p, const raw& u) { *reinterpret_cast<uint4*>(p) = u; }
};
struct F8 {
    float4 a, b;
};
template <>
struct Vec8<float> {
    using raw = F8;
    __device__ static raw load(const float* p) {
        return {__ldg(reinterpret_cast<const float4*>(p)), __ldg(reinterpret_cast<const float4*>(p) + 1)};
    }
    __device__ static void unpack(const raw& u, float* f) {
        f[0] = u.a.x, f[1] = u.a.y, f[2] = u.a.z, f[3] = u.a.w, f[4] = u.b.x, f[5] = u.b.y, f[6] = u.b.z, f[7] = u.b.w;
    }
    __device__ static raw pack(const float* f) {
        return {make_float4(f[0], f[1], f[2], f[3]), make_float4(f[4], f[5], f[6], f[7])};
    }
    __device__ static void store(float* p, const raw& u) {
        reinterpret_cast<float4*>(p)[0] = u.a;
        reinterpret_cast<float4*>(p)[1] = u.b;
    }
};

// 8 consecutive channels (one vector) of pixel `pix` from a two-segment channel
// concat; both segments are multiples of 8 channels (checked on the host)
template <typename T>
__device__ __forceinline__ typename Vec8<T>::raw cat_vec(const Cat2T<T>& x, long long pix, int v) {
    const int c = v * 8;
    return c < x.c0 ? Vec8<T>::load(x.p0 + pix * x.c0 + c) : Vec8<T>::load(x.p1 + pix * x.c1 + (c - x.c0));
}

// GroupNorm scratch: [ticket counters (64 B)][gn_fused grid barrier (64 B)][per-channel (scale, shift) float2, batch*C][partials]
constexpr int kGnMaxChunks = 148;  // one statistics CTA per SM
constexpr int kGnImageTickets = 16;  // per-image ticket counters in the scratch's first 64 B
// pixel chunks per image: one per SM for 1-2 images; a video batch shares ~2 CTAs per SM so
// the last CTA's merge reads few partials per (image, group)
inline int gn_chunk_cap(int batch) {
    static const int per_sm = [] {  // ADX_GN_CTAS_PER_SM: statistics CTAs per SM for batches > 2
        const char* e = getenv("ADX_GN_CTAS_PER_SM");
        return e ? std::max(1, atoi(e)) : 2;
    }();
    return batch <= 2 ? kGnMaxChunks : std::max(4, per_sm * kGnMaxChunks / batch);
}
struct GnLayout {
    unsigned* counter;
    float2* ab;
    float2* part;
};
__host__ __device__ inline GnLayout gn_layout(float2* scratch, int batch, int C) {
    GnLayout l;
    l.counter = reinterpret_cast<unsigned*>(scratch);
    l.ab = scratch + 16;
    l.part = l.ab + static_cast<long long>(batch) * C;
    return l;
}

// GroupNorm pass 1, one CTA per (pixel chunk, image).  Thread (r, v) owns the 8
// channels of vector v and pixels p0 + r, p0 + r + rpb, ...; per-channel partial
// (sum, sumsq) are reduced to per-group partials in a fixed order.  The last CTA
// (ticket) merges all chunks in fp64 (fixed order) and folds mean / rstd / gamma /
// beta into per-channel (a, b) with y = x * a + b.  Deterministic and independent of
// which CTA happens to finish last.
template <typename T>
__global__ void gn_stats(Cat2T<T> x, int HW, int groups, int chunk_pix, int chunks, const float* gamma,
                         const float* beta, float eps, float2* scratch) {
    pdl_wait();
    extern __shared__ __align__(16) float sm[];  // [2][rpb][C]
    const int n = blockIdx.y, ch = blockIdx.x, batch = gridDim.y;
    const int C = x.c0 + x.c1, nv = C / 8, cpg = C / groups;
    const int rpb = blockDim.x / nv, r = threadIdx.x / nv, v = threadIdx.x % nv;
    const GnLayout L = gn_layout(scratch, batch, C);
    const int p0 = ch * chunk_pix, p1 = min(HW, p0 + chunk_pix);
    if (r < rpb) {
        float s[8], ss[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = ss[i] = 0.f;
        // 4 rows in flight per thread (the loads do not depend on the running sums)
        for (int p = p0 + r; p < p1; p += 4 * rpb) {
            typename Vec8<T>::raw u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (p + k * rpb < p1) u[k] = cat_vec(x, static_cast<long long>(n) * HW + p + k * rpb, v);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (p + k * rpb >= p1) break;
                float f[8];
                Vec8<T>::unpack(u[k], f);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    s[i] += f[i];
                    ss[i] = fmaf(f[i], f[i], ss[i]);
                }
            }
        }
        // 16-byte stores (C % 8 == 0: 32-byte aligned): scalar stores at a 32-byte thread
        // stride were 8-way bank conflicts
        float4* w0 = reinterpret_cast<float4*>(sm + r * C + v * 8);
        float4* w1 = reinterpret_cast<float4*>(sm + (rpb + r) * C + v * 8);
        w0[0] = make_float4(s[0], s[1], s[2], s[3]);
        w0[1] = make_float4(s[4], s[5], s[6], s[7]);
        w1[0] = make_float4(ss[0], ss[1], ss[2], ss[3]);
        w1[1] = make_float4(ss[4], ss[5], ss[6], ss[7]);
    }
    __syncthreads();
    // rows -> per channel (one thread per channel), then channels -> per group; fixed order
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int rr = 0; rr < rpb; ++rr) {
            a += sm[rr * C + c];
            b += sm[(rpb + rr) * C + c];
        }
        sm[c] = a;
        sm[rpb * C + c] = b;  // row 0 of each half: only this thread reads / writes column c
    }
    __syncthreads();
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int c = g * cpg; c < (g + 1) * cpg; ++c) {
            a += sm[c];
            b += sm[rpb * C + c];
        }
        L.part[(static_cast<long long>(n) * chunks + ch) * groups + g] = make_float2(a, b);
    }
    // ticket: up to kGnImageTickets images, the last CTA of each image finalises that image
    // (the merges of a video batch run in parallel); larger batches: the last CTA of the grid
    // finalises every image
    __shared__ unsigned last;
    const bool per_image = batch <= kGnImageTickets;
    const int n0 = per_image ? n : 0, nb = per_image ? 1 : batch;
    unsigned* counter = L.counter + (per_image ? n : 0);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == static_cast<unsigned>(chunks * nb - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    // fp64 merge of the chunk partials: nsub threads per (image, group), each over a fixed
    // strided subset with 4 loads in flight, then combined in sub order (fixed = deterministic)
    const int ngs = nb * groups, nsub = max(1, static_cast<int>(blockDim.x) / ngs);
    // (loops: a video batch can hold more (image, group) pairs than the CTA has threads)
    double* red = reinterpret_cast<double*>(sm);  // [nsub][ngs][2], then [ngs][2] mean / rstd
    for (int idx = threadIdx.x; idx < nsub * ngs; idx += blockDim.x) {
        const int ng = idx % ngs, sub = idx / ngs, nn = n0 + ng / groups, g = ng % groups;
        const float2* pp = L.part + static_cast<long long>(nn) * chunks * groups + g;
        double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
        int k = sub;
        for (; k + 3 * nsub < chunks; k += 4 * nsub) {
            float2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcg(pp + static_cast<long long>(k + u * nsub) * groups);
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] += v[u].x, b[u] += v[u].y;
        }
        for (; k < chunks; k += nsub) {
            const float2 v = __ldcg(pp + static_cast<long long>(k) * groups);
            a[0] += v.x, b[0] += v.y;
        }
        red[2 * (sub * ngs + ng)] = (a[0] + a[1]) + (a[2] + a[3]);
        red[2 * (sub * ngs + ng) + 1] = (b[0] + b[1]) + (b[2] + b[3]);
    }
    __syncthreads();
    double* st = red + 2 * nsub * ngs;  // [ngs][2] mean / rstd
    for (int ng = threadIdx.x; ng < ngs; ng += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int sub = 0; sub < nsub; ++sub) a += red[2 * (sub * ngs + ng)], b += red[2 * (sub * ngs + ng) + 1];
        const double cnt = static_cast<double>(HW) * cpg;
        const double mu = a / cnt;
        const double var = fmax(b / cnt - mu * mu, 0.0);
        st[2 * ng] = mu;
        st[2 * ng + 1] = 1.0 / sqrt(var + static_cast<double>(eps));
    }
    __syncthreads();
    for (int nc = threadIdx.x; nc < nb * C; nc += blockDim.x) {
        const int nn = nc / C, c = nc % C, g = c / cpg;
        const double mu = st[2 * (nn * groups + g)], rs = st[2 * (nn * groups + g) + 1];
        const float a = static_cast<float>(rs * gamma[c]);
        L.ab[static_cast<long long>(n0) * C + nc] = make_float2(a, static_cast<float>(beta[c] - mu * rs * gamma[c]));
    }
    if (threadIdx.x == 0) *counter = 0u;  // re-arm for the next launch on this scratch
}

// GroupNorm pass 2: y = x * a[c] + b[c] (+SiLU).  Thread (r, v) owns the 8 channels of
// vector v for pixel rows r, r + rpb, ... of its CTA's contiguous pixel range, so its (scale,
// shift) pairs are loaded once per image, not per element; 4 rows in flight per thread
template <typename T>
__global__ void gn_apply(Cat2T<T> x, int pixels, int HW, const float2* __restrict__ ab, int act, T* out) {
    pdl_wait();
    const int C = x.c0 + x.c1, nv = C / 8, rpb = blockDim.x / nv;
    const int r = threadIdx.x / nv, v = threadIdx.x - (threadIdx.x / nv) * nv;
    if (r >= rpb) return;
    const int per = (pixels + gridDim.x - 1) / gridDim.x;
    const int p0 = blockIdx.x * per, p1 = min(pixels, p0 + per);
    int cur = -1;
    float2 q[8];
    for (int pix = p0 + r; pix < p1; pix += 4 * rpb) {
        typename Vec8<T>::raw u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (pix + k * rpb < p1) u[k] = cat_vec(x, pix + k * rpb, v);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int pk = pix + k * rpb;
            if (pk >= p1) break;
            const int img = pk / HW;
            if (img != cur) {
                cur = img;
                const float4* a4 = reinterpret_cast<const float4*>(ab + static_cast<long long>(img) * C + v * 8);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 t = __ldg(a4 + j);
                    q[2 * j] = make_float2(t.x, t.y);
                    q[2 * j + 1] = make_float2(t.z, t.w);
                }
            }
            float f[8];
            Vec8<T>::unpack(u[k], f);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                f[j] = fmaf(f[j], q[j].x, q[j].y);
                if (act) f[j] = silu(f[j]);
            }
            Vec8<T>::store(out + (static_cast<long long>(pk) * nv + v) * 8, Vec8<T>::pack(f));
        }
    }
}

// GroupNorm in one cooperative launch (batch 1): CTA c of G (<= #SMs, all co-resident)
// owns pixels [c*chunk, (c+1)*chunk): it loads them into SMEM once while accumulating
// per-channel (sum, sumsq), reduces rows -> channels -> groups in a fixed order and
// publishes its group partials; after a grid barrier every CTA folds all G partials
// in the same fixed fp64 order (identical statistics everywhere, deterministic),
// builds per-channel (a, b) and normalises its SMEM copy: one HBM read of x.
#ifdef ADX_GN_TIMELINE  // %globaltimer stamps per CTA (diagnostics; adx_gn_timeline)
__device__ unsigned long long g_gn_tl[256][8];
__device__ __forceinline__ void gn_stamp(int k) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_gn_tl[blockIdx.x][k] = t;
    }
}
#else
__device__ __forceinline__ void gn_stamp(int) {}
#endif

template <typename T>
__global__ void gn_fused(Cat2T<T> x, int HW, int groups, int chunk_pix, const float* gamma, const float* beta,
                         float eps, int act, float2* scratch, T* out) {
    extern __shared__ __align__(16) uint8_t gsm[];
    gn_stamp(0);
    pdl_wait();
    gn_stamp(1);
    const int G = gridDim.x, cta = blockIdx.x;
    const int C = x.c0 + x.c1, nv = C / 8, cpg = C / groups;
    const int rpb = blockDim.x / nv, r = threadIdx.x / nv, v = threadIdx.x % nv;
    const int p0 = cta * chunk_pix, p1 = min(HW, p0 + chunk_pix), np = max(0, p1 - p0);
    using Raw = typename Vec8<T>::raw;
    Raw* tile = reinterpret_cast<Raw*>(gsm);                                  // [chunk_pix][nv]
    float* red = reinterpret_cast<float*>(gsm + static_cast<size_t>(chunk_pix) * nv * sizeof(Raw));  // [2][rpb][C]
    float2* ab = reinterpret_cast<float2*>(red + 2 * rpb * C);               // [C]
    double* st = reinterpret_cast<double*>(ab + C);                          // [nsub][groups][2], then [groups][2]
    // header words 18-19 (bytes 72-79): clear of gn_stats' ticket counters (words 0-15)
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(scratch + 9);
    float2* part = scratch + 16;
    // (gamma, beta) staged now: their loads overlap the statistics instead of following the fold
    for (int c = threadIdx.x; c < C; c += blockDim.x) ab[c] = make_float2(__ldg(gamma + c), __ldg(beta + c));
    if (r < rpb) {
        float s[8], ss[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = ss[i] = 0.f;
        for (int q = r; q < np; q += 4 * rpb) {
            Raw u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (q + k * rpb < np) u[k] = cat_vec(x, p0 + q + k * rpb, v);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (q + k * rpb >= np) break;
                tile[(q + k * rpb) * nv + v] = u[k];
                float f[8];
                Vec8<T>::unpack(u[k], f);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    s[i] += f[i];
                    ss[i] = fmaf(f[i], f[i], ss[i]);
                }
            }
        }
        // 16-byte stores (C % 8 == 0: 32-byte aligned): scalar stores at a 32-byte thread
        // stride were 8-way bank conflicts
        float4* w0 = reinterpret_cast<float4*>(red + r * C + v * 8);
        float4* w1 = reinterpret_cast<float4*>(red + (rpb + r) * C + v * 8);
        w0[0] = make_float4(s[0], s[1], s[2], s[3]);
        w0[1] = make_float4(s[4], s[5], s[6], s[7]);
        w1[0] = make_float4(ss[0], ss[1], ss[2], ss[3]);
        w1[1] = make_float4(ss[4], ss[5], ss[6], ss[7]);
    }
    __syncthreads();
    gn_stamp(2);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int rr = 0; rr < rpb; ++rr) {
            a += red[rr * C + c];
            b += red[(rpb + rr) * C + c];
        }
        red[c] = a;
        red[rpb * C + c] = b;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int c = g * cpg; c < (g + 1) * cpg; ++c) {
            a += red[c];
            b += red[rpb * C + c];
        }
        part[static_cast<long long>(cta) * groups + g] = make_float2(a, b);
    }
    gn_stamp(3);
    // grid barrier (co-residency guaranteed by the cooperative launch): arrival count +
    // generation; the last CTA to arrive re-arms the count and bumps the generation, so
    // consecutive launches with different grid sizes reuse the same two words
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int* count = reinterpret_cast<unsigned int*>(bar);
        unsigned int* gen = count + 1;
        unsigned int g0;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
        __threadfence();
        if (atomicAdd(count, 1u) == static_cast<unsigned int>(G - 1)) {
            *count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            unsigned int cur;
            do {
                __nanosleep(64);
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
            } while (cur == g0);
        }
    }
    __syncthreads();
    gn_stamp(4);
    // statistics: nsub threads per group over a fixed strided subset of the G partials
    const int nsub = max(1, static_cast<int>(blockDim.x) / groups);
    if (threadIdx.x < nsub * groups) {
        const int g = threadIdx.x % groups, sub = threadIdx.x / groups;
        // all of this thread's partials are requested before any is summed (one L2
        // round trip instead of one per partial); summed in k order (deterministic)
        constexpr int kMaxPer = 16;
        float2 pv[kMaxPer];
#pragma unroll
        for (int i = 0; i < kMaxPer; ++i) {
            const int k = sub + i * nsub;
            pv[i] = k < G ? __ldcg(&part[static_cast<long long>(k) * groups + g]) : make_float2(0.f, 0.f);
        }
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int i = 0; i < kMaxPer; ++i) a += pv[i].x, b += pv[i].y;
        for (int k = sub + kMaxPer * nsub; k < G; k += nsub) {  // (only for > 16 * nsub partials)
            const float2 q = __ldcg(&part[static_cast<long long>(k) * groups + g]);
            a += q.x;
            b += q.y;
        }
        st[2 * (sub * groups + g)] = a;
        st[2 * (sub * groups + g) + 1] = b;
    }
    __syncthreads();
    double mv0 = 0.0, mv1 = 0.0;
    if (threadIdx.x < groups) {
        const int g = threadIdx.x;
        double a = 0.0, b = 0.0;
        for (int sub = 0; sub < nsub; ++sub) a += st[2 * (sub * groups + g)], b += st[2 * (sub * groups + g) + 1];
        const double cnt = static_cast<double>(HW) * cpg;
        mv0 = a / cnt;
        mv1 = 1.0 / sqrt(fmax(b / cnt - mv0 * mv0, 0.0) + static_cast<double>(eps));
    }
    __syncthreads();
    if (threadIdx.x < groups) st[2 * threadIdx.x] = mv0, st[2 * threadIdx.x + 1] = mv1;
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const int g = c / cpg;
        const double rs = st[2 * g + 1];
        const float2 gb = ab[c];
        ab[c] = make_float2(static_cast<float>(rs * gb.x), static_cast<float>(gb.y - st[2 * g] * rs * gb.x));
    }
    __syncthreads();
    gn_stamp(5);
    // normalise the SMEM copy, 16-byte coalesced stores.  blockDim.x = rpb * nv, so the
    // vector index i % nv of a thread is the same every iteration: its 8 (a, b) pairs are
    // read from SMEM once (per-iteration reads at a 64-byte thread stride were 16-way
    // bank conflicts, the kernel's top stall)
    T* o = out + static_cast<long long>(p0) * C;
    float2 q[8];
    {
        const float4* a4 = reinterpret_cast<const float4*>(ab + (threadIdx.x % nv) * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4 t = a4[j];
            q[2 * j] = make_float2(t.x, t.y);
            q[2 * j + 1] = make_float2(t.z, t.w);
        }
    }
    for (int i = threadIdx.x; i < np * nv; i += blockDim.x) {
        float f[8];
        Vec8<T>::unpack(tile[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            f[k] = fmaf(f[k], q[k].x, q[k].y);
            if (act) f[k] = silu(f[k]);
        }
        Vec8<T>::store(o + static_cast<long long>(i) * 8, Vec8<T>::pack(f));
    }
    gn_stamp(6);
}

// LayerNorm over C per token, one warp per token, row held in registers (C <= 2048)
// (NV: vectors of 8 per lane the instantiation holds -- C <= 256 NV; fewer registers for
// narrow rows = more warps resident = more bytes in flight)
constexpr int kLnMaxVec = 8;
template <typename T, int NV = kLnMaxVec>
__global__ void layernorm_k(const T* x, int tokens, int C, const float* gamma, const float* beta, float eps,
                            T* out) {
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= tokens) return;
    const int nv = C / 8;
    const T* r = x + static_cast<long long>(warp) * C;
    float f[NV][8];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int v = lane + 32 * j;
        if (v < nv) {
            Vec8<T>::unpack(Vec8<T>::load(r + v * 8), f[j]);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += f[j][k];
        }
    }
    const float mu = warp_sum(s) / C;
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
        if (lane + 32 * j < nv) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float d = f[j][k] - mu;
                ss = fmaf(d, d, ss);
            }
        }
    const float rstd = rsqrtf(warp_sum(ss) / C + eps);
    T* o = out + static_cast<long long>(warp) * C;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int v = lane + 32 * j;
        if (v < nv) {
            const float4* g4 = reinterpret_cast<const float4*>(gamma + v * 8);
            const float4* b4 = reinterpret_cast<const float4*>(beta + v * 8);
            const float4 ga = __ldg(g4), gb = __ldg(g4 + 1), ba = __ldg(b4), bb = __ldg(b4 + 1);
            const float gg[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
            const float be[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
            float y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = (f[j][k] - mu) * rstd * gg[k] + be[k];
            Vec8<T>::store(o + v * 8, Vec8<T>::pack(y));
        }
    }
}

// softmax over the first `valid` columns of each fp32 row (already scaled);
// P bf16 with zeros in the padding columns [valid, ldp)
__global__ void softmax_rows_k(const float* S, long long lds, int valid, bf16* P, long long ldp, int padded) {
    pdl_wait();
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

// out[t][j] = F[t][j] * gelu(F[t][j + H])   (diffusers GEGLU: hidden * gelu(gate)), 8 per thread
__global__ void geglu_k(const bf16* F, long long tokens, int H, bf16* out) {
    pdl_wait();
    const int hv = H / 8;
    const long long n = tokens * hv;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long t = i / hv;
        const int j = static_cast<int>(i - t * hv);
        const uint4* row = reinterpret_cast<const uint4*>(F + t * 2 * H);
        float a[8], g[8];
        unpack8(__ldg(row + j), a);
        unpack8(__ldg(row + hv + j), g);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] *= gelu(g[k]);
        reinterpret_cast<uint4*>(out)[i] = pack8(a);
    }
}

// nearest 2x upsample, NHWC, 8 channels per thread
__global__ void upsample2x_k(const bf16* x, int batch, int H, int W, int C, bf16* out) {
    pdl_wait();
    const int nv = C / 8;
    const long long n = static_cast<long long>(batch) * 2 * H * 2 * W * nv;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        long long p = i / nv;
        const int v = static_cast<int>(i - p * nv);
        const int w2 = static_cast<int>(p % (2 * W));
        p /= 2 * W;
        const int h2 = static_cast<int>(p % (2 * H));
        const long long b = p / (2 * H);
        reinterpret_cast<uint4*>(out)[i] =
            __ldg(reinterpret_cast<const uint4*>(x + ((b * H + h2 / 2) * W + w2 / 2) * C) + v);
    }
}

__global__ void concat_k(Cat2 x, long long pixels, bf16* out) {
    pdl_wait();
    const int nv = (x.c0 + x.c1) / 8;
    const long long n = pixels * nv;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / nv;
        reinterpret_cast<uint4*>(out)[i] = cat_vec(x, p, static_cast<int>(i - p * nv));
    }
}

// latent (fp32 or fp64, H*W*c_lat, HWC order) -> bf16 NHWC with cpad channels (zeros above c_lat)
template <typename T, typename O = bf16>
__global__ void pack_latent_k(const T* x, long long pixels, int c_lat, int cpad, O* out) {
    pdl_wait();
    const long long n = pixels * cpad;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / cpad;
        const int c = static_cast<int>(i % cpad);
        const float v = c < c_lat ? static_cast<float>(x[p * c_lat + c]) : 0.f;
        if constexpr (sizeof(O) == 2)
            out[i] = __float2bfloat16(v);
        else
            out[i] = v;
    }
}

// VT[d][k] = V[k * ldv + d] for k < L, 0 for L <= k < Lpad  (one head, head_dim rows)
__global__ void transpose_head_k(const bf16* V, long long ldv, int L, int Lpad, int hd, bf16* VT) {
    pdl_wait();
    V += static_cast<long long>(blockIdx.z) * L * ldv;  // image z of a stacked batch
    VT += static_cast<long long>(blockIdx.z) * hd * Lpad;
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

// split-bf16 operands of the ADX_F32 mode (see split3 in unet_kernels.cuh)
__global__ void split3_k(const float* x, long long rows, int cols, long long ldx, int g, int pattern, bf16* out) {
    pdl_wait();
    const int nv = cols / 8;
    const long long n = rows * nv;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = i / nv;
        const int c = static_cast<int>(i - row * nv) * 8;
        float f[8], hi[8], lo[8];
        Vec8<float>::unpack(Vec8<float>::load(x + row * ldx + c), f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            hi[k] = __bfloat162float(__float2bfloat16(f[k]));
            lo[k] = f[k] - hi[k];
        }
        const uint4 h = pack8(hi), l = pack8(lo);
        const int grp = c / g, cg = c - grp * g;
        bf16* o = out + row * 3LL * cols + 3LL * grp * g + cg;
        *reinterpret_cast<uint4*>(o) = h;
        *reinterpret_cast<uint4*>(o + g) = pattern ? l : h;
        *reinterpret_cast<uint4*>(o + 2 * g) = pattern ? h : l;
    }
}

// hi / lo planes of the fused split-operand attention (see split2 in unet_kernels.cuh)
__global__ void split2_k(const float* x, long long n8, bf16* hi, bf16* lo) {
    pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float f[8], h[8], l[8];
        Vec8<float>::unpack(Vec8<float>::load(x + 8 * i), f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h[k] = __bfloat162float(__float2bfloat16(f[k]));
            l[k] = f[k] - h[k];
        }
        *reinterpret_cast<uint4*>(hi + 8 * i) = pack8(h);
        *reinterpret_cast<uint4*>(lo + 8 * i) = pack8(l);
    }
}

// fp32 row softmax, in place (the ADX_F32 mode's unfused attention)
__global__ void softmax_rows_f32_k(float* S, long long lds, int valid, int padded) {
    pdl_wait();
    float* r = S + static_cast<long long>(blockIdx.x) * lds;
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
    for (int c = threadIdx.x; c < valid; c += blockDim.x) s += expf(r[c] - mx);
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
    for (int c = threadIdx.x; c < padded; c += blockDim.x) r[c] = c < valid ? expf(r[c] - mx) * inv : 0.f;
}

// the ADX_F32 attention's softmax fused with the split of P: row softmax over the first
// `valid` columns (same reductions as softmax_rows_f32_k) written straight as the A-side
// split operand [hi | hi | lo] (3 x padded bf16 per row): S is read, never written back
__global__ void softmax_split_rows_k(const float* S, long long lds, int valid, int padded, bf16* out) {
    pdl_wait();
    const float* r = S + static_cast<long long>(blockIdx.x) * lds;
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
    for (int c = threadIdx.x; c < valid; c += blockDim.x) s += expf(r[c] - mx);
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
    bf16* o = out + static_cast<long long>(blockIdx.x) * 3 * padded;
    for (int c = threadIdx.x * 8; c < padded; c += blockDim.x * 8) {
        float hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float p = c + k < valid ? expf(r[c + k] - mx) * inv : 0.f;
            hi[k] = __bfloat162float(__float2bfloat16(p));
            lo[k] = p - hi[k];
        }
        const uint4 h = pack8(hi), l = pack8(lo);
        *reinterpret_cast<uint4*>(o + c) = h;
        *reinterpret_cast<uint4*>(o + padded + c) = h;
        *reinterpret_cast<uint4*>(o + 2 * padded + c) = l;
    }
}

__global__ void transpose_f32_k(const float* V, long long ldv, int L, int Lpad, int hd, float* VT) {
    pdl_wait();
    __shared__ float tile[32][33];
    const int k0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, d = d0 + threadIdx.x;
        tile[i][threadIdx.x] = (k < L && d < hd) ? V[static_cast<long long>(k) * ldv + d] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int d = d0 + i, k = k0 + threadIdx.x;
        if (d < hd && k < Lpad) VT[static_cast<long long>(d) * Lpad + k] = tile[threadIdx.x][i];
    }
}

__global__ void cfg_combine_k(const float* e, long long n, float scale, float* out) {
    pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = fmaf(scale, e[n + i] - e[i], e[i]);
}

// Temporal self-attention of the video motion modules (AnimateDiff-shaped, BASELINE config
// 5): for every (pixel, 64-wide head) the NF frames attend to each other.  qkv is the
// frame-major packed projection [NF][HW][3C]; out [NF][HW][C].  Sequences are NF <= 32
// long, far below a tensor-core tile, so this runs on the CUDA cores: one warp per (pixel,
// head), K and V of all frames staged in shared memory as fp32, LPQ lanes per query frame
// each owning 64 / LPQ dimensions (scores reduced over the LPQ lanes by xor shuffles).  fp32
// scores / softmax / accumulation, one rounding at the store; fixed order (deterministic).
template <int NF>
struct TemporalShape {
    static constexpr int LPQ = NF <= 4 ? 8 : NF <= 8 ? 4 : NF <= 16 ? 2 : 1;  // lanes per query
    static constexpr int D = 64 / LPQ;                                         // dims per lane
    static constexpr int WPB = NF > 16 ? 2 : 4;                                // warps per CTA
    static constexpr int SMEM = WPB * NF * 128 * 4;                            // K + V, fp32
};

template <typename T, int NF>  // NF: frame capacity (4, 8, 16, 32); nf <= NF frames present
__global__ void __launch_bounds__(128) temporal_attn_k(const T* qkv, int nf, int HW, int C, T* out) {
    using S = TemporalShape<NF>;
    constexpr int LPQ = S::LPQ, D = S::D;
    pdl_wait();
    extern __shared__ float tsm[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, heads = C / 64;
    const long long item = static_cast<long long>(blockIdx.x) * S::WPB + warp;  // (pixel, head)
    if (item >= static_cast<long long>(HW) * heads) return;                    // warp-uniform
    const int p = static_cast<int>(item / heads), h = static_cast<int>(item % heads);
    float* Ks = tsm + warp * NF * 128;
    float* Vs = Ks + NF * 64;
    const long long ld = 3LL * C;
    {  // nf rows x (8 K + 8 V) vectors of 8: every load issued before the first store
        constexpr int IT = NF / 2;  // NF * 16 vectors / 32 lanes
        typename Vec8<T>::raw u[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int i = lane + 32 * it, f = i / 16, v = i % 16, kv = v / 8, c8 = (v % 8) * 8;
            if (f < nf) u[it] = Vec8<T>::load(qkv + (static_cast<long long>(f) * HW + p) * ld + (1 + kv) * C + h * 64 + c8);
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int i = lane + 32 * it, f = i / 16, v = i % 16, kv = v / 8, c8 = (v % 8) * 8;
            if (f >= nf) continue;
            float x[8];
            Vec8<T>::unpack(u[it], x);
            float4* dst = reinterpret_cast<float4*>((kv ? Vs : Ks) + f * 64 + c8);
            dst[0] = make_float4(x[0], x[1], x[2], x[3]);
            dst[1] = make_float4(x[4], x[5], x[6], x[7]);
        }
    }
    __syncwarp();
    const int qf = lane / LPQ, sub = lane % LPQ;
    const bool active = qf < nf;
    const int qr = active ? qf : nf - 1;  // idle lanes shadow the last query (shuffles stay full-warp)
    float q[D];
    const T* qp = qkv + (static_cast<long long>(qr) * HW + p) * ld + h * 64 + sub * D;
#pragma unroll
    for (int d = 0; d < D; d += 8) Vec8<T>::unpack(Vec8<T>::load(qp + d), q + d);
    float sc[NF];
    float mx = -3.0e38f;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
        const float4* kr = reinterpret_cast<const float4*>(Ks + j * 64 + sub * D);
        float a = 0.f;
#pragma unroll
        for (int d = 0; d < D / 4; ++d) {
            const float4 k4 = kr[d];
            a = fmaf(q[4 * d], k4.x, a);
            a = fmaf(q[4 * d + 1], k4.y, a);
            a = fmaf(q[4 * d + 2], k4.z, a);
            a = fmaf(q[4 * d + 3], k4.w, a);
        }
#pragma unroll
        for (int o = 1; o < LPQ; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        sc[j] = j < nf ? a * 0.125f : -3.0e38f;  // 1 / sqrt(64); absent frames weigh 0
        mx = fmaxf(mx, sc[j]);
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
        sc[j] = j < nf ? expf(sc[j] - mx) : 0.f;
        sum += sc[j];
    }
    const float inv = 1.f / sum;
    float o[D];
#pragma unroll
    for (int d = 0; d < D; ++d) o[d] = 0.f;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
        if (j >= nf) break;
        const float pj = sc[j] * inv;
        const float4* vr = reinterpret_cast<const float4*>(Vs + j * 64 + sub * D);
#pragma unroll
        for (int d = 0; d < D / 4; ++d) {
            const float4 v4 = vr[d];
            o[4 * d] = fmaf(pj, v4.x, o[4 * d]);
            o[4 * d + 1] = fmaf(pj, v4.y, o[4 * d + 1]);
            o[4 * d + 2] = fmaf(pj, v4.z, o[4 * d + 2]);
            o[4 * d + 3] = fmaf(pj, v4.w, o[4 * d + 3]);
        }
    }
    if (!active) return;
    T* op = out + (static_cast<long long>(qf) * HW + p) * C + h * 64 + sub * D;
#pragma unroll
    for (int d = 0; d < D; d += 8) Vec8<T>::store(op + d, Vec8<T>::pack(o + d));
}

// bf16 motion-module attention for up to 16 frames on the tensor cores (mma.sync m16n8k16):
// per (pixel, head) item one warp computes S = Q K^T (16 x 16, K = 64 dims: 2 n8 tiles x 4
// k16 steps) from fragments loaded straight from the packed QKV rows, the row softmax in
// registers (quad shuffles), then O = P V (P re-used from the S accumulators as the A
// fragment, rounded to bf16; V via ldmatrix.trans from a swizzled 2 KB SMEM copy) and
// O / rowsum.  Frames >= nf are zero rows / masked keys.
__device__ __forceinline__ uint32_t ld_b32(const bf16* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(128) temporal_mma_k(const bf16* qkv, int nf, int HW, int C, bf16* out) {
    pdl_wait();
    __shared__ __align__(128) uint8_t vsm[4][16 * 128];  // per warp: V [16 frames][64 dims] bf16, swizzled
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, heads = C / 64;
    const long long item = static_cast<long long>(blockIdx.x) * 4 + warp;
    if (item >= static_cast<long long>(HW) * heads) return;  // warp-uniform
    const int p = static_cast<int>(item / heads), h = static_cast<int>(item % heads);
    const long long fs = static_cast<long long>(HW) * 3 * C;  // frame stride (elements)
    const bf16* qb = qkv + static_cast<long long>(p) * 3 * C + h * 64;
    const int g = lane >> 2, t = lane & 3;
    // V rows -> SMEM (16-byte chunks, chunk c of frame r at (c ^ (r & 7))), zero past nf
    uint8_t* vs = vsm[warp];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int i = lane + 32 * it, r = i >> 3, c = i & 7;
        uint4 u = make_uint4(0, 0, 0, 0);
        if (r < nf) u = *reinterpret_cast<const uint4*>(qb + r * fs + 2 * C + c * 8);
        *reinterpret_cast<uint4*>(vs + r * 128 + ((c ^ (r & 7)) << 4)) = u;
    }
    // S = Q K^T
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    const bool r0ok = g < nf, r1ok = g + 8 < nf;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const int c = ks * 16 + 2 * t;
        uint32_t a[4];
        a[0] = r0ok ? ld_b32(qb + g * fs + c) : 0u;
        a[1] = r1ok ? ld_b32(qb + (g + 8) * fs + c) : 0u;
        a[2] = r0ok ? ld_b32(qb + g * fs + c + 8) : 0u;
        a[3] = r1ok ? ld_b32(qb + (g + 8) * fs + c + 8) : 0u;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int kf = nt * 8 + g;  // key frame of this lane's B column
            const bool ok = kf < nf;
            const uint32_t b0 = ok ? ld_b32(qb + kf * fs + C + c) : 0u;
            const uint32_t b1 = ok ? ld_b32(qb + kf * fs + C + c + 8) : 0u;
            mma16816(sacc[nt], a, b0, b1);
        }
    }
    // softmax over the 16 keys of rows g and g + 8 (quad lanes hold 4 keys each)
    const float sl2 = 0.125f * 1.4426950408889634f;
    float m0 = -3.0e38f, m1 = -3.0e38f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const bool kok = nt * 8 + 2 * t + e < nf;
            sacc[nt][e] = kok ? sacc[nt][e] * sl2 : -3.0e38f;
            sacc[nt][2 + e] = kok ? sacc[nt][2 + e] * sl2 : -3.0e38f;
            m0 = fmaxf(m0, sacc[nt][e]);
            m1 = fmaxf(m1, sacc[nt][2 + e]);
        }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            sacc[nt][e] = exp2f(sacc[nt][e] - m0);
            sacc[nt][2 + e] = exp2f(sacc[nt][2 + e] - m1);
            l0 += sacc[nt][e];
            l1 += sacc[nt][2 + e];
        }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    const uint32_t pa[4] = {pack_bf2(sacc[0][0], sacc[0][1]), pack_bf2(sacc[0][2], sacc[0][3]),
                            pack_bf2(sacc[1][0], sacc[1][1]), pack_bf2(sacc[1][2], sacc[1][3])};
    __syncwarp();
    // O = P V: 8 dim tiles; ldmatrix.x4.trans yields (b0, b1) of two dim tiles
    float oacc[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) oacc[dt][0] = oacc[dt][1] = oacc[dt][2] = oacc[dt][3] = 0.f;
    const uint32_t vbase = static_cast<uint32_t>(__cvta_generic_to_shared(vs));
#pragma unroll
    for (int d2 = 0; d2 < 4; ++d2) {
        const int mtx = lane >> 3, fr = (mtx & 1) * 8 + (lane & 7), ch = 2 * d2 + (mtx >> 1);
        const uint32_t addr = vbase + fr * 128 + ((ch ^ (fr & 7)) << 4);
        uint32_t b[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "r"(addr));
        mma16816(oacc[2 * d2], pa, b[0], b[1]);
        mma16816(oacc[2 * d2 + 1], pa, b[2], b[3]);
    }
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    bf16* ob = out + static_cast<long long>(p) * C + h * 64 + 2 * t;
    const long long os = static_cast<long long>(HW) * C;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
        if (r0ok)
            *reinterpret_cast<uint32_t*>(ob + g * os + dt * 8) = pack_bf2(oacc[dt][0] * i0, oacc[dt][1] * i0);
        if (r1ok)
            *reinterpret_cast<uint32_t*>(ob + (g + 8) * os + dt * 8) = pack_bf2(oacc[dt][2] * i1, oacc[dt][3] * i1);
    }
}

template <typename T, int NF>
void temporal_launch(const T* qkv, int frames, int HW, int C, T* out, cudaStream_t st) {
    if constexpr (NF > 4) {
        if (2 * frames <= NF) return temporal_launch<T, NF / 2>(qkv, frames, HW, C, out, st);
    }
    using S = TemporalShape<NF>;
    const long long items = static_cast<long long>(HW) * (C / 64);
    CKU(launch_pdl(temporal_attn_k<T, NF>, dim3(static_cast<unsigned>((items + S::WPB - 1) / S::WPB)),
                   dim3(32 * S::WPB), S::SMEM, st, 1, qkv, frames, HW, C, out));
    CKU(cudaGetLastError());
}

int grid_for(long long n, int threads = 256) {
    return static_cast<int>(std::min<long long>((n + threads - 1) / threads, 148LL * 16));
}

}  // namespace

template <typename T>
void check_vec8(const Cat2T<T>& x, const char* who) {
    if ((x.c0 % 8) || (x.c1 % 8))
        throw std::invalid_argument(std::string(who) + ": channel segments must be multiples of 8");
}


// GroupNorm(+SiLU) with one thread-block CLUSTER per (image, group): CTA r of the CS-CTA cluster
// owns pixels [r*chunk, (r+1)*chunk) of the group's channels (cpg of the concat, read as pairs
// from whichever segment holds them), keeps them in SMEM while summing (fp32 per thread, fixed
// xor-butterfly per warp, fp64 across warps), the CTAs exchange their (sum, sumsq) over DSMEM
// after one cluster barrier and every CTA folds them in rank order (identical statistics in the
// cluster, deterministic), then applies from SMEM.  No grid-wide barrier and no partials in
// global memory: the cooperative kernel spent ~4 of its ~9 us (level 0) in the grid barrier and
// the fold of 147 CTA partials.
template <typename T>
struct Pair2;
template <>
struct Pair2<bf16> {
    using raw = uint32_t;
    __device__ static raw load(const bf16* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }
    __device__ static float2 unpack(raw u) {
        return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
    }
    __device__ static void store(bf16* p, float2 f) {
        *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(f.x, f.y);
    }
};
template <>
struct Pair2<float> {
    using raw = float2;
    __device__ static raw load(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
    __device__ static float2 unpack(raw u) { return u; }
    __device__ static void store(float* p, float2 f) { *reinterpret_cast<float2*>(p) = f; }
};

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <typename T>
__global__ void __launch_bounds__(256) gn_cluster(Cat2T<T> x, int HW, int groups, int chunk, const float* gamma,
                                                  const float* beta, float eps, int act, T* out) {
    extern __shared__ __align__(16) uint8_t gsm[];
    using P2 = Pair2<T>;
    using Raw = typename P2::raw;
    pdl_wait();
    const int CS = gridDim.x, r = blockIdx.x, g = blockIdx.y, n = blockIdx.z;
    const int C = x.c0 + x.c1, cpg = C / groups, np2 = cpg / 2;
    const int p0 = r * chunk, p1 = min(HW, p0 + chunk), npx = max(0, p1 - p0);
    Raw* tile = reinterpret_cast<Raw*>(gsm);  // [npx][np2]
    double* red = reinterpret_cast<double*>(gsm + ((static_cast<size_t>(chunk) * np2 * sizeof(Raw) + 15) & ~size_t(15)));
    float2* ab = reinterpret_cast<float2*>(red + 24);  // [cpg] (scale, shift)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long base = static_cast<long long>(n) * HW + p0;
    // this thread's (gamma, beta), requested before the statistics (not after the cluster fold)
    const float gm = threadIdx.x < cpg ? __ldg(gamma + g * cpg + threadIdx.x) : 0.f;
    const float bt = threadIdx.x < cpg ? __ldg(beta + g * cpg + threadIdx.x) : 0.f;
    float s = 0.f, ss = 0.f;
    const int total = npx * np2;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int pl = e / np2, j = e - pl * np2;
        const int c = g * cpg + 2 * j;
        const long long pix = base + pl;
        const Raw v = c < x.c0 ? P2::load(x.p0 + pix * x.c0 + c) : P2::load(x.p1 + pix * x.c1 + (c - x.c0));
        tile[e] = v;
        const float2 f = P2::unpack(v);
        s += f.x + f.y;
        ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
    }
    s = warp_sum(s);
    ss = warp_sum(ss);
    if (lane == 0) red[2 * warp] = s, red[2 * warp + 1] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) a += red[2 * w], b += red[2 * w + 1];
        red[16] = a;
        red[17] = b;
    }
    cluster_barrier();  // every CTA's (sum, sumsq) is published in its SMEM
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        const uint32_t mine = static_cast<uint32_t>(__cvta_generic_to_shared(red + 16));
        for (int q = 0; q < CS; ++q) {
            uint32_t addr;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(mine), "r"(q));
            double da, db;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(da) : "r"(addr));
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(db) : "r"(addr + 8));
            a += da;
            b += db;
        }
        const double cnt = static_cast<double>(HW) * cpg;
        const double mu = a / cnt;
        red[18] = mu;
        red[19] = 1.0 / sqrt(fmax(b / cnt - mu * mu, 0.0) + static_cast<double>(eps));
    }
    __syncthreads();
    if (threadIdx.x < cpg) {
        const double rs = red[19];
        ab[threadIdx.x] = make_float2(static_cast<float>(rs * gm), static_cast<float>(bt - red[18] * rs * gm));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int pl = e / np2, j = e - pl * np2;
        const float2 q0 = ab[2 * j], q1 = ab[2 * j + 1];
        float2 f = P2::unpack(tile[e]);
        f.x = fmaf(f.x, q0.x, q0.y);
        f.y = fmaf(f.y, q1.x, q1.y);
        if (act) f.x = silu(f.x), f.y = silu(f.y);
        P2::store(out + (base + pl) * C + g * cpg + 2 * j, f);
    }
    cluster_barrier();  // peers may still read this CTA's partial
}

// cluster GroupNorm (gn_cluster): CS CTAs per (image, group), CS = 4 (8 when a CTA's share of
// the group would not fit in 200 KB of SMEM); returns false (nothing launched) when it cannot run.
// ADX_GN_CLUSTER=0 disables it, =2 uses it for every size.
template <typename T>
bool group_norm_cluster(const Cat2T<T>& x, int batch, int HW, int groups, const float* gamma, const float* beta,
                        float eps, int act, T* out, cudaStream_t st) {
    static const int mode = [] {
        const char* e = getenv("ADX_GN_CLUSTER");
        return e ? atoi(e) : 1;
    }();
    if (!mode || batch > 65535) return false;
    // measured (tools/tools_gn_bench.py): a cluster per group wins on the small low-resolution maps
    // (576 px: 7.8 vs 9.1 us, 144 px x 2560 ch: 5.6 vs 11.8) and loses on the big ones, where 128
    // CTAs reading 20-40-byte channel runs cannot match 147 CTAs streaming whole pixels
    // (9216 px x 320 ch: 20.8 vs 9.9 us) -- so it takes the maps of <= 1024 pixels
    if (mode == 1 && (HW > 1024 || batch > 1)) return false;  // (batches: the stats + apply path measured faster)
    const int C = x.c0 + x.c1, cpg = C / groups;
    if (cpg % 2 || (x.c0 % 2) || cpg > 256) return false;
    const size_t pair = sizeof(T) * 2;
    int CS = 0;
    size_t smem = 0;
    for (int cs : {4, 8}) {
        const int chunk = (HW + cs - 1) / cs;
        const size_t sm = ((static_cast<size_t>(chunk) * (cpg / 2) * pair + 15) & ~size_t(15)) + 24 * 8 + cpg * 8 + 64;
        if (sm <= 200 * 1024) {
            CS = cs;
            smem = sm;
            break;
        }
    }
    if (!CS) return false;
    const int chunk = (HW + CS - 1) / CS;
    int dev = 0;
    CKU(cudaGetDevice(&dev));
    static bool attr[64] = {};
    if (!attr[dev]) {
        CKU(cudaFuncSetAttribute(gn_cluster<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr[dev] = true;
    }
    CKU(launch_pdl(gn_cluster<T>, dim3(CS, groups, batch), dim3(256), smem, st, static_cast<unsigned>(CS), x, HW,
                   groups, chunk, gamma, beta, eps, act, out));
    return true;
}

// one-launch cooperative GroupNorm when the chunk of every SM fits in SMEM (see gn_fused);
// returns false (nothing launched) otherwise.  ADX_GN_FUSED=0 disables it.
template <typename T>
bool group_norm_fused(const Cat2T<T>& x, int HW, int groups, const float* gamma, const float* beta, float eps, int act,
                      T* out, float2* scratch, cudaStream_t st) {
    static const int mode = [] {
        const char* e = getenv("ADX_GN_FUSED");
        return e ? atoi(e) : 1;
    }();
    if (!mode) return false;
    int dev = 0, sms = 0;
    CKU(cudaGetDevice(&dev));
    CKU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int C = x.c0 + x.c1, nv = C / 8;
    if (nv > 512) return false;
    const int chunk_pix = (HW + sms - 1) / sms;
    const int G = (HW + chunk_pix - 1) / chunk_pix;
    const int rpb = std::max(1, 512 / nv), threads = rpb * nv;
    const int nsub = std::max(1, threads / groups);
    const size_t smem = static_cast<size_t>(chunk_pix) * C * sizeof(T) + static_cast<size_t>(2) * rpb * C * 4 +
                        static_cast<size_t>(C) * 8 + static_cast<size_t>(nsub) * groups * 16;
    if (smem > 200 * 1024) return false;
    static bool attr[64] = {};
    if (!attr[dev]) {
        CKU(cudaFuncSetAttribute(gn_fused<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    unsigned n = 1;
    // PDL as well: the CTAs may launch while the producer drains (they wait in pdl_wait);
    // the producer never waits on them, so the co-residency the grid barrier needs follows
    static const bool pdl_coop = [] {
        const char* e = getenv("ADX_GN_PDL");
        return !(e && *e == '0');
    }();
    if (pdl_enabled() && pdl_coop) {
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        n = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    CKU(cudaLaunchKernelEx(&cfg, gn_fused<T>, x, HW, groups, chunk_pix, gamma, beta, eps, act, scratch, out));
    return true;
}

template <typename T>
void group_norm_t(const Cat2T<T>& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                  int silu_act, T* out, float2* scratch, cudaStream_t st) {
    const int C = x.c0 + x.c1;
    if (C % groups) throw std::invalid_argument("group_norm: channels not divisible by groups");
    check_vec8(x, "group_norm");
    const int nv = C / 8;
    if (nv > 1024) throw std::invalid_argument("group_norm: more than 8192 channels");
    if (group_norm_cluster(x, batch, HW, groups, gamma, beta, eps, silu_act, out, st)) {
        tc_profile_measure(st, 3, 2.0 * batch * HW * (x.c0 + x.c1) * sizeof(T), [&](cudaStream_t s2) {
            group_norm_cluster(x, batch, HW, groups, gamma, beta, eps, silu_act, out, s2);
        });
        return;
    }
    if (batch == 1 && group_norm_fused(x, HW, groups, gamma, beta, eps, silu_act, out, scratch, st)) {
        tc_profile_measure(st, 3, 2.0 * HW * (x.c0 + x.c1) * sizeof(T), [&](cudaStream_t s2) {
            group_norm_fused(x, HW, groups, gamma, beta, eps, silu_act, out, scratch, s2);
        });
        return;
    }
    const int chunk_pix = (HW + gn_chunk_cap(batch) - 1) / gn_chunk_cap(batch);
    const int chunks = (HW + chunk_pix - 1) / chunk_pix;
    const int rpb = std::max(1, 512 / nv);
    const int threads = rpb * nv, nsub = std::max(1, threads / (batch * groups));
    size_t smem = static_cast<size_t>(2) * rpb * C * sizeof(float);
    smem = std::max(smem, static_cast<size_t>(nsub + 1) * batch * groups * 2 * sizeof(double));
    if (batch <= kGnImageTickets)  // per-image merge (gn_stats): nsub over one image's groups
        smem = std::max(smem, static_cast<size_t>(std::max(1, threads / groups) + 1) * groups * 2 * sizeof(double));
    if (smem > 48 * 1024) throw std::invalid_argument("group_norm: statistics tile exceeds 48 KB shared memory");
    auto stats = [&](cudaStream_t s2) {
        CKU(launch_pdl(gn_stats<T>, dim3(chunks, batch), dim3(threads), smem, s2, 1, x, HW, groups, chunk_pix, chunks,
                       gamma, beta, eps, scratch));
    };
    stats(st);
    CKU(cudaGetLastError());
    tc_profile_measure(st, 3, 1.0 * batch * HW * C * sizeof(T), stats);  // reads x once
    const GnLayout L = gn_layout(scratch, batch, C);
    const int pixels = batch * HW;
    const int arpb = std::max(1, 256 / nv);
    const int ablocks = static_cast<int>(std::min<long long>(148LL * 8, (pixels + 4LL * arpb - 1) / (4LL * arpb)));
    auto apply = [&](cudaStream_t s2) {
        CKU(launch_pdl(gn_apply<T>, dim3(ablocks), dim3(arpb * nv), 0, s2, 1, x, pixels, HW,
                       static_cast<const float2*>(L.ab), silu_act, out));
    };
    apply(st);
    CKU(cudaGetLastError());
    tc_profile_measure(st, 3, 2.0 * batch * HW * C * sizeof(T), apply);  // reads x, writes y
}

void group_norm(const Cat2& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, __nv_bfloat16* out, float2* scratch, cudaStream_t st) {
    group_norm_t(x, batch, HW, groups, gamma, beta, eps, silu_act, out, scratch, st);
}
void group_norm(const Cat2F& x, int batch, int HW, int groups, const float* gamma, const float* beta, float eps,
                int silu_act, float* out, float2* scratch, cudaStream_t st) {
    group_norm_t(x, batch, HW, groups, gamma, beta, eps, silu_act, out, scratch, st);
}

void gn_timeline(unsigned long long* out, int n) {
#ifdef ADX_GN_TIMELINE
    CKU(cudaDeviceSynchronize());
    CKU(cudaMemcpyFromSymbol(out, g_gn_tl, static_cast<size_t>(std::min(n, 256)) * 64));
#else
    std::memset(out, 0, static_cast<size_t>(n) * 64);
#endif
}

size_t group_norm_scratch_bytes(int batch, int HW, int groups, int C) {
    const int chunk_pix = (std::max(HW, 1) + gn_chunk_cap(batch) - 1) / gn_chunk_cap(batch);
    const int chunks = (HW + chunk_pix - 1) / chunk_pix;
    return (16 + static_cast<size_t>(batch) * C + static_cast<size_t>(batch) * chunks * groups) * sizeof(float2);
}

template <typename T>
void layer_norm_t(const T* x, int tokens, int C, const float* gamma, const float* beta, float eps, T* out,
                  cudaStream_t st) {
    if (C % 8 || C > 256 * kLnMaxVec) throw std::invalid_argument("layer_norm: C must be a multiple of 8, <= 2048");
    auto k = C <= 256 ? layernorm_k<T, 1> : C <= 512 ? layernorm_k<T, 2> : C <= 1024 ? layernorm_k<T, 4>
                                                                                  : layernorm_k<T, kLnMaxVec>;
    CKU(launch_pdl(k, dim3((tokens + 7) / 8), dim3(256), 0, st, 1, x, tokens, C, gamma, beta, eps, out));
    CKU(cudaGetLastError());
    tc_profile_measure(st, 4, 2.0 * tokens * C * sizeof(T), [&](cudaStream_t s2) {
        CKU(launch_pdl(k, dim3((tokens + 7) / 8), dim3(256), 0, s2, 1, x, tokens, C, gamma, beta, eps, out));
    });
}
void layer_norm(const __nv_bfloat16* x, int tokens, int C, const float* gamma, const float* beta, float eps,
                __nv_bfloat16* out, cudaStream_t st) {
    layer_norm_t(x, tokens, C, gamma, beta, eps, out, st);
}
void layer_norm(const float* x, int tokens, int C, const float* gamma, const float* beta, float eps, float* out,
                cudaStream_t st) {
    layer_norm_t(x, tokens, C, gamma, beta, eps, out, st);
}

void split3(const float* x, long long rows, int cols, long long ldx, int g, int pattern, __nv_bfloat16* out,
            cudaStream_t st) {
    if (cols % g || g % 8) throw std::invalid_argument("split3: group width must divide cols and be a multiple of 8");
    CKU(launch_pdl(split3_k, dim3(grid_for(rows * cols / 8)), dim3(256), 0, st, 1, x, rows, cols, ldx, g, pattern,
                   out));
    CKU(cudaGetLastError());
}

void split2(const float* x, long long n, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t st) {
    if (n % 8) throw std::invalid_argument("split2: element count must be a multiple of 8");
    CKU(launch_pdl(split2_k, dim3(grid_for(n / 8)), dim3(256), 0, st, 1, x, n / 8, hi, lo));
    CKU(cudaGetLastError());
}

template <typename T>
void temporal_attention_t(const T* qkv, int frames, int HW, int C, T* out, cudaStream_t st) {
    if (frames < 2 || frames > 32) throw std::invalid_argument("temporal_attention: frames must be in 2..32");
    if (C % 64) throw std::invalid_argument("temporal_attention: channels must be a multiple of 64");
    temporal_launch<T, 32>(qkv, frames, HW, C, out, st);
}
void temporal_attention(const __nv_bfloat16* qkv, int frames, int HW, int C, __nv_bfloat16* out, cudaStream_t st) {
    static const bool cuda_cores = [] {  // ADX_TEMPORAL=cc: the CUDA-core kernel for every frame count
        const char* e = getenv("ADX_TEMPORAL");
        return e && std::string(e) == "cc";
    }();
    if (frames <= 16 && frames >= 2 && C % 64 == 0 && !cuda_cores) {  // tensor-core path
        const long long items = static_cast<long long>(HW) * (C / 64);
        CKU(launch_pdl(temporal_mma_k, dim3(static_cast<unsigned>((items + 3) / 4)), dim3(128), 0, st, 1, qkv, frames,
                       HW, C, out));
        CKU(cudaGetLastError());
        return;
    }
    temporal_attention_t(qkv, frames, HW, C, out, st);
}
void temporal_attention(const float* qkv, int frames, int HW, int C, float* out, cudaStream_t st) {
    temporal_attention_t(qkv, frames, HW, C, out, st);
}

void cfg_combine(const float* e, long long n, float scale, float* out, cudaStream_t st) {
    CKU(launch_pdl(cfg_combine_k, dim3(grid_for(n)), dim3(256), 0, st, 1, e, n, scale, out));
    CKU(cudaGetLastError());
}

void softmax_rows_f32(float* S, long long lds, int rows, int valid, int padded, cudaStream_t st) {
    CKU(launch_pdl(softmax_rows_f32_k, dim3(rows), dim3(256), 0, st, 1, S, lds, valid, padded));
    CKU(cudaGetLastError());
}

void softmax_split_rows(const float* S, long long lds, int rows, int valid, int padded, __nv_bfloat16* out,
                        cudaStream_t st) {
    if (padded % 8) throw std::invalid_argument("softmax_split_rows: padded width must be a multiple of 8");
    CKU(launch_pdl(softmax_split_rows_k, dim3(rows), dim3(256), 0, st, 1, S, lds, valid, padded, out));
    CKU(cudaGetLastError());
}

void transpose_f32(const float* V, long long ldv, int L, int Lpad, int hd, float* VT, cudaStream_t st) {
    CKU(launch_pdl(transpose_f32_k, dim3((Lpad + 31) / 32, (hd + 31) / 32), dim3(32, 8), 0, st, 1, V, ldv, L, Lpad,
                   hd, VT));
    CKU(cudaGetLastError());
}

void pack_latent_f32(const void* x, bool f64, long long pixels, int c_lat, int cpad, float* out, cudaStream_t st) {
    if (f64)
        pack_latent_k<double, float><<<grid_for(pixels * cpad), 256, 0, st>>>(static_cast<const double*>(x), pixels,
                                                                             c_lat, cpad, out);
    else
        pack_latent_k<float, float><<<grid_for(pixels * cpad), 256, 0, st>>>(static_cast<const float*>(x), pixels,
                                                                            c_lat, cpad, out);
    CKU(cudaGetLastError());
}

void softmax_rows(const float* S, long long lds, int rows, int valid, __nv_bfloat16* P, long long ldp, int padded,
                  cudaStream_t st) {
    CKU(launch_pdl(softmax_rows_k, dim3(rows), dim3(256), 0, st, 1, S, lds, valid, P, ldp, padded));
    CKU(cudaGetLastError());
}

void geglu(const __nv_bfloat16* F, long long tokens, int H, __nv_bfloat16* out, cudaStream_t st) {
    if (H % 8) throw std::invalid_argument("geglu: hidden width must be a multiple of 8");
    CKU(launch_pdl(geglu_k, dim3(grid_for(tokens * H / 8)), dim3(256), 0, st, 1, F, tokens, H, out));
    CKU(cudaGetLastError());
}

void upsample2x(const __nv_bfloat16* x, int batch, int H, int W, int C, __nv_bfloat16* out, cudaStream_t st) {
    if (C % 8) throw std::invalid_argument("upsample2x: C must be a multiple of 8");
    CKU(launch_pdl(upsample2x_k, dim3(grid_for(4LL * batch * H * W * C / 8)), dim3(256), 0, st, 1, x, batch, H, W, C,
                   out));
    CKU(cudaGetLastError());
}

void concat_channels(const Cat2& x, long long pixels, __nv_bfloat16* out, cudaStream_t st) {
    check_vec8(x, "concat_channels");
    CKU(launch_pdl(concat_k, dim3(grid_for(pixels * (x.c0 + x.c1) / 8)), dim3(256), 0, st, 1, x, pixels, out));
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
                    cudaStream_t st, int batch) {
    CKU(launch_pdl(transpose_head_k, dim3((Lpad + 31) / 32, (hd + 31) / 32, batch), dim3(32, 8), 0, st, 1, V, ldv, L,
                   Lpad, hd, VT));
    CKU(cudaGetLastError());
}

}  // namespace adx
