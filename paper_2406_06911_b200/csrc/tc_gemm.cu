// tc_gemm.cu -- sm_100a tensor-core GEMM / implicit-GEMM conv for the
// UNet-shaped denoiser family (the conv / QKV / proj / FFN contractions the
// north_star puts on tcgen05).
//
//   D[M x N] (fp32, TMEM) = A[M x K] (bf16, K-major) . B[N x K]^T (bf16, K-major)
//
// One CTA per 128 x BN output tile, 6 warps:
//   warp 0   TMA producer: cp.async.bulk.tensor (2-D for GEMM; 4-D NHWC box
//            loads at tap-shifted coordinates for conv3x3 -- the TMA's
//            out-of-bounds zero fill *is* the conv padding, so no im2col
//            tensor is ever materialised) into a STAGES-deep SMEM ring,
//            128-byte swizzle, one full/empty mbarrier pair per stage;
//   warp 1   TMEM allocator + single-thread MMA issuer: tcgen05.mma
//            .cta_group::1.kind::f16 (M=128, N=BN, K=16 per instruction),
//            tcgen05.commit -> empty[stage] releases the SMEM stage,
//            the last commit -> tmem_full;
//   warps 2-5 epilogue: tcgen05.ld 32x32b (thread = output row), fused
//            bias / per-(image,channel) add / residual / SiLU, bf16 or fp32
//            stores.
#include "tc_gemm.cuh"

#include "pdl.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace adx {

#define CKT(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

bool tma_store_enabled();
bool tma_res_enabled();
bool n_fast_order(long long a_bytes);

namespace {

constexpr int BM = 128, BK = 64;

// -DADX_TC_TIMELINE: %globaltimer stamps per CTA (tools/tools_tc_timeline.py; diagnostics only)
#ifdef ADX_TC_TIMELINE
__device__ unsigned long long g_tl[2048][8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TL(k) (g_tl[blockIdx.x + gridDim.x * blockIdx.y][k] = gtime())
#else
#define TL(k) ((void)0)
#endif
constexpr int kMaxSplitsDev = 8;  // split-K cluster size bound (portable cluster size)
constexpr int EPW_ = 8;           // epilogue warps

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}\n" ::"r"(sa(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bar_arrive1(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sa(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(sa(b))
        : "memory");
}
// SMEM -> global bulk tensor store (bulk-group completion)
__device__ __forceinline__ void tma_store2d(const CUtensorMap* m, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(sa(src))
                 : "memory");
}
__device__ __forceinline__ void tma_store4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(src))
                 : "memory");
}
__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(sa(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(b))
        : "memory");
}
// K-major, 128-byte swizzle UMMA shared-memory descriptor (rows of 128 B,
// 8-row core groups 1024 B apart; version 1 = sm_100)
__device__ __forceinline__ uint64_t sdesc(const void* p) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((sa(p) >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;           // LBO (unused for SW128 K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO
    d |= static_cast<uint64_t>(1) << 46;           // version
    d |= static_cast<uint64_t>(2) << 61;           // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// one 64-deep k block (4 x K16) issued by the elected lane of a converged warp, then the commit
// that releases its SMEM stage: one asm block, descriptors precomputed by every lane (so the
// compiler keeps them warp-uniform), no per-instruction election loop
__device__ __forceinline__ void mma_kblock_commit(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                  uint32_t acc0, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, t;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%11];\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc0), "l"(a + 2), "l"(b + 2), "l"(a + 4), "l"(b + 4), "l"(a + 6),
        "l"(b + 6), "r"(sa(bar))
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* b) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(b))
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

template <int BN>
constexpr uint32_t idesc_bf16() {
    return (1u << 4)                               // D = f32
           | (1u << 7)                             // A = bf16
           | (1u << 10)                            // B = bf16
           | (static_cast<uint32_t>(BN >> 3) << 17)  // N
           | (static_cast<uint32_t>(BM >> 4) << 24); // M
}

template <int BN>
constexpr uint32_t tmem_cols() {
    return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

// x * sigmoid(x) with the MUFU reciprocal: an IEEE division here was a branchy ~15-instruction
// sequence per element (the GroupNorm apply phase's bottleneck); 1 / (1 + e^-x) -> 0 as x -> -inf
__device__ __forceinline__ float silu(float x) { return x * __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }


// --------------------------------------------------------------- epilogue
// output row (pixel) of tile row `row`; false when the row is padding (or an odd
// pixel of a stride-2 conv)
template <bool CONV>
__device__ __forceinline__ bool row_to_m(const TcArgs& p, int tile_m, int img, int h0, int w0, int row,
                                         long long& m) {
    if constexpr (CONV) {
        const int hh = h0 + row / p.box_w, ww = w0 + row % p.box_w;
        // rows past the box (box_w * box_h < 128) hold stale SMEM: computed, never stored
        // (stride-2 convs: H, W are the output grid's; the TMA box already skipped the odd pixels)
        const bool valid = row < p.box_w * p.box_h && hh < p.H && ww < p.W;
        m = (static_cast<long long>(img) * p.H + hh) * p.W + ww;
        return valid;
    } else {
        m = static_cast<long long>(tile_m) * BM + row;
        return m < p.M;
    }
}

__device__ __forceinline__ uint4 pack_bf16x8(const float* v) {
    uint32_t w4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
        w4[k] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    return make_uint4(w4[0], w4[1], w4[2], w4[3]);
}

// the chan_add row output row m reads (per row group, shared, or per image); resolved once
// per tile row by the caller, outside the column loop
__device__ __forceinline__ const float* chan_row(const TcArgs& p, long long m, int img) {
    if (!p.chan_add) return nullptr;
    const int r = p.chan_add_rows ? static_cast<int>(m) / p.chan_add_rows : p.chan_add_shared ? 0 : img;
    return p.chan_add + static_cast<long long>(r) * p.N;
}

// fused epilogue on 16 accumulator columns [nb, nb + 16) of output row m
// bias_base: column-indexed bias (p.bias, or the tile's SMEM-staged copy offset by -n0)
__device__ __forceinline__ void epi16(const TcArgs& p, long long m, const float* ca, int nb, float* v,
                                      const uint4* rpre = nullptr, uint4* sdst = nullptr,
                                      const float* bias_base = nullptr, const float* lncs = nullptr,
                                      float2 ln = make_float2(0.f, 1.f)) {
    const int nlim = p.n_store ? p.n_store : p.N;
    const float* bias = bias_base ? bias_base : p.bias;
    if (lncs) {  // LayerNorm fold: rstd (acc - mean colsum)
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
            const float4 c = *reinterpret_cast<const float4*>(lncs + nb + j);
            v[j] = ln.y * fmaf(-ln.x, c.x, v[j]), v[j + 1] = ln.y * fmaf(-ln.x, c.y, v[j + 1]);
            v[j + 2] = ln.y * fmaf(-ln.x, c.z, v[j + 2]), v[j + 3] = ln.y * fmaf(-ln.x, c.w, v[j + 3]);
        }
    }
    if ((((p.ldo | p.ldr) & 7) == 0) && nb + 16 <= nlim && !p.residual_f32) {
        // vectorised: 16-byte loads / stores
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
            if (bias) {
                const float4 b = *reinterpret_cast<const float4*>(bias + nb + j);
                v[j] += b.x, v[j + 1] += b.y, v[j + 2] += b.z, v[j + 3] += b.w;
            }
            if (ca) {
                const float4 b = *reinterpret_cast<const float4*>(ca + nb + j);
                v[j] += b.x, v[j + 1] += b.y, v[j + 2] += b.z, v[j + 3] += b.w;
            }
        }
        if (p.act == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = silu(v[j]);
        }
        if (p.residual) {
            const uint4* rp = rpre ? rpre : reinterpret_cast<const uint4*>(p.residual + m * p.ldr + nb);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 u = rp[h];
                const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[k]));
                    v[h * 8 + 2 * k] += f.x;
                    v[h * 8 + 2 * k + 1] += f.y;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= p.out_scale;
        if (p.out_f32) {
            float4* op = reinterpret_cast<float4*>(p.out_f32 + m * p.ldo + nb);
#pragma unroll
            for (int j = 0; j < 4; ++j) op[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
            uint4* op = sdst ? sdst : reinterpret_cast<uint4*>(p.out_bf16 + m * p.ldo + nb);
            op[0] = pack_bf16x8(v);
            op[1] = pack_bf16x8(v + 8);
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int n = nb + j;
        if (n >= nlim) continue;
        float x = v[j];
        if (bias) x += bias[n];
        if (ca) x += ca[n];
        if (p.act == 1) x = silu(x);
        if (p.residual) x += __bfloat162float(p.residual[m * p.ldr + n]);
        if (p.residual_f32) x += p.residual_f32[m * p.ldr + n];
        x *= p.out_scale;
        if (p.out_f32)
            p.out_f32[m * p.ldo + n] = x;
        else if (sdst)  // TMA-store staging: the bulk store writes this block
            reinterpret_cast<__nv_bfloat16*>(sdst)[j] = __float2bfloat16(x);
        else
            p.out_bf16[m * p.ldo + n] = __float2bfloat16(x);
    }
}

// packed fp32 pairs (FADD2 / FFMA2): the LayerNorm-fold statistics warps
__device__ __forceinline__ unsigned long long f2add(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float f2lo(unsigned long long a) { return __uint_as_float(static_cast<uint32_t>(a)); }
__device__ __forceinline__ float f2hi(unsigned long long a) { return __uint_as_float(static_cast<uint32_t>(a >> 32)); }
// a bf16 pair word -> the packed fp32 pair (lo, hi)
__device__ __forceinline__ unsigned long long bf2_to_f2(uint32_t w) {
    return static_cast<unsigned long long>(w << 16) | (static_cast<unsigned long long>(w & 0xffff0000u) << 32);
}

// bias / cs: column-indexed bases (the tile's SMEM-staged copies offset by -n0)
// (hb: hidden columns per tile, BN / 2; the gate column of hidden column c is c + hb)
__device__ __forceinline__ void epi_geglu16(const TcArgs& p, long long m, int n0, int c, int hb, float* v, float* g,
                                            const float* bias, const float* cs, float2 ln = make_float2(0.f, 1.f)) {
    if (cs) {  // LayerNorm fold on both halves
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
            const float4 ch = *reinterpret_cast<const float4*>(cs + n0 + c + j);
            const float4 cg = *reinterpret_cast<const float4*>(cs + n0 + hb + c + j);
            v[j] = ln.y * fmaf(-ln.x, ch.x, v[j]), v[j + 1] = ln.y * fmaf(-ln.x, ch.y, v[j + 1]);
            v[j + 2] = ln.y * fmaf(-ln.x, ch.z, v[j + 2]), v[j + 3] = ln.y * fmaf(-ln.x, ch.w, v[j + 3]);
            g[j] = ln.y * fmaf(-ln.x, cg.x, g[j]), g[j + 1] = ln.y * fmaf(-ln.x, cg.y, g[j + 1]);
            g[j + 2] = ln.y * fmaf(-ln.x, cg.z, g[j + 2]), g[j + 3] = ln.y * fmaf(-ln.x, cg.w, g[j + 3]);
        }
    }
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
        const float4 bh = *reinterpret_cast<const float4*>(bias + n0 + c + j);
        const float4 bg = *reinterpret_cast<const float4*>(bias + n0 + hb + c + j);
        v[j] += bh.x, v[j + 1] += bh.y, v[j + 2] += bh.z, v[j + 3] += bh.w;
        g[j] += bg.x, g[j + 1] += bg.y, g[j + 2] += bg.z, g[j + 3] += bg.w;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] *= gelu(g[j]);
    if (p.out_f32) {
        float4* op = reinterpret_cast<float4*>(p.out_f32 + m * p.ldo + n0 / 2 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) op[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        return;
    }
    uint4* op = reinterpret_cast<uint4*>(p.out_bf16 + m * p.ldo + n0 / 2 + c);
    op[0] = pack_bf16x8(v);
    op[1] = pack_bf16x8(v + 8);
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// not volatile / no memory clobber: the staged partials are immutable between the two
// cluster barriers, so the compiler may batch these remote loads (latency ~200 cycles)
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
    float4 v;
    asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
// sum of float4 #j4 of the staged row chunk over all S CTAs, in split order 0..S-1:
// all S loads are issued before the (fixed-order) additions
__device__ __forceinline__ float4 reduce_dsmem4(const uint32_t* a, int S, int off) {
    float4 x[kMaxSplitsDev];
#pragma unroll
    for (int r = 0; r < kMaxSplitsDev; ++r)
        if (r < S) x[r] = ld_dsmem4(a[r] + off);
    float4 acc = x[0];
#pragma unroll
    for (int r = 1; r < kMaxSplitsDev; ++r)
        if (r < S) acc.x += x[r].x, acc.y += x[r].y, acc.z += x[r].z, acc.w += x[r].w;
    return acc;
}

// 16 consecutive floats of the staged row chunk at byte offset `off`, summed over the S CTAs in
// split order 0..S-1 (the same order and rounding as reduce_dsmem4); two splits' 4 float4 loads
// are issued together, so a chunk costs ceil(S / 2) DSMEM round trips instead of 4 ceil(S / 2)
__device__ __forceinline__ void reduce_dsmem16(const uint32_t* a, int S, uint32_t off, float* v) {
    float4 acc[4];
#pragma unroll
    for (int r = 0; r < kMaxSplitsDev; r += 2) {
        if (r >= S) break;
        const bool two = r + 1 < S;
        float4 xa[4], xb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) xa[j] = ld_dsmem4(a[r] + off + 16 * j);
        if (two) {
#pragma unroll
            for (int j = 0; j < 4; ++j) xb[j] = ld_dsmem4(a[r + 1] + off + 16 * j);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (r == 0) {
                acc[j] = xa[j];
            } else {
                acc[j].x += xa[j].x, acc[j].y += xa[j].y, acc[j].z += xa[j].z, acc[j].w += xa[j].w;
            }
            if (two) acc[j].x += xb[j].x, acc[j].y += xb[j].y, acc[j].z += xb[j].z, acc[j].w += xb[j].w;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) v[4 * j] = acc[j].x, v[4 * j + 1] = acc[j].y, v[4 * j + 2] = acc[j].z, v[4 * j + 3] = acc[j].w;
}

// TMA-store staging chunks per epilogue warp (its share of the BN / 16 column chunks);
// BN = 256 tiles do not use the TMA store (no SMEM left beside their pipeline)
template <int BN>
constexpr int kStageChunks() { return BN > 192 ? 0 : (BN / 16 + 1) / 2; }

// SMEM ring depth: as many (A, B) stages as fit one CTA per SM (max dynamic SMEM 227 KB), up to
// 8.  The mainloop is latency-bound, not MMA-bound: a k-block's TMA round trip is ~1 us under
// load (tools/tools_tc_timeline.py), so throughput ~ stages x stage bytes / 1 us; with the
// round-1 ring of 4 every conv / GEMM ran at ~250 ns per k-block whatever its tile width.
// ADX_TC_STAGES (compile time) caps it for A/B runs.
#ifndef ADX_TC_STAGES
#define ADX_TC_STAGES 8
#endif
// PDL: the first ring of weight (B) tiles is requested before griddepcontrol.wait, and the
// MMA warp triggers the dependent launch once its last MMA is issued (A/B switches)
#ifndef ADX_TC_EARLY_B
#define ADX_TC_EARLY_B 0
#endif
#ifndef ADX_TC_TRIGGER
#define ADX_TC_TRIGGER 0
#endif
template <int BN>
constexpr int kStages() {
    constexpr int fixed = 1024 + 256 + EPW_ * kStageChunks<BN>() * 1024 + 16 * BN + 2 * BM * 8;
    constexpr int per = BM * BK * 2 + BN * BK * 2;
    constexpr int fit = (227 * 1024 - fixed) / per;
    return fit < ADX_TC_STAGES ? fit : ADX_TC_STAGES;
}
template <int BN>
constexpr size_t kGemmSmem() {
    return 1024 + static_cast<size_t>(kStages<BN>()) * (BM * BK * 2 + BN * BK * 2) + 256 +
           static_cast<size_t>(EPW_) * kStageChunks<BN>() * 1024 + 16 * BN + 2 * BM * 8;
}

// ------------------------------------------------------------------ kernel
// epilogue warps: EPW / 4 per TMEM lane quadrant, each over its share of the tile's
// 16-column chunks (more loads / stores in flight for the 1-tile-per-CTA small GEMMs)
constexpr int EPW = EPW_;
// LayerNorm-fold statistics warps: compiled in only with -DADX_TC_STATW=2 (384 threads, still 168
// registers).  The default build has none: the fold measured slower than the standalone LayerNorm
// and the two idle warps alone cost 0.2-0.5% of a pass
#ifndef ADX_TC_STATW
#define ADX_TC_STATW 0
#endif
constexpr int kStatWarps = ADX_TC_STATW;
constexpr int kGemmThreads = 64 + 32 * EPW + 32 * kStatWarps;
__device__ __forceinline__ void epi_chunks(int nch, int part, int& c0, int& c1) {
    constexpr int P = EPW / 4;
    c0 = (nch * part) / P * 16;
    c1 = (nch * (part + 1)) / P * 16;
}

template <int BN, bool CONV>
__global__ void __launch_bounds__(kGemmThreads, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ CUtensorMap tmC,
                                                         const __grid_constant__ CUtensorMap tmR, const TcArgs p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (threadIdx.x == 0) TL(0);
    // 1024-byte alignment of the swizzled tiles
    // 1024-byte aligned by offsetting the __shared__ array itself (not through an integer
    // cast), so every access through `smem` stays a shared-space LDS / STS, not a generic LD / ST
    uint8_t* smem = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGES = kStages<BN>();
    constexpr uint32_t ACC_COLS = tmem_cols<BN>();  // one accumulator; two are allocated
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2] accumulator ready for the epilogue
    uint64_t* tempty = tfull + 2;      // [2] accumulator drained by the epilogue
    uint64_t* rbar = tempty + 2;       // [EPW] residual chunks landed in an epilogue warp's staging
    uint64_t* sfull = rbar + EPW;      // [2] LayerNorm-fold row statistics of an accumulator's tile ready
    uint32_t* tptr = reinterpret_cast<uint32_t*>(sfull + 2);  // (barrier block: <= 244 of 256 B)
    // per accumulator: [bias | chan_add] of the tile's BN columns, staged by the epilogue warps
    float* sepi = reinterpret_cast<float*>(sB + STAGES * B_BYTES + 256 + EPW * kStageChunks<BN>() * 1024);
    float2* sstat = reinterpret_cast<float2*>(sepi + 4 * BN);  // [2 accumulators][BM rows] (mean, rstd)
    const bool lnf = !CONV && kStatWarps > 0 && p.ln_colsum != nullptr;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Work units.  S == 1: persistent -- CTA b takes output tiles b, b + G, ... (m fastest,
    // so the CTAs in flight share the B tile) with the TMEM accumulator double-buffered:
    // the epilogue of one tile overlaps the mainloop of the next.  S > 1 (split-K): the
    // S CTAs of one tile form a cluster along x, one unit each; CTA `split` contracts
    // k blocks [kb0, kb1) and the partials are reduced over DSMEM below.
    const int S = p.splits;
    const int split = S > 1 ? static_cast<int>(blockIdx.x % S) : 0;
    int u0, ustride, uend;
    if (S == 1) {
        u0 = blockIdx.x;
        ustride = gridDim.x;
        uend = p.m_tiles * p.n_tiles * p.batch;
    } else {
        u0 = static_cast<int>(blockIdx.x / S) + p.m_tiles * (blockIdx.y + p.n_tiles * blockIdx.z);
        ustride = 1;
        uend = u0 + 1;
    }
    const int kb0 = (p.k_blocks * split) / S, kb1 = (p.k_blocks * (split + 1)) / S;
    const int nkb = kb1 - kb0;
    auto coords = [&](int u, int& tile_m, int& tile_n, int& img, int& h0, int& w0) {
        if (p.n_fast) {  // the CTAs in flight share the A (activation) tile
            tile_n = u % p.n_tiles;
            const int r = u / p.n_tiles;
            tile_m = r % p.m_tiles;
            img = r / p.m_tiles;
        } else {  // the CTAs in flight share the B (weight) tile
            tile_m = u % p.m_tiles;
            const int r = u / p.m_tiles;
            tile_n = r % p.n_tiles;
            img = r / p.n_tiles;
        }
        h0 = w0 = 0;
        if constexpr (CONV) {  // conv tile origin: box_h rows x box_w cols of one image
            const int tiles_w = p.W / p.box_w;
            h0 = (tile_m / tiles_w) * p.box_h;
            w0 = (tile_m % tiles_w) * p.box_w;
        }
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], lnf ? 1 + kStatWarps : 1);  // + the statistics warps' reads
        }
        for (int a = 0; a < 2; ++a) {
            bar_init(&tfull[a], 1);
            bar_init(&tempty[a], EPW);  // one arrival per epilogue warp
            bar_init(&sfull[a], kStatWarps);
        }
        for (int w = 0; w < EPW; ++w) bar_init(&rbar[w], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        if (p.k_split) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmR)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tptr)),
                     "n"(2 * ACC_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tptr;
    if (threadIdx.x == 0) TL(1);
    // prologue done: wait for the producers of A / residual (the TMA thread waits below, after
    // requesting the first weight tiles, which no predecessor writes)
    if (!(warp == 0 && lane == 0)) pdl_wait();
    if (threadIdx.x == 0) TL(2);

    if (warp == 0 && lane == 0) {
        // ---------------------------------------------------------- producer
        constexpr int kEarly = ADX_TC_EARLY_B ? STAGES : 0;
        const int early = u0 < uend ? (nkb < kEarly ? nkb : kEarly) : 0;
        {
            int tile_m, tile_n, img, h0, w0;
            coords(u0, tile_m, tile_n, img, h0, w0);
            for (int i = 0; i < early; ++i) {  // fresh ring: no empty wait
                bar_expect(&full[i], (CONV ? p.box_w * p.box_h * BK * 2 : A_BYTES) + B_BYTES);
                tma2d(sB + i * B_BYTES, &tmB, (kb0 + i) * BK, tile_n * BN, &full[i]);
            }
        }
        pdl_wait();
        int it = 0;  // ring position, continuous across tiles
        for (int u = u0; u < uend; u += ustride) {
            int tile_m, tile_n, img, h0, w0;
            coords(u, tile_m, tile_n, img, h0, w0);
            const int n0 = tile_n * BN;
            for (int i = 0; i < nkb; ++i, ++it) {
                const int kb = kb0 + i, s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                const bool pre = it < early;  // B already requested (and the bytes expected)
                if (!pre) {
                    bar_wait(&empty[s], ph ^ 1);
                    bar_expect(&full[s], (CONV ? p.box_w * p.box_h * BK * 2 : A_BYTES) + B_BYTES);
                }
                if constexpr (CONV) {
                    // k block kb -> tap (r, s) and channel block; A box at the
                    // tap-shifted window (OOB rows/cols are zero-filled = padding)
                    const int cpb = p.cin / BK;
                    const int tap = kb / cpb, cb = kb - tap * cpb;
                    const int dr = tap / 3 - 1, ds = tap % 3 - 1;
                    const int st2 = p.sub2 ? 2 : 1;  // stride 2: input pixel (2h + dr, 2w + ds)
                    tma4d(sA + s * A_BYTES, &tmA, cb * BK, st2 * w0 + ds, st2 * h0 + dr, img, &full[s]);
                } else if (p.k_split && kb * BK >= p.k_split) {  // A = [A1 | A2] along K: A2 rides in tmR
                    tma2d(sA + s * A_BYTES, &tmR, kb * BK - p.k_split, tile_m * BM, &full[s]);
                } else {
                    tma2d(sA + s * A_BYTES, &tmA, kb * BK, tile_m * BM, &full[s]);
                }
                if (!pre) tma2d(sB + s * B_BYTES, &tmB, kb * BK, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        // the whole warp runs the loop (warp-uniform control flow and descriptors); one elected
        // lane issues each k block's 4 MMAs and the commit releasing its stage
        constexpr uint32_t idesc = idesc_bf16<BN>();
        const uint64_t da0 = sdesc(sA), db0 = sdesc(sB);  // stage s, k step k: + (s * bytes + 32 k) >> 4
        int it = 0, lu = 0;
        for (int u = u0; u < uend; u += ustride, ++lu) {
            const int acc = lu & 1;
            bar_wait(&tempty[acc], ((lu >> 1) & 1) ^ 1);  // the epilogue drained this accumulator
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tacc = tmem + acc * ACC_COLS;
            for (int i = 0; i < nkb; ++i, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                bar_wait(&full[s], ph);
                if (it == 0 && lane == 0) TL(3);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                mma_kblock_commit(tacc, da0 + static_cast<uint64_t>((s * A_BYTES) >> 4),
                                  db0 + static_cast<uint64_t>((s * B_BYTES) >> 4), idesc, i != 0 ? 1u : 0u, &empty[s]);
            }
            mma_commit_elect(&tfull[acc]);
        }
        // every MMA of this CTA is issued: let the next kernel of the stream start launching
        // (its CTAs take SMs as ours exit, and its weight TMA overlaps our epilogues)
        if (ADX_TC_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    } else if (warp >= 2 && warp < 2 + EPW) {
        // --------------------------------------------------------- epilogue
        const int q = warp & 3;             // TMEM lane quadrant this warp may access
        const int part = (warp - 2) >> 2;   // which share of the tile's column chunks
        const int row = q * 32 + lane;
        // TMA-store staging: per warp, one 32-row x 16-column bf16 block (1 KB) per chunk of its share
        uint8_t* stage = sB + STAGES * B_BYTES + 256 + (warp - 2) * kStageChunks<BN>() * 1024;
        int lu = 0;
        for (int u = u0; u < uend; u += ustride, ++lu) {
            int tile_m, tile_n, img, h0, w0;
            coords(u, tile_m, tile_n, img, h0, w0);
            const int n0 = tile_n * BN;
            const int acc = lu & 1;
            float2 lnr = make_float2(0.f, 1.f);
            if (p.tma_store && lu > 0) {  // the previous tile's stores have read their staging blocks
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
            }
            // while the mainloop runs: (1) the residual chunks of this warp's share arrive by TMA
            // straight into its staging blocks (the output is written over them in place);
            // (2) the tile's bias / per-image channel-add columns are staged in SMEM -- no
            // dependent global load is left inside the chunk loop
            int rcb = 0, rce = 0;
            if (S == 1 && p.act != 2) epi_chunks(BN / 16, part, rcb, rce);
            if (p.tma_res && S == 1 && p.act != 2 && lane == 0 && rcb < rce) {
                bar_expect(&rbar[warp - 2], (rce - rcb) / 16 * 1024);
                for (int c = rcb; c < rce; c += 16) {
                    uint8_t* dst = stage + ((c - rcb) >> 4) * 1024;
                    if constexpr (CONV)
                        tma4d(dst, &tmR, n0 + c, w0 + (q * 32) % p.box_w, h0 + (q * 32) / p.box_w, img, &rbar[warp - 2]);
                    else
                        tma2d(dst, &tmR, n0 + c, tile_m * BM + q * 32, &rbar[warp - 2]);
                }
            }
            float* sb = sepi + acc * 2 * BN;
#ifndef ADX_TC_GEGLU_STAGE
#define ADX_TC_GEGLU_STAGE 1
#endif
            const bool stage_cols = (ADX_TC_GEGLU_STAGE ? (!CONV || p.act != 2) : p.act != 2) &&
                                    !p.chan_add_rows;  // (S > 1: one tile, acc 0)
            if (stage_cols) {
                const float* car = p.chan_add ? p.chan_add + static_cast<long long>(p.chan_add_shared ? 0 : img) * p.N
                                              : nullptr;
                for (int cidx = threadIdx.x - 64; cidx < BN; cidx += 32 * EPW) {
                    const int n = n0 + cidx;
                    sb[cidx] = p.bias && n < p.N ? p.bias[n] : 0.f;
                    // LayerNorm-fold consumer: colsum(W') in the channel-add slot (never both)
                    sb[BN + cidx] = n >= p.N ? 0.f : !CONV && p.ln_colsum ? p.ln_colsum[n] : car ? car[n] : 0.f;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * EPW) : "memory");  // the epilogue warps
            }
            bar_wait(&tfull[acc], (lu >> 1) & 1);
            if (lu == 0 && threadIdx.x == 64) TL(4);
            if (lnf) {  // this row's LayerNorm statistics from the statistics warps
                bar_wait(&sfull[acc], (lu >> 1) & 1);
                lnr = sstat[acc * BM + row];
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t trow = tmem + acc * ACC_COLS + (static_cast<uint32_t>(q * 32) << 16);
            if (S > 1) {
                // stage this CTA's fp32 partial in its own SMEM (the drained pipeline
                // buffers), rows padded by 4 floats so 8 lanes' float4 stores hit 32 banks
                float* stg = reinterpret_cast<float*>(smem) + row * (BN + 4);
                int cb, ce;
                epi_chunks(BN / 16, part, cb, ce);
                for (int c = cb; c < ce; c += 16) {
                    float v[16];
                    tmem_ld16(trow + c, v);
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(stg + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
            } else {
                long long m;
                const bool valid = row_to_m<CONV>(p, tile_m, img, h0, w0, row, m);
                const float2 ln = lnr;
                if (!CONV && p.act == 2) {
                    int cb, ce;
                    epi_chunks(BN / 32, part, cb, ce);
                    for (int c = cb; c < ce; c += 16) {
                        // hidden and gate columns: two TMEM loads, one wait
                        uint32_t rv[16], rg[16];
                        tmem_ld16_nowait(trow + c, rv);
                        tmem_ld16_nowait(trow + BN / 2 + c, rg);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        float v[16], g[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(rv[i]), g[i] = __uint_as_float(rg[i]);
                        if (valid)
                            epi_geglu16(p, m, n0, c, BN / 2, v, g, stage_cols ? sb - n0 : p.bias,
                                        p.ln_colsum ? (stage_cols ? sb + BN - n0 : p.ln_colsum) : nullptr, ln);
                    }
                } else {
                    // the residual of chunk c+16 is requested before chunk c's TMEM read and
                    // epilogue, so its L2 latency overlaps instead of stalling every chunk
                    const int nlim = p.n_store ? p.n_store : p.N;
#if defined(ADX_EPI_DBG) && ADX_EPI_DBG == 1  // diagnostics: no residual traffic
                    TcArgs pnr = p;
                    pnr.residual = nullptr;
                    const TcArgs& pe = pnr;
#else
                    const TcArgs& pe = p;
#endif
                    // residual: TMA-staged (tma_res), else register-prefetched one chunk ahead
                    const bool tres = p.tma_res != 0;
                    const bool pre = !tres && valid && pe.residual && (((p.ldo | p.ldr) & 7) == 0);
                    const int cb = rcb, ce = rce;
                    uint4 rnext[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
                    if (pre && cb < ce && n0 + cb + 16 <= nlim) {
                        const uint4* rp = reinterpret_cast<const uint4*>(p.residual + m * p.ldr + n0 + cb);
                        rnext[0] = rp[0], rnext[1] = rp[1];
                    }
                    const float* ca = !valid ? nullptr : stage_cols ? (p.chan_add ? sb + BN - n0 : nullptr)
                                                                    : chan_row(p, m, img);
                    const float* bb = stage_cols ? (p.bias ? sb - n0 : nullptr) : p.bias;
                    const float* lncs = CONV || !p.ln_colsum ? nullptr : stage_cols ? sb + BN - n0 : p.ln_colsum;
                    if (!CONV && p.ln_colsum) ca = nullptr;
                    if (tres && cb < ce) bar_wait(&rbar[warp - 2], lu & 1);
                    if (p.tma_store) {
                        // staged epilogue: TMEM chunks in pairs (two loads, one wait), the math written
                        // over the (TMA-loaded) residual in the staging blocks, then ONE proxy fence and
                        // warp sync, and lane 0 issues every bulk store of the share in one group
                        for (int c = cb; c < ce; c += 32) {
                            const bool two = c + 16 < ce;
                            uint32_t r0[16], r1[16];
                            tmem_ld16_nowait(trow + c, r0);
                            if (two) tmem_ld16_nowait(trow + c + 16, r1);
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                if (h == 1 && !two) break;
                                const int cc = c + 16 * h;
                                float v[16];
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(h ? r1[i] : r0[i]);
                                uint4* sd = reinterpret_cast<uint4*>(stage + ((cc - cb) >> 4) * 1024 + lane * 32);
                                // the residual (used only when pe.residual): TMA-staged in sd, or from global
                                uint4 rr[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
                                if (tres) {
                                    rr[0] = sd[0], rr[1] = sd[1];
                                } else if (pre) {
                                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + m * p.ldr + n0 + cc);
                                    rr[0] = rp[0], rr[1] = rp[1];
                                }
                                if (valid) epi16(pe, m, ca, n0 + cc, v, rr, sd, bb, lncs, ln);
                            }
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0 && cb < ce) {
                            for (int c = cb; c < ce; c += 16) {
                                if constexpr (CONV)  // tile rows 32q.. = 32 pixels of the box (32 | bw or bw | 32)
                                    tma_store4d(&tmC, stage + ((c - cb) >> 4) * 1024, n0 + c, w0 + (q * 32) % p.box_w,
                                                h0 + (q * 32) / p.box_w, img);
                                else
                                    tma_store2d(&tmC, stage + ((c - cb) >> 4) * 1024, n0 + c, tile_m * BM + q * 32);
                            }
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    } else {
                        for (int c = cb; c < ce; c += 16) {
                            const uint4 rcur[2] = {rnext[0], rnext[1]};
                            const bool have = pre && n0 + c + 16 <= nlim;
                            if (pre && c + 16 < ce && n0 + c + 32 <= nlim) {
                                const uint4* rp = reinterpret_cast<const uint4*>(p.residual + m * p.ldr + n0 + c + 16);
                                rnext[0] = rp[0], rnext[1] = rp[1];
                            }
                            float v[16];
                            tmem_ld16(trow + c, v);
                            if (valid) epi16(pe, m, ca, n0 + c, v, have ? rcur : nullptr, nullptr, bb, lncs, ln);
                        }
                    }
                }
            }
            // hand the accumulator back to the MMA warp
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive1(&tempty[acc]);
        }
#if !defined(ADX_TL_CHUNK) && !defined(ADX_TL_SPLIT)
        if (threadIdx.x == 64) TL(5);
#endif
        if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#if !defined(ADX_TL_CHUNK) && !defined(ADX_TL_SPLIT)
        if (threadIdx.x == 64) TL(6);
#endif
    } else if (lnf && warp >= 2 + EPW) {
        // ------------------------------------------- LayerNorm-fold statistics (2 warps)
        // thread t owns tile rows t and t + 64: every A k-block of the tile is read from the ring
        // (the 128 B of a row, swizzle order irrelevant to a sum) as soon as it lands, then
        // released; sum x and sum (x - c)^2 with c = a value of the row (shift against
        // cancellation) in packed fp32 pairs; (mean, rstd) per row to sstat[acc]
        const int t = threadIdx.x - (64 + 32 * EPW);
        const float inv_k = 1.f / static_cast<float>(p.k_blocks * BK);
        int it = 0, lu = 0;
        for (int u = u0; u < uend; u += ustride, ++lu) {
            const int acc = lu & 1;
            bar_wait(&tempty[acc], ((lu >> 1) & 1) ^ 1);  // the epilogue read sstat[acc] two tiles ago
            unsigned long long s1[2] = {0ull, 0ull}, s2[2] = {0ull, 0ull}, c2[2] = {0ull, 0ull};
            for (int i = 0; i < nkb; ++i, ++it) {
                const int s = it % STAGES;
                bar_wait(&full[s], (it / STAGES) & 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint4* rp = reinterpret_cast<const uint4*>(sA + s * A_BYTES + (t + 64 * h) * 128);
                    uint4 q[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) q[j] = rp[j];
                    if (i == 0) {  // shift: the row's first stored pair's low value, in both halves
                        const float c = __uint_as_float(q[0].x << 16);
                        c2[h] = static_cast<unsigned long long>(__float_as_uint(-c)) |
                                (static_cast<unsigned long long>(__float_as_uint(-c)) << 32);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const unsigned long long x = bf2_to_f2(w4[k]);
                            const unsigned long long d = f2add(x, c2[h]);
                            s1[h] = f2add(s1[h], x);
                            s2[h] = f2fma(d, d, s2[h]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) bar_arrive1(&empty[s]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float mean = (f2lo(s1[h]) + f2hi(s1[h])) * inv_k;
                const float dm = mean + f2lo(c2[h]);  // mean - c
                const float var = fmaxf((f2lo(s2[h]) + f2hi(s2[h])) * inv_k - dm * dm, 0.f);
                sstat[acc * BM + t + 64 * h] = make_float2(mean, rsqrtf(var + p.ln_eps));
            }
            __syncwarp();
            if (lane == 0) bar_arrive1(&sfull[acc]);
        }
    }
    if (S > 1) {
        // split-K reduction: CTA `split` owns tile rows [r0, r1) and sums the S staged
        // partials in split order 0..S-1 over DSMEM (fixed order: deterministic)
        __syncwarp();
#ifdef ADX_TL_SPLIT
        if (threadIdx.x == 64) TL(5);
#endif
        cluster_sync_all();
#ifdef ADX_TL_SPLIT
        if (threadIdx.x == 64) TL(6);
#endif
        if (warp >= 2 && warp < 2 + EPW) {
            int tile_m, tile_n, img, h0, w0;
            coords(u0, tile_m, tile_n, img, h0, w0);
            const int n0 = tile_n * BN;
            const int r0 = (BM * split) / S, r1 = (BM * (split + 1)) / S;
            const uint32_t base = sa(smem);
            const int et = threadIdx.x - 64;  // 0 .. 32 EPW - 1
            const int cols = p.act == 2 ? BN / 2 : BN, chunks = cols / 16;
            // the S ranks' staging bases (mapa is linear in the offset); bias / channel-add come
            // from this CTA's SMEM copy, the residual is requested with the partials
            uint32_t rb[kMaxSplitsDev];
#pragma unroll
            for (int r = 0; r < kMaxSplitsDev; ++r) rb[r] = mapa(base, r < S ? r : 0);
            const bool sc = (!CONV || p.act != 2) && !p.chan_add_rows;
            const float* bb = sc && p.bias ? sepi - n0 : p.bias;
            for (int it = et; it < (r1 - r0) * chunks; it += 32 * EPW) {
                const int row = r0 + it / chunks, c = (it % chunks) * 16;
                long long m;
                const bool valid = row_to_m<CONV>(p, tile_m, img, h0, w0, row, m);
                if (!valid) continue;
                const bool rv = p.act != 2 && p.residual && !p.residual_f32 && (((p.ldo | p.ldr) & 7) == 0) &&
                                n0 + c + 16 <= (p.n_store ? p.n_store : p.N);
                uint4 res[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
                if (rv) {
                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + m * p.ldr + n0 + c);
                    res[0] = rp[0], res[1] = rp[1];
                }
                float v[16], g[16];
                uint32_t a[kMaxSplitsDev];
                const uint32_t off = static_cast<uint32_t>((row * (BN + 4) + c) * 4);
#pragma unroll
                for (int r = 0; r < kMaxSplitsDev; ++r) a[r] = rb[r] + off;
#ifdef ADX_TC_REDUCE4  // (A/B: the per-float4 reduction)
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const float4 x = reduce_dsmem4(a, S, j * 4);
                    v[j] = x.x, v[j + 1] = x.y, v[j + 2] = x.z, v[j + 3] = x.w;
                }
                if (!CONV && p.act == 2) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const float4 x = reduce_dsmem4(a, S, (BN / 2 + j) * 4);
                        g[j] = x.x, g[j + 1] = x.y, g[j + 2] = x.z, g[j + 3] = x.w;
                    }
                }
#else
                reduce_dsmem16(a, S, 0, v);
                if (!CONV && p.act == 2) reduce_dsmem16(a, S, (BN / 2) * 4, g);
#endif
                const float2 ln = make_float2(0.f, 1.f);  // (LayerNorm-fold GEMMs run unsplit)
                if (!CONV && p.act == 2) {
                    epi_geglu16(p, m, n0, c, BN / 2, v, g, sc ? sepi - n0 : p.bias, nullptr, ln);
                } else {
                    const float* ca = sc ? (p.chan_add ? sepi + BN - n0 : nullptr) : chan_row(p, m, img);
                    epi16(p, m, ca, n0 + c, v, rv ? res : nullptr, nullptr, bb, nullptr, ln);
                }
            }
        }
        __syncwarp();
#ifdef ADX_TL_SPLIT
        if (threadIdx.x == 64) TL(7);
#endif
        cluster_sync_all();  // keep every CTA's SMEM alive until all slices are reduced
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * ACC_COLS)
                     : "memory");
#if !defined(ADX_TL_CHUNK) && !defined(ADX_TL_SPLIT)
    if (threadIdx.x == 0) TL(7);
#endif
}

// --------------------------------------------------------- tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw cuda_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_map(const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                     const cuuint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                     const cuuint32_t* elem_strides = nullptr) {
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (elem_strides)
        for (int i = 0; i < rank; ++i) es[i] = elem_strides[i];
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                                   strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

template <int BN, bool CONV>
void launch_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const CUtensorMap& r, const TcArgs& p,
              dim3 grid, cudaStream_t st) {
    constexpr size_t smem = kGemmSmem<BN>();
    static_assert(static_cast<size_t>(BM) * (BN + 4) * 4 <= kStages<BN>() * (BM * BK * 2 + BN * BK * 2),
                  "split-K staging must fit in the pipeline buffers");
    static_assert(smem <= 227 * 1024, "tc_gemm: SMEM over the per-CTA limit");
    static bool attr[64] = {};
    int dev = 0;
    CKT(cudaGetDevice(&dev));
    if (!attr[dev]) {
        CKT(cudaFuncSetAttribute(tc_gemm_kernel<BN, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr[dev] = true;
    }
    CKT(launch_pdl(tc_gemm_kernel<BN, CONV>, grid, dim3(kGemmThreads), smem, st, static_cast<unsigned>(p.splits), a,
                   b, c, r, p));
}

template <bool CONV>
void dispatch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const CUtensorMap& r, const TcArgs& p,
              dim3 grid, int bn, cudaStream_t st) {
    switch (bn) {
        case 32: launch_t<32, CONV>(a, b, c, r, p, grid, st); break;
        case 64: launch_t<64, CONV>(a, b, c, r, p, grid, st); break;
        case 80: launch_t<80, CONV>(a, b, c, r, p, grid, st); break;
        case 96: launch_t<96, CONV>(a, b, c, r, p, grid, st); break;
        case 128: launch_t<128, CONV>(a, b, c, r, p, grid, st); break;
        case 160: launch_t<160, CONV>(a, b, c, r, p, grid, st); break;
        case 192: launch_t<192, CONV>(a, b, c, r, p, grid, st); break;
        case 256: launch_t<256, CONV>(a, b, c, r, p, grid, st); break;
        default: throw std::invalid_argument("tc_gemm: BN must be 32/64/80/96/128/160/192/256");
    }
}

constexpr int kSMs = 148;

// ADX_TC_TRACE=1: print every launch's tile plan to stderr
bool tc_trace_on() {
    static const bool on = [] {
        const char* e = getenv("ADX_TC_TRACE");
        return e && *e == '1';
    }();
    return on;
}
constexpr int kMaxSplits = kMaxSplitsDev;

// How many S-CTA clusters of tc_gemm_kernel<BN, CONV> the GPU holds at once
// (clusters must fit inside one GPC: e.g. 7-CTA clusters at 1 CTA/SM leave SMs idle)
template <int BN, bool CONV>
int cluster_capacity_t(int S) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    int dev = 0;
    CKT(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, S});
    if (it != cache.end()) return it->second;
    constexpr size_t smem = kGemmSmem<BN>();
    CKT(cudaFuncSetAttribute(tc_gemm_kernel<BN, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S * 64, 1, 1);
    cfg.blockDim = dim3(kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(S);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tc_gemm_kernel<BN, CONV>, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = kSMs / S;  // fall back to the ideal packing
    }
    cache[{dev, S}] = n;
    return n;
}

template <bool CONV>
int cluster_capacity(int bn, int S) {
    switch (bn) {
        case 32: return cluster_capacity_t<32, CONV>(S);
        case 64: return cluster_capacity_t<64, CONV>(S);
        case 80: return cluster_capacity_t<80, CONV>(S);
        case 96: return cluster_capacity_t<96, CONV>(S);
        case 128: return cluster_capacity_t<128, CONV>(S);
        case 160: return cluster_capacity_t<160, CONV>(S);
        case 192: return cluster_capacity_t<192, CONV>(S);
        default: return cluster_capacity_t<256, CONV>(S);
    }
}

// S == 1: persistent grid of min(tiles, resident CTAs); S > 1: one CTA per (tile, split)
template <bool CONV>
dim3 launch_grid(const TcArgs& p, int bn) {
    const long long tiles = static_cast<long long>(p.m_tiles) * p.n_tiles * p.batch;
    if (p.splits > 1) return dim3(p.m_tiles * p.splits, p.n_tiles, p.batch);
    return dim3(static_cast<unsigned>(std::min<long long>(tiles, cluster_capacity<CONV>(bn, 1))), 1, 1);
}

// N tile and split-K factor minimising the modelled time
//   waves x (BN + 64) x ceil(k_blocks / S) x (1.15 if split) (+ 2 k-blocks of reduction)
// where waves = ceil(tiles / concurrent S-clusters) (occupancy query, so GPC packing
// is accounted for) and 64 models the per-tile A-operand cost a narrower tile
// amortises worse.  Every split stages a 128 x BN fp32 partial that the cluster
// reduces over DSMEM -- only worth it when the unsplit grid leaves SMs idle.
// bn_fixed != 0 pins the tile width.
int g_override_bn = 0, g_override_splits = 0;

// Measured plans (tools/tools_tc_tune.py on B200: every (BN, S) timed per shape, best kept).
// GEMM rows: {0, M, N, K, 0, bn, S}; conv rows: {1, H, W, Cin, Cout, bn, S} (batch 1).
struct PlanRow {
    int conv, a, b, c, d, bn, s;
};
constexpr PlanRow kPlanTable[] = {
#include "tc_plan_table.inc"
    {-1, 0, 0, 0, 0, 0, 0}};

bool plan_lookup(int conv, int a, int b, int c, int d, int& bn, int& s) {
    for (const PlanRow& r : kPlanTable)
        if (r.conv == conv && r.a == a && r.b == b && r.c == c && r.d == d) {
            bn = r.bn;
            s = r.s;
            return true;
        }
    return false;
}

template <bool CONV>
void tile_plan(int m_tiles, int N, int batch, int k_blocks, int bn_fixed, int& bn_out, int& s_out) {
    double best = 1e300;
    for (int bn : {256, 192, 160, 128, 64, 32}) {
        if (bn_fixed && bn != bn_fixed) continue;
        if (!bn_fixed && bn < 128 && N > 2 * bn) continue;  // narrow tiles only for narrow outputs
        const long long tiles = static_cast<long long>(m_tiles) * ((N + bn - 1) / bn) * batch;
        for (int S = 1; S <= kMaxSplits; ++S) {
            if (S > 1 && (k_blocks / S < 4 || tiles >= kSMs)) break;
            const long long cap = std::max(1, cluster_capacity<CONV>(bn, S));
            const long long waves = (tiles + cap - 1) / cap;
            const double t = static_cast<double>(waves) * (bn + 64) * ((k_blocks + S - 1) / S) *
                                 (S > 1 ? 1.15 : 1.0) +
                             (S > 1 ? 2.0 * (bn + 64) : 0.0);
            if (t < best - 1e-9) {
                best = t;
                bn_out = bn;
                s_out = S;
            }
        }
    }
}

struct ProfRec {
    int kind;
    double flops, bytes, ms;  // bytes: compulsory HBM traffic (every operand read once, output written once)
};
bool g_prof_on = false;
std::vector<ProfRec> g_prof, g_prof_last;

}  // namespace

void tc_profile_enable(bool on) { g_prof_on = on; }


void tc_plan_override(int bn, int splits) {
    if (bn && bn != 32 && bn != 64 && bn != 80 && bn != 96 && bn != 128 && bn != 160 && bn != 192 && bn != 256)
        throw std::invalid_argument("tc_plan_override: BN must be 0/32/64/80/96/128/160/192/256");
    if (splits < 0 || splits > kMaxSplits) throw std::invalid_argument("tc_plan_override: splits must be 0..8");
    g_override_bn = bn;
    g_override_splits = splits;
}

// Profiling: after the real launch completes, the identical launch is replayed kRep times
// from a CUDA graph on a side stream and timed with events around the replay -- device time
// per launch, warm inputs (as in the pass), no host gaps, no event nodes between kernels.
void tc_profile_measure(cudaStream_t st, int kind, double flops, const std::function<void(cudaStream_t)>& launch) {
    tc_profile_measure(st, kind, flops, kind > 2 ? flops : 0.0, launch);
}
void tc_profile_measure(cudaStream_t st, int kind, double flops, double bytes,
                        const std::function<void(cudaStream_t)>& launch) {
    if (!g_prof_on) return;
    constexpr int kRep = 10;
    CKT(cudaStreamSynchronize(st));
    cudaStream_t s2;
    CKT(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    CKT(cudaStreamBeginCapture(s2, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kRep; ++i) launch(s2);
    CKT(cudaStreamEndCapture(s2, &g));
    CKT(cudaGraphInstantiate(&ge, g, 0));
    CKT(cudaGraphLaunch(ge, s2));  // warm
    cudaEvent_t a, b;
    CKT(cudaEventCreate(&a));
    CKT(cudaEventCreate(&b));
    CKT(cudaEventRecord(a, s2));
    CKT(cudaGraphLaunch(ge, s2));
    CKT(cudaEventRecord(b, s2));
    CKT(cudaEventSynchronize(b));
    float ms = 0.f;
    CKT(cudaEventElapsedTime(&ms, a, b));
    g_prof.push_back({kind, flops, bytes, ms / kRep});
    if (tc_trace_on())
        fprintf(stderr, "  prof kind=%d %.1f us %.1f %s\n", kind, 1e3 * ms / kRep, flops / (ms / kRep) / 1e9,
                kind > 2 ? "GB/s" : "TFLOP/s");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s2);
}

void tc_profile_collect(double out[3][3]) {
    for (int k = 0; k < 3; ++k) out[k][0] = out[k][1] = out[k][2] = 0.0;
    for (auto& r : g_prof) {
        if (r.kind > 2) continue;  // bandwidth kernels (3 GroupNorm, 4 LayerNorm): trace only
        out[r.kind][0] += 1;
        out[r.kind][1] += r.ms;
        out[r.kind][2] += r.flops;
    }
    g_prof_last.swap(g_prof);
    g_prof.clear();
}

int tc_profile_records(double* out, int cap) {
    const int n = static_cast<int>(g_prof_last.size());
    for (int i = 0; i < n && i < cap; ++i) {
        out[4 * i] = g_prof_last[i].kind;
        out[4 * i + 1] = g_prof_last[i].flops;
        out[4 * i + 2] = g_prof_last[i].bytes;
        out[4 * i + 3] = g_prof_last[i].ms;
    }
    return n;
}

// compulsory HBM bytes of one launch: A and B read once, the stored columns of every output
// row written once (+ the residual read); bias / per-channel adds are negligible
static double compulsory_bytes(const TcArgs& p, double a_bytes, double b_bytes, double out_rows) {
    const int cols = p.n_store ? p.n_store : (p.act == 2 ? p.N / 2 : p.N);
    const double ob = p.out_f32 ? 4.0 : 2.0;
    const double rb = p.residual_f32 ? 4.0 : (p.residual ? 2.0 : 0.0);
    return a_bytes + b_bytes + out_rows * cols * (ob + rb);
}

// the conditions under which epi16 takes its vectorised path (16-byte residual loads / stores);
// the TMA-store epilogue is only enabled when they hold (the scalar path stages too, but the
// launcher keeps the fast path the only one the bulk stores see)
static bool vec_epilogue(const TcArgs& p) {
    if (p.residual_f32) return false;
    if (p.residual && ((p.ldr & 7) || (reinterpret_cast<uintptr_t>(p.residual) & 15))) return false;
    return true;
}

// D = A[M x K] . B[N x K]^T ; A, B bf16 row-major (K contiguous), K % 64 == 0
// (bn, S) of a GEMM launch: the tuning override, else the measured plan table, else the model
static void gemm_plan(int M, int N, int K, bool geglu, int& bn, int& S) {
    S = 1;
    if (!geglu && bn == 0 && g_override_bn) {
        bn = g_override_bn;
        S = std::max(1, g_override_splits);
    } else if (geglu) {  // fixed N tile: the measured split (rows {3, ...}), else the model's
        int tbn = 0, ts = 1;
        if (plan_lookup(3, M, N, K, 0, tbn, ts) && tbn == bn)
            S = ts;
        else
            tile_plan<false>((M + BM - 1) / BM, N, 1, K / BK, bn, bn, S);
    } else if (!(bn == 0 && plan_lookup(0, M, N, K, 0, bn, S))) {
        tile_plan<false>((M + BM - 1) / BM, N, 1, K / BK, bn, bn, S);
    }
    if (geglu && g_override_splits) S = g_override_splits;  // the GEGLU tile width stays fixed
    if (S > 1 && (K / BK) / S < 1) S = std::max(1, K / BK);
}

void tc_gemm(const void* A, const void* B, int M, int N, int K, TcArgs p, cudaStream_t st, int bn) {
    tc_gemm_strided(A, K, B, K, M, N, K, p, st, bn);
}

static void gemm_impl(const void* A, long long lda, const void* A2, long long lda2, int k_split, const void* B,
                      long long ldb, int M, int N, int K, TcArgs p, cudaStream_t st, int bn);

bool tc_ln_fold_supported() { return kStatWarps > 0; }

// GEGLU weight-row interleave group (hidden rows per N tile): the N tile is twice this
#ifndef ADX_GEGLU_BN
#define ADX_GEGLU_BN 256
#endif
int tc_geglu_group() { return ADX_GEGLU_BN / 2; }

void tc_gemm_strided(const void* A, long long lda, const void* B, long long ldb, int M, int N, int K, TcArgs p,
                     cudaStream_t st, int bn) {
    gemm_impl(A, lda, nullptr, 0, 0, B, ldb, M, N, K, p, st, bn);
}

void tc_gemm_cat(const void* A1, int K1, const void* A2, int K2, const void* B, int M, int N, TcArgs p,
                 cudaStream_t st, int bn) {
    gemm_impl(A1, K1, A2, K2, K1, B, K1 + K2, M, N, K1 + K2, p, st, bn);
}

// A2 != nullptr: the A operand is [A1 | A2] concatenated along K at column k_split (A1 rows of
// lda elements, A2 rows of lda2); the A2 tensor map takes the residual map's slot (no residual)
static void gemm_impl(const void* A, long long lda, const void* A2, long long lda2, int k_split, const void* B,
                      long long ldb, int M, int N, int K, TcArgs p, cudaStream_t st, int bn) {
    if (K % BK) throw std::invalid_argument("tc_gemm: K must be a multiple of 64");
    if (A2 && (k_split % BK || k_split <= 0 || k_split >= K || lda2 % 8 || p.residual || p.residual_f32))
        throw std::invalid_argument("tc_gemm_cat: K1, K2 must be multiples of 64 and the GEMM has no residual");
    if ((lda | ldb) % 8) throw std::invalid_argument("tc_gemm: row strides must be multiples of 8 elements");
    if (p.act == 2) {  // fused GEGLU (see the epilogue): fixed tiles of [G hidden | G gate], G = tc_geglu_group()
        const int gbn = 2 * tc_geglu_group();
        if (bn && bn != gbn) throw std::invalid_argument("tc_gemm: GEGLU epilogue needs its fixed N tile");
        if (N % gbn || !(p.out_bf16 || p.out_f32) || !p.bias || p.residual || p.residual_f32 || p.chan_add ||
            (p.ldo % 8))
            throw std::invalid_argument("tc_gemm: GEGLU epilogue needs N % tile == 0, bias, no residual, ldo % 8 == 0");
        bn = gbn;
    }
    int S = 1;
    gemm_plan(M, N, K, p.act == 2, bn, S);
    if (p.ln_colsum) S = 1;  // LayerNorm fold: the statistics warps see whole rows of A
    const cuuint64_t da[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
    const cuuint64_t sa_[1] = {static_cast<cuuint64_t>(lda) * 2};
    const cuuint64_t sb_[1] = {static_cast<cuuint64_t>(ldb) * 2};
    const cuuint32_t ba[2] = {BK, BM};
    const cuuint64_t db[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
    const cuuint32_t bb[2] = {BK, static_cast<cuuint32_t>(bn)};
    const cuuint64_t da1[2] = {static_cast<cuuint64_t>(A2 ? k_split : K), static_cast<cuuint64_t>(M)};
    const CUtensorMap ma = make_map(A, 2, da1, sa_, ba), mb = make_map(B, 2, db, sb_, bb);
    p.k_split = A2 ? k_split : 0;
    p.M = M;
    p.N = N;
    p.k_blocks = K / BK;
    p.splits = S;
    p.m_tiles = (M + BM - 1) / BM;
    p.n_tiles = (N + bn - 1) / bn;
    p.batch = 1;
    p.n_fast = S == 1 && p.n_tiles > 1 && n_fast_order(2LL * M * K);
    // bf16 output through SMEM + TMA bulk stores (32 rows x 16 columns per store): full-line
    // writes instead of 32 row-scattered 16-byte stores per warp instruction
    CUtensorMap mc = ma;
    p.tma_store = 0;
    if (tma_store_enabled() && S == 1 && bn <= 192 && p.act != 2 && p.out_bf16 && !p.out_f32 && !p.n_store &&
        N % 16 == 0 && p.ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(p.out_bf16) & 15) == 0 && vec_epilogue(p)) {
        const cuuint64_t dc[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
        const cuuint64_t sc[1] = {static_cast<cuuint64_t>(p.ldo) * 2};
        const cuuint32_t bc[2] = {16, 32};
        mc = make_map(p.out_bf16, 2, dc, sc, bc, CU_TENSOR_MAP_SWIZZLE_NONE);
        p.tma_store = 1;
    }
    CUtensorMap mr = ma;
    p.tma_res = 0;
    if (p.tma_store && p.residual && tma_res_enabled()) {
        const cuuint64_t dr[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
        const cuuint64_t sr[1] = {static_cast<cuuint64_t>(p.ldr) * 2};
        const cuuint32_t br[2] = {16, 32};
        mr = make_map(p.residual, 2, dr, sr, br, CU_TENSOR_MAP_SWIZZLE_NONE);
        p.tma_res = 1;
    }
    if (A2) {  // (no residual: the map slot is free)
        const cuuint64_t da2[2] = {static_cast<cuuint64_t>(K - k_split), static_cast<cuuint64_t>(M)};
        const cuuint64_t sa2[1] = {static_cast<cuuint64_t>(lda2) * 2};
        mr = make_map(A2, 2, da2, sa2, ba);
    }
    if (p.ln_colsum && !tc_ln_fold_supported())
        throw std::invalid_argument("tc_gemm: the LayerNorm fold needs a build with -DADX_TC_STATW=2");
    if (p.ln_colsum && (p.chan_add || N % 16 || S != 1))
        throw std::invalid_argument("tc_gemm: the LayerNorm fold needs an unsplit plan and no chan_add");
    const dim3 grid = launch_grid<false>(p, bn);
    if (tc_trace_on())
        fprintf(stderr, "tc_gemm M=%d N=%d K=%d bn=%d S=%d act=%d grid=%ux%u\n", M, N, K, bn, S, p.act, grid.x, grid.y);
    dispatch<false>(ma, mb, mc, mr, p, grid, bn, st);
    tc_profile_measure(st, 1, 2.0 * M * N * K, compulsory_bytes(p, 2.0 * M * K, 2.0 * N * K, M),
                       [&](cudaStream_t s2) { dispatch<false>(ma, mb, mc, mr, p, grid, bn, s2); });
}

// 3x3 conv, stride 1, pad 1, as an implicit GEMM over NHWC bf16:
//   out[n,h,w,co] = sum_{r,s,ci} X[n,h+r-1,w+s-1,ci] . Wt[co][(r*3+s)*Cin + ci]
// A tiles are 4-D TMA boxes (64 channels x box_w x box_h x 1) at tap-shifted
// coordinates; out-of-range rows/cols arrive as zeros (the padding).
void tc_conv3x3(const void* X, const void* Wt, int batch, int H, int W, int Cin, int Cout, TcArgs p,
                cudaStream_t st, int bn) {
    if (Cin % BK) throw std::invalid_argument("tc_conv3x3: Cin must be a multiple of 64");
    if (p.ln_colsum || p.act == 2)
        throw std::invalid_argument("tc_conv3x3: the LayerNorm fold and GEGLU are GEMM-only");
    // stride 2 (p.sub2): the output grid is (H/2, W/2) and the A boxes are read with TMA element
    // strides of 2 along W and H from input pixel (2 h + dr, 2 w + ds): no discarded rows
    const int Hi = H, Wi = W;
    if (p.sub2) {
        if ((H | W) & 1) throw std::invalid_argument("tc_conv3x3: stride 2 needs even H and W");
        H /= 2;
        W /= 2;
    }
    // box = bw columns x bh rows of output pixels, bw | W, bw * bh <= 128 and a multiple
    // of 8 (whole 1024-byte swizzle atoms); minimise the MMA rows computed per image
    // (e.g. 24 x 24 -> 24 x 5 boxes: 640 rows, not 768 with 8 x 16)
    int bw = 0, bh = 0;
    long long best_rows = 0;
    for (int c = std::min(W, BM); c >= 1; --c) {
        if (W % c) continue;
        for (int r = std::min(BM / c, H); r >= 1; --r) {
            if ((c * r) % 8) continue;
            const long long rows = static_cast<long long>((H + r - 1) / r) * (W / c) * BM;
            if (!bw || rows < best_rows || (rows == best_rows && c * r > bw * bh)) {
                bw = c;
                bh = r;
                best_rows = rows;
            }
            break;  // the tallest legal box for this width
        }
    }
    if (!bw) throw std::invalid_argument("tc_conv3x3: no legal TMA box for this image width");
    const int m_tiles = ((H + bh - 1) / bh) * (W / bw);
    int S = 1;
    if (bn == 0 && g_override_bn) {
        bn = g_override_bn;
        S = std::max(1, g_override_splits);
    } else if (!(bn == 0 && batch == 1 && plan_lookup(p.sub2 ? 2 : 1, Hi, Wi, Cin, Cout, bn, S))) {
        tile_plan<true>(m_tiles, Cout, batch, 9 * Cin / BK, bn, bn, S);
    }
    const cuuint64_t dx[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(Wi), static_cast<cuuint64_t>(Hi),
                              static_cast<cuuint64_t>(batch)};
    const cuuint64_t sx[3] = {static_cast<cuuint64_t>(Cin) * 2, static_cast<cuuint64_t>(Wi) * Cin * 2,
                              static_cast<cuuint64_t>(Hi) * Wi * Cin * 2};
    const cuuint32_t f2 = p.sub2 ? 2 : 1;  // box traversal spans f2 x the loaded pixels
    const cuuint32_t bx[4] = {BK, static_cast<cuuint32_t>(bw) * f2, static_cast<cuuint32_t>(bh) * f2, 1};
    const cuuint32_t ex[4] = {1, f2, f2, 1};
    const int K = 9 * Cin;
    const cuuint64_t dw[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Cout)};
    const cuuint64_t sw[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint32_t bwb[2] = {BK, static_cast<cuuint32_t>(bn)};
    const CUtensorMap ma = make_map(X, 4, dx, sx, bx, CU_TENSOR_MAP_SWIZZLE_128B, ex), mb = make_map(Wt, 2, dw, sw, bwb);
    p.M = batch * H * W;
    p.N = Cout;
    p.k_blocks = K / BK;
    p.H = H;
    p.W = W;
    p.box_w = bw;
    p.box_h = bh;
    p.cin = Cin;
    p.splits = S;
    p.m_tiles = m_tiles;
    p.n_tiles = (Cout + bn - 1) / bn;
    p.batch = batch;
    p.n_fast = S == 1 && p.n_tiles > 1 && n_fast_order(2LL * batch * Hi * Wi * Cin);
    // bf16 NHWC output through SMEM + 4-D TMA bulk stores when a warp's 32 tile rows are one
    // box of pixels (32 | bw or bw | 32, full 128-pixel boxes): the row-per-thread epilogue
    // otherwise issues 32 row-scattered 16-byte stores per warp instruction
    CUtensorMap mc = ma;
    p.tma_store = 0;
    if (tma_store_enabled() && S == 1 && bn <= 192 && p.out_bf16 && !p.out_f32 && !p.n_store &&
        bw * bh == BM && (bw % 32 == 0 || 32 % bw == 0) && Cout % 16 == 0 && p.ldo % 8 == 0 &&
        (reinterpret_cast<uintptr_t>(p.out_bf16) & 15) == 0 && vec_epilogue(p)) {
        const int bx = bw < 32 ? bw : 32;
        const cuuint64_t dc[4] = {static_cast<cuuint64_t>(Cout), static_cast<cuuint64_t>(W),
                                  static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(batch)};
        const cuuint64_t sc[3] = {static_cast<cuuint64_t>(p.ldo) * 2, static_cast<cuuint64_t>(W) * p.ldo * 2,
                                  static_cast<cuuint64_t>(H) * W * p.ldo * 2};
        const cuuint32_t bc[4] = {16, static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(32 / bx), 1};
        mc = make_map(p.out_bf16, 4, dc, sc, bc, CU_TENSOR_MAP_SWIZZLE_NONE);
        p.tma_store = 1;
    }
    CUtensorMap mr = ma;
    p.tma_res = 0;
    if (p.tma_store && p.residual && tma_res_enabled()) {
        const int bx = bw < 32 ? bw : 32;
        const cuuint64_t dr[4] = {static_cast<cuuint64_t>(Cout), static_cast<cuuint64_t>(W),
                                  static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(batch)};
        const cuuint64_t sr[3] = {static_cast<cuuint64_t>(p.ldr) * 2, static_cast<cuuint64_t>(W) * p.ldr * 2,
                                  static_cast<cuuint64_t>(H) * W * p.ldr * 2};
        const cuuint32_t br[4] = {16, static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(32 / bx), 1};
        mr = make_map(p.residual, 4, dr, sr, br, CU_TENSOR_MAP_SWIZZLE_NONE);
        p.tma_res = 1;
    }
    const dim3 grid = launch_grid<true>(p, bn);
    if (tc_trace_on())
        fprintf(stderr, "tc_conv3x3 %s%dx%dx%d->%d box=%dx%d bn=%d S=%d grid=%ux%ux%u tma_store=%d\n",
                p.sub2 ? "stride2 " : "", H, W, Cin, Cout, bw, bh, bn, S, grid.x, grid.y, grid.z, p.tma_store);
    dispatch<true>(ma, mb, mc, mr, p, grid, bn, st);
    // algorithmic FLOPs and compulsory bytes (H, W: the output grid; the input is Hi x Wi)
    tc_profile_measure(st, 0, 2.0 * batch * H * W * Cout * 9.0 * Cin,
                       compulsory_bytes(p, 2.0 * batch * Hi * Wi * Cin, 2.0 * 9 * Cin * Cout,
                                        static_cast<double>(batch) * H * W),
                       [&](cudaStream_t s2) { dispatch<true>(ma, mb, mc, mr, p, grid, bn, s2); });
}

bool tc_trace() { return tc_trace_on(); }

// copy the per-CTA timeline stamps of the last launch (-DADX_TC_TIMELINE builds; else zeros)
void tc_timeline(unsigned long long* out, int n_ctas) {
#ifdef ADX_TC_TIMELINE
    CKT(cudaDeviceSynchronize());
    CKT(cudaMemcpyFromSymbol(out, g_tl, static_cast<size_t>(std::min(n_ctas, 2048)) * 8 * 8));
#else
    std::memset(out, 0, static_cast<size_t>(n_ctas) * 8 * 8);
#endif
}

// ADX_TC_TMA_STORE=0: the GEMM epilogue stores straight from registers
bool tma_store_enabled() {
    static const bool on = [] {
        const char* e = getenv("ADX_TC_TMA_STORE");
        return !(e && *e == '0');
    }();
    return on;
}

// ADX_TC_TMA_RES=0: the residual is register-prefetched from global one chunk ahead instead
bool tma_res_enabled() {
    static const bool on = [] {
        const char* e = getenv("ADX_TC_TMA_RES");
        return !(e && *e == '0');
    }();
    return on;
}

// persistent tile order: n fastest, so the CTAs in flight share (and L2-hit) one A
// (activation) tile and each A tile is consumed while hot -- with m fastest the CTAs sweep
// every A tile once per N tile.  Measured per pass: c2 5.85 -> 5.81 ms, c4 21.68 -> 21.39,
// c5 30.81 -> 30.55 (the weights are small enough to stay L2-resident either way).
// ADX_TC_NFAST=0 restores m-fastest.
bool n_fast_order(long long /*a_bytes*/) {
    static const bool on = [] {
        const char* e = getenv("ADX_TC_NFAST");
        return !(e && *e == '0');
    }();
    return on;
}

}  // namespace adx
