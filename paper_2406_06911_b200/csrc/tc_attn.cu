// tc_attn.cu -- fused multi-head attention on tcgen05 (flash style) for the
// UNet-shaped family: out = softmax(Q K^T / sqrt(64)) V per 64-wide head.
//
// attn_kernel_v2 (default): one CTA per (128-query tile, head, KV split), 10 warps, two CTAs
// per SM (64-key KV blocks, 256 TMEM columns per CTA):
//   warp 0     TMA: the Q tile once; K and V [64 keys x 64 dims] per KV block, straight from
//              the row-major projection output, into a 3-stage SW128 ring;
//   warp 1     TMEM alloc + MMA issue: S = Q K^T (M128 N64 K64) into one of two TMEM S
//              buffers; O_h += P_h V_h with the A operand P read from TMEM (P written over
//              the half's own S columns) and V as an MN-major B operand (no V^T pass);
//   warps 2-9  softmax, two warps per TMEM lane quadrant, each owning half of every block's
//              keys with its own running max / sum and O accumulator (O_0, O_1 in TMEM),
//              merged once after the last block; lazy O rescale (row max grows by > 2^8).
// A (tile, head) grid with a wave tail is split over KV; the last split (ticket) combines
// the partial O / max / sum in split order.  attn_kernel_v2<true> is the f32 mode's
// split-operand variant: Q, K, V as bf16 hi / lo planes, three MMAs per product, P split
// into hi / lo in registers, fp32 output.  attn_kernel (ADX_ATTN_V=1) is the round-1 kernel.
// S never touches HBM.
#include "tc_attn.cuh"

#include "pdl.cuh"

#include "tc_gemm.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <mutex>
#include <stdexcept>
#include <string>

namespace adx {

#define CKA(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

namespace {

// KT = 64 keys per KV block: 100 KB of SMEM and 256 TMEM columns per CTA, so two CTAs
// (20 warps) share an SM and hide each other's barrier / TMEM / MUFU latencies
#ifndef ADX_ATTN_STG
#define ADX_ATTN_STG 3
#endif
constexpr int QT = 128, KT = 64, HD = 64, STG = ADX_ATTN_STG;
// the split-operand kernel carries hi and lo planes of Q, K and V (2x the SMEM per stage):
// a 2-deep KV ring keeps it at two CTAs per SM
constexpr int XSTG = 2;
constexpr int HK = KT / 2;                            // keys per softmax warp (two warps per row)
// V tiles are [KT keys][64 dims] straight from the V rows (SW128, dims contiguous) and feed
// the PV MMA as an MN-major B operand (idesc bit 16; a K=16 step = 16 key rows = 2048 B,
// SBO 1024 B between 8-row swizzle atoms; checked by tools/mn_mma_test.cu): no V^T pass
constexpr int TP_COL = 2 * KT + HD;                  // P[2] (bf16 pairs: KT/2 columns each) after S[2], O
constexpr uint32_t TM_COLS = (TP_COL + KT) <= 256 ? 256 : 512;  // S[2] + O + P[2], power of two

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
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
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
__device__ __forceinline__ uint64_t sdesc(const void* p) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((sa(p) >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(b))
                 : "memory");
}
__device__ __forceinline__ void tld16(uint32_t taddr, float* v) {
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
// 64 consecutive TMEM columns of this thread's lane; no wait (caller batches tcgen05.wait::ld)
#define TLD64_REGS(P)                                                                                          \
    "=r"(P[0]), "=r"(P[1]), "=r"(P[2]), "=r"(P[3]), "=r"(P[4]), "=r"(P[5]), "=r"(P[6]), "=r"(P[7]), "=r"(P[8]), \
        "=r"(P[9]), "=r"(P[10]), "=r"(P[11]), "=r"(P[12]), "=r"(P[13]), "=r"(P[14]), "=r"(P[15]), "=r"(P[16]),  \
        "=r"(P[17]), "=r"(P[18]), "=r"(P[19]), "=r"(P[20]), "=r"(P[21]), "=r"(P[22]), "=r"(P[23]), "=r"(P[24]), \
        "=r"(P[25]), "=r"(P[26]), "=r"(P[27]), "=r"(P[28]), "=r"(P[29]), "=r"(P[30]), "=r"(P[31]), "=r"(P[32]), \
        "=r"(P[33]), "=r"(P[34]), "=r"(P[35]), "=r"(P[36]), "=r"(P[37]), "=r"(P[38]), "=r"(P[39]), "=r"(P[40]), \
        "=r"(P[41]), "=r"(P[42]), "=r"(P[43]), "=r"(P[44]), "=r"(P[45]), "=r"(P[46]), "=r"(P[47]), "=r"(P[48]), \
        "=r"(P[49]), "=r"(P[50]), "=r"(P[51]), "=r"(P[52]), "=r"(P[53]), "=r"(P[54]), "=r"(P[55]), "=r"(P[56]), \
        "=r"(P[57]), "=r"(P[58]), "=r"(P[59]), "=r"(P[60]), "=r"(P[61]), "=r"(P[62]), "=r"(P[63])
__device__ __forceinline__ void tld64_nowait(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,"
        "%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : TLD64_REGS(r)
        : "r"(taddr));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tld32_nowait(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void tst16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 2^x on the FMA / integer pipes: x = n + f, n = rint(x) via the 1.5 * 2^23 trick,
// 2^f on [-0.5, 0.5] by a degree-3 minimax fit (max rel. error 7.5e-5 << bf16's
// 3.9e-3), 2^n added to the exponent field; x clamped at -126 (P ~1e-38: negligible)
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -126.f);
    const float t = x + 12582912.f;
    const int n = __float_as_int(t) - 0x4B400000;
    const float f = x - (t - 12582912.f);
    const float p = fmaf(f, fmaf(f, fmaf(f, 0.05517132f, 0.24261054f), 0.69326097f), 0.99992812f);
    return __int_as_float(__float_as_int(p) + (n << 23));
}
// every POLY_EVERY-th exponential goes to the FMA pipe (0: all on MUFU ex2)
#ifndef ADX_ATTN_POLY_EVERY
#define ADX_ATTN_POLY_EVERY 0
#endif
constexpr int POLY_EVERY = ADX_ATTN_POLY_EVERY;
__device__ __forceinline__ float ex2_mix(float x, int i) {
    if constexpr (POLY_EVERY > 0) {
        constexpr int kEvery = POLY_EVERY > 0 ? POLY_EVERY : 1;
        if (i % kEvery == kEvery - 1) return ex2_poly(x);
    }
    return ex2(x);
}

constexpr uint32_t idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// this warp's HK columns of its S row
__device__ __forceinline__ void tld_hk_nowait(uint32_t taddr, uint32_t* r) {
    if constexpr (HK == 64)
        tld64_nowait(taddr, r);
    else
        tld32_nowait(taddr, r);
}

// D (+)= A . B^T with A (M x K bf16, K-major) read from TMEM: lane = row, one 32-bit
// column = two consecutive K elements, 8 columns per K=16 instruction (checked by
// tools/ts_mma_test.cu); B from SMEM as usual
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
template <int N>
__device__ __forceinline__ void tst_u32(uint32_t taddr, const uint32_t* r) {
    static_assert(N == 16 || N == 32, "tst_u32: 16 or 32 columns");
    if constexpr (N == 16) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                taddr),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
    } else {
        tst_u32<16>(taddr, r);
        tst_u32<16>(taddr + 16, r + 16);
    }
}

struct AttnArgs {
    int L, Lk, C;  // query tokens, key tokens, model width (heads * 64)
    __nv_bfloat16* out;
    long long ldo;
    // split-KV (load balance): nsplit CTAs share one (query tile, head) item, each over a
    // contiguous range of KV blocks; partial O / row max / row sum go to `part`, and the
    // last CTA of the item (ticket in `counters`) combines them in split order
    int nsplit = 1;
    float* part = nullptr;         // [item][split] records of kRecFloats
    float* out_f32 = nullptr;      // split-operand (fp32-exact) kernel: fp32 output instead of `out`
    unsigned* counters = nullptr;  // [item], zero at allocation, re-armed by the combiner
    // stream-K (attn_kernel_sk): the items' KV blocks laid end to end (item = (query tile, head,
    // image), nkv blocks each) and cut into gridDim.x equal ranges, one per CTA; an item cut
    // across ranges is combined like a split-KV item (nsplit = record slots per item)
    int qtiles = 0, heads = 0;
    long long total_blocks = 0;
};
constexpr int kRecFloats = QT * HD + 2 * QT;  // O [128][64] fp32, then m[128], l[128]

__global__ void __launch_bounds__(320, TM_COLS == 256 ? 2 : 1) attn_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                      const __grid_constant__ CUtensorMap tmK,
                                                      const __grid_constant__ CUtensorMap tmV, const AttnArgs p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned by offsetting the __shared__ array itself (not through an integer
    // cast), so every access through `smem` stays a shared-space LDS / STS, not a generic LD / ST
    uint8_t* smem = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
    constexpr int Q_B = QT * HD * 2, K_B = KT * HD * 2, V_B = HD * KT * 2;
    constexpr int XCH_OFF = Q_B + STG * (K_B + V_B) + 256;  // after the barriers
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + Q_B;        // STG x K_B
    uint8_t* sV = sK + STG * K_B;  // STG x (2 halves of [64 dims x 64 keys])
    // P lives in TMEM (the PV MMA's A operand), not SMEM
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + STG * V_B);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;         // [STG]
    uint64_t* kv_empty = kv_full + STG;   // [STG]
    uint64_t* s_full = kv_empty + STG;    // [2] MMA -> softmax
    uint64_t* s_free = s_full + 2;        // [2] softmax -> MMA (S buffer read)
    uint64_t* p_full = s_free + 2;        // [2] softmax -> MMA (P buffer written, O rescaled)
    uint64_t* pv_done = p_full + 2;       // [2] MMA -> softmax: PV_j done (P buffer j&1 free)
    uint32_t* tptr = reinterpret_cast<uint32_t*>(pv_done + 2);
    float* xmax = reinterpret_cast<float*>(smem + XCH_OFF);  // [2 tiles][2 halves][128 rows] partial row max,
                                                             // then [2 halves][128 rows] row sums

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qt = blockIdx.x / p.nsplit, split = blockIdx.x - qt * p.nsplit, head = blockIdx.y, img = blockIdx.z;
    const int nkv_all = (p.Lk + KT - 1) / KT;
    const int j0 = (nkv_all * split) / p.nsplit;  // this CTA's KV blocks [j0, j0 + nkv)
    const int nkv = (nkv_all * (split + 1)) / p.nsplit - j0;

    if (warp == 0 && lane == 0) {
        bar_init(q_full, 1);
        for (int s = 0; s < STG; ++s) {
            bar_init(&kv_full[s], 1);
            bar_init(&kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            bar_init(&s_full[b], 1);
            bar_init(&s_free[b], 8);
            bar_init(&p_full[b], 8);
            bar_init(&pv_done[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tptr)), "n"(TM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pdl_wait();  // prologue done: wait for the producers of Q / K / V^T
    const uint32_t tmem = *tptr;
    // TMEM columns: S buffers [0,KT) and [KT,2KT); O accumulator [2KT, 2KT+64)

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------------------ TMA
        bar_expect(q_full, Q_B);
        tma2d(sQ, &tmQ, head * HD, img * p.L + qt * QT, q_full);  // (a ragged tile reads the next
                                                                   // image's rows; never stored)
        for (int j = 0; j < nkv; ++j) {
            const int s = j % STG;
            bar_wait(&kv_empty[s], ((j / STG) & 1) ^ 1);
            bar_expect(&kv_full[s], K_B + V_B);
            tma2d(sK + s * K_B, &tmK, head * HD, img * p.Lk + (j0 + j) * KT, &kv_full[s]);  // (masked past Lk)
            // V^T rows = this head's 64 dims, one box per 64-key block (128-byte rows)
            tma2d(sV + s * V_B, &tmV, head * HD, img * p.Lk + (j0 + j) * KT, &kv_full[s]);  // (P = 0 past Lk)
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------------------ MMA
        // iteration j issues S_j (overlapping the softmax of S_{j-1}) and PV_{j-1}
        auto issue_s = [&](int j) {
            const int s = j % STG, b = j & 1;
            bar_wait(&kv_full[s], (j / STG) & 1);
            bar_wait(&s_free[b], ((j >> 1) & 1) ^ 1);  // softmax read S_{j-2}
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int k = 0; k < HD / 16; ++k)
                mma(tmem + b * KT, sdesc(sQ + k * 32), sdesc(sK + s * K_B + k * 32), idesc(QT, KT), k > 0);
            commit(&s_full[b]);
        };
        bar_wait(q_full, 0);
        issue_s(0);
        // S_{j+1} is issued before waiting for P_j, so it runs under the softmax of tile j
        for (int j = 1; j <= nkv; ++j) {
            if (j < nkv) issue_s(j);
            {
                const int jj = j - 1, s = jj % STG, b = jj & 1;
                bar_wait(&p_full[b], (jj >> 1) & 1);  // P_jj in SMEM (and O rescaled if needed)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int k = 0; k < KT / 16; ++k)
                    mma_ts(tmem + 2 * KT, tmem + TP_COL + b * (KT / 2) + k * 8, sdesc(sV + s * V_B + k * 2048),
                           idesc(QT, HD) | (1u << 16), (jj | k) > 0);
                commit(&pv_done[b]);
                commit(&kv_empty[s]);
            }
        }
    } else if (warp >= 2) {
        // --------------------------------------------------- softmax + epilogue
        // 8 warps: warp pair (w, w+4) shares TMEM lane quadrant q (rows 32q..32q+31) and
        // splits the 128 keys of a tile in two 64-key halves (two warps per SM
        // sub-partition on one tile); the pair exchanges partial row maxima through
        // SMEM (named barrier 1+q, 64 threads).  O accumulates in TMEM across KV tiles;
        // m is the max the exponentials use and only moves when the row max grows by
        // > 8 (log2 units): the O rescale is rare and P stays <= 2^8.
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = q * 32 + lane;  // query row within the tile
        const uint32_t lrow = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t tO = tmem + 2 * KT + lrow;
        const float sl2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
        auto pair_sync = [&] { asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory"); };
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            const uint32_t tS = tmem + b * KT + half * HK + lrow;
            bar_wait(&s_full[b], (j >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t sr[HK];
            tld_hk_nowait(tS, sr);
            tld_wait();
            // S_j is in registers: release its TMEM buffer to the MMA warp (S_{j+2}) now
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&s_free[b]);
            // ragged last tile: mask the dead keys to -inf once so the hot loops carry no predicates
            const int valid = min(KT, p.Lk - (j0 + j) * KT) - half * HK;
            if (valid < HK) {
#pragma unroll
                for (int i = 0; i < HK; ++i)
                    if (i >= valid) sr[i] = 0xff800000u;
            }
            float mp[8];  // 8 independent max chains
#pragma unroll
            for (int a = 0; a < 8; ++a) mp[a] = __uint_as_float(sr[a]);
#pragma unroll
            for (int i = 8; i < HK; ++i) mp[i & 7] = fmaxf(mp[i & 7], __uint_as_float(sr[i]));
            const float mh = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                   fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            xmax[(b * 2 + half) * QT + r] = mh;
            pair_sync();
            const float mx = fmaxf(mh, xmax[(b * 2 + (half ^ 1)) * QT + r]);
            // P buffer b was last read by PV_{j-2}
            if (j >= 2) bar_wait(&pv_done[b], ((j >> 1) & 1) ^ 1);
            if (j == 0) {
                m = mx;
            } else {
                const bool need = (mx - m) * sl2 > 8.f;
                if (__any_sync(0xffffffffu, need)) {  // rare: rescale O and l to the new max
                    const int qb = (j - 1) & 1;        // O must be final for PV_{j-1}
                    bar_wait(&pv_done[qb], ((j - 1) >> 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const float alpha = need ? ex2((m - mx) * sl2) : 1.f;
#pragma unroll
                    for (int c = 0; c < HD / 2; c += 16) {  // this warp's 32 of the 64 O columns
                        float ov[16];
                        tld16(tO + half * (HD / 2) + c, ov);
#pragma unroll
                        for (int i = 0; i < 16; ++i) ov[i] *= alpha;
                        tst16(tO + half * (HD / 2) + c, ov);
                    }
                    tst_wait();
                    l *= alpha;
                    if (need) m = mx;
                }
            }
            const float off = -m * sl2;
            // P = exp2(s*scale*log2e - m*scale*log2e) as bf16 pairs (keys 2c, 2c+1 in one 32-bit
            // column) straight into this row's TMEM lane: the PV MMA reads its A operand from there
            float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent sum chains
            uint32_t pk[HK / 2];
#pragma unroll
            for (int c = 0; c < HK; c += 2) {
                const float v0 = ex2_mix(fmaf(__uint_as_float(sr[c]), sl2, off), c);
                const float v1 = ex2_mix(fmaf(__uint_as_float(sr[c + 1]), sl2, off), c + 1);
                sp[c & 7] += v0;
                sp[(c + 1) & 7] += v1;
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v0, v1);
                pk[c / 2] = *reinterpret_cast<uint32_t*>(&h2);
            }
            tst_u32<HK / 2>(tmem + TP_COL + b * (KT / 2) + half * (HK / 2) + lrow, pk);
            tst_wait();
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&p_full[b]);
            l += ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
        }
        // epilogue: row sum = half 0 + half 1 (fixed order); O final after the last PV,
        // each warp of the pair normalises and stores 32 of the 64 columns
        float* xsum = xmax + 4 * QT;  // own region: the partner may still read tile nkv-1's maxima
        xsum[half * QT + r] = l;
        pair_sync();
        float lt = xsum[r] + xsum[QT + r];
        bar_wait(&pv_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float ov[HD / 2];
        tld16(tO + half * (HD / 2), ov);
        tld16(tO + half * (HD / 2) + 16, ov + 16);
        const long long row = static_cast<long long>(qt) * QT + r;
        bool write_out = true;
        if (p.nsplit > 1) {
            // publish this split's partial: O (unnormalised), the row max m it used, row sum
            const long long item =
                qt + static_cast<long long>(gridDim.x / p.nsplit) * (head + static_cast<long long>(gridDim.y) * img);
            float* rec = p.part + (item * p.nsplit + split) * kRecFloats;
#pragma unroll
            for (int c = 0; c < HD / 2; c += 4)
                *reinterpret_cast<float4*>(rec + r * HD + half * (HD / 2) + c) =
                    make_float4(ov[c], ov[c + 1], ov[c + 2], ov[c + 3]);
            if (half == 0) rec[QT * HD + r] = m, rec[QT * HD + QT + r] = lt;
            __threadfence();
            __shared__ unsigned last;
            asm volatile("bar.sync 5, 256;" ::: "memory");  // the 8 softmax warps
            if (threadIdx.x == 64)
                last = atomicAdd(p.counters + item, 1u) == static_cast<unsigned>(p.nsplit - 1);
            asm volatile("bar.sync 5, 256;" ::: "memory");
            write_out = last != 0u;
            if (write_out) {
                __threadfence();
                // combine in split order: M = max m_s, w_s = 2^((m_s - M) * scale * log2e),
                // O = sum w_s O_s / sum w_s l_s (deterministic whichever split finishes last)
                const float* base = p.part + item * p.nsplit * kRecFloats;
                float M = -INFINITY;
                for (int s2 = 0; s2 < p.nsplit; ++s2) M = fmaxf(M, __ldcg(base + s2 * kRecFloats + QT * HD + r));
                float acc[HD / 2], den = 0.f;
#pragma unroll
                for (int c = 0; c < HD / 2; ++c) acc[c] = 0.f;
                for (int s2 = 0; s2 < p.nsplit; ++s2) {
                    const float* rs = base + s2 * kRecFloats;
                    const float w = ex2((__ldcg(rs + QT * HD + r) - M) * sl2);
                    den = fmaf(w, __ldcg(rs + QT * HD + QT + r), den);
#pragma unroll
                    for (int c = 0; c < HD / 2; c += 4) {
                        const float4 o4 = __ldcg(reinterpret_cast<const float4*>(rs + r * HD + half * (HD / 2) + c));
                        acc[c] = fmaf(w, o4.x, acc[c]), acc[c + 1] = fmaf(w, o4.y, acc[c + 1]);
                        acc[c + 2] = fmaf(w, o4.z, acc[c + 2]), acc[c + 3] = fmaf(w, o4.w, acc[c + 3]);
                    }
                }
#pragma unroll
                for (int c = 0; c < HD / 2; ++c) ov[c] = acc[c];
                lt = den;
                if (threadIdx.x == 64) p.counters[item] = 0u;  // re-arm for the next launch
            }
        }
        if (write_out && row < p.L) {
            const float inv = 1.0f / lt;
            __nv_bfloat16* dst = p.out + (static_cast<long long>(img) * p.L + row) * p.ldo + head * HD + half * (HD / 2);
#pragma unroll
            for (int c = 0; c < HD / 2; c += 8) {
                uint4 v;
                __nv_bfloat162 b0 = __floats2bfloat162_rn(ov[c] * inv, ov[c + 1] * inv);
                __nv_bfloat162 b1 = __floats2bfloat162_rn(ov[c + 2] * inv, ov[c + 3] * inv);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(ov[c + 4] * inv, ov[c + 5] * inv);
                __nv_bfloat162 b3 = __floats2bfloat162_rn(ov[c + 6] * inv, ov[c + 7] * inv);
                v.x = *reinterpret_cast<uint32_t*>(&b0);
                v.y = *reinterpret_cast<uint32_t*>(&b1);
                v.z = *reinterpret_cast<uint32_t*>(&b2);
                v.w = *reinterpret_cast<uint32_t*>(&b3);
                *reinterpret_cast<uint4*>(dst + c) = v;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS) : "memory");
}

// ---------------------------------------------------------------------------- v2
// Same CTA shape (one 128-query tile x one head x KV split, 10 warps, 2 CTAs per SM, 64-key
// KV blocks), but the two softmax warps of a TMEM lane quadrant no longer meet every block:
// warp half h owns keys [32h, 32h + 32) of every block with its OWN running max m_h, sum l_h
// and O accumulator O_h (TMEM [2KT + 64h, 2KT + 64h + 64)).  O_h = sum_j P_j,h V_j,h is the
// product over that half's keys only; the two partial softmaxes are merged once, after the
// last block (the split-KV combine rule inside the CTA).  P_j,h (bf16 pairs) is written over
// the half's own S_j columns (TMEM budget: S[2] 128 + O[2] 128 = 256 columns).  S_{j+2}
// reuses that buffer: the MMA warp issues it after PV_j (tcgen05.mma from one thread
// execute in issue order), and after the softmax has read S_j (p_full_j precedes PV_j).
template <bool X>
__global__ void __launch_bounds__(320, 2) attn_kernel_v2(const __grid_constant__ CUtensorMap tmQ,
                                                         const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV,
                                                         const __grid_constant__ CUtensorMap tmQl,
                                                         const __grid_constant__ CUtensorMap tmKl,
                                                         const __grid_constant__ CUtensorMap tmVl, const AttnArgs p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
    constexpr int Q_B = QT * HD * 2, K_B = KT * HD * 2, V_B = HD * KT * 2;
    constexpr int XS = X ? 2 : 1;            // operand planes: hi (+ lo)
    constexpr int NS = X ? XSTG : STG;       // KV ring depth
    constexpr int XCH_OFF = XS * Q_B + NS * XS * (K_B + V_B) + 256;
    uint8_t* sQ = smem;                      // [hi | lo]
    uint8_t* sK = sQ + XS * Q_B;             // stage s: [hi | lo] at s * XS * K_B
    uint8_t* sV = sK + NS * XS * K_B;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NS * XS * V_B);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;       // [NS]
    uint64_t* kv_empty = kv_full + NS;  // [NS]
    uint64_t* s_full = kv_empty + NS;   // [2]
    uint64_t* p_full = s_full + 2;       // [2 buffers][2 halves]
    uint64_t* pv_done = p_full + 4;      // [2 buffers][2 halves]
    uint32_t* tptr = reinterpret_cast<uint32_t*>(pv_done + 4);
    float* xml = reinterpret_cast<float*>(smem + XCH_OFF);  // [2 halves][2 (m, l)][128 rows]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qt = blockIdx.x / p.nsplit, split = blockIdx.x - qt * p.nsplit, head = blockIdx.y, img = blockIdx.z;
    const int nkv_all = (p.Lk + KT - 1) / KT;
    const int j0 = (nkv_all * split) / p.nsplit;
    const int nkv = (nkv_all * (split + 1)) / p.nsplit - j0;

    if (warp == 0 && lane == 0) {
        bar_init(q_full, 1);
        for (int s = 0; s < NS; ++s) {
            bar_init(&kv_full[s], 1);
            bar_init(&kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) bar_init(&s_full[b], 1);
        for (int i = 0; i < 4; ++i) {
            bar_init(&p_full[i], 4);  // the 4 warps of one half
            bar_init(&pv_done[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tptr)), "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pdl_wait();
    const uint32_t tmem = *tptr;

    if (warp == 0 && lane == 0) {
        bar_expect(q_full, XS * Q_B);
        tma2d(sQ, &tmQ, head * HD, img * p.L + qt * QT, q_full);
        if constexpr (X) tma2d(sQ + Q_B, &tmQl, head * HD, img * p.L + qt * QT, q_full);
        for (int j = 0; j < nkv; ++j) {
            const int s = j % NS, row = img * p.Lk + (j0 + j) * KT;
            bar_wait(&kv_empty[s], ((j / NS) & 1) ^ 1);
            bar_expect(&kv_full[s], XS * (K_B + V_B));
            tma2d(sK + s * XS * K_B, &tmK, head * HD, row, &kv_full[s]);
            tma2d(sV + s * XS * V_B, &tmV, head * HD, row, &kv_full[s]);
            if constexpr (X) {
                tma2d(sK + s * XS * K_B + K_B, &tmKl, head * HD, row, &kv_full[s]);
                tma2d(sV + s * XS * V_B + V_B, &tmVl, head * HD, row, &kv_full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {
        auto issue_s = [&](int j) {
            const int s = j % NS, b = j & 1;
            bar_wait(&kv_full[s], (j / NS) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint8_t* kh = sK + s * XS * K_B;
#pragma unroll
            for (int k = 0; k < HD / 16; ++k) {
                mma(tmem + b * KT, sdesc(sQ + k * 32), sdesc(kh + k * 32), idesc(QT, KT), k > 0);
                if constexpr (X) {  // S = Qh Kh^T + Qh Kl^T + Ql Kh^T (fp32 in TMEM)
                    mma(tmem + b * KT, sdesc(sQ + k * 32), sdesc(kh + K_B + k * 32), idesc(QT, KT), 1u);
                    mma(tmem + b * KT, sdesc(sQ + Q_B + k * 32), sdesc(kh + k * 32), idesc(QT, KT), 1u);
                }
            }
            commit(&s_full[b]);
        };
        bar_wait(q_full, 0);
        issue_s(0);
        for (int j = 1; j <= nkv; ++j) {
            if (j < nkv) issue_s(j);  // after PV_{j-2} in issue order: S_j may overwrite P_{j-2}
            const int jj = j - 1, s = jj % NS, b = jj & 1;
            const uint8_t* vh = sV + s * XS * V_B;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                bar_wait(&p_full[b * 2 + h], (jj >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int k = 2 * h; k < 2 * h + 2; ++k) {  // keys [16k, 16k + 16) of the block
                    const uint32_t ph = tmem + b * KT + h * HK + (k & 1) * 8, od = tmem + 2 * KT + h * HD;
                    constexpr uint32_t id = idesc(QT, HD) | (1u << 16);
                    mma_ts(od, ph, sdesc(vh + k * 2048), id, (jj > 0 || (k & 1)) ? 1u : 0u);
                    if constexpr (X) {  // O += Ph Vl + Pl Vh (P lo 16 columns after P hi)
                        mma_ts(od, ph, sdesc(vh + V_B + k * 2048), id, 1u);
                        mma_ts(od, ph + HK / 2, sdesc(vh + k * 2048), id, 1u);
                    }
                }
                commit(&pv_done[b * 2 + h]);
            }
            commit(&kv_empty[s]);
        }
    } else if (warp >= 2) {
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = q * 32 + lane;
        const uint32_t lrow = static_cast<uint32_t>(q * 32) << 16;
        const float sl2 = 0.125f * 1.4426950408889634f;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            const uint32_t tS = tmem + b * KT + half * HK + lrow;
            bar_wait(&s_full[b], (j >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t sr[HK];
            tld_hk_nowait(tS, sr);
            tld_wait();
            const int valid = min(KT, p.Lk - (j0 + j) * KT) - half * HK;
            if (valid < HK) {
#pragma unroll
                for (int i = 0; i < HK; ++i)
                    if (i >= valid) sr[i] = 0xff800000u;
            }
            float mp[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) mp[a] = __uint_as_float(sr[a]);
#pragma unroll
            for (int i = 8; i < HK; ++i) mp[i & 7] = fmaxf(mp[i & 7], __uint_as_float(sr[i]));
            const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                   fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            // lazy rescale of this half's O: only when its row max grows by > 2^8
            const bool need = mx > m && (m == -INFINITY || (mx - m) * sl2 > 8.f);
            if (__any_sync(0xffffffffu, need)) {
                if (j > 0) {  // O_h must hold PV_{j-1},h
                    bar_wait(&pv_done[((j - 1) & 1) * 2 + half], ((j - 1) >> 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const float alpha = need ? (m == -INFINITY ? 0.f : ex2((m - mx) * sl2)) : 1.f;
                    const uint32_t tO = tmem + 2 * KT + half * HD + lrow;
#pragma unroll
                    for (int c = 0; c < HD; c += 16) {
                        float ov[16];
                        tld16(tO + c, ov);
#pragma unroll
                        for (int i = 0; i < 16; ++i) ov[i] *= alpha;
                        tst16(tO + c, ov);
                    }
                    tst_wait();
                    l *= alpha;
                }
                if (need) m = mx;
            }
            const float off = m == -INFINITY ? 0.f : -m * sl2;  // (a fully masked half: P = 0)
            float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            uint32_t pk[HK / 2], pl[X ? HK / 2 : 1];
#pragma unroll
            for (int c = 0; c < HK; c += 2) {
                const float v0 = ex2_mix(fmaf(__uint_as_float(sr[c]), sl2, off), c);
                const float v1 = ex2_mix(fmaf(__uint_as_float(sr[c + 1]), sl2, off), c + 1);
                sp[c & 7] += v0;
                sp[(c + 1) & 7] += v1;
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v0, v1);
                pk[c / 2] = *reinterpret_cast<uint32_t*>(&h2);
                if constexpr (X) {  // P = hi + lo to ~2^-17
                    __nv_bfloat162 l2 = __floats2bfloat162_rn(v0 - __low2float(h2), v1 - __high2float(h2));
                    pl[c / 2] = *reinterpret_cast<uint32_t*>(&l2);
                }
            }
            tst_u32<HK / 2>(tS, pk);  // P_j,h over the S_j,h columns just read
            if constexpr (X) tst_u32<HK / 2>(tS + HK / 2, pl);
            tst_wait();
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&p_full[b * 2 + half]);
            l += ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
        }
        // merge the two halves: M = max(m0, m1), w_h = 2^((m_h - M) log2e / 8), O = w0 O0 + w1 O1,
        // row sum w0 l0 + w1 l1; warp half h finishes output columns [32h, 32h + 32)
        xml[(half * 2 + 0) * QT + r] = m;
        xml[(half * 2 + 1) * QT + r] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        const float m0 = xml[0 * QT + r], l0 = xml[1 * QT + r], m1 = xml[2 * QT + r], l1 = xml[3 * QT + r];
        const float M = fmaxf(m0, m1);
        const float w0 = m0 == -INFINITY ? 0.f : ex2((m0 - M) * sl2);
        const float w1 = m1 == -INFINITY ? 0.f : ex2((m1 - M) * sl2);
        float lt = w0 * l0 + w1 * l1;
        const int lb = (nkv - 1) & 1;
        bar_wait(&pv_done[lb * 2 + 0], ((nkv - 1) >> 1) & 1);
        bar_wait(&pv_done[lb * 2 + 1], ((nkv - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float ov[HD / 2];
        const uint32_t tO0 = tmem + 2 * KT + lrow + half * (HD / 2);
        {  // both halves' O columns: two TMEM loads, one wait
            uint32_t r0[HD / 2], r1[HD / 2];
            tld32_nowait(tO0, r0);
            tld32_nowait(tO0 + HD, r1);
            tld_wait();
#pragma unroll
            for (int c = 0; c < HD / 2; ++c) ov[c] = w0 * __uint_as_float(r0[c]) + w1 * __uint_as_float(r1[c]);
        }
        const float mrow = M;
        const long long row = static_cast<long long>(qt) * QT + r;
        bool write_out = true;
        if (p.nsplit > 1) {
            const long long item =
                qt + static_cast<long long>(gridDim.x / p.nsplit) * (head + static_cast<long long>(gridDim.y) * img);
            float* rec = p.part + (item * p.nsplit + split) * kRecFloats;
#pragma unroll
            for (int c = 0; c < HD / 2; c += 4)
                *reinterpret_cast<float4*>(rec + r * HD + half * (HD / 2) + c) =
                    make_float4(ov[c], ov[c + 1], ov[c + 2], ov[c + 3]);
            if (half == 0) rec[QT * HD + r] = mrow, rec[QT * HD + QT + r] = lt;
            __threadfence();
            __shared__ unsigned last2;
            asm volatile("bar.sync 5, 256;" ::: "memory");
            if (threadIdx.x == 64)
                last2 = atomicAdd(p.counters + item, 1u) == static_cast<unsigned>(p.nsplit - 1);
            asm volatile("bar.sync 5, 256;" ::: "memory");
            write_out = last2 != 0u;
            if (write_out) {
                __threadfence();
                const float* base = p.part + item * p.nsplit * kRecFloats;
                float MM = -INFINITY;
                for (int s2 = 0; s2 < p.nsplit; ++s2) MM = fmaxf(MM, __ldcg(base + s2 * kRecFloats + QT * HD + r));
                float acc[HD / 2], den = 0.f;
#pragma unroll
                for (int c = 0; c < HD / 2; ++c) acc[c] = 0.f;
                for (int s2 = 0; s2 < p.nsplit; ++s2) {
                    const float* rs = base + s2 * kRecFloats;
                    const float ms = __ldcg(rs + QT * HD + r);
                    const float w = ms == -INFINITY ? 0.f : ex2((ms - MM) * sl2);
                    den = fmaf(w, __ldcg(rs + QT * HD + QT + r), den);
#pragma unroll
                    for (int c = 0; c < HD / 2; c += 4) {
                        const float4 o4 = __ldcg(reinterpret_cast<const float4*>(rs + r * HD + half * (HD / 2) + c));
                        acc[c] = fmaf(w, o4.x, acc[c]), acc[c + 1] = fmaf(w, o4.y, acc[c + 1]);
                        acc[c + 2] = fmaf(w, o4.z, acc[c + 2]), acc[c + 3] = fmaf(w, o4.w, acc[c + 3]);
                    }
                }
#pragma unroll
                for (int c = 0; c < HD / 2; ++c) ov[c] = acc[c];
                lt = den;
                if (threadIdx.x == 64) p.counters[item] = 0u;
            }
        }
        if (X && write_out && row < p.L) {
            const float inv = 1.0f / lt;
            float* dst = p.out_f32 + (static_cast<long long>(img) * p.L + row) * p.ldo + head * HD + half * (HD / 2);
#pragma unroll
            for (int c = 0; c < HD / 2; c += 4)
                *reinterpret_cast<float4*>(dst + c) =
                    make_float4(ov[c] * inv, ov[c + 1] * inv, ov[c + 2] * inv, ov[c + 3] * inv);
        } else if (write_out && row < p.L) {
            const float inv = 1.0f / lt;
            __nv_bfloat16* dst = p.out + (static_cast<long long>(img) * p.L + row) * p.ldo + head * HD + half * (HD / 2);
#pragma unroll
            for (int c = 0; c < HD / 2; c += 8) {
                uint4 v;
                __nv_bfloat162 b0 = __floats2bfloat162_rn(ov[c] * inv, ov[c + 1] * inv);
                __nv_bfloat162 b1 = __floats2bfloat162_rn(ov[c + 2] * inv, ov[c + 3] * inv);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(ov[c + 4] * inv, ov[c + 5] * inv);
                __nv_bfloat162 b3 = __floats2bfloat162_rn(ov[c + 6] * inv, ov[c + 7] * inv);
                v.x = *reinterpret_cast<uint32_t*>(&b0);
                v.y = *reinterpret_cast<uint32_t*>(&b1);
                v.z = *reinterpret_cast<uint32_t*>(&b2);
                v.w = *reinterpret_cast<uint32_t*>(&b3);
                *reinterpret_cast<uint4*>(dst + c) = v;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
}


// ---------------------------------------------------------------------- stream-K
// -DADX_SK_TIMELINE: %globaltimer stamps of the first softmax thread of every CTA (diagnostics)
#ifdef ADX_SK_TIMELINE
__device__ unsigned long long g_sk_tl[512 * 16];
__device__ __forceinline__ void sk_stamp(int i) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (i < 16) g_sk_tl[blockIdx.x * 16 + i] = t;
}
#define SK_TL(i) \
    if (threadIdx.x == 64) sk_stamp(i)
#else
#define SK_TL(i)
#endif
// attn_kernel_v2's CTA (10 warps, two per SM, same TMEM / SMEM plan) run persistently over a
// contiguous range of the (item, KV block) sequence instead of one item: every CTA gets the
// same number of KV blocks (+-1), so a grid of items that does not fill the SMs evenly (level 0:
// 360 items over 296 slots; SDXL level 2: 320) has no wave tail.  Per segment (the part of
// one item inside the range): Q is loaded into one of two Q buffers (the next segment's Q
// overlaps this one's MMAs), the softmax state restarts, and at its end the output is written
// (whole item) or published as a partial record whose last-arriving segment combines all of
// them in segment order (deterministic).  Barrier phases run on the CTA's global block count.
// K/V ring depth of the stream-K kernel (ADX_ATTN_SKSTG for A/B)
#ifndef ADX_ATTN_SKSTG
#define ADX_ATTN_SKSTG 3
#endif
constexpr int SKSTG = ADX_ATTN_SKSTG;
// (block counts fit 32 bits: the launcher checks total < 2^31 / G)
__device__ __forceinline__ int sk_b0(int c, int total, int G) {
    return static_cast<int>(static_cast<long long>(c) * total / G);
}
// the CTA whose range holds block x
__device__ __forceinline__ int sk_cta(int x, int total, int G) {
    int c = static_cast<int>(static_cast<long long>(x) * G / total);
    while (c + 1 < G && sk_b0(c + 1, total, G) <= x) ++c;
    while (c > 0 && sk_b0(c, total, G) > x) --c;
    return c;
}

__global__ void __launch_bounds__(320, 2) attn_kernel_sk(const __grid_constant__ CUtensorMap tmQ,
                                                         const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV, const AttnArgs p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
    constexpr int Q_B = QT * HD * 2, K_B = KT * HD * 2, V_B = HD * KT * 2;
    constexpr int XCH_OFF = 2 * Q_B + SKSTG * (K_B + V_B) + 256;
    uint8_t* sQ = smem;  // [2] Q buffers
    uint8_t* sK = sQ + 2 * Q_B;
    uint8_t* sV = sK + SKSTG * K_B;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + SKSTG * V_B);
    uint64_t* q_full = bars;              // [2]
    uint64_t* q_empty = q_full + 2;       // [2] the S MMAs of the buffer's segment are done
    uint64_t* kv_full = q_empty + 2;      // [SKSTG]
    uint64_t* kv_empty = kv_full + SKSTG;   // [SKSTG]
    uint64_t* s_full = kv_empty + SKSTG;    // [2]
    uint64_t* p_full = s_full + 2;        // [2 buffers][2 halves]
    uint64_t* pv_done = p_full + 4;       // [2 buffers][2 halves]
    uint32_t* tptr = reinterpret_cast<uint32_t*>(pv_done + 4);
    float* xml = reinterpret_cast<float*>(smem + XCH_OFF);  // [2 segment parities][2 halves][2][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nkv = (p.Lk + KT - 1) / KT;
    const int total = static_cast<int>(p.total_blocks);
    const int b_lo = sk_b0(cta, total, G), b_hi = sk_b0(cta + 1, total, G);

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            bar_init(&q_full[i], 1);
            bar_init(&q_empty[i], 1);
        }
        for (int s = 0; s < SKSTG; ++s) {
            bar_init(&kv_full[s], 1);
            bar_init(&kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) bar_init(&s_full[b], 1);
        for (int i = 0; i < 4; ++i) {
            bar_init(&p_full[i], 4);
            bar_init(&pv_done[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tptr)), "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pdl_wait();
    const uint32_t tmem = *tptr;
    // item -> (query tile, head, image)
    auto decode = [&](int it, int& qt, int& head, int& img) {
        qt = it % p.qtiles;
        const int r = it / p.qtiles;
        head = r % p.heads;
        img = r / p.heads;
    };

    if (warp == 0 && lane == 0) {
        int g = 0;  // the CTA's KV block count
        int q = 0;        // segment count
        for (int b = b_lo; b < b_hi; ++q) {
            const int it = b / nkv, kb0 = b - it * nkv, end = min(b_hi, (it + 1) * nkv);
            int qt, head, img;
            decode(it, qt, head, img);
            const int qb = q & 1;
            bar_wait(&q_empty[qb], ((q >> 1) & 1) ^ 1);
            bar_expect(&q_full[qb], Q_B);
            tma2d(sQ + qb * Q_B, &tmQ, head * HD, img * p.L + qt * QT, &q_full[qb]);
            for (int kb = kb0; kb < kb0 + (end - b); ++kb, ++g) {
                const int s = g % SKSTG;
                bar_wait(&kv_empty[s], ((g / SKSTG) & 1) ^ 1);
                bar_expect(&kv_full[s], K_B + V_B);
                const int row = img * p.Lk + kb * KT;
                tma2d(sK + s * K_B, &tmK, head * HD, row, &kv_full[s]);
                tma2d(sV + s * V_B, &tmV, head * HD, row, &kv_full[s]);
            }
            b = end;
        }
    } else if (warp == 1 && lane == 0) {
        int g = 0;
        int q = 0;
        auto issue_s = [&](int gg, int qb) {
            const int s = gg % SKSTG, b = gg & 1;
            bar_wait(&kv_full[s], (gg / SKSTG) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int k = 0; k < HD / 16; ++k)
                mma(tmem + b * KT, sdesc(sQ + qb * Q_B + k * 32), sdesc(sK + s * K_B + k * 32), idesc(QT, KT), k > 0);
            commit(&s_full[b]);
        };
        for (int b = b_lo; b < b_hi; ++q) {
            const int it = b / nkv, end = min(b_hi, (it + 1) * nkv);
            const int n = end - b, qb = q & 1;
            bar_wait(&q_full[qb], (q >> 1) & 1);
            issue_s(g, qb);
            if (n == 1) commit(&q_empty[qb]);
            for (int j = 1; j <= n; ++j) {
                if (j < n) {
                    issue_s(g + j, qb);
                    if (j == n - 1) commit(&q_empty[qb]);  // every S of this segment issued
                }
                const int jj = g + j - 1;
                const int s = jj % SKSTG, bb = jj & 1;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    bar_wait(&p_full[bb * 2 + h], (jj >> 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int k = 2 * h; k < 2 * h + 2; ++k)
                        mma_ts(tmem + 2 * KT + h * HD, tmem + bb * KT + h * HK + (k & 1) * 8,
                               sdesc(sV + s * V_B + k * 2048), idesc(QT, HD) | (1u << 16),
                               (j > 1 || (k & 1)) ? 1u : 0u);
                    commit(&pv_done[bb * 2 + h]);
                }
                commit(&kv_empty[s]);
            }
            g += n;
            b = end;
        }
    } else if (warp >= 2) {
        const int qq = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = qq * 32 + lane;
        const uint32_t lrow = static_cast<uint32_t>(qq * 32) << 16;
        const float sl2 = 0.125f * 1.4426950408889634f;
        int g = 0;
        int q = 0;
        SK_TL(0);
        for (int b = b_lo; b < b_hi; ++q) {
            const int it = b / nkv, kb0 = b - it * nkv, end = min(b_hi, (it + 1) * nkv);
            const int n = end - b;
            int qt, head, img;
            decode(it, qt, head, img);
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < n; ++j) {
                const int gg = g + j;
                const int bb = gg & 1;
                const uint32_t tS = tmem + bb * KT + half * HK + lrow;
                bar_wait(&s_full[bb], (gg >> 1) & 1);
                if (j == 0) SK_TL(1 + 3 * q);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t sr[HK];
                tld_hk_nowait(tS, sr);
                tld_wait();
                const int valid = min(KT, p.Lk - (kb0 + j) * KT) - half * HK;
                if (valid < HK) {
#pragma unroll
                    for (int i = 0; i < HK; ++i)
                        if (i >= valid) sr[i] = 0xff800000u;
                }
                float mp[8];
#pragma unroll
                for (int a = 0; a < 8; ++a) mp[a] = __uint_as_float(sr[a]);
#pragma unroll
                for (int i = 8; i < HK; ++i) mp[i & 7] = fmaxf(mp[i & 7], __uint_as_float(sr[i]));
                const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                       fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
                const bool need = mx > m && (m == -INFINITY || (mx - m) * sl2 > 8.f);
                if (__any_sync(0xffffffffu, need)) {
                    if (j > 0) {  // O_h must hold PV_{j-1},h of this segment
                        const int gp = gg - 1;
                        bar_wait(&pv_done[(gp & 1) * 2 + half], (gp >> 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const float alpha = need ? (m == -INFINITY ? 0.f : ex2((m - mx) * sl2)) : 1.f;
                        const uint32_t tO = tmem + 2 * KT + half * HD + lrow;
#pragma unroll
                        for (int c = 0; c < HD; c += 16) {
                            float ov[16];
                            tld16(tO + c, ov);
#pragma unroll
                            for (int i = 0; i < 16; ++i) ov[i] *= alpha;
                            tst16(tO + c, ov);
                        }
                        tst_wait();
                        l *= alpha;
                    }
                    if (need) m = mx;
                }
                const float off = m == -INFINITY ? 0.f : -m * sl2;
                float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                uint32_t pk[HK / 2];
#pragma unroll
                for (int c = 0; c < HK; c += 2) {
                    const float v0 = ex2(fmaf(__uint_as_float(sr[c]), sl2, off));
                    const float v1 = ex2(fmaf(__uint_as_float(sr[c + 1]), sl2, off));
                    sp[c & 7] += v0;
                    sp[(c + 1) & 7] += v1;
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(v0, v1);
                    pk[c / 2] = *reinterpret_cast<uint32_t*>(&h2);
                }
                tst_u32<HK / 2>(tS, pk);
                tst_wait();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) bar_arrive(&p_full[bb * 2 + half]);
                l += ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
            }
            SK_TL(2 + 3 * q);
            // merge the halves (xml double-buffered by segment parity: the partner warp may still
            // read the previous segment's values)
            float* xm = xml + (q & 1) * 4 * QT;
            xm[(half * 2 + 0) * QT + r] = m;
            xm[(half * 2 + 1) * QT + r] = l;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + qq) : "memory");
            const float m0 = xm[0 * QT + r], l0 = xm[1 * QT + r], m1 = xm[2 * QT + r], l1 = xm[3 * QT + r];
            const float M = fmaxf(m0, m1);
            const float w0 = m0 == -INFINITY ? 0.f : ex2((m0 - M) * sl2);
            const float w1 = m1 == -INFINITY ? 0.f : ex2((m1 - M) * sl2);
            float lt = w0 * l0 + w1 * l1;
            const int gl = g + n - 1;
            const int lb = gl & 1;
            bar_wait(&pv_done[lb * 2 + 0], (gl >> 1) & 1);
            bar_wait(&pv_done[lb * 2 + 1], (gl >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float ov[HD / 2], o1[HD / 2];
            const uint32_t tO0 = tmem + 2 * KT + lrow + half * (HD / 2);
            tld16(tO0, ov);
            tld16(tO0 + 16, ov + 16);
            tld16(tO0 + HD, o1);
            tld16(tO0 + HD + 16, o1 + 16);
#pragma unroll
            for (int c = 0; c < HD / 2; ++c) ov[c] = w0 * ov[c] + w1 * o1[c];
            const long long row = static_cast<long long>(qt) * QT + r;
            // segments of this item: CTAs sk_cta(first block) .. sk_cta(last block)
            const int c_first = sk_cta(it * nkv, total, G);
            const int nseg = sk_cta((it + 1) * nkv - 1, total, G) - c_first + 1;
            bool write_out = true;
            if (nseg > 1) {
                const int seg = cta - c_first;
                float* rec = p.part + (static_cast<long long>(it) * p.nsplit + seg) * kRecFloats;
#pragma unroll
                for (int c = 0; c < HD / 2; c += 4)
                    *reinterpret_cast<float4*>(rec + r * HD + half * (HD / 2) + c) =
                        make_float4(ov[c], ov[c + 1], ov[c + 2], ov[c + 3]);
                if (half == 0) rec[QT * HD + r] = M, rec[QT * HD + QT + r] = lt;
                // release: the barrier orders every softmax thread's record stores before thread 64's
                // gpu-scope fence and ticket (one fence per CTA, not one per thread); acquire: the
                // last arrival fences again before the barrier that releases the combine reads
                __shared__ unsigned last_sk;
                asm volatile("bar.sync 5, 256;" ::: "memory");
                if (threadIdx.x == 64) {
                    __threadfence();
                    last_sk = atomicAdd(p.counters + it, 1u) == static_cast<unsigned>(nseg - 1);
                    __threadfence();
                }
                asm volatile("bar.sync 5, 256;" ::: "memory");
                write_out = last_sk != 0u;
                if (write_out) {
                    const float* base = p.part + static_cast<long long>(it) * p.nsplit * kRecFloats;
                    float MM = -INFINITY;
                    for (int s2 = 0; s2 < nseg; ++s2) MM = fmaxf(MM, __ldcg(base + s2 * kRecFloats + QT * HD + r));
                    float acc[HD / 2], den = 0.f;
#pragma unroll
                    for (int c = 0; c < HD / 2; ++c) acc[c] = 0.f;
                    for (int s2 = 0; s2 < nseg; ++s2) {
                        const float* rs = base + s2 * kRecFloats;
                        const float ms = __ldcg(rs + QT * HD + r);
                        const float w = ms == -INFINITY ? 0.f : ex2((ms - MM) * sl2);
                        den = fmaf(w, __ldcg(rs + QT * HD + QT + r), den);
#pragma unroll
                        for (int c = 0; c < HD / 2; c += 4) {
                            const float4 o4 =
                                __ldcg(reinterpret_cast<const float4*>(rs + r * HD + half * (HD / 2) + c));
                            acc[c] = fmaf(w, o4.x, acc[c]), acc[c + 1] = fmaf(w, o4.y, acc[c + 1]);
                            acc[c + 2] = fmaf(w, o4.z, acc[c + 2]), acc[c + 3] = fmaf(w, o4.w, acc[c + 3]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < HD / 2; ++c) ov[c] = acc[c];
                    lt = den;
                    if (threadIdx.x == 64) p.counters[it] = 0u;
                }
            }
            if (write_out && row < p.L) {
                const float inv = 1.0f / lt;
                __nv_bfloat16* dst =
                    p.out + (static_cast<long long>(img) * p.L + row) * p.ldo + head * HD + half * (HD / 2);
#pragma unroll
                for (int c = 0; c < HD / 2; c += 8) {
                    uint4 v;
                    __nv_bfloat162 b0 = __floats2bfloat162_rn(ov[c] * inv, ov[c + 1] * inv);
                    __nv_bfloat162 b1 = __floats2bfloat162_rn(ov[c + 2] * inv, ov[c + 3] * inv);
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(ov[c + 4] * inv, ov[c + 5] * inv);
                    __nv_bfloat162 b3 = __floats2bfloat162_rn(ov[c + 6] * inv, ov[c + 7] * inv);
                    v.x = *reinterpret_cast<uint32_t*>(&b0);
                    v.y = *reinterpret_cast<uint32_t*>(&b1);
                    v.z = *reinterpret_cast<uint32_t*>(&b2);
                    v.w = *reinterpret_cast<uint32_t*>(&b3);
                    *reinterpret_cast<uint4*>(dst + c) = v;
                }
            }
            SK_TL(3 + 3 * q);
            g += n;
            b = end;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    });
    if (!fn) throw cuda_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D bf16 map: rows x cols (cols contiguous, row stride ld elements), box (64 cols, box_rows)
CUtensorMap map2d(const void* base, long long rows, long long cols, long long ld, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r =
        encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("attention: cuTensorMapEncodeTiled failed " + std::to_string(r));
    return m;
}

}  // namespace

namespace {
// split-KV factor: the (query tile, head) items fill 2 CTAs per SM unevenly (e.g. 360
// items over 296 slots = a 22% second wave); minimise rounds x (KV blocks per CTA + fixed
// per-CTA cost, + the combine when split)
int attn_splits(int L, int Lk, int C, int sms, int batch) {
    static const int forced = [] {  // ADX_ATTN_SPLITS=S forces the split factor (tuning)
        const char* e = getenv("ADX_ATTN_SPLITS");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) return std::min(forced, std::max(1, (Lk + KT - 1) / KT));
    const long long items = static_cast<long long>((L + QT - 1) / QT) * (C / HD) * batch;
    const int nkv = (Lk + KT - 1) / KT, slots = 2 * sms;
    // the partial publish + fence + ticket + combine costs about ten KV blocks (measured:
    // splitting the 100-item L=576 grid doubled its time), so only long grids with a bad
    // wave tail split (level 0: 360 items over 296 slots); the smallest S within 5% of the
    // best modelled time wins (level 0 measured: S=1 227 us, S=2 200 us, S=3 206 us)
    double t[9] = {};
    double best = 1e300;
    for (int S = 1; S <= 8 && S <= nkv; ++S) {
        const long long rounds = (items * S + slots - 1) / slots;
        t[S] = static_cast<double>(rounds) * ((nkv + S - 1) / S + 3 + (S > 1 ? 10 : 0));
        best = std::min(best, t[S]);
    }
    for (int S = 1; S <= 8 && S <= nkv; ++S)
        if (t[S] <= 1.05 * best) return S;
    return 1;
}
int device_sms() {
    int dev = 0, sms = 0;
    CKA(cudaGetDevice(&dev));
    CKA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}
// stream-K plan: grid G (0 = use the per-item grid of attn_splits) and the record slots per item.
// Modelled in KV-block times like attn_splits: ceil(total / G) + 3 per CTA, + 10 when items are
// cut (partial publish + ticket + combine, as for split-KV); taken only when it beats the best
// split plan by 15% (measured: c2 level 0, 360 items x 144 blocks, 188.9 -> 183.7 us; level 1,
// 180 x 36, 38.3 -> 43.8 us -- the cut items' combine costs more than the model says).
// ADX_ATTN_SK=0 / 1 disables / forces it.
int attn_sk_plan(int L, int Lk, int C, int sms, int batch, int& slots) {
    static const int mode = [] {
        const char* e = getenv("ADX_ATTN_SK");
        return e ? atoi(e) : -1;
    }();
    slots = 0;
    if (mode == 0) return 0;
    const long long items = static_cast<long long>((L + QT - 1) / QT) * (C / HD) * batch;
    const int nkv = (Lk + KT - 1) / KT;
    const long long total = items * nkv;
    const int G = static_cast<int>(std::min<long long>(2LL * sms, total));
    const long long rmin = total / G;
    if (rmin < 1 || total >= (1LL << 31) / G) return 0;
    const int S = attn_splits(L, Lk, C, sms, batch);
    const long long rounds = (items * S + 2LL * sms - 1) / (2LL * sms);
    const double t_split = static_cast<double>(rounds) * ((nkv + S - 1) / S + 3 + (S > 1 ? 10 : 0));
    const bool cut = total % G != 0 || (total / G) % nkv != 0;
    const double t_sk = static_cast<double>((total + G - 1) / G) + 3 + (cut ? 10 : 0);
    // long items only (a combine per cut item is amortised over >= 96 blocks): measured gains
    // at c2 level 0 (144 blocks per item), losses at SDXL's L = 1024 (16) and the cross attention
    if (mode != 1 && (t_sk > 0.85 * t_split || nkv < 96)) return 0;
    slots = static_cast<int>((nkv + rmin - 1) / rmin) + 1;
    return G;
}
}  // namespace

size_t tc_attention_ws_bytes(int L, int Lk, int C, int batch) {
    const size_t items = static_cast<size_t>((L + QT - 1) / QT) * (C / HD) * batch;
    int slots = 0;
    if (attn_sk_plan(L, Lk, C, device_sms(), batch, slots) > 0)
        return 256 * ((items * 4 + 255) / 256) + items * slots * kRecFloats * sizeof(float);
    const int S = attn_splits(L, Lk, C, device_sms(), batch);
    if (S == 1) return 0;
    return 256 * ((items * 4 + 255) / 256) + items * S * kRecFloats * sizeof(float);
}

void tc_attention(const void* Q, long long ldq, const void* K, long long ldk, const void* V, long long ldv, int L,
                  int Lk, int C, __nv_bfloat16* out, long long ldo, cudaStream_t st, void* ws, size_t ws_bytes,
                  int batch) {
    if (C % HD) throw std::invalid_argument("attention: C must be a multiple of 64");
    if ((ldq | ldk | ldv | ldo) % 8) throw std::invalid_argument("attention: strides must be multiples of 8");
    if (batch < 1 || batch > 65535) throw std::invalid_argument("attention: batch must be in 1..65535");
    const CUtensorMap mq = map2d(Q, static_cast<long long>(batch) * L, C, ldq, QT);
    const CUtensorMap mk = map2d(K, static_cast<long long>(batch) * Lk, C, ldk, KT);
    const CUtensorMap mv = map2d(V, static_cast<long long>(batch) * Lk, C, ldv, KT);  // rows = keys, like K
    AttnArgs a{L, Lk, C, out, ldo};
    const size_t need = tc_attention_ws_bytes(L, Lk, C, batch);
    const size_t items = static_cast<size_t>((L + QT - 1) / QT) * (C / HD) * batch;
    int sk_slots = 0;
    const int sk_grid = ws && ws_bytes >= need ? attn_sk_plan(L, Lk, C, device_sms(), batch, sk_slots) : 0;
    static const int ver = [] {  // ADX_ATTN_V=1: the round-1 kernel (per-block max exchange)
        const char* e = getenv("ADX_ATTN_V");
        return e && *e == '1' ? 1 : 2;
    }();
    if (sk_grid > 0 && ver == 2) {  // stream-K over the items' KV blocks (see attn_kernel_sk)
        a.nsplit = sk_slots;
        a.counters = static_cast<unsigned*>(ws);
        a.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256 * ((items * 4 + 255) / 256));
        a.qtiles = (L + QT - 1) / QT;
        a.heads = C / HD;
        a.total_blocks = static_cast<long long>(items) * ((Lk + KT - 1) / KT);
        constexpr size_t smem_sk =
            1024 + 2 * QT * HD * 2 + SKSTG * (KT * HD * 2 + HD * KT * 2) + 256 + 8 * QT * sizeof(float);
        static bool attr_sk[64] = {};
        int dev = 0;
        CKA(cudaGetDevice(&dev));
        if (!attr_sk[dev]) {
            CKA(cudaFuncSetAttribute(attn_kernel_sk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_sk));
            attr_sk[dev] = true;
        }
        if (tc_trace())
            fprintf(stderr, "tc_attention L=%d Lk=%d C=%d batch=%d stream-K grid=%d slots=%d\n", L, Lk, C, batch,
                    sk_grid, sk_slots);
        auto launch = [&](cudaStream_t s2) {
            CKA(launch_pdl(attn_kernel_sk, dim3(sk_grid), dim3(320), smem_sk, s2, 1, mq, mk, mv, a));
        };
        launch(st);
        tc_profile_measure(st, 2, 4.0 * L * Lk * C * batch, 2.0 * batch * C * (2.0 * L + 2.0 * Lk), launch);
        CKA(cudaGetLastError());
        return;
    }
    const int S = attn_splits(L, Lk, C, device_sms(), batch);
    if (S > 1 && ws && ws_bytes >= need) {  // without a (large enough) workspace: unsplit
        a.nsplit = S;
        a.counters = static_cast<unsigned*>(ws);
        a.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256 * ((items * 4 + 255) / 256));
    }
    constexpr size_t smem = 1024 + QT * HD * 2 + STG * (KT * HD * 2 + HD * KT * 2) + 256 + 6 * QT * sizeof(float);
    static bool attr[64] = {};
    int dev = 0;
    CKA(cudaGetDevice(&dev));
    if (!attr[dev]) {
        CKA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr[dev] = true;
    }
    static bool attr2[64] = {};
    if (!attr2[dev]) {
        CKA(cudaFuncSetAttribute(attn_kernel_v2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr2[dev] = true;
    }
    dim3 grid(((L + QT - 1) / QT) * a.nsplit, C / HD, batch);
    if (tc_trace()) fprintf(stderr, "tc_attention L=%d Lk=%d C=%d batch=%d S=%d v%d\n", L, Lk, C, batch, a.nsplit, ver);
    auto launch = [&](cudaStream_t s2) {
        if (ver == 1)
            CKA(launch_pdl(attn_kernel, grid, dim3(320), smem, s2, 1, mq, mk, mv, a));
        else
            CKA(launch_pdl(attn_kernel_v2<false>, grid, dim3(320), smem, s2, 1, mq, mk, mv, mq, mk, mv, a));
    };
    launch(st);
    tc_profile_measure(st, 2, 4.0 * L * Lk * C * batch, 2.0 * batch * C * (2.0 * L + 2.0 * Lk), launch);
    CKA(cudaGetLastError());
}

// the stream-K kernel's per-CTA stamps of the last launch (-DADX_SK_TIMELINE builds; else zeros)
void tc_sk_timeline(unsigned long long* out, int n_ctas) {
#ifdef ADX_SK_TIMELINE
    CKA(cudaDeviceSynchronize());
    CKA(cudaMemcpyFromSymbol(out, g_sk_tl, static_cast<size_t>(std::min(n_ctas, 512)) * 16 * 8));
#else
    std::fill(out, out + static_cast<size_t>(n_ctas) * 16, 0ull);
#endif
}

void tc_attention_x(const void* Qh, const void* Ql, long long ldq, const void* Kh, const void* Kl, long long ldk,
                    const void* Vh, const void* Vl, long long ldv, int L, int Lk, int C, float* out, long long ldo,
                    cudaStream_t st, void* ws, size_t ws_bytes, int batch) {
    if (C % HD) throw std::invalid_argument("attention: C must be a multiple of 64");
    if ((ldq | ldk | ldv) % 8 || ldo % 4) throw std::invalid_argument("attention: bad strides");
    if (batch < 1 || batch > 65535) throw std::invalid_argument("attention: batch must be in 1..65535");
    const long long rq = static_cast<long long>(batch) * L, rk = static_cast<long long>(batch) * Lk;
    const CUtensorMap mqh = map2d(Qh, rq, C, ldq, QT), mql = map2d(Ql, rq, C, ldq, QT);
    const CUtensorMap mkh = map2d(Kh, rk, C, ldk, KT), mkl = map2d(Kl, rk, C, ldk, KT);
    const CUtensorMap mvh = map2d(Vh, rk, C, ldv, KT), mvl = map2d(Vl, rk, C, ldv, KT);
    AttnArgs a{L, Lk, C, nullptr, ldo};
    a.out_f32 = out;
    const int S = attn_splits(L, Lk, C, device_sms(), batch);
    const size_t need = tc_attention_ws_bytes(L, Lk, C, batch);
    if (S > 1 && ws && ws_bytes >= need) {
        const size_t items = static_cast<size_t>((L + QT - 1) / QT) * (C / HD) * batch;
        a.nsplit = S;
        a.counters = static_cast<unsigned*>(ws);
        a.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256 * ((items * 4 + 255) / 256));
    }
    constexpr size_t smem =
        1024 + 2 * QT * HD * 2 + XSTG * 2 * (KT * HD * 2 + HD * KT * 2) + 256 + 6 * QT * sizeof(float);
    static bool attr[64] = {};
    int dev = 0;
    CKA(cudaGetDevice(&dev));
    if (!attr[dev]) {
        CKA(cudaFuncSetAttribute(attn_kernel_v2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr[dev] = true;
    }
    dim3 grid(((L + QT - 1) / QT) * a.nsplit, C / HD, batch);
    if (tc_trace()) fprintf(stderr, "tc_attention_x L=%d Lk=%d C=%d batch=%d S=%d\n", L, Lk, C, batch, a.nsplit);
    auto launch = [&](cudaStream_t s2) {
        CKA(launch_pdl(attn_kernel_v2<true>, grid, dim3(320), smem, s2, 1, mqh, mkh, mvh, mql, mkl, mvl, a));
    };
    launch(st);
    tc_profile_measure(st, 2, 3 * 4.0 * L * Lk * C * batch, 2.0 * batch * C * (2.0 * L + 4.0 * Lk + 2.0 * L),
                       launch);
    CKA(cudaGetLastError());
}

}  // namespace adx
