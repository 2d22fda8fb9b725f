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

#include <cuda.h>
#include <cuda_bf16.h>

#include <cstring>
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

namespace {

constexpr int BM = 128, BK = 64, STAGES = 4;

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

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// ------------------------------------------------------------------ kernel
template <int BN, bool CONV>
__global__ void __launch_bounds__(192, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, const TcArgs p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment of the swizzled tiles
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint32_t* tptr = reinterpret_cast<uint32_t*>(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile_m = blockIdx.x, tile_n = blockIdx.y, img = blockIdx.z;
    const int n0 = tile_n * BN;
    const int nkb = p.k_blocks;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tptr)),
                     "n"(tmem_cols<BN>())
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tptr;

    // conv tile origin (output pixels of one image: box_h rows x box_w cols)
    int h0 = 0, w0 = 0;
    if constexpr (CONV) {
        const int tiles_w = p.W / p.box_w;
        h0 = (tile_m / tiles_w) * p.box_h;
        w0 = (tile_m % tiles_w) * p.box_w;
    }

    if (warp == 0 && lane == 0) {
        // ---------------------------------------------------------- producer
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            bar_wait(&empty[s], ph ^ 1);
            bar_expect(&full[s], A_BYTES + B_BYTES);
            if constexpr (CONV) {
                // k block kb -> tap (r, s) and channel block; A box at the
                // tap-shifted window (OOB rows/cols are zero-filled = padding)
                const int cpb = p.cin / BK;
                const int tap = kb / cpb, cb = kb - tap * cpb;
                const int dr = tap / 3 - 1, ds = tap % 3 - 1;
                tma4d(sA + s * A_BYTES, &tmA, cb * BK, w0 + ds, h0 + dr, img, &full[s]);
                tma2d(sB + s * B_BYTES, &tmB, kb * BK, n0, &full[s]);
            } else {
                tma2d(sA + s * A_BYTES, &tmA, kb * BK, tile_m * BM, &full[s]);
                tma2d(sB + s * B_BYTES, &tmB, kb * BK, n0, &full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16<BN>();
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            bar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                const uint64_t a = sdesc(sA + s * A_BYTES + k * 32);
                const uint64_t b = sdesc(sB + s * B_BYTES + k * 32);
                mma_bf16(tmem, a, b, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            mma_commit(&empty[s]);
        }
        mma_commit(tfull);
    } else if (warp >= 2) {
        // --------------------------------------------------------- epilogue
        bar_wait(tfull, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int row = q * 32 + lane;
        long long m;  // output row (pixel) index
        bool valid;
        if constexpr (CONV) {
            const int hh = h0 + row / p.box_w, ww = w0 + row % p.box_w;
            valid = hh < p.H && ww < p.W;
            m = (static_cast<long long>(img) * p.H + hh) * p.W + ww;
            if (p.sub2) {  // stride-2 conv: keep even pixels, write the half-resolution grid
                valid = valid && !(hh & 1) && !(ww & 1);
                m = (static_cast<long long>(img) * (p.H / 2) + hh / 2) * (p.W / 2) + ww / 2;
            }
        } else {
            m = static_cast<long long>(tile_m) * BM + row;
            valid = m < p.M;
        }
        const int nlim = p.n_store ? p.n_store : p.N;
        const bool vec_ok = ((p.ldo | p.ldr) & 7) == 0;
        if (p.act == 2) {
            // GEGLU: the host interleaved the weight rows per tile, so columns [0, BN/2)
            // of this tile are hidden units n0/2 + c and [BN/2, BN) their gates;
            // out[m][n0/2 + c] = (h + bh) * gelu(g + bg)  (the 2x-wide product never reaches HBM)
            for (int c = 0; c < BN / 2; c += 16) {
                float v[16], g[16];
                tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
                tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + BN / 2 + c, g);
                if (!valid) continue;
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const float4 bh = *reinterpret_cast<const float4*>(p.bias + n0 + c + j);
                    const float4 bg = *reinterpret_cast<const float4*>(p.bias + n0 + BN / 2 + c + j);
                    v[j] += bh.x, v[j + 1] += bh.y, v[j + 2] += bh.z, v[j + 3] += bh.w;
                    g[j] += bg.x, g[j + 1] += bg.y, g[j + 2] += bg.z, g[j + 3] += bg.w;
                }
                uint4* op = reinterpret_cast<uint4*>(p.out_bf16 + m * p.ldo + n0 / 2 + c);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t w4[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int j = h * 8 + 2 * k;
                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[j] * gelu(g[j]), v[j + 1] * gelu(g[j + 1]));
                        w4[k] = *reinterpret_cast<const uint32_t*>(&b2);
                    }
                    op[h] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                }
            }
        } else
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
            if (!valid) continue;
            const int nb = n0 + c;
            if (vec_ok && nb + 16 <= nlim) {
                // vectorised epilogue: 16 consecutive columns of this row, 16-byte loads / stores
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    if (p.bias) {
                        const float4 b = *reinterpret_cast<const float4*>(p.bias + nb + j);
                        v[j] += b.x, v[j + 1] += b.y, v[j + 2] += b.z, v[j + 3] += b.w;
                    }
                    if (p.chan_add) {
                        const float4 b =
                            *reinterpret_cast<const float4*>(p.chan_add + static_cast<long long>(img) * p.N + nb + j);
                        v[j] += b.x, v[j + 1] += b.y, v[j + 2] += b.z, v[j + 3] += b.w;
                    }
                }
                if (p.act == 1) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = silu(v[j]);
                }
                if (p.residual) {
                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + m * p.ldr + nb);
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
                    uint4* op = reinterpret_cast<uint4*>(p.out_bf16 + m * p.ldo + nb);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t w4[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[h * 8 + 2 * k], v[h * 8 + 2 * k + 1]);
                            w4[k] = *reinterpret_cast<const uint32_t*>(&b2);
                        }
                        op[h] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                    }
                }
                continue;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int n = n0 + c + j;
                if (n >= (p.n_store ? p.n_store : p.N)) continue;
                float x = v[j];
                if (p.bias) x += p.bias[n];
                if (p.chan_add) x += p.chan_add[static_cast<long long>(img) * p.N + n];
                if (p.act == 1) x = silu(x);
                if (p.residual) x += __bfloat162float(p.residual[m * p.ldr + n]);
                x *= p.out_scale;
                if (p.out_f32)
                    p.out_f32[m * p.ldo + n] = x;
                else
                    p.out_bf16[m * p.ldo + n] = __float2bfloat16(x);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols<BN>())
                     : "memory");
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
                     const cuuint32_t* box) {
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                                   strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

template <int BN, bool CONV>
void launch_t(const CUtensorMap& a, const CUtensorMap& b, const TcArgs& p, dim3 grid, cudaStream_t st) {
    constexpr size_t smem = 1024 + STAGES * (BM * BK * 2 + BN * BK * 2) + 256;
    static bool attr[64] = {};
    int dev = 0;
    CKT(cudaGetDevice(&dev));
    if (!attr[dev]) {
        CKT(cudaFuncSetAttribute(tc_gemm_kernel<BN, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr[dev] = true;
    }
    tc_gemm_kernel<BN, CONV><<<grid, 192, smem, st>>>(a, b, p);
    CKT(cudaGetLastError());
}

template <bool CONV>
void dispatch(const CUtensorMap& a, const CUtensorMap& b, const TcArgs& p, dim3 grid, int bn, cudaStream_t st) {
    switch (bn) {
        case 32: launch_t<32, CONV>(a, b, p, grid, st); break;
        case 64: launch_t<64, CONV>(a, b, p, grid, st); break;
        case 128: launch_t<128, CONV>(a, b, p, grid, st); break;
        case 160: launch_t<160, CONV>(a, b, p, grid, st); break;
        case 192: launch_t<192, CONV>(a, b, p, grid, st); break;
        case 256: launch_t<256, CONV>(a, b, p, grid, st); break;
        default: throw std::invalid_argument("tc_gemm: BN must be 32/64/128/160/192/256");
    }
}

// N tile: least padded columns, ties to the wider tile (fewer CTAs re-reading A)
int pick_bn(int N) {
    if (N <= 32) return 32;
    if (N <= 64) return 64;
    int best = 256;
    long long waste = (N + 255) / 256 * 256LL - N;
    for (int bn : {192, 160, 128}) {
        const long long w = (N + bn - 1) / bn * static_cast<long long>(bn) - N;
        if (w < waste) {
            waste = w;
            best = bn;
        }
    }
    return best;
}

struct ProfRec {
    int kind;
    double flops;
    cudaEvent_t a, b;
};
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_open;

}  // namespace

void tc_profile_enable(bool on) { g_prof_on = on; }

void tc_profile_record_begin(cudaStream_t st) {
    if (!g_prof_on) return;
    cudaEvent_t e;
    CKT(cudaEventCreate(&e));
    CKT(cudaEventRecord(e, st));
    g_prof_open.push_back(e);
}

void tc_profile_record_end(cudaStream_t st, int kind, double flops) {
    if (!g_prof_on || g_prof_open.empty()) return;
    cudaEvent_t e;
    CKT(cudaEventCreate(&e));
    CKT(cudaEventRecord(e, st));
    g_prof.push_back({kind, flops, g_prof_open.back(), e});
    g_prof_open.pop_back();
}

void tc_profile_collect(double out[3][3]) {
    for (int k = 0; k < 3; ++k) out[k][0] = out[k][1] = out[k][2] = 0.0;
    for (auto& r : g_prof) {
        CKT(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CKT(cudaEventElapsedTime(&ms, r.a, r.b));
        out[r.kind][0] += 1;
        out[r.kind][1] += ms;
        out[r.kind][2] += r.flops;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
}

// D = A[M x K] . B[N x K]^T ; A, B bf16 row-major (K contiguous), K % 64 == 0
void tc_gemm(const void* A, const void* B, int M, int N, int K, TcArgs p, cudaStream_t st, int bn) {
    tc_gemm_strided(A, K, B, K, M, N, K, p, st, bn);
}

void tc_gemm_strided(const void* A, long long lda, const void* B, long long ldb, int M, int N, int K, TcArgs p,
                     cudaStream_t st, int bn) {
    if (K % BK) throw std::invalid_argument("tc_gemm: K must be a multiple of 64");
    if ((lda | ldb) % 8) throw std::invalid_argument("tc_gemm: row strides must be multiples of 8 elements");
    if (p.act == 2) {  // fused GEGLU (see the epilogue): fixed 256-wide tiles of [128 hidden | 128 gate]
        if (bn && bn != 256) throw std::invalid_argument("tc_gemm: GEGLU epilogue needs 256-wide N tiles");
        if (N % 256 || !p.out_bf16 || !p.bias || p.residual || p.chan_add || (p.ldo % 8))
            throw std::invalid_argument("tc_gemm: GEGLU epilogue needs N % 256 == 0, bias, bf16 output, ldo % 8 == 0");
        bn = 256;
    }
    if (bn == 0) bn = pick_bn(N);
    const cuuint64_t da[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
    const cuuint64_t sa_[1] = {static_cast<cuuint64_t>(lda) * 2};
    const cuuint64_t sb_[1] = {static_cast<cuuint64_t>(ldb) * 2};
    const cuuint32_t ba[2] = {BK, BM};
    const cuuint64_t db[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
    const cuuint32_t bb[2] = {BK, static_cast<cuuint32_t>(bn)};
    const CUtensorMap ma = make_map(A, 2, da, sa_, ba), mb = make_map(B, 2, db, sb_, bb);
    p.M = M;
    p.N = N;
    p.k_blocks = K / BK;
    dim3 grid((M + BM - 1) / BM, (N + bn - 1) / bn, 1);
    tc_profile_record_begin(st);
    dispatch<false>(ma, mb, p, grid, bn, st);
    tc_profile_record_end(st, 1, 2.0 * M * N * K);
}

// 3x3 conv, stride 1, pad 1, as an implicit GEMM over NHWC bf16:
//   out[n,h,w,co] = sum_{r,s,ci} X[n,h+r-1,w+s-1,ci] . Wt[co][(r*3+s)*Cin + ci]
// A tiles are 4-D TMA boxes (64 channels x box_w x box_h x 1) at tap-shifted
// coordinates; out-of-range rows/cols arrive as zeros (the padding).
void tc_conv3x3(const void* X, const void* Wt, int batch, int H, int W, int Cin, int Cout, TcArgs p,
                cudaStream_t st, int bn) {
    if (Cin % BK) throw std::invalid_argument("tc_conv3x3: Cin must be a multiple of 64");
    int bw = 0;
    for (int c : {128, 64, 32, 16, 8, 4})
        if (W % c == 0 && c <= W && BM % c == 0) {
            bw = c;
            break;
        }
    if (!bw) throw std::invalid_argument("tc_conv3x3: W must be divisible by 8, 16, 32, 64 or 128");
    const int bh = BM / bw;
    if (bn == 0) bn = pick_bn(Cout);
    const cuuint64_t dx[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(batch)};
    const cuuint64_t sx[3] = {static_cast<cuuint64_t>(Cin) * 2, static_cast<cuuint64_t>(W) * Cin * 2,
                              static_cast<cuuint64_t>(H) * W * Cin * 2};
    const cuuint32_t bx[4] = {BK, static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
    const int K = 9 * Cin;
    const cuuint64_t dw[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Cout)};
    const cuuint64_t sw[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint32_t bwb[2] = {BK, static_cast<cuuint32_t>(bn)};
    const CUtensorMap ma = make_map(X, 4, dx, sx, bx), mb = make_map(Wt, 2, dw, sw, bwb);
    p.M = batch * H * W;
    p.N = Cout;
    p.k_blocks = K / BK;
    p.H = H;
    p.W = W;
    p.box_w = bw;
    p.box_h = bh;
    p.cin = Cin;
    dim3 grid(((H + bh - 1) / bh) * (W / bw), (Cout + bn - 1) / bn, batch);
    tc_profile_record_begin(st);
    dispatch<true>(ma, mb, p, grid, bn, st);
    // algorithmic FLOPs (a stride-2 conv does a quarter of the work it launches)
    tc_profile_record_end(st, 0, 2.0 * batch * H * W * Cout * 9.0 * Cin / (p.sub2 ? 4.0 : 1.0));
}

}  // namespace adx
