// kernels.cu -- sm_100a kernels of the async denoising hot path (see kernels.cuh).
//
// Stage GEMV design (batch-1 dense layer, HBM-bound):
//  * weights row-major with a zero-padded pitch (multiple of 8 elements) so every
//    lane streams 16-byte vectors: ld.global.nc.L1::no_allocate (read once, keep
//    L1 for the activations);
//  * one warp per output row, 4 warps per CTA, grid = rows/4: on 148 SMs a 4096-row
//    layer lands 27.7 rows per SM with <2% quantisation;
//  * prologue BEFORE griddepcontrol.wait (programmatic dependent launch): each warp
//    issues its first 8 weight vectors per lane and an L2 bulk prefetch of its row,
//    so HBM stays busy across the kernel boundary of the dependent GEMV chain;
//  * the skip-concat input is gathered from its segments into shared memory once
//    per CTA (no concat tensor in HBM);
//  * fixed per-lane order + butterfly shuffle: results do not depend on grid size,
//    device or stream -> run_parallel is bit-identical to run_serial.
#include "kernels.cuh"

#include <cuda_bf16.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace adx {

namespace {

constexpr int kWarps = 4;
constexpr int kPre = 8;  // weight vectors per lane issued in the prologue / per batch

#define ADX_CUDA(x)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                             \
    } while (0)

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

template <typename WT>
struct Acc;
template <>
struct Acc<double> {
    using T = double;
};
template <>
struct Acc<float> {
    using T = float;
};
template <>
struct Acc<__nv_bfloat16> {
    using T = float;
};

// acc += W-vector . x[col .. col+VEC), in element order
__device__ __forceinline__ double dot16(uint4 w, const double* x, double acc) {
    const double2 xv = *reinterpret_cast<const double2*>(x);
    const double w0 = __hiloint2double(static_cast<int>(w.y), static_cast<int>(w.x));
    const double w1 = __hiloint2double(static_cast<int>(w.w), static_cast<int>(w.z));
    acc = fma(w0, xv.x, acc);
    acc = fma(w1, xv.y, acc);
    return acc;
}
__device__ __forceinline__ float dot16(uint4 w, const float* x, float acc) {
    const float4 xv = *reinterpret_cast<const float4*>(x);
    acc = fmaf(__uint_as_float(w.x), xv.x, acc);
    acc = fmaf(__uint_as_float(w.y), xv.y, acc);
    acc = fmaf(__uint_as_float(w.z), xv.z, acc);
    acc = fmaf(__uint_as_float(w.w), xv.w, acc);
    return acc;
}
__device__ __forceinline__ float dot16_bf16(uint4 w, const float* x, float acc) {
    const float4 xa = *reinterpret_cast<const float4*>(x);
    const float4 xb = *reinterpret_cast<const float4*>(x + 4);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    const float xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float lo = __uint_as_float(u[k] << 16);
        const float hi = __uint_as_float(u[k] & 0xffff0000u);
        acc = fmaf(lo, xs[2 * k], acc);
        acc = fmaf(hi, xs[2 * k + 1], acc);
    }
    return acc;
}

template <typename WT, typename AT>
__device__ __forceinline__ typename Acc<WT>::T dot_vec(uint4 w, const AT* x, typename Acc<WT>::T acc) {
    if constexpr (sizeof(WT) == 2)
        return dot16_bf16(w, x, acc);
    else
        return dot16(w, x, acc);
}

template <typename WT, typename AT>
__global__ void __launch_bounds__(kWarps * 32) gemv_kernel(const GemvArgs a) {
    using AccT = typename Acc<WT>::T;
    constexpr int VEC = 16 / sizeof(WT);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AT* sx = reinterpret_cast<AT*>(smem_raw);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nvec = a.pitch / VEC;
    const int stride = gridDim.x * kWarps;
    int row = blockIdx.x * kWarps + warp;

    // ---- prologue (independent of the previous kernel): stream in weights
    uint4 pre[kPre];
    if (row < a.rows) {
        const uint4* wrow = reinterpret_cast<const uint4*>(static_cast<const WT*>(a.W) + (size_t)row * a.pitch);
        if (lane == 0 && nvec > kPre * 32) {
            const char* p = reinterpret_cast<const char*>(wrow + kPre * 32);
            const unsigned bytes = static_cast<unsigned>((nvec - kPre * 32) * 16);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
        }
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            const int v = lane + u * 32;
            pre[u] = v < nvec ? ld_stream(wrow + v) : make_uint4(0, 0, 0, 0);
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- gather the concatenated input into shared memory (zero padded)
    int off = 0;
    for (int s = 0; s < a.nseg; ++s) {
        const AT* src = static_cast<const AT*>(a.seg[s]);
        for (int i = threadIdx.x; i < a.seg_len[s]; i += blockDim.x) sx[off + i] = src[i];
        off += a.seg_len[s];
    }
    for (int i = off + threadIdx.x; i < a.pitch; i += blockDim.x) sx[i] = AT(0);
    __syncthreads();

    bool first = true;
    for (; row < a.rows; row += stride) {
        const uint4* wrow = reinterpret_cast<const uint4*>(static_cast<const WT*>(a.W) + (size_t)row * a.pitch);
        AccT acc = AccT(0);
        int v = lane;
        if (first) {
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                const int vv = lane + u * 32;
                if (vv < nvec) acc = dot_vec<WT, AT>(pre[u], sx + (size_t)vv * VEC, acc);
            }
            v = lane + kPre * 32;
            first = false;
        }
        for (; v + (kPre - 1) * 32 < nvec; v += kPre * 32) {
            uint4 buf[kPre];
#pragma unroll
            for (int u = 0; u < kPre; ++u) buf[u] = ld_stream(wrow + v + u * 32);
#pragma unroll
            for (int u = 0; u < kPre; ++u) acc = dot_vec<WT, AT>(buf[u], sx + (size_t)(v + u * 32) * VEC, acc);
        }
        for (; v < nvec; v += 32) acc = dot_vec<WT, AT>(ld_stream(wrow + v), sx + (size_t)v * VEC, acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            AccT val = acc;
            if (a.bias) val += static_cast<AccT>(static_cast<const AT*>(a.bias)[row]);
            if (a.act) val = val > AccT(0) ? val : AccT(0.1) * val;
            static_cast<AT*>(a.out)[row] = static_cast<AT>(val);
            if (a.bad && !isfinite(val)) atomicMin(a.bad, a.bad_key);
        }
    }
}

// ---------------------------------------------------------------------------
// TMA-streamed GEMV (the production kernel).
//
// One persistent CTA per SM, kTWarps warps.  Every warp owns a ring of kSlots
// shared-memory chunk buffers (kChunk bytes) with one mbarrier each; its lane 0
// streams the warp's rows through the ring with cp.async.bulk (1-D TMA,
// complete_tx on the slot's mbarrier), so the bytes in flight per SM are fixed
// by the ring (kTWarps*kSlots*kChunk = 128 KB) instead of by the compiler's load
// scheduling.  The first kSlots chunks are issued before griddepcontrol.wait,
// overlapping the previous kernel of the dependent GEMV chain.  Rows are dealt
// to warps round-robin across SMs (warp g = local*grid + cta) so the last,
// partial pass is spread over the whole chip.  Each row is reduced by one warp
// in a fixed order (per-lane chunk/vector order, then a butterfly), so the
// result is independent of grid size and placement.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_row_chunk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

template <typename WT, typename AT, int kTWarps, int kSlots, int kChunk>
__global__ void __launch_bounds__(kTWarps * 32, 1) gemv_tma_kernel(const GemvArgs a) {
    using AccT = typename Acc<WT>::T;
    constexpr int VEC = 16 / sizeof(WT);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t x_bytes = (static_cast<size_t>(a.pitch) * sizeof(AT) + 127) & ~size_t(127);
    AT* sx = reinterpret_cast<AT*>(smem_raw);
    unsigned char* ring = smem_raw + x_bytes + static_cast<size_t>(warp) * kSlots * kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + x_bytes + static_cast<size_t>(kTWarps) * kSlots * kChunk) +
                     warp * kSlots;

    const int G = gridDim.x * kTWarps;
    const int g = warp * gridDim.x + blockIdx.x;
    const int my_rows = g < a.rows ? (a.rows - 1 - g) / G + 1 : 0;
    const uint32_t row_bytes = static_cast<uint32_t>(a.pitch) * sizeof(WT);
    const int cpr = static_cast<int>((row_bytes + kChunk - 1) / kChunk);  // chunks per row
    const int nchunks = my_rows * cpr;
    const char* Wb = static_cast<const char*>(a.W);

    auto chunk_src = [&](int i, uint32_t& bytes) {
        const int rk = i / cpr, j = i - rk * cpr;
        const size_t row = static_cast<size_t>(g) + static_cast<size_t>(rk) * G;
        const uint32_t off = static_cast<uint32_t>(j) * kChunk;
        bytes = min(static_cast<uint32_t>(kChunk), row_bytes - off);
        return Wb + row * row_bytes + off;
    };

    // x-gather barrier lives after the ring barriers
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + x_bytes + static_cast<size_t>(kTWarps) * kSlots * kChunk) +
                     kTWarps * kSlots;

    // ---- prologue: barriers + first kSlots chunks (weights only; independent of
    // the producer kernel, so it runs before griddepcontrol.wait)
    if (lane == 0) {
        for (int s = 0; s < kSlots; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
        if (warp == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(xbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < kSlots && i < nchunks; ++i) {
            uint32_t bytes;
            const char* src = chunk_src(i, bytes);
            tma_row_chunk(smem_u32(ring + i * kChunk), src, bytes, smem_u32(&bars[i]));
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- gather the concatenated input into shared memory (zero padded):
    // 16-byte-aligned segments by one bulk TMA copy each (a single L2 round
    // trip), the rest element-wise.
    int off = 0;
    uint32_t tx = 0;
    for (int s = 0; s < a.nseg; ++s) {
        const uint32_t nb = static_cast<uint32_t>(a.seg_len[s]) * sizeof(AT);
        const bool bulk = ((reinterpret_cast<uintptr_t>(a.seg[s]) | nb | (off * sizeof(AT))) & 15u) == 0 && nb > 0;
        if (bulk) {
            tx += nb;
        } else {
            const AT* src = static_cast<const AT*>(a.seg[s]);
            for (int i = threadIdx.x; i < a.seg_len[s]; i += blockDim.x) sx[off + i] = src[i];
        }
        off += a.seg_len[s];
    }
    for (int i = off + threadIdx.x; i < a.pitch; i += blockDim.x) sx[i] = AT(0);
    if (threadIdx.x == 0) {
        __syncwarp(1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(xbar)), "r"(tx)
                     : "memory");
        int o = 0;
        for (int s = 0; s < a.nseg; ++s) {
            const uint32_t nb = static_cast<uint32_t>(a.seg_len[s]) * sizeof(AT);
            const bool bulk = ((reinterpret_cast<uintptr_t>(a.seg[s]) | nb | (o * sizeof(AT))) & 15u) == 0 && nb > 0;
            if (bulk)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sx + o)),
                    "l"(a.seg[s]), "r"(nb), "r"(smem_u32(xbar))
                    : "memory");
            o += a.seg_len[s];
        }
    }
    __syncthreads();
    mbar_wait(smem_u32(xbar), 0u);

    AccT acc = AccT(0);
    for (int i = 0; i < nchunks; ++i) {
        const int slot = i % kSlots;
        mbar_wait(smem_u32(&bars[slot]), static_cast<uint32_t>((i / kSlots) & 1));
        const int rk = i / cpr, j = i - rk * cpr;
        const uint32_t cbytes = min(static_cast<uint32_t>(kChunk), row_bytes - static_cast<uint32_t>(j) * kChunk);
        const int nv = static_cast<int>(cbytes / 16);
        const uint4* wv = reinterpret_cast<const uint4*>(ring + slot * kChunk);
        const AT* xs = sx + static_cast<size_t>(j) * (kChunk / sizeof(WT));
#pragma unroll 4
        for (int v = lane; v < nv; v += 32) acc = dot_vec<WT, AT>(wv[v], xs + static_cast<size_t>(v) * VEC, acc);
        if (j == cpr - 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                const int row = g + rk * G;
                AccT val = acc;
                if (a.bias) val += static_cast<AccT>(static_cast<const AT*>(a.bias)[row]);
                if (a.act) val = val > AccT(0) ? val : AccT(0.1) * val;
                static_cast<AT*>(a.out)[row] = static_cast<AT>(val);
                if (a.bad && !isfinite(val)) atomicMin(a.bad, a.bad_key);
            }
            acc = AccT(0);
        }
        // release the slot to the async proxy, then refill it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && i + kSlots < nchunks) {
            uint32_t bytes;
            const char* src = chunk_src(i + kSlots, bytes);
            tma_row_chunk(smem_u32(ring + slot * kChunk), src, bytes, smem_u32(&bars[slot]));
        }
    }
}

// DDIM: x0 = (x - s1*eps)/s2 ; out = s3*x0 + s4*eps, every op rounded exactly
// as the reference's fp64 expression (no FMA contraction).
template <typename AT>
__global__ void ddim_kernel(const DdimArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.d; i += gridDim.x * blockDim.x) {
        const double x = static_cast<double>(static_cast<const AT*>(a.x)[i]);
        const double e = static_cast<double>(static_cast<const AT*>(a.eps)[i]);
        if (a.bad && !isfinite(e)) atomicMin(a.bad, a.bad_key);
        const double x0 = __ddiv_rn(__dsub_rn(x, __dmul_rn(a.s1, e)), a.s2);
        const double o = __dadd_rn(__dmul_rn(a.s3, x0), __dmul_rn(a.s4, e));
        static_cast<AT*>(a.out)[i] = static_cast<AT>(o);
    }
}

__global__ void delay_kernel(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(20000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

template <typename AT>
__global__ void from_f64_kernel(const double* src, AT* dst, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = static_cast<AT>(src[i]);
}

int g_num_sms[64] = {0};
bool g_attr_done[64][3] = {};

int num_sms() {
    int dev = 0;
    ADX_CUDA(cudaGetDevice(&dev));
    if (!g_num_sms[dev]) ADX_CUDA(cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev));
    return g_num_sms[dev];
}

bool use_ldg_gemv() {
    static const bool v = [] {
        const char* e = getenv("ADX_GEMV");
        return e && std::string(e) == "ldg";
    }();
    return v;
}

// (warps per CTA, ring slots per warp, chunk bytes, CTAs per SM) of the TMA GEMV;
// ADX_GEMV_CFG=<index> selects one for tuning runs.
struct TmaCfg {
    int warps, slots, chunk, ctas_per_sm;
};
constexpr TmaCfg kTmaCfgs[] = {{8, 4, 4096, 1}, {8, 2, 8192, 1}, {4, 4, 4096, 2}, {8, 8, 2048, 1},
                               {16, 2, 4096, 1}, {4, 2, 8192, 2}};
constexpr int kNumTmaCfgs = sizeof(kTmaCfgs) / sizeof(kTmaCfgs[0]);

int tma_cfg_index() {
    static int forced = -2;
    if (forced == -2) {
        const char* e = getenv("ADX_GEMV_CFG");
        forced = e ? std::max(0, std::min(kNumTmaCfgs - 1, atoi(e))) : -1;
    }
    return forced < 0 ? 4 : forced;  // 16 warps x 2 slots x 4 KB: best of the B200 sweep
}

template <typename WT, typename AT, int W, int S, int CH>
void launch_tma(const GemvArgs& a, cudaLaunchConfig_t& cfg, int ctas_per_sm) {
    static bool attr_done[64] = {};
    int dev = 0;
    ADX_CUDA(cudaGetDevice(&dev));
    if (!attr_done[dev]) {
        ADX_CUDA(cudaFuncSetAttribute(gemv_tma_kernel<WT, AT, W, S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
        attr_done[dev] = true;
    }
    const size_t x_bytes = (static_cast<size_t>(a.pitch) * sizeof(AT) + 127) & ~size_t(127);
    const size_t smem = x_bytes + static_cast<size_t>(W) * S * (CH + 8) + 16;
    if (smem * ctas_per_sm > 227 * 1024) ctas_per_sm = 1;
    if (smem > 227 * 1024) throw std::invalid_argument("gemv: input width too large for shared memory");
    const int want = (a.rows + W - 1) / W;
    cfg.gridDim = dim3(std::max(1, std::min(want, num_sms() * ctas_per_sm)));
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    ADX_CUDA(cudaLaunchKernelEx(&cfg, gemv_tma_kernel<WT, AT, W, S, CH>, a));
}

template <typename WT, typename AT>
void launch_gemv_t(int prec, const GemvArgs& a, cudaStream_t stream, bool pdl) {
    int dev = 0;
    ADX_CUDA(cudaGetDevice(&dev));
    if (!g_attr_done[dev][prec]) {
        ADX_CUDA(cudaFuncSetAttribute(gemv_kernel<WT, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        g_attr_done[dev][prec] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cfg.stream = stream;
    if (use_ldg_gemv()) {
        const size_t smem = static_cast<size_t>(a.pitch) * sizeof(AT);
        if (smem > 200 * 1024) throw std::invalid_argument("gemv: input width too large for shared memory");
        cfg.gridDim = dim3((a.rows + kWarps - 1) / kWarps);
        cfg.blockDim = dim3(kWarps * 32);
        cfg.dynamicSmemBytes = smem;
        ADX_CUDA(cudaLaunchKernelEx(&cfg, gemv_kernel<WT, AT>, a));
        return;
    }
    const TmaCfg& c = kTmaCfgs[tma_cfg_index()];
    switch (tma_cfg_index()) {
        case 0: launch_tma<WT, AT, 8, 4, 4096>(a, cfg, c.ctas_per_sm); break;
        case 1: launch_tma<WT, AT, 8, 2, 8192>(a, cfg, c.ctas_per_sm); break;
        case 2: launch_tma<WT, AT, 4, 4, 4096>(a, cfg, c.ctas_per_sm); break;
        case 3: launch_tma<WT, AT, 8, 8, 2048>(a, cfg, c.ctas_per_sm); break;
        case 4: launch_tma<WT, AT, 16, 2, 4096>(a, cfg, c.ctas_per_sm); break;
        default: launch_tma<WT, AT, 4, 2, 8192>(a, cfg, c.ctas_per_sm); break;
    }
}

}  // namespace

int act_bytes(int prec) { return prec == kF64 ? 8 : 4; }
int weight_bytes(int prec) { return prec == kF64 ? 8 : prec == kF32 ? 4 : 2; }

size_t gemv_weight_bytes(int prec, int rows, int pitch) {
    return static_cast<size_t>(rows) * pitch * weight_bytes(prec);
}

void launch_gemv(int prec, const GemvArgs& a, cudaStream_t stream, bool pdl) {
    if (a.nseg < 1 || a.nseg > kMaxSegs) throw std::invalid_argument("gemv: bad segment count");
    if (a.pitch % 8 != 0 || a.pitch < a.K) throw std::invalid_argument("gemv: bad pitch");
    switch (prec) {
        case kF64: launch_gemv_t<double, double>(prec, a, stream, pdl); break;
        case kF32: launch_gemv_t<float, float>(prec, a, stream, pdl); break;
        case kBF16: launch_gemv_t<__nv_bfloat16, float>(prec, a, stream, pdl); break;
        default: throw std::invalid_argument("gemv: bad precision");
    }
}

// Microbenchmark: a dependent chain of `chain` square GEMVs (n x n, distinct
// weight buffers so the chain streams chain*n*n*wb bytes from HBM), captured in
// one CUDA graph and launched `iters` times; returns device ms per GEMV.
double bench_gemv_chain(int prec, int n, int chain, int iters, bool pdl) {
    const int pitch = (n + 7) & ~7;
    const size_t wbytes = static_cast<size_t>(n) * pitch * weight_bytes(prec);
    std::vector<void*> W(chain), v(chain + 1);
    void* bad = nullptr;
    for (int i = 0; i < chain; ++i) {
        ADX_CUDA(cudaMalloc(&W[i], wbytes));
        ADX_CUDA(cudaMemset(W[i], 0x11, wbytes));  // small finite values in every dtype
    }
    for (int i = 0; i <= chain; ++i) {
        ADX_CUDA(cudaMalloc(&v[i], static_cast<size_t>(pitch) * act_bytes(prec)));
        ADX_CUDA(cudaMemset(v[i], 0, static_cast<size_t>(pitch) * act_bytes(prec)));
    }
    ADX_CUDA(cudaMalloc(&bad, 8));
    cudaStream_t st;
    ADX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    ADX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < chain; ++i) {
        GemvArgs a = {};
        a.W = W[i];
        a.rows = n;
        a.pitch = pitch;
        a.K = n;
        a.nseg = 1;
        a.seg[0] = v[i];
        a.seg_len[0] = n;
        a.out = v[i + 1];
        a.act = 1;
        launch_gemv(prec, a, st, pdl);
    }
    ADX_CUDA(cudaStreamEndCapture(st, &g));
    ADX_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1;
    ADX_CUDA(cudaEventCreate(&e0));
    ADX_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) ADX_CUDA(cudaGraphLaunch(ge, st));
    ADX_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) ADX_CUDA(cudaGraphLaunch(ge, st));
    ADX_CUDA(cudaEventRecord(e1, st));
    ADX_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    ADX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    for (void* p : W) cudaFree(p);
    for (void* p : v) cudaFree(p);
    cudaFree(bad);
    return ms / (static_cast<double>(iters) * chain);
}

void launch_ddim(int prec, const DdimArgs& a, cudaStream_t stream) {
    const int threads = 256;
    const int blocks = std::max(1, std::min((a.d + threads - 1) / threads, num_sms() * 4));
    if (prec == kF64)
        ddim_kernel<double><<<blocks, threads, 0, stream>>>(a);
    else
        ddim_kernel<float><<<blocks, threads, 0, stream>>>(a);
    ADX_CUDA(cudaGetLastError());
}

void launch_delay(double seconds, cudaStream_t stream) {
    if (seconds <= 0.0) return;
    delay_kernel<<<1, 1, 0, stream>>>(static_cast<unsigned long long>(seconds * 1e9));
    ADX_CUDA(cudaGetLastError());
}

void launch_from_f64(int prec, const double* src, void* dst, int n, cudaStream_t stream) {
    const int threads = 256;
    const int blocks = std::max(1, std::min((n + threads - 1) / threads, 1024));
    if (prec == kF64)
        from_f64_kernel<double><<<blocks, threads, 0, stream>>>(src, static_cast<double*>(dst), n);
    else
        from_f64_kernel<float><<<blocks, threads, 0, stream>>>(src, static_cast<float*>(dst), n);
    ADX_CUDA(cudaGetLastError());
}

}  // namespace adx
