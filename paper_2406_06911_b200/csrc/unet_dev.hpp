// unet_dev.hpp -- per-GPU state of the UNet-shaped family (see unet_dev.cu).
#pragma once

#include "engine.hpp"
#include "tc_gemm.cuh"
#include "unet.hpp"
#include "unet_kernels.cuh"

#include <cuda_bf16.h>

#include <map>
#include <string>
#include <vector>

namespace adx {

struct UDevStage {
    bool ready = false;
    std::map<std::string, void*> p;  // matrices bf16 (row-major [out][in]), vectors fp32
    std::map<std::string, long long> bytes;
    float* chan_add = nullptr;       // [(T+1)][cout] time-embedding projection per t
    int chan_T = -1;
    // cross-attention keys [ctx_pad][C] and values, per (transformer block, context): index
    // block * contexts + context; values row-major [ctx_pad][C] (bf16 mode) or V^T split
    // along the keys [C][3 ctx_pad] (ADX_F32 mode)
    std::vector<__nv_bfloat16*> k2, vt2;
    // ADX_F32 mode, fused attention: per (block, context) the planes [Kh | Kl | Vh | Vl], each
    // [ctx_pad][C] bf16 row-major (x = hi + lo)
    std::vector<__nv_bfloat16*> kv2x;
    // video motion module: per temporal attention, the frame positional encoding through the
    // QKV projection, PE . Wqkv^T [frames][3C] fp32 (added per frame in the GEMM epilogue)
    std::vector<float*> pe_proj;
};

struct UScratch {
    __nv_bfloat16 *a = nullptr, *b = nullptr, *c = nullptr, *r = nullptr, *qkv = nullptr, *att = nullptr,
                  *ff = nullptr, *ff2 = nullptr, *P = nullptr, *VT = nullptr;
    float* S = nullptr;
    float2* gn = nullptr;
    float* eps2 = nullptr;    // CFG: [eps_u | eps_c] before the guidance combine
    void* attn_ws = nullptr;  // split-KV workspace of the fused attention (zeroed counters)
    size_t attn_ws_bytes = 0;
    // ADX_F32 mode: fp32 activations and split-bf16 operands (3 columns per column)
    float *fa = nullptr, *fb = nullptr, *fc = nullptr, *fr = nullptr, *fqkv = nullptr, *fatt = nullptr, *fff = nullptr,
          *fvt = nullptr;
    __nv_bfloat16 *sa = nullptr, *sq = nullptr, *sk = nullptr, *sv = nullptr;
};

class UNetDevice {
public:
    // exact = ADX_F32 mode: fp32 activations, split-bf16 tensor-core products (rel-L2 <= 1e-3
    // vs the fp64 oracle); otherwise ADX_BF16: bf16 activations
    UNetDevice(const Model& m, int ordinal, bool exact);
    ~UNetDevice();
    void ensure_stage(int stage);
    void ensure_tables(int T);
    bool ready(int stage) const { return st_[stage].ready; }
    long long param_bytes(int stage) const;
    // one stage on `st`: in[0] = main input (latent for stage 1), in[1] = skip
    void enqueue(int stage, const std::vector<Seg>& in, int t, void* y, bool latent_f64, cudaStream_t st);

private:
    UScratch& scratch(cudaStream_t st);
    const void* P(int stage, const char* name) const;
    const float* F(int stage, const char* name) const;
    void attention(UScratch& s, const __nv_bfloat16* q, long long ldq, const __nv_bfloat16* k, long long ldk,
                   const __nv_bfloat16* v, long long ldv, int L, int Lk, int C, __nv_bfloat16* out, cudaStream_t st,
                   int batch = 1);
    void transformer(int stage, const __nv_bfloat16* x, int H, int W, int C, __nv_bfloat16* y, cudaStream_t st);
    void motion(int stage, const __nv_bfloat16* x, int H, int W, int C, __nv_bfloat16* y, cudaStream_t st);
    void motion_exact(int stage, const float* x, int H, int W, int C, float* y, cudaStream_t st);
    // GroupNorm of every image of the batch: the fused single launch for one image, one
    // batched two-kernel launch for CFG pairs and video frames
    template <typename T>
    void gn_images(const Cat2T<T>& x, int HW, const float* gamma, const float* beta, float eps, int act, T* out,
                   UScratch& s, cudaStream_t st);
    // ADX_F32 mode
    void enqueue_exact(int stage, const std::vector<Seg>& in, int t, void* y, bool latent_f64, cudaStream_t st);
    void transformer_exact(int stage, const float* x, int H, int W, int C, float* y, cudaStream_t st);
    void attention_exact(UScratch& s, const float* q, long long ldq, const __nv_bfloat16* ks, const float* v,
                         long long ldv, const __nv_bfloat16* vts, int L, int Lk, int C, float* out, cudaStream_t st);
    // split-bf16 GEMM / conv: out = act(split(x) . W'^T + ...) with W' stored split on the device
    void gemm_x(UScratch& s, const float* x, int M, int K, const char* wname, int stage, int N, TcArgs a,
                cudaStream_t st);
    void conv_x(UScratch& s, const float* x, int H, int W, int Cin, const char* wname, int stage, int Cout, TcArgs a,
                cudaStream_t st);
    bool exact_ = false;

    const Model& m_;
    const UNetDesc& d_;
    int ordinal_;
    std::vector<UDevStage> st_;
    std::map<cudaStream_t, UScratch> scratch_;
};

}  // namespace adx
