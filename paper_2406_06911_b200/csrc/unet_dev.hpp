// unet_dev.hpp -- per-GPU state of the UNet-shaped family (see unet_dev.cu).
#pragma once

#include "engine.hpp"
#include "unet.hpp"

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
    __nv_bfloat16* k2 = nullptr;     // cross-attention keys   [ctx_pad][C]
    __nv_bfloat16* vt2 = nullptr;    // cross-attention values [C][ctx_pad] (transposed per head)
};

struct UScratch {
    __nv_bfloat16 *a = nullptr, *b = nullptr, *c = nullptr, *r = nullptr, *qkv = nullptr, *att = nullptr,
                  *ff = nullptr, *ff2 = nullptr, *P = nullptr, *VT = nullptr;
    float* S = nullptr;
    float2* gn = nullptr;
};

class UNetDevice {
public:
    UNetDevice(const Model& m, int ordinal);
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
                   const __nv_bfloat16* v, long long ldv, const __nv_bfloat16* v_t, int L, int Lk, int C,
                   __nv_bfloat16* out, cudaStream_t st);
    void transformer(int stage, const __nv_bfloat16* x, int H, int W, int C, __nv_bfloat16* y, cudaStream_t st);

    const Model& m_;
    const UNetDesc& d_;
    int ordinal_;
    std::vector<UDevStage> st_;
    std::map<cudaStream_t, UScratch> scratch_;
};

}  // namespace adx
