// tc_attn.cuh -- fused tcgen05 multi-head attention (see tc_attn.cu).
#pragma once

#include "host.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace adx {

// out[L x C] (row stride ldo) = per 64-wide head softmax(Q K^T / 8) V, with
// Q [L x C] (ldq), K [Lk x C] (ldk) and V [Lk x C] (ldv): every operand row-major as the
// projections write it (V feeds the PV MMA MN-major; no transpose)
// ws: zero-initialised workspace of tc_attention_ws_bytes(L, Lk, C, batch) bytes (per stream;
// its counters re-arm themselves) enabling split-KV load balancing; nullptr runs unsplit.
// batch > 1: independent images in one launch, stacked: Q / out rows [b * L, (b + 1) * L),
// K and V rows [b * Lk, (b + 1) * Lk)
void tc_attention(const void* Q, long long ldq, const void* K, long long ldk, const void* V, long long ldv, int L,
                  int Lk, int C, __nv_bfloat16* out, long long ldo, cudaStream_t st, void* ws = nullptr,
                  size_t ws_bytes = 0, int batch = 1);
size_t tc_attention_ws_bytes(int L, int Lk, int C, int batch = 1);
// per-CTA %globaltimer stamps of the last stream-K launch (16 per CTA; -DADX_SK_TIMELINE builds)
void tc_sk_timeline(unsigned long long* out, int n_ctas);

// the ADX_F32 mode's attention: every operand as bf16 hi and lo planes (x = hi + lo, same
// layout and strides each), S = Qh Kh^T + Qh Kl^T + Ql Kh^T and O = Ph Vh + Ph Vl + Pl Vh with
// fp32 accumulation in TMEM, fp32 softmax, P split in registers; fp32 output (ldo floats).
// Same grid, split-KV workspace and batching rules as tc_attention.
void tc_attention_x(const void* Qh, const void* Ql, long long ldq, const void* Kh, const void* Kl, long long ldk,
                    const void* Vh, const void* Vl, long long ldv, int L, int Lk, int C, float* out, long long ldo,
                    cudaStream_t st, void* ws = nullptr, size_t ws_bytes = 0, int batch = 1);

}  // namespace adx
