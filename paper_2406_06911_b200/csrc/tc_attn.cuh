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

}  // namespace adx
