// kernels.cuh -- sm_100a kernels of the async denoising hot path.
//
//  * stage GEMV  (run_stage_range's two dense layers, proj/src/denoiser.cpp:182-184):
//      out[r] = act( W[r,:] . concat(seg_0 .. seg_{n-1}) + bias[r] )
//    HBM-bound at batch 1; the skip concat (denoiser.cpp:159-177) is never
//    materialised in HBM -- the segments are gathered straight into shared
//    memory as the column blocks of W.  Finite check (denoiser.cpp:185-187)
//    is an epilogue atomicMin into a device word.
//  * DDIM update (proj/src/diffusion.cpp:95-116), IEEE-exact in fp64.
//  * delay kernel (InstrumentedDenoiser, executor.hpp:53-59) and converts.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace adx {

enum Precision { kF64 = 0, kF32 = 1, kBF16 = 2 };

constexpr int kMaxSegs = 8;

struct GemvArgs {
    const void* W;      // rows x pitch, weight dtype
    int rows;
    int pitch;          // elements per row (multiple of 8, >= K, zero padded)
    int K;              // logical input width = sum(seg_len)
    int nseg;
    const void* seg[kMaxSegs];  // activation dtype
    int seg_len[kMaxSegs];
    const void* bias;   // rows, activation dtype
    void* out;          // rows, activation dtype
    int act;            // 1 = leaky relu (slope 0.1)
    int* bad;           // finite check target (nullptr = off)
    int bad_key;
};

// Bytes of weights the kernel streams per launch (the roofline unit).
size_t gemv_weight_bytes(int prec, int rows, int pitch);

// Launch on `stream` (current device must own it).  pdl=true sets
// programmatic stream serialization so the weight prologue overlaps the
// previous kernel's tail.
void launch_gemv(int prec, const GemvArgs& a, cudaStream_t stream, bool pdl);

struct DdimArgs {
    const void* x;
    const void* eps;
    void* out;
    int d;
    double s1, s2, s3, s4;  // sqrt(1-abar_t), sqrt(abar_t), sqrt(abar_{t-1}), sqrt(1-abar_{t-1})
    int* bad;
    int bad_key;
};
void launch_ddim(int prec, const DdimArgs& a, cudaStream_t stream);

void launch_delay(double seconds, cudaStream_t stream);
// fp64 -> activation dtype (fp64 copy or fp32 round)
void launch_from_f64(int prec, const double* src, void* dst, int n, cudaStream_t stream);

// dependent chain of square GEMVs in one CUDA graph: device ms per GEMV
double bench_gemv_chain(int prec, int n, int chain, int iters, bool pdl);

int act_bytes(int prec);     // activation element size
int weight_bytes(int prec);  // weight element size

}  // namespace adx
