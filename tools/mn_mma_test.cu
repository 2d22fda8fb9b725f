// micro-test (tools/mn_mma_test.cu): tcgen05.mma kind::f16, A in TMEM, B MN-major (N contiguous, SW128):
// which LBO / SBO / K-step the attention PV MMA needs for V tiles loaded [keys][64 dims]
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((sa(p) >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(lbo >> 4) << 16;
    d |= static_cast<uint64_t>(sbo >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
__device__ float aval(int i, int k) { return (float)(((i * 3 + k) % 7) - 3); }
__device__ float bval(int n, int k) { return (float)(((n + 2 * k) % 5) - 2); }
__global__ void k(float* out, uint32_t lbo, uint32_t sbo, int step_bytes) {
    __shared__ __align__(1024) uint8_t sB[64 * 128];
    __shared__ uint32_t tptr;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // B: 64 rows (n) x 64 K bf16, SW128 K-major: chunk c (8 elems) of row n at (c ^ (n & 7))
    for (int e = t; e < 64 * 64; e += blockDim.x) {  // MN-major: row = k, 64 n contiguous, SW128
        const int kk = e / 64, n = e % 64, c = n / 8, w = n % 8;
        reinterpret_cast<__nv_bfloat16*>(sB + kk * 128 + ((c ^ (kk & 7)) * 16))[w] = __float2bfloat16(bval(n, kk));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tptr)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tptr;
    // A row i = thread t (4 warps x 32 lanes = 128 lanes), K = 32 -> 16 columns of bf16x2 at col 64
    {
        uint32_t r[16];
        for (int c = 0; c < 16; ++c) {
            __nv_bfloat162 h = __floats2bfloat162_rn(aval(t, 2 * c), aval(t, 2 * c + 1));
            r[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        const uint32_t ta = tmem + 64 + (static_cast<uint32_t>(warp * 32) << 16);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (t == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(64 >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
        for (int kb = 0; kb < 2; ++kb) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                "r"(tmem + 64 + kb * 8), "l"(sdesc(sB + kb * step_bytes, lbo, sbo)), "r"(idesc), "r"(kb)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    {
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    for (int c = 0; c < 64; c += 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + c + (static_cast<uint32_t>(warp * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) out[t * 64 + c + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}
int main() {
    float* d; cudaMalloc(&d, 128 * 64 * 4);
    // measured on B200: SBO 1024 (8 key rows) works whatever the LBO (N = 64 is one swizzle
    // atom wide); SBO 16 does not
    const uint32_t cand[][3] = {{16, 1024, 2048}, {1024, 16, 2048}, {1024, 1024, 2048}, {8192, 1024, 2048}};
    int rc = 1;
    for (auto& cv : cand) {
    k<<<1, 128>>>(d, cv[0], cv[1], cv[2]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    float h[128 * 64]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0; double maxerr = 0;
    for (int i = 0; i < 128; ++i) for (int n = 0; n < 64; ++n) {
        float ref = 0; for (int kk = 0; kk < 32; ++kk) ref += (float)(((i * 3 + kk) % 7) - 3) * (float)(((n + 2 * kk) % 5) - 2);
        double err = fabs(ref - h[i * 64 + n]); if (err > maxerr) maxerr = err; if (err > 1e-3) ++bad;
    }
    printf("lbo %u sbo %u step %u: %d mismatches of %d, max err %g\n", cv[0], cv[1], cv[2], bad, 128 * 64, maxerr);
    if (!bad) rc = 0;
    }
    return rc;
}
