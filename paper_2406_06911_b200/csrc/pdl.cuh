// pdl.cuh -- Programmatic Dependent Launch for the UNet-pass kernels.
//
// Every kernel of the pass is launched with programmatic stream serialization and
// calls pdl_wait() after its prologue (barrier init, TMEM alloc, tensor-map
// prefetch) and before touching any data a predecessor produced: the launch and
// prologue overlap the previous kernel's tail (~430 kernel boundaries per pass),
// and because every kernel waits before it can finish, completion stays ordered
// transitively along the stream.  ADX_PDL=0 launches without the attribute
// (griddepcontrol.wait is then a no-op).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

namespace adx {

// (no early griddepcontrol.launch_dependents: measured no gain on the graph-replayed
// UNet pass, 6.88 ms either way, and it would let successors occupy SM resources early)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ADX_PDL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

// cudaLaunchKernelEx with the PDL attribute (plus an optional cluster size)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster_x > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster_x;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace adx
