// Programmatic dependent launch (sm_90+): every kernel of a frame is launched
// with programmatic stream serialization and starts with pdl_enter(), so the
// next kernel's launch and CTA rasterization overlap the tail of the current
// one instead of leaving the GPU idle at every kernel boundary.
//
// Safety: griddepcontrol.wait blocks until the preceding grid has COMPLETED and
// its memory is visible, and every kernel waits before touching any data, so
// the stream order of the frame is preserved transitively. The trigger only
// lets the dependent grid launch once every CTA of this grid has started.
#pragma once

#include <cuda_runtime.h>
#include <stdlib.h>

#include <utility>

namespace dfx {

__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static const int on = [] {
        const char* e = getenv("DFX_PDL");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dfx
