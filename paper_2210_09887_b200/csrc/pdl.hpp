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

#include <atomic>
#include <utility>

namespace dfx {

// Chain trace (DFX_KTRACE=1, development only): CTA 0 of every kernel stamps
// %globaltimer when its dependency wait returns, i.e. when the previous kernel
// of the stream has completed; consecutive stamps are the per-kernel time in
// the real (overlapped) launch chain. TU-local pointers, set per translation
// unit by its DFX_KTRACE_SETTER.
namespace {
__device__ unsigned long long* g_kt_buf;
__device__ unsigned* g_kt_ctr;
}  // namespace
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long* b = g_kt_buf;
        if (b) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            b[atomicAdd(g_kt_ctr, 1u) & 4095u] = t;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define DFX_KTRACE_SETTER(name)                                     \
    void name(unsigned long long* b, unsigned* c) {                 \
        cudaMemcpyToSymbol(g_kt_buf, &b, sizeof b);                 \
        cudaMemcpyToSymbol(g_kt_ctr, &c, sizeof c);                 \
    }

inline bool pdl_enabled() {
    static const int on = [] {
        const char* e = getenv("DFX_PDL");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return on != 0;
}

// One-time setup per device (kernel attributes belong to a device context, so
// an engine on a second GPU of the same process needs its own): runs f() once
// for the calling thread's current device. Concurrent first calls may both run
// f(); the setups used here are idempotent.
template <typename F>
inline void once_per_device(std::atomic<unsigned long long>& done, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_acq_rel);
}

// SM count of the calling thread's current device (cached per device).
inline int device_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int n = cache[dev & 63].load(std::memory_order_relaxed);
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev & 63].store(n, std::memory_order_relaxed);
    }
    return n;
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
