// Microbenchmark: back-to-back tcgen05.mma.kind::tf32 issue rate per SM
// (M = 128, A from TMEM or shared memory, B from shared memory), to know the
// floor of the conv kernels' K-block pacing (dev tool, not part of the product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mma_rate.cu -o tools/mma_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ uint32_t idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f800000u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    long long t0 = 0, t1 = 0;
    if (warp == 1) {
        const uint32_t sb = smem_u32(smem);
        const uint32_t lbo_b = N * 16;
        uint32_t pred;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        t0 = clock64();
        if (pred) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint64_t db = desc(sb + 2 * j * lbo_b, lbo_b, 128);
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        if (A_TMEM) {
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                                "r"(tmem + 256 + 8 * j), "l"(db), "r"(idesc(N)), "r"(1)
                                : "memory");
                        } else {
                            const uint64_t da = desc(sb + 32768 + 2 * j * 2048, 2048, 128);
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                "l"(da), "l"(db), "r"(idesc(N)), "r"(1)
                                : "memory");
                        }
                    }
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar))
                         : "memory");
        }
        __syncwarp();
        asm volatile(
            "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                smem_u32(&bar))
            : "memory");
        t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool AT>
void run(long long* d) {
    cudaFuncSetAttribute(k_rate<N, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 2000;
    for (int rep = 0; rep < 3; ++rep) k_rate<N, AT><<<148, 128, 64 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double per = (double)mx / (iters * 12.0);
    printf("N=%3d A=%s: %.1f cycles per M128xN%dxK8 tf32 MMA (%.0f%% of the 128*N/256 floor)\n", N, AT ? "tmem" : "smem",
           per, N, 100.0 * (128.0 * N / 256.0) / per);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    run<64, true>(d);
    run<128, true>(d);
    run<256, true>(d);
    run<64, false>(d);
    run<128, false>(d);
    run<256, false>(d);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
