// Microbenchmark (dev tool, not part of the product): the per-K-block
// handshake skeleton of k_conv_dense in isolation, to find what paces a
// K-block when neither the tensor pipe nor memory does.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/skel_bench.cu -o /tmp/skel && /tmp/skel
// Roles as in k_conv_dense: NWG producer warpgroups take K-blocks round robin
// (wait empty -> [split + tcgen05.st] -> fence -> arrive full, 4 warps), one
// weight lane (wait empty -> arrive [+ 16 KB bulk copy]), NISS MMA issuers
// taking groups of PAIR K-blocks alternately (wait full -> [6 MMAs / K-block]
// -> commit empty), a ring of NST stages. Reports cycles per K-block.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

struct Cfg {
    int nwg, niss, pair, nst, weights, mma, sttm, n, kb, extra_warps;
};

constexpr int kMaxThreads = 736;

__global__ void __launch_bounds__(kMaxThreads, 1) k_skel(Cfg cfg, const float* wsrc, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[8], empty[8], done;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NST = cfg.nst, KB = cfg.kb;
    const int wp = 4 * cfg.nwg;  // producer warps
    const int w_iss0 = wp, w_w = wp + cfg.niss;  // issuers, weight warp
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&full[i]), 4 + (cfg.weights ? 1 : 0));
            mbar_init(smem_u32(&empty[i]), 1);
        }
        mbar_init(smem_u32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f800000u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase, sb = smem_u32(smem);
    const uint32_t a_col0 = 256, w_stage = (uint32_t)cfg.n * 16 * 8;
    long long t0 = clock64();
    if (warp < wp) {
        const int wg = warp >> 2, wq = warp & 3;
        uint32_t st = 0, ph = 0;
        for (int g = 0; g < KB; ++g) {
            const uint32_t s = st, q = ph;
            if (++st == (uint32_t)NST) st = 0, ph ^= 1;
            if (g % cfg.nwg != wg) continue;
            mbar_wait(smem_u32(&empty[s]), q ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (cfg.sttm) {
                uint32_t hv[16], lv[16];
                const uint32_t src = sb + (uint32_t)(tid & 127) * 80 + (uint32_t)(g & 7) * 16;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(hv[4 * q4]), "=r"(hv[4 * q4 + 1]), "=r"(hv[4 * q4 + 2]), "=r"(hv[4 * q4 + 3])
                                 : "r"(src + 16 * q4));
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float x = __uint_as_float(hv[e]);
                    hv[e] &= 0xffffe000u;
                    lv[e] = __float_as_uint(__fsub_rn(x, __uint_as_float(hv[e])));
                }
                const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + a_col0 + s * 32;
                st16(taddr, hv);
                st16(taddr + 16, lv);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&full[s]));
        }
    } else if (warp >= w_iss0 && warp < w_iss0 + cfg.niss) {
        const int mw = warp - w_iss0;
        const uint32_t id = idesc(cfg.n), lbo = (uint32_t)cfg.n * 16;
        uint32_t st = 0, ph = 0;
        for (int kb = 0, q = 0; kb < KB; kb += cfg.pair, ++q) {
            const int cnt = kb + cfg.pair <= KB ? cfg.pair : KB - kb;
            if (q % cfg.niss != mw) {
                for (int h = 0; h < cnt; ++h)
                    if (++st == (uint32_t)NST) st = 0, ph ^= 1;
                continue;
            }
            uint32_t s = st, p = ph;
            for (int h = 0; h < cnt; ++h) {
                mbar_wait(smem_u32(&full[s]), p);
                if (++s == (uint32_t)NST) s = 0, p ^= 1;
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (elect_one()) {
                for (int h = 0; h < cnt; ++h) {
                    const uint32_t wb = sb + 64 * 1024 + st * w_stage;
                    if (cfg.mma) {
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const uint64_t dh = desc(wb + 2 * j * lbo, lbo, 128), dl = desc(wb + w_stage / 2 + 2 * j * lbo, lbo, 128);
                            const uint32_t d = tmem + mw * cfg.n, at = tmem + a_col0 + st * 32;
                            mma_ts(d, at + 16 + 8 * j, dh, id, 1u);
                            mma_ts(d, at + 8 * j, dl, id, 1u);
                            mma_ts(d, at + 8 * j, dh, id, 1u);
                        }
                    }
                    commit(smem_u32(&empty[st]));
                    if (++st == (uint32_t)NST) st = 0, ph ^= 1;
                }
            } else {
                for (int h = 0; h < cnt; ++h)
                    if (++st == (uint32_t)NST) st = 0, ph ^= 1;
            }
            __syncwarp();
        }
        if (mw == 0 && lane == 0) mbar_arrive(smem_u32(&done));
    } else if (warp == w_w && cfg.weights) {
        if (lane == 0) {
            uint32_t st = 0, ph = 0;
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(smem_u32(&empty[st]), ph ^ 1);
                if (cfg.weights == 2) {
                    mbar_arrive_tx(smem_u32(&full[st]), w_stage);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            sb + 64 * 1024 + st * w_stage),
                        "l"(wsrc + (size_t)(kb % 64) * (w_stage / 4)), "r"(w_stage), "r"(smem_u32(&full[st]))
                        : "memory");
                } else {
                    mbar_arrive(smem_u32(&full[st]));
                }
                if (++st == (uint32_t)NST) st = 0, ph ^= 1;
            }
        }
        __syncwarp();
    } else if (warp >= w_w + 1 && warp < w_w + 1 + cfg.extra_warps) {
        // idle warps parked on a barrier that completes at the end (epilogue / loader stand-ins)
        mbar_wait(smem_u32(&done), 0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    float* w;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&w, 64 * 128 * 16 * 8 + 1024);
    cudaMemset(w, 0, 64 * 128 * 16 * 8 + 1024);
    cudaFuncSetAttribute(k_skel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto run = [&](const char* name, Cfg c) {
        const int threads = (4 * c.nwg + c.niss + 1 + c.extra_warps) * 32;
        long long best = 1LL << 60;
        for (int rep = 0; rep < 3; ++rep) {
            k_skel<<<148, threads, 200 * 1024>>>(c, w, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("%s: %s\n", name, cudaGetErrorString(e));
                exit(1);
            }
            long long h[148];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            best = mx < best ? mx : best;
        }
        printf("%-44s %7.1f cycles / K-block  (MMA floor %d)\n", name, (double)best / c.kb, c.mma ? 6 * c.n / 2 : 0);
    };
    const int KB = 2880;
    //            nwg niss pair nst weights mma sttm n   kb  extra
    run("skeleton: 3 WG, 2 iss x2, 8 st, no work", {3, 2, 2, 8, 1, 0, 0, 128, KB, 0});
    run("skeleton, 1 issuer x2", {3, 1, 2, 8, 1, 0, 0, 128, KB, 0});
    run("skeleton, 2 issuers x4", {3, 2, 4, 8, 1, 0, 0, 128, KB, 0});
    run("skeleton, 1 WG", {1, 2, 2, 8, 1, 0, 0, 128, KB, 0});
    run("skeleton + sttm", {3, 2, 2, 8, 1, 0, 1, 128, KB, 0});
    run("MMA only N=128 (no sttm, no weights)", {3, 2, 2, 8, 0, 1, 0, 128, KB, 0});
    run("MMA only N=128 x4", {3, 2, 4, 8, 0, 1, 0, 128, KB, 0});
    for (int n : {64, 128})
        for (int st : {6, 8})
            for (int pr : {2, 3, 4, 6, 8}) {
                if (pr > st) continue;
                char name[96];
                snprintf(name, sizeof name, "full N=%d, %d stages, 1 issuer x%d", n, st, pr);
                run(name, {3, 1, pr, st, 2, 1, 1, n, KB, 0});
            }
    run("full N=128, 8 stages, 2 issuers x4 (ref)", {3, 2, 4, 8, 2, 1, 1, 128, KB, 0});
    return 0;
}
