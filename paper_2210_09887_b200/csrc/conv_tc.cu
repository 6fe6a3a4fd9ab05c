// Sparse DeltaConv on the 5th-gen tensor cores (tcgen05, sm_100a).
//
// Replaces padded_delta_conv's target loop (reference src/delta_layers.cpp:
// 100-147). The conv is an implicit GEMM over the COMPACTED target pixels of
// the layer (k_conv_targets builds the list):
//     D[p, o] = sum_{tap, i} X[p @ tap, i] * W[o, i, tap]
// M = 128 gathered target pixels per tile (any shape: tiles of every size,
// partial tiles, ring pixels), N = Cout (<= 256 per MMA), K = k*k*Cin walked
// as K-blocks of (tap, 32 input channels).
//
// Arithmetic: 3xTF32 (x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi);
// D += Ahi*Bhi + Ahi*Blo + Alo*Bhi, fp32 accumulate in TMEM) — fp32-grade
// accuracy (|err| ~1e-6 relative), within the stated 1e-4 tolerance of the
// reference's fp32 outputs.
//
// Pipeline (per CTA, persistent over M x N work items), 2 smem stages:
//   * B (weights, pre-split hi/lo and pre-laid-out in the UMMA canonical
//     K-major SWIZZLE_NONE image on the host) arrives by one cp.async.bulk per
//     stage, completing on an mbarrier with transaction bytes;
//   * A is gathered by all 256 threads from the HWC delta packet (zero for
//     samples outside the packet's written tiles), split hi/lo in registers and
//     stored in the canonical layout; fence.proxy.async hands it to the tensor
//     core;
//   * one thread issues the tcgen05.mma chain and tcgen05.commit's the stage's
//     mbarrier, so the gather of K-block kb+1 overlaps the MMAs of kb;
//   * epilogue: tcgen05.ld 32x32b.x32 from TMEM, 128-byte stores of each
//     pixel's channels into the output packet.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace dfx {

namespace {

constexpr int kM = 128;      // target pixels per tile (MMA M)
constexpr int kKC = 32;      // input channels per K-block
constexpr int kThreadsTC = 256;
constexpr int kAStage = kM * kKC * 4 * 2;  // hi + lo = 32 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical
// ((8,m),(T,2)):((1T,SBO),(1,LBO)) in 16-byte units), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// Instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, M=128.
__host__ __device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool valid_px(const PktDev& p, int th, int tw, int y, int x) {
    if (y < -p.halo || y >= th * p.t + p.halo || x < -p.halo || x >= tw * p.t + p.halo) return false;
    return p.ext[ext_idx(p, floor_div32(y, p.t), floor_div32(x, p.t))] != 0;
}

__global__ void __launch_bounds__(kThreadsTC, 1)
    k_conv_tc(Ctx c, PktDev in, const float* __restrict__ wsplit, int cin, int cin_pad, int cout, int cout_pad, int k,
              int s, int r, PktDev out, int hg, const int* __restrict__ list, const int* __restrict__ count) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[2], bar_mma[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int s_py[kM], s_px[kM];

    const FrameDev& F = *c.f;
    const int n = *count;
    const int nCB = (cin_pad + kKC - 1) / kKC;
    const int nKB = k * k * nCB;
    const int nNB = (cout_pad + 255) / 256;
    const int items = ((n + kM - 1) / kM) * nNB;
    if ((int)blockIdx.x >= items) return;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NBmax = cout_pad < 256 ? cout_pad : 256;
    const uint32_t b_stage_bytes = (uint32_t)NBmax * kKC * 4 * 2;
    const uint32_t stage_bytes = kAStage + b_stage_bytes;
    uint32_t ncols = 32;
    while ((int)ncols < NBmax) ncols <<= 1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(smem_u32(&bar_full[0]), 1);
        mbar_init(smem_u32(&bar_full[1]), 1);
        mbar_init(smem_u32(&bar_mma[0]), 1);
        mbar_init(smem_u32(&bar_mma[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t smem_base = smem_u32(smem);

    const int row = tid & (kM - 1), half = tid >> 7;  // gather: 2 threads per row, 16 channels each
    uint32_t g = 0;                                   // global K-block counter (stage / parity bookkeeping)

    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int mb = item / nNB, nb = item % nNB;
        const int NB = (cout_pad - nb * 256) < 256 ? (cout_pad - nb * 256) : 256;
        const uint32_t idesc = idesc_tf32(NB);
        if (tid < kM) {
            const int idx = mb * kM + tid;
            if (idx < n) {
                const int v = list[idx];
                s_py[tid] = (v >> 16) - hg;
                s_px[tid] = (v & 0xffff) - hg;
            } else {
                s_py[tid] = -(1 << 20);
                s_px[tid] = -(1 << 20);
            }
        }
        __syncthreads();
        const int py = s_py[row], px = s_px[row];
        const float* wblk = wsplit + (size_t)nb * 256 * nKB * kKC * 2;

        for (int kb = 0; kb < nKB; ++kb, ++g) {
            const uint32_t st = g & 1, q = g >> 1;
            const uint32_t a_base = smem_base + st * stage_bytes;
            const uint32_t b_base = a_base + kAStage;
            if (g >= 2) mbar_wait(smem_u32(&bar_mma[st]), (q - 1) & 1);
            const int tap = kb / nCB, cb = kb - tap * nCB;
            const int c0 = cb * kKC;
            if (tid == 0) {
                mbar_expect_tx(smem_u32(&bar_full[st]), (uint32_t)NB * kKC * 8);
                bulk_g2s(b_base, wblk + (size_t)kb * NB * kKC * 2, (uint32_t)NB * kKC * 8, smem_u32(&bar_full[st]));
            }
            // ---- gather + split A (rows = target pixels, K = 32 channels at this tap)
            {
                float v[16];
                const int ky = tap / k, kx = tap - ky * k;
                const int iy = py * s - r + ky, ix = px * s - r + kx;
                const int cbeg = c0 + half * 16;
                const bool ok = py > -(1 << 19) && valid_px(in, F.th, F.tw, iy, ix);
                if (ok && (in.C & 3) == 0 && cbeg + 16 <= cin) {
                    const float4* src = reinterpret_cast<const float4*>(in.d + pkt_off(in, iy, ix) + cbeg);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 t = __ldg(src + j);
                        v[4 * j] = t.x, v[4 * j + 1] = t.y, v[4 * j + 2] = t.z, v[4 * j + 3] = t.w;
                    }
                } else {
                    const float* src = ok ? in.d + pkt_off(in, iy, ix) : nullptr;
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = (ok && cbeg + j < cin) ? src[cbeg + j] : 0.0f;
                }
                uint8_t* a_hi = smem + st * stage_bytes;
                uint8_t* a_lo = a_hi + kM * kKC * 4;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint4 hi, lo;
                    hi.x = to_tf32(v[4 * j]);
                    hi.y = to_tf32(v[4 * j + 1]);
                    hi.z = to_tf32(v[4 * j + 2]);
                    hi.w = to_tf32(v[4 * j + 3]);
                    lo.x = to_tf32(__fsub_rn(v[4 * j], __uint_as_float(hi.x)));
                    lo.y = to_tf32(__fsub_rn(v[4 * j + 1], __uint_as_float(hi.y)));
                    lo.z = to_tf32(__fsub_rn(v[4 * j + 2], __uint_as_float(hi.z)));
                    lo.w = to_tf32(__fsub_rn(v[4 * j + 3], __uint_as_float(hi.w)));
                    const int kc = half * 4 + j;  // 16-byte K chunk within the block
                    const uint32_t off = (uint32_t)kc * (kM * 16) + (uint32_t)row * 16;
                    *reinterpret_cast<uint4*>(a_hi + off) = hi;
                    *reinterpret_cast<uint4*>(a_lo + off) = lo;
                }
            }
            fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                mbar_wait(smem_u32(&bar_full[st]), q & 1);
                tc_fence_after();
                const int nsteps = (cin_pad - c0) / 8 < 4 ? (cin_pad - c0) / 8 : 4;
                const uint32_t lbo_a = kM * 16, lbo_b = (uint32_t)NB * 16;
                for (int j = 0; j < nsteps; ++j) {
                    const uint64_t dah = umma_desc(a_base + 2 * j * lbo_a, lbo_a, 128);
                    const uint64_t dal = umma_desc(a_base + kM * kKC * 4 + 2 * j * lbo_a, lbo_a, 128);
                    const uint64_t dbh = umma_desc(b_base + 2 * j * lbo_b, lbo_b, 128);
                    const uint64_t dbl = umma_desc(b_base + (uint32_t)NB * kKC * 4 + 2 * j * lbo_b, lbo_b, 128);
                    mma_tf32(tmem, dal, dbh, idesc, (kb > 0 || j > 0) ? 1u : 0u);
                    mma_tf32(tmem, dah, dbl, idesc, 1u);
                    mma_tf32(tmem, dah, dbh, idesc, 1u);
                }
                mma_commit(smem_u32(&bar_mma[st]));
            }
        }
        // ---- epilogue: wait for the last commit (covers all earlier MMAs)
        {
            const uint32_t gl = g - 1;
            mbar_wait(smem_u32(&bar_mma[gl & 1]), (gl >> 1) & 1);
            tc_fence_after();
            const int lq = warp & 3, chalf = warp >> 2;
            const int prow = lq * 32 + lane;
            const int oy = s_py[prow], ox = s_px[prow];
            const bool valid = oy > -(1 << 19);
            for (int cc = chalf * 32; cc < NB; cc += 64) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)cc, v);
                if (valid) {
                    const int o0 = nb * 256 + cc;
                    float* dst = out.d + pkt_off(out, oy, ox) + o0;
                    if ((out.C & 3) == 0 && o0 + 32 <= cout) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    } else {
                        for (int j = 0; j < 32 && o0 + j < cout; ++j) dst[j] = v[j];
                    }
                }
            }
            tc_fence_before();
            __syncthreads();
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

uint32_t rna_tf32_host(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return u;
    return (u + 0x1000u) & 0xffffe000u;
}

}  // namespace

size_t conv_tc_weight_floats(int cin_pad, int cout_pad, int k) {
    const int nCB = (cin_pad + kKC - 1) / kKC;
    return (size_t)k * k * nCB * kKC * cout_pad * 2;
}

// Host: O-I-Kh-Kw fp32 weights -> per (N-block, K-block) smem images
// [hi: 8 chunks x NB rows x 4 ch][lo: same], zero padded.
void conv_tc_prepare_weights(const float* w, int cin, int cout, int k, int cin_pad, int cout_pad, float* outp) {
    const int nCB = (cin_pad + kKC - 1) / kKC, K2 = k * k, nKB = K2 * nCB;
    const int nNB = (cout_pad + 255) / 256;
    memset(outp, 0, conv_tc_weight_floats(cin_pad, cout_pad, k) * sizeof(float));
    for (int nb = 0; nb < nNB; ++nb) {
        const int NB = std::min(256, cout_pad - nb * 256);
        float* base = outp + (size_t)nb * 256 * nKB * kKC * 2;
        for (int kb = 0; kb < nKB; ++kb) {
            const int tap = kb / nCB, cb = kb % nCB;
            float* blob = base + (size_t)kb * NB * kKC * 2;
            for (int nn = 0; nn < NB; ++nn) {
                const int o = nb * 256 + nn;
                for (int ci = 0; ci < kKC; ++ci) {
                    const int i = cb * kKC + ci;
                    float x = 0.0f;
                    if (o < cout && i < cin) x = w[((size_t)o * cin + i) * K2 + tap];
                    const uint32_t hb = rna_tf32_host(x);
                    float hi;
                    memcpy(&hi, &hb, 4);
                    const uint32_t lb = rna_tf32_host(x - hi);
                    float lo;
                    memcpy(&lo, &lb, 4);
                    const size_t off = ((size_t)(ci / 4) * NB + nn) * 4 + (ci % 4);
                    blob[off] = hi;
                    blob[(size_t)NB * kKC + off] = lo;
                }
            }
        }
    }
}

void launch_conv_tc(const Ctx& c, cudaStream_t s, PktDev in, const float* wsplit, int cin, int cin_pad, int cout,
                    int cout_pad, int k, int st, int r, PktDev out, int hg, const int* list, const int* count,
                    int max_targets, int num_sms) {
    const int NBmax = cout_pad < 256 ? cout_pad : 256;
    const size_t smem = 2 * ((size_t)kAStage + (size_t)NBmax * kKC * 8);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = 200 * 1024;
    }
    if (smem > 200 * 1024) throw std::runtime_error("conv_tc: smem too large");
    const int nNB = (cout_pad + 255) / 256;
    const long long items = (long long)((max_targets + kM - 1) / kM) * nNB;
    int grid = num_sms;
    if (items < grid) grid = (int)(items < 1 ? 1 : items);
    k_conv_tc<<<grid, kThreadsTC, smem, s>>>(c, in, wsplit, cin, cin_pad, cout, cout_pad, k, st, r, out, hg, list,
                                             count);
}

}  // namespace dfx
