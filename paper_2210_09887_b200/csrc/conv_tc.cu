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
// Arithmetic: 3xTF32 (x = hi + lo with hi = x truncated to TF32, lo = x - hi;
// D += Ahi*Bhi + Ahi*Blo + Alo*Bhi, fp32 accumulate in TMEM) — fp32-grade
// accuracy (|err| ~1e-6 relative), within the stated 1e-4 tolerance of the
// reference's fp32 outputs.
//
// Pipeline (per CTA, persistent over M x N work items), 2-4 smem stages:
//   * B (weights, pre-split hi/lo and pre-laid-out in the UMMA canonical
//     K-major SWIZZLE_NONE image on the host) arrives by one cp.async.bulk per
//     stage, completing on the stage's mbarrier with transaction bytes;
//   * A is gathered by 8 producer warps from the HWC delta packet (zero for
//     samples outside the packet's written tiles), split hi/lo in registers and
//     stored in the canonical layout; fence.proxy.async hands it to the tensor
//     core;
//   * one thread issues the tcgen05.mma chain and tcgen05.commit's the stage's
//     "empty" mbarrier; the producers run up to nstages K-blocks ahead;
//   * accumulators are double-buffered in TMEM (when 2*N <= 512 columns) so the
//     4 epilogue warps (tcgen05.ld 32x32b.x32 -> 128-byte stores of each
//     pixel's channels) drain tile i while the MMAs of tile i+1 run.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "pdl.hpp"

namespace dfx {

namespace {

constexpr int kM = 128;      // target pixels per tile (MMA M)
constexpr int kKC = 32;      // input channels per K-block
constexpr int kAStage = kM * kKC * 4 * 2;  // hi + lo = 32 KiB
// K-block geometry. Input-channel counts of 8 or 16 (padded from an RGB frame's
// 3, say) pack several taps into one 32-channel K-block (tap-major: tpk taps x
// cin_pad channels) instead of padding every tap to 32 channels; wider inputs
// take one (32-channel block, tap) per K-block.
struct KGeom {
    int tpk;  // taps per K-block (1: channel block outer, tap inner)
    int nCB;  // channel blocks
    int nKB;  // K-blocks
};
__host__ __device__ __forceinline__ KGeom k_geom(int cin_pad, int k) {
    const int K2 = k * k;
    KGeom g;
    g.tpk = (cin_pad == 8 || cin_pad == 16) ? kKC / cin_pad : 1;
    g.nCB = g.tpk > 1 ? 1 : (cin_pad + kKC - 1) / kKC;
    g.nKB = g.tpk > 1 ? (K2 + g.tpk - 1) / g.tpk : K2 * g.nCB;
    return g;
}

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
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
        "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
        "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
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

// Warp roles (416 threads): warps 0-7 are two producer warpgroups that gather
// A for alternating K-blocks (one thread per row, 32 channels = 8 x 16 B
// loads, the next K-block of the same group prefetched into registers); warps
// 8-11 epilogue (TMEM lane quarter = warp % 4); warp 12 issues the MMAs.
// Barriers: full[s] (4 producer-warp arrivals, the weight bulk copy's
// transaction bytes), empty[s] (tcgen05.commit), acc_full[b] (commit after a
// work unit's last K-block), acc_empty[b] (4 epilogue warps).
// Work unit = (128-row M tile, 256-wide N block, K split). K order: channel
// block outer, tap inner. Each row's per-tap validity (packet tile written /
// inside the grown extent) is resolved once per unit into a bitmask, so the
// K loop issues no dependent loads. Split-K (layers with few target tiles)
// writes fp32 partials to a workspace reduced in fixed order by
// k_conv_splitk_reduce (deterministic).
constexpr int kProdWarps = 8, kEpiWarps = 4;
constexpr int kThreadsV2 = (kProdWarps + kEpiWarps + 1) * 32;

// expect_tx WITHOUT an arrival (the issuing warp arrives after its own stores)
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

struct ConvArgs {
    PktDev in, out;
    const float* wsplit;
    const int* list;
    const int* count;
    float* ws;  // split-K workspace [splits][n][cout_pad] or nullptr
    int cin, cin_pad, cout, cout_pad, k, s, r, hg, splits;
};

template <int NST>
__global__ void __launch_bounds__(kThreadsV2, 1) k_conv_tc(Ctx c, ConvArgs a) {
    pdl_enter();
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[NST], bar_empty[NST], bar_accf[2], bar_acce[2];
    __shared__ uint32_t tmem_base_sh;

    const FrameDev& F = *c.f;
    const int n = *a.count;
    const KGeom kg = k_geom(a.cin_pad, a.k);
    const int K2 = a.k * a.k;
    const int nKB = kg.nKB;
    const int nNB = (a.cout_pad + 255) / 256;
    const int S = a.splits;
    const int units = ((n + kM - 1) / kM) * nNB * S;
    if ((int)blockIdx.x >= units) return;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NBmax = a.cout_pad < 256 ? a.cout_pad : 256;
    const uint32_t stage_bytes = (uint32_t)NBmax * kKC * 8;  // smem: weights only
    // TMEM (512 columns): accumulators [0, nbuf*acc_cols), then NST A stages of
    // 64 columns (32 hi + 32 lo tf32 columns per row / lane).
    uint32_t acc_cols = 32;
    while ((int)acc_cols < NBmax) acc_cols <<= 1;
    const int nbuf = acc_cols * 2 + NST * 64 <= 512 ? 2 : 1;
    const uint32_t ncols = 512;
    const uint32_t a_col0 = nbuf * acc_cols;

    if (warp == kProdWarps + kEpiWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_full[i]), 4);
            mbar_init(smem_u32(&bar_empty[i]), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_accf[i]), 1);
            mbar_init(smem_u32(&bar_acce[i]), kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t smem_base = smem_u32(smem);

    // unit -> (m tile, n block, split) and its K-block range
    auto unit_info = [&](int u, int& mb, int& nb, int& kb0, int& kb1) {
        const int sp = u % S, t = u / S;
        mb = t / nNB;
        nb = t % nNB;
        kb0 = (int)(((long long)nKB * sp) / S);
        kb1 = (int)(((long long)nKB * (sp + 1)) / S);
    };

    if (warp < kProdWarps) {
        // ------------------------------------------------ producers
        const int wg = warp >> 2;      // warpgroup: K-blocks with g % 2 == wg
        const int row = tid & (kM - 1);
        const int wid_in_wg = warp & 3;
        // state of the K-block this thread gathers next
        int u = blockIdx.x, mb, nb, kb0, kb1;
        unit_info(u, mb, nb, kb0, kb1);
        int kb = kb0;
        uint32_t g = 0;  // CTA-global K-block sequence number of (u, kb)
        int py = 0, px = 0;
        uint64_t vmask = 0;
        auto load_rows = [&]() {
            const int idx = mb * kM + row;
            py = -(1 << 20), px = -(1 << 20);
            vmask = 0;
            if (idx < n) {
                const int v = __ldg(a.list + idx);
                py = (v >> 16) - a.hg;
                px = (v & 0xffff) - a.hg;
                for (int tp = 0; tp < K2; ++tp) {
                    const int ky = tp / a.k, kx = tp - ky * a.k;
                    if (valid_px(a.in, F.th, F.tw, py * a.s - a.r + ky, px * a.s - a.r + kx)) vmask |= 1ull << tp;
                }
            }
        };
        auto advance = [&]() {  // move (u, kb, g) one K-block forward in the CTA sequence
            ++g;
            if (++kb == kb1) {
                u += gridDim.x;
                if (u < units) {
                    unit_info(u, mb, nb, kb0, kb1);
                    kb = kb0;
                    load_rows();
                }
            }
        };
        auto gather = [&](float* v) {
            if (kg.tpk > 1) {  // tpk taps x cin_pad channels of this K-block
                const int cp = a.cin_pad;
#pragma unroll
                for (int q = 0; q < kKC; q += 8) {
                    const int tap = kb * kg.tpk + q / cp, c0 = q % cp;
                    const bool ok = tap < K2 && ((vmask >> tap) & 1ull);
                    const int ky = ok ? tap / a.k : 0, kx = ok ? tap - ky * a.k : 0;
                    const float* src = ok ? a.in.d + pkt_off(a.in, py * a.s - a.r + ky, px * a.s - a.r + kx) : nullptr;
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[q + j] = (ok && c0 + j < a.cin) ? __ldg(src + c0 + j) : 0.0f;
                }
                return;
            }
            const int cb = kb / K2, tap = kb - cb * K2;
            const int ky = tap / a.k, kx = tap - ky * a.k;
            const int cbeg = cb * kKC;
            const bool ok = (vmask >> tap) & 1ull;
            if (ok && (a.in.C & 3) == 0 && cbeg + kKC <= a.cin) {
                const float4* src = reinterpret_cast<const float4*>(
                    a.in.d + pkt_off(a.in, py * a.s - a.r + ky, px * a.s - a.r + kx) + cbeg);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 t = __ldg(src + j);
                    v[4 * j] = t.x, v[4 * j + 1] = t.y, v[4 * j + 2] = t.z, v[4 * j + 3] = t.w;
                }
            } else {
                const float* src = ok ? a.in.d + pkt_off(a.in, py * a.s - a.r + ky, px * a.s - a.r + kx) : nullptr;
#pragma unroll
                for (int j = 0; j < kKC; ++j) v[j] = (ok && cbeg + j < a.cin) ? __ldg(src + cbeg + j) : 0.0f;
            }
        };
        load_rows();
        if (wg == 1) advance();  // warpgroup 1 starts at the second K-block
        float cur[kKC];
        bool have = u < units;
        if (have) gather(cur);
        while (have) {
            const uint32_t my_g = g;
            const int my_kb = kb, my_nb = nb;
            // prefetch this warpgroup's next K-block (two ahead in the CTA sequence)
            advance();
            if (u < units) advance();
            const bool has_next = u < units;
            float nxt[kKC];
            if (has_next) gather(nxt);
            const uint32_t st = my_g % NST, q = my_g / NST;
            const int NB = (a.cout_pad - my_nb * 256) < 256 ? (a.cout_pad - my_nb * 256) : 256;
            mbar_wait(smem_u32(&bar_empty[st]), (q & 1) ^ 1);
            tc_fence_after();
            const uint32_t b_base = smem_base + st * stage_bytes;
            if (wid_in_wg == 0 && lane == 0) {
                const float* wblk = a.wsplit + (size_t)my_nb * 256 * nKB * kKC * 2;
                mbar_expect_tx_only(smem_u32(&bar_full[st]), (uint32_t)NB * kKC * 8);
                bulk_g2s(b_base, wblk + (size_t)my_kb * NB * kKC * 2, (uint32_t)NB * kKC * 8, smem_u32(&bar_full[st]));
            }
            {
                uint32_t part[kKC];
                const uint32_t taddr = tmem + ((uint32_t)(wid_in_wg * 32) << 16) + a_col0 + st * 64;
                // hi = x with the 13 low mantissa bits cleared (exact TF32); lo = x - hi is
                // exact in fp32 and the tensor core reads its top 19 bits.
#pragma unroll
                for (int j = 0; j < kKC; ++j) part[j] = __float_as_uint(cur[j]) & 0xffffe000u;
                tmem_st32(taddr, part);
#pragma unroll
                for (int j = 0; j < kKC; ++j)
                    part[j] = __float_as_uint(__fsub_rn(cur[j], __uint_as_float(__float_as_uint(cur[j]) & 0xffffe000u)));
                tmem_st32(taddr + 32, part);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_full[st]));
            have = has_next;
            if (have) {
#pragma unroll
                for (int j = 0; j < kKC; ++j) cur[j] = nxt[j];
            }
        }
    } else if (warp < kProdWarps + kEpiWarps) {
        // ------------------------------------------------ epilogue: TMEM -> packet / workspace
        const int lq = warp & 3;
        uint32_t ui = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ui) {
            int mb, nb, kb0, kb1;
            unit_info(u, mb, nb, kb0, kb1);
            const int NB = (a.cout_pad - nb * 256) < 256 ? (a.cout_pad - nb * 256) : 256;
            const uint32_t b = nbuf == 2 ? (ui & 1) : 0, ub = nbuf == 2 ? (ui >> 1) : ui;
            mbar_wait(smem_u32(&bar_accf[b]), ub & 1);
            tc_fence_after();
            const int idx = mb * kM + lq * 32 + lane;
            const bool valid = idx < n;
            float* dst_row = nullptr;
            int lim = a.cout;
            if (valid) {
                if (S > 1) {
                    dst_row = a.ws + ((size_t)(u % S) * n + idx) * a.cout_pad;
                    lim = a.cout_pad;
                } else {
                    const int v = __ldg(a.list + idx);
                    dst_row = a.out.d + pkt_off(a.out, (v >> 16) - a.hg, (v & 0xffff) - a.hg);
                }
            }
            for (int cc = 0; cc < NB; cc += 32) {
                float v[32];
                tmem_ld32(tmem + b * acc_cols + ((uint32_t)(lq * 32) << 16) + (uint32_t)cc, v);
                if (valid) {
                    const int o0 = nb * 256 + cc;
                    float* dst = dst_row + o0;
                    if (((S > 1) || (a.out.C & 3) == 0) && o0 + 32 <= lim) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (o0 + j < lim) dst[j] = v[j];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_acce[b]));
        }
    } else {
        // ------------------------------------------------ MMA issuer
        // Warp-uniform loop (descriptors in uniform registers); one elected
        // lane issues the MMAs and commits.
        uint32_t st = 0, ph = 0, ui = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ui) {
            int mb, nb, kb0, kb1;
            unit_info(u, mb, nb, kb0, kb1);
            const int NB = (a.cout_pad - nb * 256) < 256 ? (a.cout_pad - nb * 256) : 256;
            const uint32_t idesc = idesc_tf32(NB);
            const uint32_t lbo_b = (uint32_t)NB * 16;
            const uint32_t b = nbuf == 2 ? (ui & 1) : 0, ub = nbuf == 2 ? (ui >> 1) : ui;
            mbar_wait(smem_u32(&bar_acce[b]), (ub & 1) ^ 1);
            tc_fence_after();
            const uint32_t dtm = tmem + b * acc_cols;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(smem_u32(&bar_full[st]), ph);
                tc_fence_after();
                const int c0 = kg.tpk > 1 ? 0 : (kb / K2) * kKC;
                const int nsteps = kg.tpk > 1 ? 4 : ((a.cin_pad - c0) / 8 < 4 ? (a.cin_pad - c0) / 8 : 4);
                const uint32_t b_base = smem_base + st * stage_bytes;
                const uint32_t a_tm = tmem + a_col0 + st * 64;
                if (elect_one()) {
                    for (int j = 0; j < nsteps; ++j) {
                        const uint64_t dbh = umma_desc(b_base + 2 * j * lbo_b, lbo_b, 128);
                        const uint64_t dbl = umma_desc(b_base + (uint32_t)NB * kKC * 4 + 2 * j * lbo_b, lbo_b, 128);
                        mma_tf32_ts(dtm, a_tm + 32 + 8 * j, dbh, idesc, (kb > kb0 || j > 0) ? 1u : 0u);
                        mma_tf32_ts(dtm, a_tm + 8 * j, dbl, idesc, 1u);
                        mma_tf32_ts(dtm, a_tm + 8 * j, dbh, idesc, 1u);
                    }
                    mma_commit(smem_u32(&bar_empty[st]));
                }
                __syncwarp();
                if (++st == (uint32_t)NST) st = 0, ph ^= 1;
            }
            if (elect_one()) mma_commit(smem_u32(&bar_accf[b]));
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kProdWarps + kEpiWarps)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// Fixed-order split-K reduction into the output packet (deterministic).
__global__ void k_conv_splitk_reduce(ConvArgs a) {
    pdl_enter();
    const int n = *a.count;
    const long long total = (long long)n * a.cout;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int idx = (int)(e / a.cout), o = (int)(e % a.cout);
        float sum = a.ws[(size_t)idx * a.cout_pad + o];
        for (int sp = 1; sp < a.splits; ++sp) sum = __fadd_rn(sum, a.ws[((size_t)sp * n + idx) * a.cout_pad + o]);
        const int v = __ldg(a.list + idx);
        a.out.d[pkt_off(a.out, (v >> 16) - a.hg, (v & 0xffff) - a.hg) + o] = sum;
    }
}

uint32_t rna_tf32_host(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return u;
    return (u + 0x1000u) & 0xffffe000u;
}

}  // namespace

size_t conv_tc_weight_floats(int cin_pad, int cout_pad, int k) {
    return (size_t)k_geom(cin_pad, k).nKB * kKC * cout_pad * 2;
}

// Host: O-I-Kh-Kw fp32 weights -> per (N-block, K-block) smem images
// [hi: 8 chunks x NB rows x 4 ch][lo: same], zero padded.
void conv_tc_prepare_weights(const float* w, int cin, int cout, int k, int cin_pad, int cout_pad, float* outp) {
    const KGeom kg = k_geom(cin_pad, k);
    const int K2 = k * k, nKB = kg.nKB;
    const int nNB = (cout_pad + 255) / 256;
    memset(outp, 0, conv_tc_weight_floats(cin_pad, cout_pad, k) * sizeof(float));
    for (int nb = 0; nb < nNB; ++nb) {
        const int NB = std::min(256, cout_pad - nb * 256);
        float* base = outp + (size_t)nb * 256 * nKB * kKC * 2;
        for (int kb = 0; kb < nKB; ++kb) {
            const int cb = kb / K2;
            float* blob = base + (size_t)kb * NB * kKC * 2;
            for (int nn = 0; nn < NB; ++nn) {
                const int o = nb * 256 + nn;
                for (int ci = 0; ci < kKC; ++ci) {
                    // K row ci of block kb: (tap, channel) = tap-packed or (block channel, one tap)
                    const int tap = kg.tpk > 1 ? kb * kg.tpk + ci / cin_pad : kb % K2;
                    const int i = kg.tpk > 1 ? ci % cin_pad : cb * kKC + ci;
                    float x = 0.0f;
                    if (o < cout && i < cin && tap < K2) x = w[((size_t)o * cin + i) * K2 + tap];
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

int conv_tc_splits(int max_targets, int cin_pad, int cout_pad, int k, int num_sms) {
    const int nKB = k_geom(cin_pad, k).nKB;
    const int nNB = (cout_pad + 255) / 256;
    const long long tiles = (long long)((max_targets + kM - 1) / kM) * nNB;
    // split K when the layer cannot give every SM a tile; keep >= 4 K-blocks per split
    int S = 1;
    while (tiles * S * 2 <= num_sms && nKB / (S * 2) >= 4 && S < 16) S *= 2;
    return S;
}

bool conv_tc_supported(int k) { return k * k <= 64; }

template <int NST>
static void launch_nst(int grid, size_t smem, cudaStream_t s, const Ctx& c, const ConvArgs& a) {
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [] {
        cudaFuncSetAttribute(k_conv_tc<NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    launch_pdl(k_conv_tc<NST>, grid, kThreadsV2, smem, s, c, a);
}

void launch_conv_tc(const Ctx& c, cudaStream_t s, PktDev in, const float* wsplit, int cin, int cin_pad, int cout,
                    int cout_pad, int k, int st, int r, PktDev out, int hg, const int* list, const int* count,
                    int max_targets, int num_sms, float* ws, int splits) {
    const int NBmax = cout_pad < 256 ? cout_pad : 256;
    const size_t stage = (size_t)NBmax * kKC * 8;
    const size_t budget = 200 * 1024;
    int nstages = (int)(budget / stage);
    if (nstages > 4) nstages = 4;
    {
        int acc = 32;
        while (acc < NBmax) acc <<= 1;
        while (nstages > 2 && acc + nstages * 64 > 512) --nstages;  // TMEM: acc + A stages
    }
    if (nstages < 2) throw std::runtime_error("conv_tc: Cout too large for two pipeline stages");
    if (k * k > 64) throw std::runtime_error("conv_tc: kernel larger than 7x7 is not supported");
    ConvArgs a{in, out, wsplit, list, count, splits > 1 ? ws : nullptr, cin, cin_pad, cout, cout_pad, k, st, r, hg,
               splits > 1 ? splits : 1};
    const int nNB = (cout_pad + 255) / 256;
    const long long units = (long long)((max_targets + kM - 1) / kM) * nNB * a.splits;
    int grid = num_sms;
    if (units < grid) grid = (int)(units < 1 ? 1 : units);
    const size_t smem = nstages * stage;
    if (nstages == 4) launch_nst<4>(grid, smem, s, c, a);
    else if (nstages == 3) launch_nst<3>(grid, smem, s, c, a);
    else launch_nst<2>(grid, smem, s, c, a);
    if (a.splits > 1) {
        long long total = (long long)max_targets * cout;
        int rg = (int)((total + 255) / 256);
        if (rg > num_sms * 8) rg = num_sms * 8;
        launch_pdl(k_conv_splitk_reduce, rg < 1 ? 1 : rg, 256, 0, s, a);
    }
}

DFX_KTRACE_SETTER(ktrace_set_tc)

}  // namespace dfx
