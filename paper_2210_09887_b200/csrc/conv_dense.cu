// Dense-unit sparse DeltaConv on tcgen05 (sm_100a): a stride-1
// padded_delta_conv (reference src/delta_layers.cpp:100-147).
//
// Work units (built by k_conv_plan, plan_block.inc.cuh): one unit = one MMA M
// tile of 128 output pixels, either a 16 x 8-pixel block of the grown extent
// (t >= 16) or 128 / t^2 ACTIVE output tiles gathered from anywhere in the
// extent (t in {2, 4, 8}, "tile units"). Every unit holding at least one conv
// target (tau = 1 by default) is computed whole here.
//
// Why whole units are exact: a non-target pixel's window touches no masked
// input tile (grown by the input halo), and unmasked packet tiles are zero by
// definition (delta_layers.hpp:37-41), so computing it yields exactly the 0
// the reference stores there; target pixels get the full window sum.
//
// Data movement: per (unit, KC = 16-channel chunk; 8 for Cin % 16 != 0) the
// unit's raw fp32 input patch ((16+2r) x (8+2r) pixels, or one (t+2r)^2 patch
// per tile) is copied ONCE into a ring of npb shared-memory patch buffers with
// 16-byte cp.async (zero fill via src-size 0 outside the grown extent or in
// unwritten tiles). For every tap, each A-producer thread reads its output
// pixel's shifted patch row, splits it into TF32 hi / lo in registers and
// tcgen05.st's both halves into a TMEM A stage. Weights (pre-split hi / lo,
// one image per (N block, K block = (channel chunk, tap))) are streamed by one
// thread with cp.async.bulk into a ring of nstw stages.
//
// Arithmetic: 3xTF32 (Ahi*Bhi + Ahi*Blo + Alo*Bhi, fp32 accumulation in TMEM;
// A from TMEM, B from shared memory). Two MMA-issuer warps alternate K-block
// pairs into their own accumulators; the epilogue sums the two partials in a
// fixed order. Split-K over CTAs (small layers) writes fp32 partials that the
// last-arriving CTA reduces in fixed order (deterministic).
//
// Warp roles (736 threads, kProdWG = 3): warps 0-11 A producers (three
// warpgroups taking taps round robin), 12-15 patch loaders, 16-19 epilogue
// (TMEM lane quarter = warp % 4, double-buffered accumulators when TMEM
// allows: nbuf), 20 and 22 MMA issuers, 21 weight producer. One unit per work item
// (umax = 1). The plan (dense_conv_plan) picks NBD = min(Cout, 128) columns per
// N block, nbuf and nstw to fit 200 KB of shared memory and 512 TMEM columns.
#include <cuda.h>  // CUtensorMap (the encoder is reached through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <stdexcept>

#include "kernels.hpp"
#include "pdl.hpp"

namespace dfx {

namespace {

#include "plan_block.inc.cuh"  // kUY / kUX, FDiv, target test, plan_block (shared with kernels_hbm.cu)
constexpr int kThreads = 320;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
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
// TMA: one 3-D box (channels, x, y) of the input packet into shared memory.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// mbarrier wait that traps instead of hanging (a malformed TMA would never complete)
__device__ __forceinline__ void mbar_wait_bounded(uint32_t bar, uint32_t parity) {
    for (long long it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (it > (1LL << 26)) __trap();
    }
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

template <bool TM>
__global__ void __launch_bounds__(kPlanThreads) k_conv_plan(Ctx c, PlanArgs pa) {
    pdl_enter();
    __shared__ PlanSmem sm;
    plan_block<kPlanThreads, TM>(c, pa, blockIdx.x, sm);
}

struct DenseArgs {
    PktDev in, out;
    const float* w;  // [nNB][nKB][hi: KC/4 x NBD x 4][lo: same]
    const int* units;
    const int* nunits;
    float* ws;       // split-K partials [S][n*128][cout_pad] (smax > 1)
    int* cnt;        // split-K arrival counters per (unit group, N-block); self-resetting
    int cin, cout, cout_pad, k, r;
    int KC, nCB, NBD, nNB, nst;
    int smax, sms;
    uint32_t pstr;         // bytes per patch pixel (KC fp32 + 16 B pad: conflict-free row reads)
    uint32_t patch_bytes;  // one patch buffer
    uint32_t w_stage;      // bytes of one weight stage (hi + lo)
    uint32_t acc_cols, nbuf, a_col0;  // TMEM plan
    int umax;              // units per item the TMEM / smem plan allows (1 or 2)
    int tpu, tsh;          // tile-unit mode (tpu tiles of 2^tsh px per unit), tpu = 0: 16x8-px units
    int ppx;               // pixels of one unit's patch
    int npb;               // patch ring depth (raw fp32 patches; the producers split hi / lo)
    int nmma;              // MMA issuer warps (2: K-block pairs alternate, one accumulator each)
    int tma;               // patches by TMA boxes (64-B pixel rows, SWIZZLE_64B) instead of cp.async
    BufDev nxt_acc, nxt_trunc;  // the consuming activation's state (L2 prefetch of this CTA's tiles), .d = null: none
    unsigned* tmax;        // fused tile max (pass 1 of the consuming activation): max |trunc + delta| per
                           // placement tile, atomicMax on the float bits; null: the activation computes it
    long long* trace;      // microbenchmark (dbg & 64): per-K-block clock64 stamps of CTA 0
    int dbg;               // microbenchmark knobs (tools/conv_trace*.py): 1 no MMA, 2 no patch loads, 4 no
                           // weights, 8 no A stores, 64 clock stamps (DFX_CONV_DBG, DFX_CONV_TRACE_IDX)
};

// Work decomposition for n units x nNB N-blocks x nKB K-blocks, chosen on
// device from the frame's unit count (the same in every CTA and the reduce):
// U units per item (2 share each weight stage: half the weight traffic; 1
// spreads small layers over more SMs) and S K-splits. Cost model in K-block
// time units: waves x K-blocks per item x (MMA time + ~300 cycles of per-K-block
// handshake, relative), + a penalty per split for the partials' traffic.
// Unit count of the frame: 16x8-px units are listed one by one; in tile-unit
// mode the list holds active tiles and a unit is tpu consecutive entries.
__device__ __forceinline__ int dense_units(const DenseArgs& a, int listed) {
    return a.tpu ? (listed + a.tpu - 1) / a.tpu : listed;
}
// Output pixel of row m of unit u (false: padding row of a partial tile unit).
__device__ __forceinline__ bool unit_pixel(const DenseArgs& a, int listed, int u, int m, int& y, int& x) {
    if (a.tpu == 0) {
        const int uv = __ldcg(a.units + u);
        y = ((uv >> 16) - 1) * kUY + (m >> 3), x = ((uv & 0xffff) - 1) * kUX + (m & 7);
        return true;
    }
    const int s = m >> (2 * a.tsh), l = m & ((1 << (2 * a.tsh)) - 1);
    const int li = u * a.tpu + s;
    if (li >= listed) return false;
    const int tv = __ldcg(a.units + li);
    y = (((tv >> 16) - 8) << a.tsh) + (l >> a.tsh);
    x = (((tv & 0xffff) - 8) << a.tsh) + (l & ((1 << a.tsh) - 1));
    return true;
}

// Fused pass 1 of the consuming activation (delta_layers.cpp:194-201):
// max |trunc + delta| over channels [o0, o0 + 4*n4) of placement pixel (y, x)
// of the activation's truncated state (slot-major, channels innermost).
template <int N4>
__device__ __forceinline__ float trunc_amax(const Ctx& c, const FrameDev& F, const BufDev& tr, int y, int x, int o0,
                                            const float* v) {
    const int t = tr.t, qy = y / t, qx = x / t;
    const float4* p = reinterpret_cast<const float4*>(tr.d + (size_t)slot_of(F, c.rows, c.cols, qy, qx) * t * t * tr.C +
                                                      ((size_t)(y - qy * t) * t + (x - qx * t)) * tr.C + o0);
    float4 tv[N4];
#pragma unroll
    for (int k4 = 0; k4 < N4; ++k4) tv[k4] = __ldcg(p + k4);  // all loads in flight first
    float m = 0.0f;
#pragma unroll
    for (int k4 = 0; k4 < N4; ++k4) {
        m = fmaxf(m, fabsf(__fadd_rn(tv[k4].x, v[4 * k4])));
        m = fmaxf(m, fabsf(__fadd_rn(tv[k4].y, v[4 * k4 + 1])));
        m = fmaxf(m, fabsf(__fadd_rn(tv[k4].z, v[4 * k4 + 2])));
        m = fmaxf(m, fabsf(__fadd_rn(tv[k4].w, v[4 * k4 + 3])));
    }
    return m;
}
// Lanes with the same tile key (-1: none) reduce their maxima (non-negative
// floats order as their bits) and the group leader folds it into tile_max.
__device__ __forceinline__ void tile_max_fold(unsigned* tmax, unsigned lanes, int key, float m) {
    const unsigned grp = __match_any_sync(lanes, key);
    const unsigned mx = __reduce_max_sync(grp, __float_as_uint(m));
    if (key >= 0 && mx != 0u && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) atomicMax(tmax + key, mx);
}

struct DenseSched {
    int U, S, items;
};
// Work decomposition, chosen on device from the frame's unit count n (the same
// in every CTA and in the reduce): two units per item (they share each weight
// stage: half the weight traffic) when there is at least a wave of such items,
// else one; split-K only when even single-unit items leave most SMs idle
// (partials cost a workspace round trip).
__host__ __device__ __forceinline__ DenseSched dense_sched(int n, int nNB, int nKB, int smax, int sms, int umax) {
    // two units per item whenever the plan allows it (weight streaming from L2
    // is the limit: it halves the bytes per FLOP); split-K fills idle SMs
    DenseSched d{umax >= 2 ? 2 : 1, 1, 0};
    const int groups = (n + d.U - 1) / d.U;
    while (d.S * 2 <= smax && (long long)groups * nNB * d.S * 2 <= sms && nKB / (d.S * 2) >= 4) d.S *= 2;
    d.items = groups * nNB * d.S;
    return d;
}

// Warp roles: 0..4*kProdWG-1 A producers, kProdWG warpgroups taking K-blocks
// round robin (row m = thread; per K-block the pixel's KC hi and lo channels at
// the tap offset are read from the shared-memory patch and tcgen05.st'ed into
// the TMEM A stage), then 4 patch loaders (cp.async + TF32 split, one patch per
// (unit, channel chunk), double buffered), 4 epilogue warps, the MMA issuer and
// the weight producer.
constexpr int kProdWG = 3;
constexpr int kMaxPB = 4;  // patch ring depth limit
// dynamic shared-memory plan of k_conv_dense (<= 224 KB = 227 KB per CTA minus
// ~3 KB static); measured: 200 KB beats 224 KB on C2 (more weight stages do not pay)
#ifndef DFX_DENSE_SMEM_KB
#define DFX_DENSE_SMEM_KB 200
#endif
constexpr size_t kDenseSmemBudget = (size_t)DFX_DENSE_SMEM_KB * 1024;
constexpr int kDenseThreads = (4 * kProdWG + 11) * 32;  // + loaders, epilogue, 2 MMA issuers, weights

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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

// Store KC 32-bit columns of this warp's lane quarter into TMEM.
template <int KC>
__device__ __forceinline__ void store_cols(uint32_t taddr, const uint32_t* v) {
    if constexpr (KC == 32) tmem_st32(taddr, v);
    else if constexpr (KC == 16) tmem_st16(taddr, v);
    else tmem_st8(taddr, v);
}

template <int KC>
__global__ void __launch_bounds__(kDenseThreads, 1)
    k_conv_dense(Ctx c, DenseArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[8], bar_empty[8], bar_pf[kMaxPB], bar_pe[kMaxPB], bar_af[2], bar_ae[2],
        bar_tma[kMaxPB];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int s_last;
    __shared__ int s_red_it;  // item whose split-K partials this CTA reduces at the end (-1: none)
    __shared__ int s_poff[2 * 22 * 14];  // per-pixel patch source offsets (k <= 7, two units)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K2 = a.k * a.k;
    const int nKB = a.nCB * K2;
    // Before the dependency wait (nothing here reads the previous kernel's
    // output): start the layer's weights towards L2 (one bulk prefetch per CTA
    // over its slice), allocate TMEM and initialise the barriers, so the wait
    // is followed directly by the first patch.
    if (tid == 0) {
        const size_t wbytes = (size_t)a.nNB * nKB * a.w_stage;
        const size_t per = ((wbytes + gridDim.x - 1) / gridDim.x + 255) / 256 * 256;
        const size_t o0 = per * blockIdx.x;
        if (o0 < wbytes) {
            const uint32_t sz = (uint32_t)(o0 + per <= wbytes ? per : wbytes - o0);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const uint8_t*>(a.w) + o0),
                         "r"(sz)
                         : "memory");
        }
    }
    const int PW = a.tpu ? (1 << a.tsh) + 2 * a.r : kUX + 2 * a.r;  // patch row pitch (pixels)
    const int NST = a.nst;
    // TMEM: accumulators [nbuf][2 units][NBD] then NST A stages of [2 units][hi KC | lo KC]
    const uint32_t acc_buf = a.nmma * a.umax * a.NBD;  // [nmma issuers][umax units][NBD]

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) s_red_it = -1;
    if (tid == 32) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_full[i]), 5);  // 4 A-producer warps + the weight bytes
            mbar_init(smem_u32(&bar_empty[i]), 1);
        }
        for (int i = 0; i < a.npb; ++i) {
            mbar_init(smem_u32(&bar_pf[i]), 4);
            mbar_init(smem_u32(&bar_pe[i]), 4 * kProdWG);
            mbar_init(smem_u32(&bar_tma[i]), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_af[i]), a.nmma);
            mbar_init(smem_u32(&bar_ae[i]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_enter();
    const FrameDev& F = *c.f;
    const int listed = __ldcg(a.nunits);
    const int n = dense_units(a, listed);
    const DenseSched sch = dense_sched(n, a.nNB, nKB, a.smax, a.sms, a.umax);
    const int S = sch.S, UPI = sch.U, items = sch.items;
    if ((int)blockIdx.x >= items) {  // no work this frame: give the TMEM back
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "r"(512));
        return;
    }
    const uint32_t tmem = tmem_base_sh;
    const uint32_t sbase = smem_u32(smem);
    if ((a.dbg & 64) && blockIdx.x == 0 && tid == 0) {
        a.trace[500] = clock64();
        a.trace[590] = n, a.trace[591] = S, a.trace[592] = items, a.trace[593] = UPI, a.trace[594] = listed;
    }
    if ((a.dbg & 64) && tid == 0 && blockIdx.x < 400) {  // per-CTA start (after the wait), %globaltimer
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[1100 + 2 * blockIdx.x] = (long long)t;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (blockIdx.x < 148) a.trace[1900 + blockIdx.x] = smid;
    }
    // smem: patches [2 buffers][2 units][hi, lo] planes, then the weight stages
    const uint32_t unit_bytes = a.patch_bytes, buf_bytes = a.umax * unit_bytes;
    const uint32_t w_base = sbase + a.npb * buf_bytes;

    // item -> (unit pair, N-block, K split) and its K-block range (channel chunk outer, tap inner)
    auto item_info = [&](int it, int& pr, int& nb, int& kb0, int& kb1) {
        const int per = a.nNB * S;
        pr = it / per;
        const int rem = it - pr * per;
        nb = rem / S;
        const int ks = rem - nb * S;
        kb0 = (int)(((long long)nKB * ks) / S);
        kb1 = (int)(((long long)nKB * (ks + 1)) / S);
    };

    // Patch loading (loader warps, and every thread in the prologue below):
    // per-pixel source offsets (-1: zero) of an item's patches, then one
    // channel chunk of the raw fp32 patch with cp.async (zero fill via src-size 0).
    const int c4n = KC / 4;
    const int P = a.ppx;  // patch pixels per unit
    const int E1 = P * c4n;
    const bool vec = (a.in.C & 3) == 0;
    auto patch_offsets = [&](int pr, int nu, int t0, int stride) {
        int y0[2] = {0, 0}, x0[2] = {0, 0};
        if (!a.tpu) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int uv = __ldcg(a.units + UPI * pr + (j < nu ? j : 0));
                y0[j] = ((uv >> 16) - 1) * kUY - a.r;
                x0[j] = ((uv & 0xffff) - 1) * kUX - a.r;
            }
        }
        for (int q = t0; q < P * nu; q += stride) {
            const int j = q >= P ? 1 : 0, p = q - j * P;
            int y, x;
            bool ok = true;
            if (a.tpu) {  // tile s of the unit, (T + 2r)^2-pixel patch per tile
                const int s = p / (PW * PW), l = p - s * PW * PW;
                const int py = l / PW, px = l - py * PW;
                const int li = pr * a.tpu + s;
                ok = li < listed;
                const int tv = ok ? __ldcg(a.units + li) : 0;
                y = (((tv >> 16) - 8) << a.tsh) - a.r + py;
                x = (((tv & 0xffff) - 8) << a.tsh) - a.r + px;
            } else {
                const int py = p / PW, px = p - py * PW;
                y = (j ? y0[1] : y0[0]) + py, x = (j ? x0[1] : x0[0]) + px;
            }
            s_poff[q] = ok && pkt_ok(a.in, F.th, F.tw, y, x) ? (int)pkt_off(a.in, y, x) : -1;
        }
    };
    auto copy_chunk = [&](uint32_t buf, int cbase, int nu, int t0, int stride) {
        for (int e = t0; e < E1 * nu; e += stride) {
            const int j = e >= E1 ? 1 : 0;
            const int e1 = e - j * E1;
            const int p = e1 / c4n, c4 = e1 - p * c4n;
            const int ch = cbase + c4 * 4;
            const uint32_t dst = buf + j * unit_bytes + p * a.pstr + c4 * 16;
            const int off = s_poff[j * P + p];
            const bool ok = off >= 0;
            if (vec) {
                const bool v = ok && ch < a.cin;
                cp_async16(dst, v ? a.in.d + off + ch : a.in.d, v ? 16u : 0u);
            } else {
                const float* src = ok ? a.in.d + off : a.in.d;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool v = ok && ch + q < a.cin;
                    cp_async4(dst + 4 * q, v ? src + ch + q : a.in.d, v ? 4u : 0u);
                }
            }
        }
    };
    // TMA staging (16x8-px units, one unit per item): the patch box (KC channels
    // x (8+2r) x (16+2r) pixels, 64-B pixel rows, SWIZZLE_64B) of channel chunk
    // cbase is one cp.async.bulk.tensor; samples outside the stored packet come
    // back zero from the TMA unit itself, samples inside it but outside the grown
    // extent or in unwritten tiles (s_poff < 0) are zeroed afterwards (fixup).
    const uint32_t box_bytes = (uint32_t)KC * 4 * PW * (kUY + 2 * a.r);
    auto tma_chunk = [&](uint32_t buf, int pr, int cbase, uint32_t bar) {
        const int uv = __ldcg(a.units + UPI * pr);
        const int y0 = ((uv >> 16) - 1) * kUY - a.r, x0 = ((uv & 0xffff) - 1) * kUX - a.r;
        mbar_arrive_tx(bar, box_bytes);
        tma_load_3d(buf, &tmap, cbase, x0 + a.in.halo, y0 + a.in.halo, bar);
    };
    auto fixup = [&](uint32_t buf, int t0, int stride) {
        for (int p = t0; p < P; p += stride)
            if (s_poff[p] < 0) {
                const uint32_t d = buf + (uint32_t)p * 64;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(d + 16 * q), "r"(0) : "memory");
            }
    };
    if (a.tma && (sbase & 511u)) __trap();  // the swizzle pattern below assumes 512-B aligned patch buffers

    // Prologue: the CTA's first patch (offsets + first channel chunk) is built by
    // ALL threads, so the first MMA is not gated by 4 loader warps walking a
    // dependent chain alone (~4-6 us per launch before).
    int w_pre = 0;  // weight stages of the first item already requested (weight-producer lane only)
    {
        int pr, nb, kb0, kb1;
        item_info(blockIdx.x, pr, nb, kb0, kb1);
        const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
        if (warp == 4 * kProdWG + 9 && lane == 0 && !(a.dbg & 4)) {
            // the first stages' weights are requested before the patch is built (the
            // stages are free at kernel start): they land while the prologue runs
            const float* wnb = a.w + (size_t)nb * nKB * (a.w_stage / 4);
            w_pre = min(NST, kb1 - kb0);
            for (int i = 0; i < w_pre; ++i) {
                mbar_arrive_tx(smem_u32(&bar_full[i]), a.w_stage);
                bulk_g2s(w_base + i * a.w_stage, wnb + (size_t)(kb0 + i) * (a.w_stage / 4), a.w_stage,
                         smem_u32(&bar_full[i]));
            }
        }
        if (a.tma && tid == 0) tma_chunk(sbase, pr, (kb0 / K2) * KC, smem_u32(&bar_tma[0]));
        patch_offsets(pr, nu, tid, kDenseThreads);
        __syncthreads();
        if (a.tma) {
            mbar_wait_bounded(smem_u32(&bar_tma[0]), 0);
            fixup(sbase, tid, kDenseThreads);
        } else {
            copy_chunk(sbase, (kb0 / K2) * KC, nu, tid, kDenseThreads);
            cp_async_wait_all();
        }
        __syncthreads();
        if (tid == 0)
            for (int i = 0; i < 4; ++i) mbar_arrive(smem_u32(&bar_pf[0]));  // the 4 loader-warp arrivals
    }

    if (warp < 4 * kProdWG) {
        // ------------------------------------------------ A producers (patch rows -> TMEM)
        // kProdWG warpgroups take K-blocks round robin (tcgen05.st + wait::st is
        // latency-bound); each writes both units' A rows of its K-block.
        const int wg = warp >> 2, wq = warp & 3;
        const int m = tid & 127;  // row = unit pixel (m >> 3, m & 7)
        const uint32_t row_off =
            a.tpu ? (uint32_t)((m >> (2 * a.tsh)) * PW * PW + ((m >> a.tsh) & ((1 << a.tsh) - 1)) * PW +
                               (m & ((1 << a.tsh) - 1))) * a.pstr
                  : (uint32_t)((m >> 3) * PW + (m & 7)) * a.pstr;
        uint32_t g = 0, pseq = 0, pst = 0, pph = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int pr, nb, kb0, kb1;
            item_info(it, pr, nb, kb0, kb1);
            const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
            for (int cb = kb0 / K2; cb <= (kb1 - 1) / K2; ++cb, ++pseq) {
                const uint32_t pb = pseq % a.npb;
                mbar_wait(smem_u32(&bar_pf[pb]), (pseq / a.npb) & 1);
                const uint32_t patch = sbase + pb * buf_bytes + row_off;
                const int t0 = max(kb0 - cb * K2, 0), t1 = min(kb1 - cb * K2, K2);
                for (int tap = t0; tap < t1; ++tap, ++g) {
                    const uint32_t st = pst, q = pph;
                    if (++pst == (uint32_t)NST) pst = 0, pph ^= 1;
                    if ((int)(g % kProdWG) != wg) continue;
                    const int ky = tap / a.k, kx = tap - ky * a.k;
                    const uint32_t src0 = patch + (uint32_t)(ky * PW + kx) * a.pstr;
                    // TMA patches are SWIZZLE_64B: 16-B chunk bits [4:5] ^= address bits [7:8]
                    // (buffer bases are 512-B aligned, so the relative offset decides)
                    const uint32_t swz = a.tma ? (((src0 - sbase) >> 7) & 3u) << 4 : 0u;
                    const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + a.a_col0 + st * 2 * a.umax * KC;
                    const long long t_a = clock64();
                    mbar_wait(smem_u32(&bar_empty[st]), q ^ 1);
                    const long long t_b = clock64();
                    tc_fence_after();
                    for (int j = 0; j < nu && !(a.dbg & 8); ++j) {  // dbg & 8: no A stores (microbenchmark)
                        // raw fp32 row -> hi = x with 13 low mantissa bits cleared (exact
                        // TF32), lo = x - hi (exact; the tensor core reads its top 19 bits)
                        uint32_t hv[KC], lv[KC];
                        const uint32_t src = src0 + j * unit_bytes;
#pragma unroll
                        for (int q4 = 0; q4 < KC / 4; ++q4)
                            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(hv[4 * q4]), "=r"(hv[4 * q4 + 1]), "=r"(hv[4 * q4 + 2]),
                                           "=r"(hv[4 * q4 + 3])
                                         : "r"(src + ((16 * q4) ^ swz)));
#pragma unroll
                        for (int e = 0; e < KC; ++e) {
                            const float x = __uint_as_float(hv[e]);
                            hv[e] &= 0xffffe000u;
                            lv[e] = __float_as_uint(__fsub_rn(x, __uint_as_float(hv[e])));
                        }
                        store_cols<KC>(taddr + j * 2 * KC, hv);
                        store_cols<KC>(taddr + j * 2 * KC + KC, lv);
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&bar_full[st]));
                    if ((a.dbg & 64) && blockIdx.x == 0 && tid == 128 * wg && g < 64) {
                        a.trace[g * 8 + 0] = t_a;
                        a.trace[g * 8 + 1] = t_b;
                        a.trace[g * 8 + 2] = clock64();
                    }
                }
                __syncwarp();  // every producer warp is done reading this patch
                if (lane == 0) mbar_arrive(smem_u32(&bar_pe[pb]));
            }
        }
    } else if (warp < 4 * kProdWG + 4) {
        // ------------------------------------------------ patch loaders (cp.async, zero fill)
        const int lt = tid - 128 * kProdWG;
        uint32_t pseq = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int pr, nb, kb0, kb1;
            item_info(it, pr, nb, kb0, kb1);
            const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
            const bool first = it == (int)blockIdx.x;  // its offsets and first chunk came from the prologue
            if (!first) {
                asm volatile("bar.sync 2, 128;" ::: "memory");  // previous item's copy loop is done with s_poff
                patch_offsets(pr, nu, lt, 128);
                asm volatile("bar.sync 2, 128;" ::: "memory");
            }
            for (int cb = kb0 / K2 + (first ? 1 : 0); cb <= (kb1 - 1) / K2; ++cb) {
                if (first && pseq == 0) pseq = 1;
                const uint32_t pb = pseq % a.npb;
                mbar_wait(smem_u32(&bar_pe[pb]), ((pseq / a.npb) & 1) ^ 1);
                if (a.dbg & 2) {  // microbenchmark: no patch loads
                } else if (a.tma) {
                    if (lt == 0) tma_chunk(sbase + pb * buf_bytes, pr, cb * KC, smem_u32(&bar_tma[pb]));
                    mbar_wait_bounded(smem_u32(&bar_tma[pb]), (pseq / a.npb) & 1);
                    fixup(sbase + pb * buf_bytes, lt, 128);
                } else {
                    copy_chunk(sbase + pb * buf_bytes, cb * KC, nu, lt, 128);
                    cp_async_wait_all();
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_pf[pb]));
                ++pseq;
            }
            if (first && pseq == 0) pseq = 1;  // single-chunk first item
        }
    } else if (warp < 4 * kProdWG + 8) {
        // ------------------------------------------------ epilogue: TMEM -> packet / split-K workspace
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int hs = a.out.halo;
        const int eh = F.th * a.out.t + hs, ew = F.tw * a.out.t + hs;
        uint32_t ui = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++ui) {
            int pr, nb, kb0, kb1;
            item_info(it, pr, nb, kb0, kb1);
            const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
            // while this item's MMAs run: tile units start the consuming activation's acc / trunc tiles of this
            // item towards L2 (its first, latency-bound pass reads them right after)
            // (16x8 units: the one 16-px-or-larger output tile the unit lies in)
            if (a.nxt_acc.d && m < 2 * (a.tpu ? a.tpu : UPI)) {
                const int s = m >> 1, li = a.tpu ? pr * a.tpu + s : UPI * pr + s;
                if (li < (a.tpu ? listed : n)) {
                    const int tv = __ldcg(a.units + li);
                    const int T = a.out.t;
                    const int tr = a.tpu ? (tv >> 16) - 8 : floor_div32(((tv >> 16) - 1) * kUY, T);
                    const int tc = a.tpu ? (tv & 0xffff) - 8 : floor_div32(((tv & 0xffff) - 1) * kUX, T);
                    const BufDev& bd = (m & 1) ? a.nxt_trunc : a.nxt_acc;
                    const uint32_t bytes = (uint32_t)bd.t * bd.t * bd.C * 4;
                    if (tr >= 0 && tr < F.th && tc >= 0 && tc < F.tw && (bytes & 15) == 0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                         bd.d + (size_t)slot_of(F, c.rows, c.cols, tr, tc) * bd.t * bd.t * bd.C),
                                     "r"(bytes)
                                     : "memory");
                }
            }
            const uint32_t b = a.nbuf == 2 ? (ui & 1) : 0, ub = a.nbuf == 2 ? (ui >> 1) : ui;
            mbar_wait(smem_u32(&bar_af[b]), ub & 1);
            const long long t_e0 = clock64();
            if ((a.dbg & 64) && ui == 0 && tid == 128 * kProdWG + 128 && blockIdx.x < 400) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                a.trace[3100 + blockIdx.x] = (long long)t;  // first accumulator ready
            }
            tc_fence_after();
            for (int j = 0; j < nu; ++j) {
                const int u = UPI * pr + j;
                int y, x;
                const bool row = unit_pixel(a, listed, u, m, y, x);
                const bool valid = row && y >= -hs && y < eh && x >= -hs && x < ew;  // stored grown extent
                float* dst_row = nullptr;
                int lim = a.cout;
                if (S > 1) {
                    dst_row = a.ws + ((size_t)((it % S) * n + u) * 128 + m) * a.cout_pad;
                    lim = a.cout_pad;
                } else if (valid) {
                    dst_row = a.out.d + pkt_off(a.out, y, x);
                }
                const uint32_t tcol = tmem + b * acc_buf + j * a.NBD + ((uint32_t)(q * 32) << 16);
                const bool two_acc = a.nmma == 2 && kb1 - kb0 > 2;  // the second issuer had K-blocks
                for (int cc = 0; cc < a.NBD; cc += 32) {
                    float v[32];
                    tmem_ld32(tcol + (uint32_t)cc, v);
                    if (two_acc) {  // fixed order: issuer 0 partial + issuer 1 partial
                        float v1[32];
                        tmem_ld32(tcol + (uint32_t)(a.umax * a.NBD) + (uint32_t)cc, v1);
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __fadd_rn(v[i], v1[i]);
                    }
                    const int o0 = nb * a.NBD + cc;
                    if (dst_row) {
                        float* dst = dst_row + o0;
                        if ((S > 1 || (a.out.C & 3) == 0) && o0 + 32 <= lim) {
#pragma unroll
                            for (int k4 = 0; k4 < 8; ++k4)
                                reinterpret_cast<float4*>(dst)[k4] =
                                    make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
                        } else {
#pragma unroll
                            for (int k4 = 0; k4 < 32; ++k4)
                                if (o0 + k4 < lim) dst[k4] = v[k4];
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_ae[b]));
            if (S > 1) {
                // split-K: the CTA whose partial arrives last sums all S partials of
                // this (unit group, N-block) in split order (deterministic) into the packet
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (q == 0 && lane == 0) {
                    __threadfence();
                    s_last = atomicAdd(a.cnt + it / S, 1) == S - 1;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                // the CTA whose partial arrives last sums all S partials at the end
                // of the kernel with ALL its threads (no CTA ever waits for another:
                // safe with several engines sharing the GPU, where not every CTA of
                // a grid need be resident at once)
                if (s_last && q == 0 && lane == 0) s_red_it = it;
            }
            if ((a.dbg & 64) && blockIdx.x == 0 && tid == 128 * kProdWG + 128 && ui < 4) {
                a.trace[504 + 2 * ui] = t_e0;
                a.trace[505 + 2 * ui] = clock64();
            }
        }
    } else if (warp == 4 * kProdWG + 8 || (warp == 4 * kProdWG + 10 && a.nmma == 2)) {
        // ------------------------------------------------ MMA issuers
        // Warp-uniform loop (descriptors in uniform registers); one elected
        // lane issues the MMAs and commits. Both units use the same weight stage.
        // With two issuers, K-block pairs alternate between them, each into its
        // own accumulator (summed in fixed order by the epilogue): one issuer's
        // barrier waits overlap the other's MMAs, so the tensor pipe stays fed.
        const int mw = warp == 4 * kProdWG + 8 ? 0 : 1;
        const uint32_t idesc = idesc_tf32(a.NBD);
        const uint32_t lbo_b = (uint32_t)a.NBD * 16, half_w = a.w_stage / 2;
        uint32_t st = 0, ph = 0, ui = 0, tq = 0;
        const bool trc = (a.dbg & 64) && blockIdx.x == 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++ui) {
            int pr, nb, kb0, kb1;
            item_info(it, pr, nb, kb0, kb1);
            const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
            const uint32_t b = a.nbuf == 2 ? (ui & 1) : 0, ub = a.nbuf == 2 ? (ui >> 1) : ui;
            mbar_wait(smem_u32(&bar_ae[b]), (ub & 1) ^ 1);
            tc_fence_after();
            const uint32_t dtm = tmem + b * acc_buf + mw * a.umax * a.NBD;
            // two K-blocks per handshake: wait for both stages, issue both MMA
            // chains back to back (the per-K-block wait/fence overhead is
            // otherwise a bubble in the tensor pipe)
            for (int kb = kb0, q = 0; kb < kb1; kb += 2, ++q) {
                const bool two = kb + 1 < kb1;
                const uint32_t st1 = st + 1 == (uint32_t)NST ? 0 : st + 1;
                const uint32_t ph1 = st + 1 == (uint32_t)NST ? ph ^ 1 : ph;
                if (q % a.nmma != mw) {  // the other issuer's pair: advance the ring only
                    if (two) {
                        st = st1 + 1 == (uint32_t)NST ? 0 : st1 + 1;
                        ph = st1 + 1 == (uint32_t)NST ? ph1 ^ 1 : ph1;
                    } else {
                        st = st1, ph = ph1;
                    }
                    continue;
                }
                const long long m_a = trc ? clock64() : 0;
                mbar_wait(smem_u32(&bar_full[st]), ph);
                if (two) mbar_wait(smem_u32(&bar_full[st1]), ph1);
                const long long m_b = trc ? clock64() : 0;
                tc_fence_after();
                if (elect_one()) {
#pragma unroll 1
                    for (int h = 0; h < (two ? 2 : 1); ++h) {
                        const uint32_t sh = h ? st1 : st;
                        const uint32_t wb = w_base + sh * a.w_stage;
                        const uint32_t a_tm = tmem + a.a_col0 + sh * 2 * a.umax * KC;
                        if (!(a.dbg & 1)) {
#pragma unroll
                            for (int j = 0; j < KC / 8; ++j) {
                                const uint64_t dbh = umma_desc(wb + 2 * j * lbo_b, lbo_b, 128);
                                const uint64_t dbl = umma_desc(wb + half_w + 2 * j * lbo_b, lbo_b, 128);
                                const uint32_t acc = (q > mw || h > 0 || j > 0) ? 1u : 0u;
                                for (int uu = 0; uu < nu; ++uu) {
                                    const uint32_t d = dtm + uu * a.NBD, at = a_tm + uu * 2 * KC;
                                    mma_tf32_ts(d, at + KC + 8 * j, dbh, idesc, acc);
                                    mma_tf32_ts(d, at + 8 * j, dbl, idesc, 1u);
                                    mma_tf32_ts(d, at + 8 * j, dbh, idesc, 1u);
                                }
                            }
                        }
                        mma_commit(smem_u32(&bar_empty[sh]));
                    }
                }
                __syncwarp();
                if (trc && mw == 0 && lane == 0 && tq < 100) {  // microbenchmark stamps (dbg & 64)
                    a.trace[600 + 3 * tq] = m_a;
                    a.trace[601 + 3 * tq] = m_b;
                    a.trace[602 + 3 * tq] = clock64();
                    ++tq;
                }
                if (two) {
                    st = st1 + 1 == (uint32_t)NST ? 0 : st1 + 1;
                    ph = st1 + 1 == (uint32_t)NST ? ph1 ^ 1 : ph1;
                } else {
                    st = st1, ph = ph1;
                }
            }
            if (elect_one()) mma_commit(smem_u32(&bar_af[b]));
            __syncwarp();
        }
    } else if (warp == 4 * kProdWG + 9) {
        // ------------------------------------------------ weight producer
        if (lane == 0) {
            uint32_t st = 0, ph = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                int pr, nb, kb0, kb1;
                item_info(it, pr, nb, kb0, kb1);
                const float* wnb = a.w + (size_t)nb * nKB * (a.w_stage / 4);
                if (it == (int)blockIdx.x && w_pre > 0) {  // skip the stages the prologue requested
                    kb0 += w_pre;
                    st = (uint32_t)(w_pre % NST);
                    ph = w_pre == NST ? 1u : 0u;
                }
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(smem_u32(&bar_empty[st]), ph ^ 1);
                    if (a.dbg & 4) {
                        mbar_arrive(smem_u32(&bar_full[st]));
                    } else {
                        mbar_arrive_tx(smem_u32(&bar_full[st]), a.w_stage);
                        bulk_g2s(w_base + st * a.w_stage, wnb + (size_t)kb * (a.w_stage / 4), a.w_stage,
                                 smem_u32(&bar_full[st]));
                    }
                    if (++st == (uint32_t)NST) st = 0, ph ^= 1;
                }
            }
        }
        __syncwarp();
    }
    if ((a.dbg & 64) && blockIdx.x == 0 && lane == 0 && warp < 32) a.trace[520 + warp] = clock64();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if ((a.dbg & 64) && tid == 0 && blockIdx.x < 400) {  // items done; does this CTA reduce?
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[2100 + blockIdx.x] = (long long)t;
        a.trace[2600 + blockIdx.x] = s_red_it >= 0 ? 1 : 0;
    }
    if (s_red_it >= 0) {
        // fixed-order (split 0, 1, ...) sum of the S partials of one (unit group,
        // N-block) tile into the packet: every thread float4 columns of rows, all
        // S loads of a float4 in flight before the adds (deterministic order)
        const int it = s_red_it;
        __threadfence();
        const int m0 = 0, nm = 128;
        int pr, nb, kb0, kb1;
        item_info(it, pr, nb, kb0, kb1);
        const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
        const int hs = a.out.halo;
        const int eh = F.th * a.out.t + hs, ew = F.tw * a.out.t + hs;
        const int o0 = nb * a.NBD, o1 = min(a.cout, (nb + 1) * a.NBD);
        const int nq = (o1 - o0 + 3) / 4;  // float4 columns per row
        const size_t sstride = (size_t)n * 128 * a.cout_pad;
        const bool vec = (a.out.C & 3) == 0;
        const int ntot = nu * nm * nq;
        for (int e0 = tid & ~31; e0 < ntot; e0 += blockDim.x) {  // warp-uniform trip count (tile max fold)
            const int e = e0 + lane;
            const int j = e / (nm * nq), rem = e - j * nm * nq;
            const int m = m0 + rem / nq, c4 = rem - (rem / nq) * nq;
            const int u = UPI * pr + j;
            int y = 0, x = 0;
            const bool live = e < ntot && unit_pixel(a, listed, u, m, y, x) && y >= -hs && y < eh && x >= -hs && x < ew;
            if (!live) {
                if (a.tmax) tile_max_fold(a.tmax, 0xffffffffu, -1, 0.0f);
                continue;
            }
            const int o = o0 + 4 * c4;
            const float* src = a.ws + ((size_t)u * 128 + m) * a.cout_pad + o;
            float4 v[8];
#pragma unroll
            for (int sp = 0; sp < 8; ++sp)
                if (sp < S) v[sp] = __ldcg(reinterpret_cast<const float4*>(src + sp * sstride));
            float4 acc4 = v[0];
#pragma unroll
            for (int sp = 1; sp < 8; ++sp)
                if (sp < S) {
                    acc4.x = __fadd_rn(acc4.x, v[sp].x), acc4.y = __fadd_rn(acc4.y, v[sp].y);
                    acc4.z = __fadd_rn(acc4.z, v[sp].z), acc4.w = __fadd_rn(acc4.w, v[sp].w);
                }
            float* dst = a.out.d + pkt_off(a.out, y, x) + o;
            if (vec && o + 4 <= o1) {
                *reinterpret_cast<float4*>(dst) = acc4;
            } else {
                const float vv[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
                for (int q = 0; q < 4 && o + q < o1; ++q) dst[q] = vv[q];
            }
            if (a.tmax) {  // fused activation pass 1 on the final sums
                const bool in_ext = y >= 0 && y < F.th * a.out.t && x >= 0 && x < F.tw * a.out.t && o + 4 <= o1;
                const float vv[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
                const float m4 = in_ext ? trunc_amax<1>(c, F, a.nxt_trunc, y, x, o, vv) : 0.0f;
                tile_max_fold(a.tmax, 0xffffffffu, in_ext ? (y / a.out.t) * F.tw + x / a.out.t : -1, m4);
            }
        }
        if (tid == 0) a.cnt[it / S] = 0;  // re-arm for the next frame
    }
    if (a.tmax && S == 1) {
        // fused pass 1 of the consuming activation (delta_layers.cpp:194-201) over
        // this CTA's items, by ALL threads once the items are done (the epilogue
        // warps alone keep too few loads in flight, and in-loop work would hold up
        // the next item): max |trunc + delta| per placement tile from the delta
        // just stored by this CTA and the activation's truncated state
        const int np = a.NBD / 32;  // 32-channel parts per pixel: one thread, 8 + 8 float4 loads in flight
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int pr, nb, kb0, kb1;
            item_info(it, pr, nb, kb0, kb1);
            const int nu = (UPI == 2 && 2 * pr + 1 < n) ? 2 : 1;
            const int ntot = nu * 128 * np;
            for (int e0 = tid & ~31; e0 < ntot; e0 += blockDim.x) {  // warp-uniform trip count
                const int e = e0 + lane;
                const int j = e / (128 * np), rem = e - j * 128 * np;
                const int m = rem / np, part = rem - m * np;
                int y = 0, x = 0;
                const bool in_ext = e < ntot && unit_pixel(a, listed, UPI * pr + j, m, y, x) && y >= 0 &&
                                    y < F.th * a.out.t && x >= 0 && x < F.tw * a.out.t;
                float mt = 0.0f;
                if (in_ext) {
                    const int o = nb * a.NBD + 32 * part;
                    const float4* d4 = reinterpret_cast<const float4*>(a.out.d + pkt_off(a.out, y, x) + o);
                    float v[32];
#pragma unroll
                    for (int k4 = 0; k4 < 8; ++k4) {
                        const float4 q4 = __ldcg(d4 + k4);
                        v[4 * k4] = q4.x, v[4 * k4 + 1] = q4.y, v[4 * k4 + 2] = q4.z, v[4 * k4 + 3] = q4.w;
                    }
                    mt = trunc_amax<8>(c, F, a.nxt_trunc, y, x, o, v);
                }
                tile_max_fold(a.tmax, 0xffffffffu, in_ext ? (y / a.out.t) * F.tw + x / a.out.t : -1, mt);
            }
        }
    }
    if ((a.dbg & 64) && blockIdx.x == 0 && tid == 0) a.trace[501] = clock64();
    if ((a.dbg & 64) && tid == 0 && blockIdx.x < 400) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[1101 + 2 * blockIdx.x] = (long long)t;
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Fixed-order split-K reduction of the dense partials into the packet.
__global__ void k_conv_dense_reduce(Ctx c, DenseArgs a) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int listed = *a.nunits;
    const int n = dense_units(a, listed);
    const int S = dense_sched(n, a.nNB, a.nCB * a.k * a.k, a.smax, a.sms, a.umax).S;
    if (S <= 1) return;
    const int hs = a.out.halo;
    const int eh = F.th * a.out.t + hs, ew = F.tw * a.out.t + hs;
    const long long total = (long long)n * 128 * a.cout;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long row = e / a.cout;
        const int o = (int)(e - row * a.cout);
        const int u = (int)(row >> 7), m = (int)(row & 127);
        int y, x;
        if (!unit_pixel(a, listed, u, m, y, x)) continue;
        if (y < -hs || y >= eh || x < -hs || x >= ew) continue;
        float sum = a.ws[(size_t)row * a.cout_pad + o];
        for (int sp = 1; sp < S; ++sp) sum = __fadd_rn(sum, a.ws[((size_t)sp * n * 128 + row) * a.cout_pad + o]);
        a.out.d[pkt_off(a.out, y, x) + o] = sum;
    }
}

uint32_t rna_tf32_bits(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return u;
    return (u + 0x1000u) & 0xffffe000u;
}

}  // namespace

// ------------------------------------------------------------------ host side
DenseConvPlan dense_conv_plan(int cin, int cout, int k, int t_out, int rows, int cols, size_t ws_budget_bytes) {
    DenseConvPlan p{};
    p.cin_pad = (cin + 7) / 8 * 8;
    p.cout_pad = (cout + 31) / 32 * 32;
    p.NBD = p.cout_pad < 128 ? p.cout_pad : 128;
    if (const char* nb = getenv("DFX_DENSE_NBD")) {  // experiments: N = 256 MMAs for wide layers
        if (atoi(nb) == 256 && p.cout_pad % 256 == 0) p.NBD = 256;
    }
    if (p.cout_pad % p.NBD) p.NBD = 32;
    p.nNB = p.cout_pad / p.NBD;
    // One unit per item: measured best on the C2 layers (more SMs busy). Two
    // units sharing a weight stage (umax = 2) was measured slower earlier and is
    // not kept working with the raw patch ring / split producers, so it is not
    // selectable.
    p.umax = 1;
    // 16-channel K-blocks: 16 KB weight stages, a deeper ring hides the bulk-copy latency (measured +2-4%)
    p.KC = p.cin_pad % 16 == 0 ? 16 : 8;
    p.r = k / 2;
    p.k = k;
    // Tile units (T = t_out in {2, 4, 8}): a unit is 128 / T^2 ACTIVE output
    // tiles gathered from anywhere in the extent, each with its own
    // (T + 2r)^2-pixel patch, instead of a 16 x 8-pixel block that at small T
    // mostly covers inactive tiles (measured 2.2-3.4x computed / target pixels
    // on the C2 deep layers). DFX_TILE_UNITS=0 restores block units.
    p.tpu = 0;
    p.tsh = 0;
    {
        const char* e = getenv("DFX_TILE_UNITS");
        const bool on = !(e && e[0] == '0');
        if (on && (t_out == 2 || t_out == 4 || t_out == 8)) {
            p.tpu = 128 / (t_out * t_out);
            p.tsh = t_out == 2 ? 1 : (t_out == 4 ? 2 : 3);
            p.umax = 1;
        }
    }
    const int PW = p.tpu ? t_out + 2 * p.r : kUX + 2 * p.r, PH = p.tpu ? t_out + 2 * p.r : kUY + 2 * p.r;
    p.patch_px = p.tpu ? p.tpu * PW * PH : PW * PH;
    const unsigned acc = (unsigned)p.umax * p.NBD;
    size_t budget = kDenseSmemBudget;
    if (const char* e = getenv("DFX_DENSE_SMEM_KB")) {  // experiments: smaller shared-memory plans
        const size_t v = (size_t)atoi(e) * 1024;
        if (v >= 64 * 1024 && v <= 220 * 1024) budget = v;
    }
    // TMA patch boxes for 16x8-px units with 16-channel K-blocks (64-B pixel rows,
    // SWIZZLE_64B instead of the cp.async layout's 16-B pad); DFX_DENSE_TMA=0: cp.async
    const char* te = getenv("DFX_DENSE_TMA");
    const bool tma_ok = !(te && te[0] == '0') && !p.tpu && cin % 4 == 0;
    auto set_kc = [&](int kc) {
        p.KC = kc;
        p.nCB = p.cin_pad / p.KC;
        p.tma = tma_ok && kc == 16;
        // pixel stride in a patch plane: TMA rows are dense (swizzled); cp.async rows
        // carry a 16-B pad (conflict-free row reads)
        p.s_c4 = p.tma ? 64u : (unsigned)p.KC * 4 + 16;
        p.patch_bytes = p.tma ? ((unsigned)p.patch_px * 64 + 511) / 512 * 512
                              : ((unsigned)p.patch_px * p.s_c4 + 127) / 128 * 128;
        p.w_stage = (uint32_t)p.NBD * p.KC * 8;
    };
    // raw patches (one fp32 plane each) in a ring of npb buffers: the loaders
    // run up to npb - 1 channel chunks ahead of the A producers
    p.npb = 2;
    p.nmma = 1;
    auto fits = [&](int nst, unsigned nbuf) {
        return (size_t)p.npb * p.umax * p.patch_bytes + (size_t)nst * p.w_stage <= budget &&
               nbuf * acc * p.nmma + (unsigned)nst * 2 * p.umax * p.KC <= 512;
    };
    set_kc(p.KC);
    if (const char* e = getenv("DFX_DENSE_NPB")) {  // experiments: patch ring depth 2..4
        const int v = atoi(e);
        if (v >= 2 && v <= kMaxPB) p.npb = v;
    }
    if (p.npb > 2 && !fits(4, 2) && !fits(4, 1)) p.npb = 2;
    if (p.KC > 8 && !fits(4, 2) && !fits(4, 1)) set_kc(8);  // large tile-unit patches: 8-channel K-blocks
    // two MMA issuers (one accumulator each) when TMEM holds them with >= 4 stages
    {
        int want = 2;
        if (const char* e = getenv("DFX_DENSE_NMMA")) want = atoi(e) == 1 ? 1 : 2;
        p.nmma = want;
        if (!fits(4, 2) && !fits(4, 1)) p.nmma = 1;
    }
    // prefer double-buffered accumulators with >= 6 weight stages, else a single
    // accumulator buffer with up to 8 stages
    // DFX_DENSE_MAXST (6..8): experiments with fewer weight stages (a smaller
    // shared-memory footprint lets the next kernel's CTAs become resident earlier)
    int maxst = 8;
    if (const char* e = getenv("DFX_DENSE_MAXST")) maxst = atoi(e) >= 6 && atoi(e) <= 8 ? atoi(e) : 8;
    p.nbuf = 2;
    p.nstw = maxst;
    while (p.nstw > 6 && !fits(p.nstw, 2)) --p.nstw;
    if (!fits(p.nstw, 2)) {
        p.nbuf = 1;
        p.nstw = maxst;
        while (p.nstw > 2 && !fits(p.nstw, 1)) --p.nstw;
    }
    p.acc_cols = acc * p.nmma;
    p.smem = (size_t)p.npb * p.umax * p.patch_bytes + (size_t)p.nstw * p.w_stage;
    const int BH = t_out > kUY ? t_out : kUY, BW = t_out > kUX ? t_out : kUX;
    p.ok = fits(p.nstw, p.nbuf) && k * k <= 49 && (k & 1) && t_out <= 64 && (BH / kUY) * (BW / kUX) <= 32 &&
           (BH / t_out) * (BW / t_out) <= 32 && p.patch_px * p.umax <= 2 * 22 * 14;
    // Pipelines of 4-5 weight stages (plans under a reduced shared-memory budget,
    // DFX_DENSE_SMEM_KB=100 / 120) are parity-tested; round 1 saw them fail to
    // launch, which no longer reproduces after this round's fixes (per-device
    // kernel attributes among them). Fewer than 4 stages are untested: such
    // layers take the gathered-target conv.
    if (p.nstw < 4) p.ok = false;
    if (getenv("DFX_PLAN_DUMP"))
        fprintf(stderr, "plan cin=%d cout=%d k=%d t=%d KC=%d nbuf=%d nstw=%d nmma=%d npb=%d tpu=%d tma=%d ok=%d\n", cin,
                cout, k, t_out, p.KC, p.nbuf, p.nstw, p.nmma, p.npb, p.tpu, p.tma, (int)p.ok);
    // units over [-16, rows*t + hg) x [-8, cols*t + hg) (hg <= 8 px of grown halo)
    p.nux_max = (cols * t_out + 8 + kUX - 1) / kUX + 1;
    p.nuy_max = (rows * t_out + 8 + kUY - 1) / kUY + 1;
    p.units_max = p.nux_max * p.nuy_max;
    p.ws_units = p.units_max;
    if (p.tpu) {  // the list holds tiles (ring tiles included): size it for all of them
        const int tiles = (rows + 16) * (cols + 16);
        p.units_max = tiles > p.units_max ? tiles : p.units_max;
        p.ws_units = (tiles + p.tpu - 1) / p.tpu;
    }
    p.nbh = (rows * t_out + 8 + BH - 1) / BH + 1;
    p.nbw = (cols * t_out + 8 + BW - 1) / BW + 1;
    p.t_out = t_out;
    p.smax = 8;
    if (const char* e = getenv("DFX_DENSE_SMAX")) {  // experiments: cap the split-K factor (1, 2, 4, 8)
        const int v = atoi(e);
        if (v >= 1 && v <= 8) p.smax = v;
    }
    while (p.smax > 1 && (size_t)p.smax * p.ws_units * 128 * p.cout_pad * 4 > ws_budget_bytes) p.smax /= 2;
    return p;
}

size_t dense_conv_weight_floats(const DenseConvPlan& p) {
    return (size_t)p.nNB * p.nCB * p.k * p.k * p.NBD * p.KC * 2;
}

void dense_conv_prepare_weights(const DenseConvPlan& p, const float* w, int cin, int cout, float* outp) {
    const int K2 = p.k * p.k, nKB = p.nCB * K2;
    memset(outp, 0, dense_conv_weight_floats(p) * sizeof(float));
    const size_t blob = (size_t)p.NBD * p.KC * 2;
    for (int nb = 0; nb < p.nNB; ++nb)
        for (int kb = 0; kb < nKB; ++kb) {
            const int cb = kb / K2, tap = kb % K2;
            float* b = outp + ((size_t)nb * nKB + kb) * blob;
            for (int nn = 0; nn < p.NBD; ++nn) {
                const int o = nb * p.NBD + nn;
                for (int ci = 0; ci < p.KC; ++ci) {
                    const int i = cb * p.KC + ci;
                    float x = 0.0f;
                    if (o < cout && i < cin) x = w[((size_t)o * cin + i) * K2 + tap];
                    const uint32_t hb = rna_tf32_bits(x);
                    float hi;
                    memcpy(&hi, &hb, 4);
                    const uint32_t lb = rna_tf32_bits(x - hi);
                    float lo;
                    memcpy(&lo, &lb, 4);
                    const size_t off = ((size_t)(ci / 4) * p.NBD + nn) * 4 + (ci % 4);
                    b[off] = hi;
                    b[(size_t)p.NBD * p.KC + off] = lo;
                }
            }
        }
}

void launch_conv_plan(const Ctx& c, cudaStream_t s, const DenseConvPlan& p, PktDev in, PktDev out, int hg, int* units,
                      int* nunits, unsigned long long* flop_px, int tau, int* list, int* lcount, unsigned* tmax,
                      BufDev tm_trunc) {
    if (hg > 8) throw std::runtime_error("conv_plan: grown halo > 8 px");
    if (p.tpu && out.RT >= 8) throw std::runtime_error("conv_plan: tile ring too wide for tile units");
    const PlanArgs pa{in,   out,  p.k,    p.r,    hg,          p.nbw, p.nbh * p.nbw, units, nunits,
                      flop_px, tau, list, lcount, p.tpu ? 1 : 0, tmax,  tm_trunc};
    // the zero-fill tile max exists only for 16x8-px units (tile units leave no zero fill)
    if (tmax && !p.tpu) launch_pdl(k_conv_plan<true>, p.nbh * p.nbw, kPlanThreads, 0, s, c, pa);
    else launch_pdl(k_conv_plan<false>, p.nbh * p.nbw, kPlanThreads, 0, s, c, pa);
}

template <int KC>
static void launch_kc(int grid, size_t smem, cudaStream_t s, const Ctx& c, const DenseArgs& a, const CUtensorMap& tm) {
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [] {
        cudaFuncSetAttribute(k_conv_dense<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    });
    launch_pdl(k_conv_dense<KC>, grid, kDenseThreads, smem, s, c, a, tm);
}

bool dense_conv_tensor_map(const DenseConvPlan& p, PktDev in, int rows, void* out) {
    if (!p.tma || (in.C & 3) != 0) return false;
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<Encode>(fn);
    }();
    if (!enc) return false;
    // the packet as a 3-D tensor (channels, x, y) over its whole stored array;
    // coordinates are packet coordinates + halo (TMA fills outside with zeros)
    const cuuint64_t dims[3] = {(cuuint64_t)in.C, (cuuint64_t)in.pitch_w, (cuuint64_t)(rows * in.t + 2 * in.halo)};
    const cuuint64_t strides[2] = {(cuuint64_t)in.C * 4, (cuuint64_t)in.pitch_w * in.C * 4};
    const cuuint32_t box[3] = {(cuuint32_t)p.KC, (cuuint32_t)(kUX + 2 * p.r), (cuuint32_t)(kUY + 2 * p.r)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, in.d, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static long long* g_trace = nullptr;
long long* dense_conv_trace_buffer() { return g_trace; }
void launch_conv_dense(const Ctx& c, cudaStream_t s, const DenseConvPlan& p, PktDev in, PktDev out, const float* w,
                       int cin, int cout, const int* units, const int* nunits, float* ws, int* cnt, int num_sms,
                       BufDev nxt_acc, BufDev nxt_trunc, unsigned* tmax, const void* tmap) {
    if (!p.ok) throw std::runtime_error("conv_dense: unsupported layer shape");
    DenseArgs a{in, out, w, units, nunits, p.smax > 1 ? ws : nullptr, cnt, cin, cout, p.cout_pad, p.k, p.r,
                p.KC, p.nCB, p.NBD, p.nNB, p.nstw, p.smax > 1 ? p.smax : 1, num_sms, p.s_c4, p.patch_bytes,
                p.w_stage, p.acc_cols, p.nbuf, p.nbuf * p.acc_cols, p.umax, p.tpu, p.tsh, p.patch_px, p.npb,
                p.nmma, tmap != nullptr ? 1 : 0, nxt_acc, nxt_trunc, tmax, nullptr, 0};
    if (getenv("DFX_CONV_DBG") && !g_trace) cudaMalloc(&g_trace, 4096 * 8);
    a.trace = g_trace;
    if (const char* d = getenv("DFX_CONV_DBG")) a.dbg = atoi(d);
    if (const char* d = getenv("DFX_CONV_TRACE_IDX")) {  // trace only the i-th dense launch of every 8
        static int seq = 0;
        if (seq++ % 8 != atoi(d)) a.dbg = 0;  // every debug bit applies to the traced launch only
    }
    DenseConvPlan pp = p;
    if (a.dbg & 128) a.smax = 1;  // microbenchmark: no split-K
    if (const char* d = getenv("DFX_CONV_NST")) {  // microbenchmark: fewer pipeline stages (>= 4, see the plan)
        const int v = atoi(d);
        if (v >= 4 && v < pp.nstw) a.nst = v;
    }
    const long long max_items = (long long)p.ws_units * p.nNB * a.smax;
    const int grid = (int)(max_items < num_sms ? (max_items < 1 ? 1 : max_items) : num_sms);
    CUtensorMap tm;
    if (tmap) memcpy(&tm, tmap, sizeof tm);
    else memset(&tm, 0, sizeof tm);
    if (p.KC == 32) launch_kc<32>(grid, p.smem, s, c, a, tm);
    else if (p.KC == 16) launch_kc<16>(grid, p.smem, s, c, a, tm);
    else launch_kc<8>(grid, p.smem, s, c, a, tm);
    // split-K partials are reduced inside k_conv_dense (last-arriving CTA)
}

DFX_KTRACE_SETTER(ktrace_set_dense)

}  // namespace dfx
