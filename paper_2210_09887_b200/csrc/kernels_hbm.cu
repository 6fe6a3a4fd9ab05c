// Streaming (HBM-bound) kernels of the delta activation and max pooling,
// written for bandwidth: warps are the work units, each takes a 16 KB chunk of
// a masked tile, every access is a 16-byte vector, and a persistent grid keeps
// ~64 warps per SM with several KB of loads in flight each. A work item is
// 4 KB of one tile (one round of 8 float4 per lane), so even a few masked
// tiles spread over every SM.
//
// Truncation (delta_activation_truncate, reference src/delta_layers.cpp:
// 185-228) needs the max over a WHOLE tile before any write, so it is two
// passes:
//   k_trunc_tilemax  max |trunc + delta| per masked owned tile (read only,
//                    atomicMax on the float bits: values are >= 0);
//   k_trunc_commit   fire (acc += trunc + delta, trunc = 0, out = relu(acc') -
//                    relu(acc) or the candidate) or fold (trunc += delta).
// The second pass re-reads trunc and delta from L2 (a layer's masked tiles are
// far smaller than the 126 MB L2), so DRAM sees the algorithmic traffic.
// Arithmetic is the reference's fp32 order with explicit rounding intrinsics.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "kernels.hpp"
#include "pdl.hpp"

namespace dfx {

namespace {

#include "output.inc.cuh"
#include "plan_block.inc.cuh"  // the next conv's plan, run by extra blocks of a commit launch

#ifndef DFX_TRUNC_MINB  // CTAs per SM of k_trunc_coop (measured: 3 -> 80 registers with spills, slower)
#define DFX_TRUNC_MINB 2
#endif
constexpr int kSub = 8;               // float4s per lane in flight per array
constexpr int kChunkF4 = 32 * kSub;
#ifndef DFX_TRUNC_PREFETCH
#define DFX_TRUNC_PREFETCH 1
#endif
constexpr bool kTruncPrefetch = DFX_TRUNC_PREFETCH != 0;   // float4s per warp work item (4 KB): one round, all loads issued up front

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
// Placement tile (qy, qx) owns its slot (TileLedger::holds, buffer_manager.hpp:41-44).
__device__ __forceinline__ bool holds_t(const Ctx& c, const FrameDev& F, int qy, int qx) {
    return c.own[qy * F.tw + qx] != 0;
}
// Any tile, ring tiles outside the placement included (slot table).
__device__ __forceinline__ bool holds_any(const Ctx& c, const FrameDev& F, int qy, int qx) {
    if (qy >= 0 && qy < F.th && qx >= 0 && qx < F.tw) return c.own[qy * F.tw + qx] != 0;
    const SlotDev& sl = c.slots[slot_of(F, c.rows, c.cols, qy, qx)];
    return sl.used && sl.ty == F.oty + qy && sl.tx == F.otx + qx;
}

// Halo stash (delta_layers.cpp:168-183; maxpool acc :262-275): every written
// ring pixel of the grown packet is added into the wrapped buffer when its
// slot is owned. Ring pixels map to distinct buffer pixels, so this is a plain
// vectorised read-modify-write (no atomics, deterministic). Spread over all
// threads of the grid (tid0 / nthr).
__device__ void ring_add_part(const Ctx& c, const FrameDev& F, const PktDev& in, BufDev dst, long long tid0,
                              long long nthr) {
    const int h = in.halo, t = in.t, C4 = in.C / 4;
    if (h <= 0) return;
    const int eh = F.th * t, ew = F.tw * t, gw = ew + 2 * h;
    const long long npx = 2LL * h * gw + 2LL * eh * h;
    for (long long i = tid0; i < npx * C4; i += nthr) {
        const long long p = i / C4;
        const int c4 = (int)(i - p * C4);
        int y, x;
        if (p < (long long)h * gw) {
            y = -h + (int)(p / gw), x = -h + (int)(p % gw);
        } else if (p < 2LL * h * gw) {
            const long long q = p - (long long)h * gw;
            y = eh + (int)(q / gw), x = -h + (int)(q % gw);
        } else if (p < 2LL * h * gw + (long long)eh * h) {
            const long long q = p - 2LL * h * gw;
            y = (int)(q / h), x = -h + (int)(q % h);
        } else {
            const long long q = p - 2LL * h * gw - (long long)eh * h;
            y = (int)(q / h), x = ew + (int)(q % h);
        }
        const int qy = floor_div32(y, t), qx = floor_div32(x, t);
        if (!in.ext[ext_idx(in, qy, qx)] || !holds_any(c, F, qy, qx)) continue;
        float4* b = reinterpret_cast<float4*>(
                        dst.d + (size_t)slot_of(F, c.rows, c.cols, qy, qx) * dst.t * dst.t * dst.C +
                        ((size_t)(y - qy * t) * t + (x - qx * t)) * dst.C) + c4;
        const float4 dv = reinterpret_cast<const float4*>(in.d + pkt_off(in, y, x))[c4];
        *b = add4(*b, dv);
    }
}
__device__ __forceinline__ float* tile_base(const Ctx& c, const FrameDev& F, BufDev b, int qy, int qx) {
    return b.d + (size_t)slot_of(F, c.rows, c.cols, qy, qx) * b.t * b.t * b.C;
}
__device__ __forceinline__ float amax4(float m, float4 v) {
    return fmaxf(fmaxf(fmaxf(m, fabsf(v.x)), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

// Masked (and, if own, owned) placement tiles of packet p, in tile order, into
// shared memory: one ballot + prefix per 256 tiles. Returns the count, or -1
// when the placement has more tiles than the list holds (callers then test
// every tile).
constexpr int kMaxList = 2048;
// zero_out (CTA 0 only): write ext = 0 of zero_out for every tile NOT in the
// list (their final output mask; listed tiles are written by their owner).
// Phase trace (DFX_TRUNC_TRACE=1, development only): %globaltimer stamps per CTA.
__device__ __forceinline__ void tstamp(unsigned long long* tr, int ph) {
    if (tr && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[blockIdx.x * 16 + ph] = t;
    }
}

__device__ __forceinline__ void tstamp_dep(unsigned long long* tr, int ph, unsigned dep) {
    if (tr && threadIdx.x == 0) {
        unsigned long long t;
        if (dep == 0x7fc00001u) tr[blockIdx.x * 16 + 15] = 0;  // in-order issue: the stamp waits for dep
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[blockIdx.x * 16 + ph] = t;
    }
}
constexpr int kPer = kMaxList / 256;  // tiles per thread in the list builder
// Owned bits of this thread's kPer tiles. Per-frame parameters are uploaded by a
// copy that precedes the frame's first kernel, so this may run BEFORE
// griddepcontrol.wait (it overlaps the previous kernel's tail).
__device__ __forceinline__ unsigned own_bits_pre(const Ctx& c, const FrameDev& F) {
    const int nt = F.th * F.tw, t0 = threadIdx.x * kPer;
    unsigned b = 0;
    if (nt > kMaxList) return 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if (t0 + j < nt && c.own[t0 + j] != 0) b |= 1u << j;
    return b;
}
__device__ int build_tile_list(const Ctx& c, const FrameDev& F, const PktDev& p, bool own, int* s_list, int* s_warp,
                               const PktDev* zero_out = nullptr, const unsigned* own_pre = nullptr,
                               unsigned long long* tr = nullptr) {
    const int nt = F.th * F.tw;
    if (nt > kMaxList) return -1;
    // each thread owns up to 8 consecutive tiles: all loads in one round
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int t0 = threadIdx.x * kPer;
    // (row, col) of the thread's tiles: one division, then an incremental walk;
    // branch-free loads (clamped index) so all kPer issue back to back
    int pk[kPer];
    {
        int r = t0 / F.tw, q = t0 - r * F.tw;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            pk[j] = r << 16 | q;
            if (++q == F.tw) q = 0, ++r;
        }
    }
    uint8_t ev[kPer], ov[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const bool ok = t0 + j < nt;
        ev[j] = p.ext[ok ? ext_idx(p, pk[j] >> 16, pk[j] & 0xffff) : 0] & (ok ? 0xff : 0);
        ov[j] = (!own || own_pre) ? 1 : c.own[ok ? t0 + j : 0];
    }
    unsigned bits = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const bool o = !own || (own_pre ? (*own_pre >> j & 1u) != 0 : ov[j] != 0);
        if (ev[j] != 0 && o) bits |= 1u << j;
    }
    tstamp_dep(tr, 8, bits);
    if (zero_out && blockIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < kPer; ++j)
            if (t0 + j < nt && !(bits >> j & 1u)) zero_out->ext[ext_idx(*zero_out, pk[j] >> 16, pk[j] & 0xffff)] = 0;
    }
    // block exclusive prefix of the per-thread counts
    int v = __popc(bits), incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[w] = incl;
    tstamp_dep(tr, 9, incl);
    __syncthreads();
    tstamp(tr, 10);
    int off = 0, tot = 0;
    for (int j = 0; j < nwb; ++j) {
        off += j < w ? s_warp[j] : 0;
        tot += s_warp[j];
    }
    off += incl - v;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if (bits >> j & 1u) s_list[off++] = pk[j];  // packed (row << 16 | col)
    __syncthreads();
    return tot;
}

// Tile li of a list built by build_tile_list (or every placement tile when nl < 0).
__device__ __forceinline__ void list_tile(const FrameDev& F, const int* s_list, int nl, int li, int& ti, int& tr,
                                          int& tc) {
    if (nl >= 0) {
        const int v = s_list[li];
        tr = v >> 16, tc = v & 0xffff, ti = tr * F.tw + tc;
    } else {
        ti = li, tr = ti / F.tw, tc = ti - tr * F.tw;
    }
}

// Delta packet float4 of tile element e4 (tile row-major [yy][xx][c]).
struct Div {
    int d, sh;
    __device__ __forceinline__ explicit Div(int v) : d(v), sh(-1) {
        if (v > 0 && (v & (v - 1)) == 0) sh = __ffs(v) - 1;
    }
    __device__ __forceinline__ int operator()(int x) const { return sh >= 0 ? (x >> sh) : x / d; }
};
__device__ __forceinline__ const float4* pkt_f4(const PktDev& p, int tr, int tc, int e4, const Div& row4) {
    const int yy = row4(e4), rem = e4 - yy * row4.d;
    return reinterpret_cast<const float4*>(p.d + pkt_off(p, tr * p.t + yy, tc * p.t)) + rem;
}

// Pass 1 of the truncation: max |trunc + delta| per masked owned tile.
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ void tilemax_body(const Ctx& c, const FrameDev& F, const PktDev& in, BufDev trunc,
                             unsigned* __restrict__ tile_max, const int* s_list, int nl,
                             const float* acc_prefetch = nullptr, int acc_C = 0, unsigned long long* trc = nullptr) {
    bool first = true;
    const int T = in.t, E4 = T * T * in.C / 4;
    const Div row4(T * in.C / 4), nch((E4 + kChunkF4 - 1) / kChunkF4);
    const int items = (nl < 0 ? F.th * F.tw : nl) * nch.d;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int it = gw; it < items; it += nw) {
        const int li = nch(it), ch = it - li * nch.d;
        int ti, tr, tc;
        list_tile(F, s_list, nl, li, ti, tr, tc);
        if (nl < 0 && (!in.ext[ext_idx(in, tr, tc)] || !holds_t(c, F, tr, tc))) continue;
        const float4* tb = reinterpret_cast<const float4*>(tile_base(c, F, trunc, tr, tc));
        const int q0 = ch * kChunkF4, q1 = min(E4, q0 + kChunkF4);
        if (first) tstamp_dep(trc, 11, (unsigned)(size_t)tb);
        if (acc_prefetch) {  // the commit pass reads acc of fired tiles: start it towards L2 now
            const float4* ab = reinterpret_cast<const float4*>(acc_prefetch + (size_t)slot_of(F, c.rows, c.cols, tr, tc) *
                                                                               T * T * acc_C);
            for (int q = q0 + lane * 8; q < q1; q += 256) prefetch_l2(ab + q);
        }
        float m = 0.0f;
        for (int qs = q0; qs < q1; qs += 32 * kSub) {
            float4 tv[kSub], dv[kSub];
#pragma unroll
            for (int j = 0; j < kSub; ++j) {
                const int q = qs + j * 32 + lane;
                if (q < q1) {
                    tv[j] = __ldcg(tb + q);
                    dv[j] = __ldcg(pkt_f4(in, tr, tc, q, row4));
                }
            }
            if (first) tstamp_dep(trc, 12, __float_as_uint(tv[0].x) ^ __float_as_uint(dv[0].x));
#pragma unroll
            for (int j = 0; j < kSub; ++j)
                if (qs + j * 32 + lane < q1) m = amax4(m, add4(tv[j], dv[j]));
        }
        if (first) tstamp_dep(trc, 13, __float_as_uint(m));
        first = false;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0 && m > 0.0f) atomicMax(tile_max + ti, __float_as_uint(m));
    }
}

#ifndef DFX_TILEMAX_MINB  // resident CTAs per SM of the tile-max pass (register cap)
#define DFX_TILEMAX_MINB 1
#endif
__global__ void __launch_bounds__(256, DFX_TILEMAX_MINB)
    k_trunc_tilemax(Ctx c, PktDev in, BufDev trunc, unsigned* __restrict__ tile_max) {
    pdl_enter();
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    const FrameDev& F = *c.f;
    // the halo stash touches ring slots only (never this frame's placement tiles): independent work
    ring_add_part(c, F, in, trunc, blockIdx.x * (long long)blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
    const int nl = build_tile_list(c, F, in, true, s_list, s_warp);
    tilemax_body(c, F, in, trunc, tile_max, s_list, nl);
}

// Pass 2: output mask of every placement tile, then fire / fold of the masked ones.
__device__ void commit_body(const Ctx& c, const FrameDev& F, const PktDev& in, BufDev acc, BufDev trunc,
                            const unsigned* __restrict__ tile_max, float thr, int relu, const PktDev& out,
                            const int* s_list, int nl, bool ext_by_items = false,
                            const BufDev* pf0 = nullptr, const BufDev* pf1 = nullptr, int B = -1, int NB = 0) {
    if (B < 0) B = blockIdx.x, NB = gridDim.x;  // blocks [0, NB) of the launch do the commit
    const int T = in.t, E4 = T * T * in.C / 4;
    const Div row4(T * in.C / 4), nch((E4 + kChunkF4 - 1) / kChunkF4);
    // output mask = fired tiles (delta_layers.cpp:203-204), every placement tile
    if (!ext_by_items || nl < 0)
    for (int ti = B * blockDim.x + threadIdx.x; ti < F.th * F.tw; ti += NB * blockDim.x) {
        const int tr = ti / F.tw, tc = ti - tr * F.tw;
        const float tm = __uint_as_float(__ldcg(tile_max + ti));
        out.ext[ext_idx(out, tr, tc)] =
            (in.ext[ext_idx(in, tr, tc)] && holds_t(c, F, tr, tc) && tm >= thr && tm > 0.0f) ? 1 : 0;
    }
    const int items = (nl < 0 ? F.th * F.tw : nl) * nch.d;
    const int lane = threadIdx.x & 31;
    const int gw = (B * blockDim.x + threadIdx.x) >> 5, nw = (NB * blockDim.x) >> 5;
    for (int it = gw; it < items; it += nw) {
        const int li = nch(it), ch = it - li * nch.d;
        int ti, tr, tc;
        list_tile(F, s_list, nl, li, ti, tr, tc);
        if (nl < 0 && (!in.ext[ext_idx(in, tr, tc)] || !holds_t(c, F, tr, tc))) continue;
        const float tm = __uint_as_float(__ldcg(tile_max + ti));
        const bool fire = tm >= thr && tm > 0.0f;
        if (ext_by_items && nl >= 0 && ch == 0 && lane == 0) {
            out.ext[ext_idx(out, tr, tc)] = fire ? 1 : 0;
            if (fire && pf0) {  // the consuming pool's state tiles of this fired tile, towards L2
                const int sl = slot_of(F, c.rows, c.cols, tr, tc);
                const uint32_t b0 = (uint32_t)pf0->t * pf0->t * pf0->C * 4, b1 = (uint32_t)pf1->t * pf1->t * pf1->C * 4;
                if ((b0 & 15) == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf0->d + (size_t)sl * b0 / 4), "r"(b0)
                                 : "memory");
                if ((b1 & 15) == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf1->d + (size_t)sl * b1 / 4), "r"(b1)
                                 : "memory");
            }
        }
        float4* tb = reinterpret_cast<float4*>(tile_base(c, F, trunc, tr, tc));
        float4* ab = reinterpret_cast<float4*>(tile_base(c, F, acc, tr, tc));
        const int q0 = ch * kChunkF4, q1 = min(E4, q0 + kChunkF4);
        for (int qs = q0; qs < q1; qs += 32 * kSub) {
            constexpr int kS = kSub / 2;  // three arrays in flight: keep registers (occupancy) in check
#pragma unroll
            for (int h = 0; h < 2; ++h) {
            float4 tv[kS], dv[kS], pv[kS];
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int q = qs + (h * kS + j) * 32 + lane;
                if (q < q1) {
                    tv[j] = __ldcg(tb + q);
                    dv[j] = __ldcg(pkt_f4(in, tr, tc, q, row4));
                    if (kTruncPrefetch) pv[j] = __ldcg(ab + q);  // L2 hit: prefetched in pass 1, no wait on tile_max
                    else if (fire) pv[j] = __ldcs(ab + q);
                }
            }
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int q = qs + (h * kS + j) * 32 + lane;
                if (q >= q1) continue;
                const float4 cd = add4(tv[j], dv[j]);
                if (fire) {
                    const float4 nv = add4(pv[j], cd);
                    float4 o = cd;
                    if (relu) {
                        o.x = __fsub_rn(fmaxf(nv.x, 0.f), fmaxf(pv[j].x, 0.f));
                        o.y = __fsub_rn(fmaxf(nv.y, 0.f), fmaxf(pv[j].y, 0.f));
                        o.z = __fsub_rn(fmaxf(nv.z, 0.f), fmaxf(pv[j].z, 0.f));
                        o.w = __fsub_rn(fmaxf(nv.w, 0.f), fmaxf(pv[j].w, 0.f));
                    }
                    __stcs(ab + q, nv);
                    __stcs(tb + q, make_float4(0.f, 0.f, 0.f, 0.f));
                    const int yy = row4(q), rem = q - yy * row4.d;
                    reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + yy, tc * T))[rem] = o;
                } else {
                    __stcs(tb + q, cd);
                }
            }
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_trunc_commit(Ctx c, PktDev in, BufDev acc, BufDev trunc,
                                                      const unsigned* __restrict__ tile_max, float thr, int relu,
                                                      PktDev out, BufDev pf0, BufDev pf1, int stash) {
    pdl_enter();
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    const FrameDev& F = *c.f;
    // pass 1 ran inside the producing conv: the halo stash (ring slots only,
    // disjoint from every tile the commit touches) moves here
    if (stash)
        ring_add_part(c, F, in, trunc, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                      (long long)gridDim.x * blockDim.x);
    const int nl = build_tile_list(c, F, in, true, s_list, s_warp);
    commit_body(c, F, in, acc, trunc, tile_max, thr, relu, out, s_list, nl, false, pf0.d ? &pf0 : nullptr,
                pf1.d ? &pf1 : nullptr);
}

// Pass 2 of the activation fused with its sole consumer, a 2x2 / stride-2 max
// pool (delta_layers.cpp:149-232 then :234-318). Both are tile-local: a pool
// output pixel's window lies inside one activation tile (k == stride, halo 0),
// and the pool's input mask is the activation's fired mask. Work item = (listed
// tile, pool output row); unfired tiles fold (trunc += delta) their two input
// rows; fired tiles commit the 2x2 input pixels of each pool output float4 and
// immediately fold the activation output into the pool state:
//   act:  cand = trunc + delta; acc' = acc + cand; trunc = 0; o = relu(acc') - relu(acc)
//   pool: pacc += o; m = max over the window (first-element init, std::max order);
//         pool out = m - prev; prev = m
// The activation output packet is still written (its consumers' readers and the
// parity tests see it), the pool never re-reads it. Same fp32 operations in the
// same order as the two kernels, so results are identical.
__device__ void commit_pool_body(const Ctx& c, PktDev in, BufDev acc, BufDev trunc, const unsigned* __restrict__ tile_max,
                                 float thr, int relu, PktDev out, BufDev pacc, BufDev pprev, PktDev pout, int* s_list,
                                 int* s_warp, int B, int NB) {
    const FrameDev& F = *c.f;
    const int T = in.t, to = T / 2, C4 = in.C / 4;
    // output masks of every placement tile: activation out = fired, pool out = the same
    for (int ti = B * blockDim.x + threadIdx.x; ti < F.th * F.tw; ti += NB * blockDim.x) {
        const int tr = ti / F.tw, tc = ti - tr * F.tw;
        const float tm = __uint_as_float(__ldcg(tile_max + ti));
        const uint8_t f = (in.ext[ext_idx(in, tr, tc)] && holds_t(c, F, tr, tc) && tm >= thr && tm > 0.0f) ? 1 : 0;
        out.ext[ext_idx(out, tr, tc)] = f;
        pout.ext[ext_idx(pout, tr, tc)] = f;
    }
    const int nl = build_tile_list(c, F, in, true, s_list, s_warp);
    const int items = (nl < 0 ? F.th * F.tw : nl) * to;
    const int lane = threadIdx.x & 31;
    const int gw = (B * blockDim.x + threadIdx.x) >> 5, nw = (NB * blockDim.x) >> 5;
    const int row4 = T * C4;  // float4s per input tile row
    for (int it = gw; it < items; it += nw) {
        const int li = it / to, oy = it - li * to;
        int ti, tr, tc;
        list_tile(F, s_list, nl, li, ti, tr, tc);
        if (nl < 0 && (!in.ext[ext_idx(in, tr, tc)] || !holds_t(c, F, tr, tc))) continue;
        const float tm = __uint_as_float(__ldcg(tile_max + ti));
        const bool fire = tm >= thr && tm > 0.0f;
        float4* tb = reinterpret_cast<float4*>(tile_base(c, F, trunc, tr, tc));
        float4* ab = reinterpret_cast<float4*>(tile_base(c, F, acc, tr, tc));
        if (!fire) {  // fold both input rows of this output row
            for (int q = 2 * oy * row4 + lane; q < (2 * oy + 2) * row4; q += 32) {
                const int yy = q / row4, rem = q - yy * row4;
                const float4 dv = __ldcg(reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * T + yy, tc * T)) + rem);
                __stcs(tb + q, add4(__ldcg(tb + q), dv));
            }
            continue;
        }
        float4* pab = reinterpret_cast<float4*>(tile_base(c, F, pacc, tr, tc));
        float4* ppb = reinterpret_cast<float4*>(tile_base(c, F, pprev, tr, tc));
        for (int q = lane; q < to * C4; q += 32) {
            const int ox = q / C4, c4 = q - ox * C4;
            size_t e[4];
            float4 tv[4], dv[4], av[4], pv[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {  // all loads of the window in flight first
                const int iy = 2 * oy + (w >> 1), ix = 2 * ox + (w & 1);
                e[w] = ((size_t)iy * T + ix) * C4 + c4;
                tv[w] = __ldcg(tb + e[w]);
                av[w] = __ldcg(ab + e[w]);
                pv[w] = __ldcs(pab + e[w]);
                dv[w] = __ldcg(reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * T + iy, tc * T + ix)) + c4);
            }
            float4* pp = ppb + ((size_t)oy * to + ox) * C4 + c4;
            const float4 prev = __ldcs(pp);
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int iy = 2 * oy + (w >> 1), ix = 2 * ox + (w & 1);
                const float4 cd = add4(tv[w], dv[w]);
                const float4 nv = add4(av[w], cd);
                float4 o = cd;
                if (relu) {
                    o.x = __fsub_rn(fmaxf(nv.x, 0.f), fmaxf(av[w].x, 0.f));
                    o.y = __fsub_rn(fmaxf(nv.y, 0.f), fmaxf(av[w].y, 0.f));
                    o.z = __fsub_rn(fmaxf(nv.z, 0.f), fmaxf(av[w].z, 0.f));
                    o.w = __fsub_rn(fmaxf(nv.w, 0.f), fmaxf(av[w].w, 0.f));
                }
                __stcs(ab + e[w], nv);
                __stcs(tb + e[w], make_float4(0.f, 0.f, 0.f, 0.f));
                reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + iy, tc * T + ix))[c4] = o;
                const float4 v = add4(pv[w], o);  // pool: acc += delta (delta_layers.cpp:253-261)
                __stcs(pab + e[w], v);
                if (w == 0) {
                    m = v;
                } else {  // std::max(m, v) == (m < v) ? v : m
                    m.x = m.x < v.x ? v.x : m.x;
                    m.y = m.y < v.y ? v.y : m.y;
                    m.z = m.z < v.z ? v.z : m.z;
                    m.w = m.w < v.w ? v.w : m.w;
                }
            }
            reinterpret_cast<float4*>(pout.d + pkt_off(pout, tr * to + oy, tc * to + ox))[c4] =
                make_float4(__fsub_rn(m.x, prev.x), __fsub_rn(m.y, prev.y), __fsub_rn(m.z, prev.z),
                            __fsub_rn(m.w, prev.w));
            __stcs(pp, m);
        }
    }
}

__global__ void __launch_bounds__(256) k_trunc_commit_pool(Ctx c, PktDev in, BufDev acc, BufDev trunc,
                                                           const unsigned* __restrict__ tile_max, float thr, int relu,
                                                           PktDev out, BufDev pacc, BufDev pprev, PktDev pout) {
    pdl_enter();
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    commit_pool_body(c, in, acc, trunc, tile_max, thr, relu, out, pacc, pprev, pout, s_list, s_warp, blockIdx.x,
                     gridDim.x);
}

// The activation's commit (optionally with its fused max pool) and the NEXT
// stride-1 conv's plan in one launch: blocks [0, nplan) run plan blocks whose
// input mask comes from the activation's tile maxima (MaskSrc), blocks
// [nplan, nplan + ncommit) run the commit. The two touch disjoint memory (the
// plan writes the conv's target list, output ext and zero fill; the commit the
// activation's / pool's state and packets), so no ordering is needed between them.
template <bool POOL>
__global__ void __launch_bounds__(256, 2) k_trunc_commit_plan(Ctx c, PktDev in, BufDev acc, BufDev trunc,
                                                             const unsigned* __restrict__ tile_max, float thr, int relu,
                                                             PktDev out, BufDev pacc, BufDev pprev, PktDev pout,
                                                             BufDev pf0, BufDev pf1, PlanArgs pa, int nplan) {
    pdl_enter();
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    __shared__ PlanSmem sm;
    if ((int)blockIdx.x < nplan) {
        plan_block<256>(c, pa, blockIdx.x, sm);
        return;
    }
    const int B = blockIdx.x - nplan, NB = gridDim.x - nplan;
    if (POOL) {
        commit_pool_body(c, in, acc, trunc, tile_max, thr, relu, out, pacc, pprev, pout, s_list, s_warp, B, NB);
    } else {
        const FrameDev& F = *c.f;
        const int nl = build_tile_list(c, F, in, true, s_list, s_warp);
        commit_body(c, F, in, acc, trunc, tile_max, thr, relu, out, s_list, nl, false, pf0.d ? &pf0 : nullptr,
                    pf1.d ? &pf1 : nullptr, B, NB);
    }
}

// Both passes in ONE cooperative persistent launch (every CTA resident): the
// tile list is built once, and a grid barrier separates the tile maxima from
// their use, saving a kernel boundary and its latency chain per layer.
// One arrival per CTA (release), then acquire LOADS while waiting: polling with
// read-modify-write atomics from every CTA would serialise at the L2 slice.
__device__ __forceinline__ void grid_barrier(unsigned* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= gridDim.x) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256, DFX_TRUNC_MINB) k_trunc_coop(Ctx c, PktDev in, BufDev acc, BufDev trunc,
                                                    unsigned* __restrict__ tile_max, float thr, int relu, PktDev out,
                                                    unsigned* __restrict__ gbar, unsigned long long* tr, int dry,
                                                    DenseOut dz, BufDev pf0, BufDev pf1) {
    tstamp(tr, 0);
    // touch every kernel parameter up front: their constant-bank lines miss once, together
    asm volatile("" ::"l"(in.d), "l"(in.ext), "r"(in.C), "r"(in.t), "r"(in.halo), "r"(in.RT), "r"(in.pitch_w),
                 "r"(in.ext_pitch), "l"(acc.d), "r"(acc.C), "r"(acc.t), "l"(trunc.d), "l"(tile_max), "f"(thr), "r"(relu));
    asm volatile("" ::"l"(out.d), "l"(out.ext), "r"(out.C), "r"(out.halo), "r"(out.RT), "r"(out.pitch_w),
                 "r"(out.ext_pitch), "l"(gbar), "r"(c.rows), "r"(c.cols), "l"(c.slots), "l"(c.own), "l"(c.f), "r"(dry));
    const FrameDev F = *c.f;  // per-frame data: safe before the dependency wait (see own_bits_pre)
    const unsigned own_pre = own_bits_pre(c, F);
    tstamp_dep(tr, 7, own_pre);
    pdl_enter();
    tstamp(tr, 1);
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    const int nl = build_tile_list(c, F, in, true, s_list, s_warp, dry ? nullptr : &out, &own_pre, dry ? nullptr : tr);
    if (dry) return;
    tstamp(tr, 2);
    tilemax_body(c, F, in, trunc, tile_max, s_list, nl, kTruncPrefetch ? acc.d : nullptr, acc.C, tr);
    tstamp(tr, 3);
    // split grid barrier: arrive, do the halo stash (ring slots only, independent of both passes), wait
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
    ring_add_part(c, F, in, trunc, blockIdx.x * (long long)blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
    tstamp(tr, 4);
    if (threadIdx.x == 0) {
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
            if (v >= gridDim.x) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
    tstamp(tr, 5);
    commit_body(c, F, in, acc, trunc, tile_max, thr, relu, out, s_list, nl, true, pf0.d ? &pf0 : nullptr,
                pf1.d ? &pf1 : nullptr);
    if (dz.out) {
        // output layer: densify acc + trunc into the frame's output after a
        // second grid barrier (same counter), saving the densify launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
            unsigned v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
                if (v >= 2 * gridDim.x) break;
                __nanosleep(32);
            }
        }
        __syncthreads();
        wait_flag(dz.rb.out_flag, dz.rb.out_val);  // host path: the output slot's previous copy-out is done
        frame_readback(dz.rb);
        densify8_body(c, acc, trunc, dz.out, (blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                      (gridDim.x * blockDim.x) >> 5);
    }
    __syncthreads();
    tstamp(tr, 6);
}

// Max pool, halo-free input, k == stride (network.cpp:164-166), C % 4 == 0:
// acc += delta over the window (delta_layers.cpp:253-261), window max of acc
// initialised from the first element (:294-306), out = max - prev, prev = max
// (:308-310); outputs of masked, non-owned tiles are 0. Work unit: a warp takes
// a chunk of a masked tile's output float4s.
__global__ void __launch_bounds__(256) k_maxpool_vec(Ctx c, PktDev in, BufDev acc, BufDev prev, int k, PktDev out) {
    pdl_enter();
    __shared__ int s_list[kMaxList];
    __shared__ int s_warp[8];
    const FrameDev& F = *c.f;
    const int to = out.t, ti_ = in.t, C4 = in.C / 4;
    const int E4 = to * to * C4;
    const int nch = (E4 + 63) / 64;
    for (int ti = blockIdx.x * blockDim.x + threadIdx.x; ti < F.th * F.tw; ti += gridDim.x * blockDim.x) {
        const int tr = ti / F.tw, tc = ti - tr * F.tw;
        out.ext[ext_idx(out, tr, tc)] = in.ext[ext_idx(in, tr, tc)] ? 1 : 0;
    }
    const int nl = build_tile_list(c, F, in, false, s_list, s_warp);
    const int items = (nl < 0 ? F.th * F.tw : nl) * nch;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int it = gw; it < items; it += nw) {
        const int li = it / nch, ch = it - li * nch;
        int tix, tr, tc;
        list_tile(F, s_list, nl, li, tix, tr, tc);
        if (nl < 0 && !in.ext[ext_idx(in, tr, tc)]) continue;
        const bool owned = holds_t(c, F, tr, tc);
        float4* ab = owned ? reinterpret_cast<float4*>(tile_base(c, F, acc, tr, tc)) : nullptr;
        float4* pb = owned ? reinterpret_cast<float4*>(tile_base(c, F, prev, tr, tc)) : nullptr;
        const int q0 = ch * 64, q1 = min(E4, q0 + 64);
#pragma unroll 2
        for (int q = q0 + lane; q < q1; q += 32) {
            const int px = q / C4, c4 = q - px * C4;
            const int y = px / to, x = px - y * to;
            float4* d = reinterpret_cast<float4*>(out.d + pkt_off(out, tr * to + y, tc * to + x)) + c4;
            if (!owned) {
                *d = make_float4(0.f, 0.f, 0.f, 0.f);
                continue;
            }
            if (k == 2) {
                // 2x2 window: all nine loads (4 acc, 4 delta, prev) in flight before any use
                float4* ap[4];
                float4 av[4], dv[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const int iy = y * 2 + (w >> 1), ix = x * 2 + (w & 1);
                    ap[w] = ab + ((size_t)iy * ti_ + ix) * C4 + c4;
                    av[w] = __ldcs(ap[w]);
                    dv[w] = __ldcg(reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * ti_ + iy, tc * ti_ + ix)) + c4);
                }
                float4* pp = pb + ((size_t)y * to + x) * C4 + c4;
                const float4 pv = __ldcs(pp);
                float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const float4 v = add4(av[w], dv[w]);
                    __stcs(ap[w], v);
                    if (w == 0) {
                        m = v;
                    } else {  // std::max(m, v) == (m < v) ? v : m
                        m.x = m.x < v.x ? v.x : m.x;
                        m.y = m.y < v.y ? v.y : m.y;
                        m.z = m.z < v.z ? v.z : m.z;
                        m.w = m.w < v.w ? v.w : m.w;
                    }
                }
                *d = make_float4(__fsub_rn(m.x, pv.x), __fsub_rn(m.y, pv.y), __fsub_rn(m.z, pv.z), __fsub_rn(m.w, pv.w));
                __stcs(pp, m);
                continue;
            }
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    const int iy = y * k + ky, ix = x * k + kx;
                    float4* ap = ab + ((size_t)iy * ti_ + ix) * C4 + c4;
                    const float4 dv = __ldcg(reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * ti_ + iy, tc * ti_ + ix)) + c4);
                    const float4 v = add4(__ldcs(ap), dv);
                    __stcs(ap, v);
                    if (ky == 0 && kx == 0) {
                        m = v;
                    } else {  // std::max(m, v) == (m < v) ? v : m
                        m.x = m.x < v.x ? v.x : m.x;
                        m.y = m.y < v.y ? v.y : m.y;
                        m.z = m.z < v.z ? v.z : m.z;
                        m.w = m.w < v.w ? v.w : m.w;
                    }
                }
            float4* pp = pb + ((size_t)y * to + x) * C4 + c4;
            const float4 pv = __ldcs(pp);
            *d = make_float4(__fsub_rn(m.x, pv.x), __fsub_rn(m.y, pv.y), __fsub_rn(m.z, pv.z), __fsub_rn(m.w, pv.w));
            __stcs(pp, m);
        }
    }
}

// Persistent grid: SMs x resident CTAs per SM for this kernel, on the calling
// thread's current device (the carveout attribute and the SM count are per
// device: `cache` is the call site's per-device memo).
template <typename K>
int stream_grid(K kernel, std::atomic<int> (&cache)[64]) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    const int hit = cache[dev & 63].load(std::memory_order_relaxed);
    if (hit) return hit;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 256, 0);
    const int g = sms * (per < 1 ? 1 : per);
    cache[dev & 63].store(g, std::memory_order_relaxed);
    return g;
}

}  // namespace

static unsigned long long* g_trunc_trace = nullptr;
unsigned long long* trunc_trace_buffer() { return g_trunc_trace; }

// Work-proportional grids: an upper bound on the warp work items of the next
// activation launches (placement tiles x chunks, set by the engine per layer);
// the persistent grids shrink to ceil(items / 8 warps) so small layers leave SMs
// to concurrent streams / engines. 0: no bound.
static thread_local long long g_item_hint = 0;
void set_trunc_work_hint(long long items) { g_item_hint = items; }
static int capped(int g) {
    if (g_item_hint <= 0) return g;
    const long long need = (g_item_hint + 7) / 8;
    return need < g ? (int)(need < 1 ? 1 : need) : g;
}

int launch_trunc_two_pass(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc, unsigned* tile_max,
                           float thr, int relu, PktDev out, unsigned* gbar, const DenseOut* dzp, bool* dz_done,
                           BufDev pf0, BufDev pf1) {
    if (dz_done) *dz_done = false;
    const DenseOut dz = (dzp && (acc.C & 7) == 0) ? *dzp : DenseOut{nullptr, Readback{}};
    if ((in.C & 3) != 0) return 0;
    static std::atomic<int> gc_cache[64];
    const int gc = stream_grid(k_trunc_coop, gc_cache);
    // two launches by default: at the C2 ~10 % update rate the cooperative
    // single launch (co-residency wait, no programmatic overlap) measured
    // 1.5-2.5 % slower; DFX_TRUNC_COOP=1 selects it (it also hosts the output
    // densify and the pool-state prefetch)
    static const bool coop_ok = [] {
        const char* e = getenv("DFX_TRUNC_COOP");
        return e && e[0] == '1';
    }();
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (getenv("DFX_TRUNC_TRACE")) cudaMalloc(&p, sizeof(unsigned long long) * 64 * 1024 * 16);
        return p;
    }();
    static int seq = 0;
    unsigned long long* tr = trace ? trace + (size_t)(seq++ % 64) * 1024 * 16 : nullptr;
    g_trunc_trace = trace;
    static const bool warm = getenv("DFX_TRUNC_WARM") != nullptr;  // experiment
    if (warm) launch_pdl(k_trunc_coop, gc, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out, gbar,
                         (unsigned long long*)nullptr, 1, DenseOut{nullptr, Readback{}}, BufDev{nullptr, 0, 0},
                         BufDev{nullptr, 0, 0});
    if (gbar && coop_ok) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(gc);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        if (cudaLaunchKernelEx(&cfg, k_trunc_coop, c, in, acc, trunc, tile_max, thr, relu, out, gbar, tr, 0, dz, pf0, pf1) ==
            cudaSuccess) {
            if (dz_done) *dz_done = dz.out != nullptr;
            return 1;
        }
        cudaGetLastError();  // fall back to two launches
    }
    static std::atomic<int> g1_cache[64], g2_cache[64];
    const int g1 = capped(stream_grid(k_trunc_tilemax, g1_cache)), g2 = capped(stream_grid(k_trunc_commit, g2_cache));
    launch_pdl(k_trunc_tilemax, g1, 256, 0, s, c, in, trunc, tile_max);
    launch_pdl(k_trunc_commit, g2, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out, pf0, pf1, 0);
    return 2;
}

void launch_trunc_tilemax(const Ctx& c, cudaStream_t s, PktDev in, BufDev trunc, unsigned* tile_max) {
    static std::atomic<int> g_cache[64];
    launch_pdl(k_trunc_tilemax, capped(stream_grid(k_trunc_tilemax, g_cache)), 256, 0, s, c, in, trunc, tile_max);
}

void launch_trunc_commit_pool(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                              const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pacc, BufDev pprev,
                              PktDev pout) {
    static std::atomic<int> g_cache[64];
    const int g = capped(stream_grid(k_trunc_commit_pool, g_cache));
    launch_pdl(k_trunc_commit_pool, g, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out, pacc, pprev, pout);
}

void launch_trunc_commit_plan(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                              const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pacc, BufDev pprev,
                              PktDev pout, const DenseConvPlan& p, PktDev cin, PktDev cout, int hg, int* units,
                              int* nunits, unsigned long long* flop_px, int* list, int* lcount) {
    static std::atomic<int> g0[64], g1[64];
    const bool pool = pacc.d != nullptr;
    const int gcommit =
        capped(pool ? stream_grid(k_trunc_commit_plan<true>, g1) : stream_grid(k_trunc_commit_plan<false>, g0));
    PlanArgs pa{cin, cout, p.k, p.r, hg, p.nbw, p.nbh * p.nbw, units, nunits, flop_px, 1, list, lcount,
                p.tpu ? 1 : 0, nullptr, BufDev{nullptr, 0, 0},
                MaskSrc{in.ext, in.RT, in.ext_pitch, tile_max, thr}};
    const int nplan = p.nbh * p.nbw;
    if (pool)
        launch_pdl(k_trunc_commit_plan<true>, nplan + gcommit, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out,
                   pacc, pprev, pout, BufDev{nullptr, 0, 0}, BufDev{nullptr, 0, 0}, pa, nplan);
    else
        launch_pdl(k_trunc_commit_plan<false>, nplan + gcommit, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out,
                   pacc, pprev, pout, BufDev{nullptr, 0, 0}, BufDev{nullptr, 0, 0}, pa, nplan);
}

void launch_trunc_commit_stash(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                               const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pf0, BufDev pf1) {
    static std::atomic<int> g_cache[64];
    const int g = capped(stream_grid(k_trunc_commit, g_cache));
    launch_pdl(k_trunc_commit, g, 256, 0, s, c, in, acc, trunc, tile_max, thr, relu, out, pf0, pf1, 1);
}

bool launch_maxpool_vec(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, PktDev out) {
    if ((in.C & 3) != 0) return false;
    static std::atomic<int> g_cache[64];
    const int g = stream_grid(k_maxpool_vec, g_cache);
    launch_pdl(k_maxpool_vec, g, 256, 0, s, c, in, acc, prev, k, out);
    return true;
}

DFX_KTRACE_SETTER(ktrace_set_hbm)

}  // namespace dfx
