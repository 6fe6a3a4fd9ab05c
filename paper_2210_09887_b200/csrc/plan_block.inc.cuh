// Conv planning block (target bits, exact output TileMask, FLOP pixels, dense
// unit / tile list, gathered list, zero fill) of k_conv_plan, as a block
// function over PlanArgs so other kernels can embed it (measured on C2:
// running it inside the persistent dense-conv or activation kernels loses to
// the standalone launch, plan blocks need many resident CTAs). Textually
// included INSIDE the translation unit's anonymous namespace; the includer
// provides kernels.hpp / dfx_types.hpp.
#pragma once

constexpr int kUY = 16, kUX = 8;  // unit = 16 rows x 8 cols = 128 pixels

// Floor division by a runtime divisor: an arithmetic shift (exact floor for
// negative values too) when the divisor is a power of two, which every tile
// size and block width of a network with pow2 tiles is.
struct FDiv {
    int d, sh;
    __device__ __forceinline__ explicit FDiv(int v) : d(v), sh(-1) {
        if (v > 0 && (v & (v - 1)) == 0) {
            sh = 0;
            while ((1 << sh) < v) ++sh;
        }
    }
    __device__ __forceinline__ int operator()(int x) const { return sh >= 0 ? (x >> sh) : floor_div32(x, d); }
};

__device__ __forceinline__ bool pkt_ok(const PktDev& p, int th, int tw, int y, int x) {
    if (y < -p.halo || y >= th * p.t + p.halo || x < -p.halo || x >= tw * p.t + p.halo) return false;
    return p.ext[ext_idx(p, floor_div32(y, p.t), floor_div32(x, p.t))] != 0;
}

// Source of the conv input's tile mask: the input packet's ext bytes, or -
// when the plan runs inside the producing activation's commit launch, whose
// blocks write that ext concurrently - the activation's fire rule evaluated
// from its tile maxima (delta_layers.cpp:203-204): masked and owned input tile
// with tile_max >= thr and > 0.
struct MaskSrc {
    const uint8_t* act_ext;  // the activation's INPUT packet ext (null: use the conv input's ext)
    int act_RT, act_pitch;
    const unsigned* tmax;
    float thr;
};
__device__ __forceinline__ bool tile_masked(const Ctx& c, const PktDev& in, const MaskSrc& ms, int tw, int tr,
                                            int tc) {
    if (!ms.act_ext) return in.ext[ext_idx(in, tr, tc)] != 0;
    const int ti = tr * tw + tc;
    if (!ms.act_ext[(tr + ms.act_RT) * ms.act_pitch + tc + ms.act_RT] || !c.own[ti]) return false;
    const float tm = __uint_as_float(__ldcg(ms.tmax + ti));
    return tm >= ms.thr && tm > 0.0f;
}

// Target test of a stride-1 window (delta_layers.cpp:34-45, :60-70).
__device__ __forceinline__ bool is_target_s1(const Ctx& c, const MaskSrc& ms, const PktDev& in, int th, int tw, int oy,
                                             int ox, int k, int r, const FDiv& dt) {
    const int iy0 = oy - r - in.halo, iy1 = oy - r + k - 1 + in.halo;
    const int ix0 = ox - r - in.halo, ix1 = ox - r + k - 1 + in.halo;
    const int tr0 = max(dt(iy0), 0), tr1 = min(dt(iy1), th - 1);
    const int tc0 = max(dt(ix0), 0), tc1 = min(dt(ix1), tw - 1);
    for (int tr = tr0; tr <= tr1; ++tr)
        for (int tc = tc0; tc <= tc1; ++tc)
            if (tile_masked(c, in, ms, tw, tr, tc)) return true;
    return false;
}

// Conv planning for the dense path (replaces target compaction for stride-1
// convs; delta_layers.cpp:34-83). One CTA per BLOCK = the union of whole units
// and whole tiles: a tile when t >= 16 (t/16 x t/8 units), a unit when t < 16
// (16/t x 8/t tiles). Blocks are aligned at pixel (0, 0); block row/col 0 is
// the one above/left of the extent, so the grown ring [-hg, 0) is covered.
// Per block: the target bit of every pixel of the geometric grown extent
// (FLOPs count all of them, :139-145), the exact output TileMask / ext byte of
// every stored tile (any target inside the stored extent, :72-83), every unit
// with >= 1 target appended to the dense list (units encoded
// (uy + 1) << 16 | (ux + 1)), and zeros for the pixels of active stored tiles
// that no dense unit covers (possible only when a tile holds several units).
constexpr int kPlanThreads = 256;
struct PlanArgs {
    PktDev in, out;
    int k, r, hg, nbw, nblocks;
    int* units;
    int* nunits;
    unsigned long long* flop_px;
    int tau;
    int* list;
    int* lcount;
    int tile_units;
    // fused activation pass 1 (k_conv_dense epilogue): zero-filled pixels of
    // active placement tiles fold max |trunc| into tile_max here (null: off)
    unsigned* tile_max;
    BufDev tm_trunc;
    MaskSrc ms;  // zero: the conv input packet's ext is final (standalone k_conv_plan)
};
struct PlanSmem {
    uint32_t bits[4096 / 32];
    int ucnt[32];
    int tstore[32];
    int geo[32];
};
// One plan block, executed by the NT threads of the calling CTA (the
// k_conv_plan CTA; NT = threads taking part).
template <int NT, bool TM = false>
__device__ void plan_block(const Ctx& c, const PlanArgs& pa, int blk, PlanSmem& sm) {
    const PktDev& in = pa.in;
    const PktDev& out = pa.out;
    const int k = pa.k, r = pa.r, hg = pa.hg, nbw = pa.nbw, tau = pa.tau, tile_units = pa.tile_units;
    int* __restrict__ units = pa.units;
    int* __restrict__ nunits = pa.nunits;
    unsigned long long* __restrict__ flop_px = pa.flop_px;
    int* __restrict__ list = pa.list;
    int* __restrict__ lcount = pa.lcount;
    uint32_t* s_bits = sm.bits;
    int* s_ucnt = sm.ucnt;
    int* s_tstore = sm.tstore;
    int* s_geo = sm.geo;
    const FrameDev& F = *c.f;
    const int t = out.t;
    const int BH = t > kUY ? t : kUY, BW = t > kUX ? t : kUX;
    const int by = blk / nbw, bx = blk - (blk / nbw) * nbw;
    const int Y0 = (by - 1) * BH, X0 = (bx - 1) * BW;
    const int eh = F.th * t, ew = F.tw * t;
    const int hs = out.halo;
    // block entirely outside the grown extent: nothing to do (its tiles are beyond ext)
    if (Y0 >= eh + hg || X0 >= ew + hg || Y0 + BH <= -hg || X0 + BW <= -hg) return;
    const int upr = BW / kUX, nun = (BH / kUY) * upr;  // units in block
    const int tpr = BW / t, ntl = (BH / t) * tpr;        // tiles in block
    const FDiv dbw(BW), dt(t), din(in.t), dtpr(tpr);
    if (threadIdx.x < 32) {
        s_ucnt[threadIdx.x] = 0;
        s_tstore[threadIdx.x] = 0;
    }
    __syncthreads();
    const int npx = BH * BW;
    int geo = 0;
    for (int p0 = 0; p0 < npx; p0 += NT) {
        const int p = p0 + threadIdx.x;
        bool tgt = false;
        int uid = -1;
        if (p < npx) {
            const int ly = dbw(p), lx = p - ly * BW;
            const int y = Y0 + ly, x = X0 + lx;
            if (y >= -hg && y < eh + hg && x >= -hg && x < ew + hg) tgt = is_target_s1(c, pa.ms, in, F.th, F.tw, y, x, k, r, din);
            if (tgt) {
                ++geo;
                uid = (ly / kUY) * upr + lx / kUX;
                if (y >= -hs && y < eh + hs && x >= -hs && x < ew + hs) s_tstore[dt(ly) * tpr + dt(lx)] = 1;
            }
        }
        // per-unit target counts, aggregated per warp (one shared atomic per unit and warp)
        const unsigned grp = __match_any_sync(0xffffffffu, uid);
        if (uid >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&s_ucnt[uid], __popc(grp));
        const unsigned m = __ballot_sync(0xffffffffu, tgt);
        if ((threadIdx.x & 31) == 0 && p < npx) s_bits[p >> 5] = m;
    }
    for (int o = 16; o > 0; o >>= 1) geo += __shfl_xor_sync(0xffffffffu, geo, o);
    if ((threadIdx.x & 31) == 0) s_geo[threadIdx.x >> 5] = geo;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < NT / 32; ++w) tot += s_geo[w];
        if (tot) atomicAdd(flop_px, (unsigned long long)tot);  // one global atomic per block
    }
    // units with >= tau targets are computed whole by k_conv_dense (tile-unit
    // mode: every active stored tile is listed instead, see below)
    if (!tile_units && threadIdx.x < nun && s_ucnt[threadIdx.x] >= tau) {
        const int uy = Y0 / kUY + threadIdx.x / upr, ux = X0 / kUX + threadIdx.x % upr;
        units[atomicAdd(nunits, 1)] = ((uy + 1) << 16) | (ux + 1);
    }
    // targets of sparser units go to the gathered kernel (stored extent only)
    if (tau > 1) {
        for (int p0 = 0; p0 < npx; p0 += NT) {
            const int p = p0 + threadIdx.x;
            bool g = false;
            int y = 0, x = 0;
            if (p < npx && ((s_bits[p >> 5] >> (p & 31)) & 1u)) {
                const int ly = dbw(p), lx = p - ly * BW;
                y = Y0 + ly, x = X0 + lx;
                g = s_ucnt[(ly / kUY) * upr + lx / kUX] < tau && y >= -hs && y < eh + hs && x >= -hs && x < ew + hs;
            }
            const unsigned m = __ballot_sync(0xffffffffu, g);
            int base = 0;
            if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(lcount, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (g) list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = ((y + hg) << 16) | (x + hg);
        }
    }
    if (threadIdx.x < ntl) {
        const int ti = dt(Y0) + dtpr((int)threadIdx.x), tj = dt(X0) + (int)threadIdx.x - dtpr((int)threadIdx.x) * tpr;
        if (ti >= -out.RT && ti < F.th + out.RT && tj >= -out.RT && tj < F.tw + out.RT) {
            out.ext[ext_idx(out, ti, tj)] = s_tstore[threadIdx.x] ? 1 : 0;
            if (tile_units && s_tstore[threadIdx.x]) units[atomicAdd(nunits, 1)] = ((ti + 8) << 16) | (tj + 8);
        }
    }
    // zero fill: non-target stored pixels of active tiles outside dense units
    const bool sparse_unit = __syncthreads_or(threadIdx.x < nun && s_ucnt[threadIdx.x] < tau);
    const bool active_tile = __syncthreads_or(threadIdx.x < ntl && s_tstore[threadIdx.x]);
    if ((nun > 1 || tau > 1) && sparse_unit && active_tile) {
        const int C = out.C;
        if ((C & 3) == 0) {
            // warp-cooperative: each warp ballots which of its 32 pixels need zeros,
            // then writes two pixels' float4 rows per instruction (coalesced)
            const int C4 = C / 4, lane = threadIdx.x & 31;
            for (int p0 = (threadIdx.x & ~31); p0 < npx; p0 += NT) {
                const int p = p0 + lane;
                bool z = false;
                int y = 0, x = 0;
                if (p < npx) {
                    const int ly = dbw(p), lx = p - ly * BW;
                    y = Y0 + ly, x = X0 + lx;
                    z = s_ucnt[(ly / kUY) * upr + lx / kUX] < tau && s_tstore[dt(ly) * tpr + dt(lx)] &&
                        !((s_bits[p >> 5] >> (p & 31)) & 1u) && y >= -hs && y < eh + hs && x >= -hs && x < ew + hs;
                }
                unsigned m = __ballot_sync(0xffffffffu, z);
                while (m) {
                    const int a0 = __ffs(m) - 1;
                    m &= m - 1;
                    int a1 = -1;
                    if (m) a1 = __ffs(m) - 1, m &= m - 1;
                    const int src = lane < 16 ? a0 : a1;
                    const int yy = __shfl_sync(0xffffffffu, y, src < 0 ? 0 : src);
                    const int xx = __shfl_sync(0xffffffffu, x, src < 0 ? 0 : src);
                    if (src >= 0) {
                        float4* row = reinterpret_cast<float4*>(out.d + pkt_off(out, yy, xx));
                        for (int q = lane & 15; q < C4; q += 16) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    if (TM) {  // delta is 0 here: max |trunc| of the pixel's channels
                        const bool in_ext = src >= 0 && yy >= 0 && yy < eh && xx >= 0 && xx < ew;
                        float mt = 0.0f;
                        int key = -1;
                        if (in_ext) {
                            const int qy = dt(yy), qx = dt(xx);
                            const BufDev& tb = pa.tm_trunc;
                            const float4* tp = reinterpret_cast<const float4*>(
                                tb.d + (size_t)slot_of(F, c.rows, c.cols, qy, qx) * t * t * C +
                                ((size_t)(yy - qy * t) * t + (xx - qx * t)) * C);
                            for (int q = lane & 15; q < C4; q += 16) {
                                const float4 tv = __ldcg(tp + q);
                                mt = fmaxf(fmaxf(fmaxf(mt, fabsf(tv.x)), fabsf(tv.y)), fmaxf(fabsf(tv.z), fabsf(tv.w)));
                            }
                            key = qy * F.tw + qx;
                        }
                        const unsigned grp = __match_any_sync(0xffffffffu, key);
                        const unsigned mx = __reduce_max_sync(grp, __float_as_uint(mt));
                        if (key >= 0 && mx != 0u && lane == __ffs(grp) - 1) atomicMax(pa.tile_max + key, mx);
                    }
                }
            }
        } else {
            for (int e = threadIdx.x; e < npx * C; e += NT) {
                const int p = e / C, q = e - p * C;
                const int ly = dbw(p), lx = p - ly * BW;
                if (s_ucnt[(ly / kUY) * upr + lx / kUX] >= tau || !s_tstore[dt(ly) * tpr + dt(lx)] ||
                    ((s_bits[p >> 5] >> (p & 31)) & 1u))
                    continue;
                const int y = Y0 + ly, x = X0 + lx;
                if (y < -hs || y >= eh + hs || x < -hs || x >= ew + hs) continue;
                out.d[pkt_off(out, y, x) + q] = 0.0f;
            }
        }
    }
}

