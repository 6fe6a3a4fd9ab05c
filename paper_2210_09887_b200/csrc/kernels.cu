// B200 (sm_100a) kernels of the sparse frame-difference path: input stage,
// claim reset / bias init, fused delta activation (truncation), sparse
// pooling, linear packet ops, conv target compaction, exact-order CUDA-core
// DeltaConv and the dense output. The tensor-core DeltaConv is conv_tc.cu.
//
// Bit-exactness: every arithmetic step that the reference performs in fp32 is
// done here with explicitly rounded intrinsics (__fadd_rn / __fmul_rn /
// __fdiv_rn, __dadd_rn / __dmul_rn) so nvcc cannot contract to FMA; the
// reference's x86-64 build has no FMA (SURVEY §7 hard part 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "kernels.hpp"
#include "pdl.hpp"

namespace dfx {

namespace {

#include "output.inc.cuh"

constexpr int kThreads = 256;

// TileLedger::holds (buffer_manager.hpp:41-44): placement tiles read the
// per-frame owned map (one byte, uploaded with the frame parameters); ring
// tiles outside the placement read the slot table.
__device__ __forceinline__ bool holds(const Ctx& c, const FrameDev& F, int qy, int qx) {
    if (qy >= 0 && qy < F.th && qx >= 0 && qx < F.tw) return c.own[qy * F.tw + qx] != 0;
    const SlotDev& s = c.slots[slot_of(F, c.rows, c.cols, qy, qx)];
    return s.used && s.ty == F.oty + qy && s.tx == F.otx + qx;
}

// Base pointer of the slot tile holding placement-relative tile (qy, qx).
__device__ __forceinline__ float* tile_ptr(const Ctx& c, const FrameDev& F, BufDev b, int qy, int qx) {
    return b.d + (size_t)slot_of(F, c.rows, c.cols, qy, qx) * b.t * b.t * b.C;
}

// Value of a wrapped buffer at extent-relative pixel (y, x) of layer tile t.
__device__ __forceinline__ float* buf_px(const Ctx& c, const FrameDev& F, BufDev b, int y, int x) {
    const int qy = floor_div32(y, b.t), qx = floor_div32(x, b.t);
    return tile_ptr(c, F, b, qy, qx) + ((size_t)(y - qy * b.t) * b.t + (x - qx * b.t)) * b.C;
}

// Packet sample with the reference's zero-fill semantics (delta_layers.hpp:37-41):
// zero beyond the grown extent and in tiles the packet never wrote.
__device__ __forceinline__ bool pkt_valid(const PktDev& p, int th, int tw, int y, int x) {
    if (y < -p.halo || y >= th * p.t + p.halo || x < -p.halo || x >= tw * p.t + p.halo) return false;
    const int i = floor_div32(y, p.t), j = floor_div32(x, p.t);
    return p.ext[ext_idx(p, i, j)] != 0;
}

__device__ __forceinline__ float block_max(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : 0.0f;
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

int grid_for(long long n, int per_block = kThreads) {
    long long g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > (1LL << 30)) g = 1LL << 30;
    return (int)g;
}

// ----------------------------------------------------------------- warp
// alignment.cpp:58-104, bilinear branch: inverse mapping in double, float
// weights. Source position of frame pixel (x, y); false if outside the frame.
struct WarpTap {
    int x0, y0, x1, y1;
    float fx, fy, gx, gy;
};
__device__ __forceinline__ bool warp_tap(const FrameDev& F, int x, int y, WarpTap& w4) {
    const int H = F.frame_h, W = F.frame_w;
    const double xd = x, yd = y;
    const double w = __dadd_rn(__dadd_rn(__dmul_rn((double)F.inv[6], xd), __dmul_rn((double)F.inv[7], yd)),
                               (double)F.inv[8]);
    const double sx = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)F.inv[0], xd), __dmul_rn((double)F.inv[1], yd)),
                                          (double)F.inv[2]), w);
    const double sy = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)F.inv[3], xd), __dmul_rn((double)F.inv[4], yd)),
                                          (double)F.inv[5]), w);
    if (sx < 0.0 || sx > W - 1 || sy < 0.0 || sy > H - 1) return false;
    w4.x0 = (int)floor(sx), w4.y0 = (int)floor(sy);
    w4.fx = (float)(sx - w4.x0), w4.fy = (float)(sy - w4.y0);
    w4.x1 = min(w4.x0 + 1, W - 1), w4.y1 = min(w4.y0 + 1, H - 1);
    w4.gx = __fsub_rn(1.0f, w4.fx), w4.gy = __fsub_rn(1.0f, w4.fy);
    return true;
}
__device__ __forceinline__ float warp_sample(const float* p, int W, const WarpTap& w4) {
    const float v00 = p[(size_t)w4.y0 * W + w4.x0], v01 = p[(size_t)w4.y0 * W + w4.x1];
    const float v10 = p[(size_t)w4.y1 * W + w4.x0], v11 = p[(size_t)w4.y1 * W + w4.x1];
    const float top = __fadd_rn(__fmul_rn(w4.gx, v00), __fmul_rn(w4.fx, v01));
    const float bot = __fadd_rn(__fmul_rn(w4.gx, v10), __fmul_rn(w4.fx, v11));
    return __fadd_rn(__fmul_rn(w4.gy, top), __fmul_rn(w4.fy, bot));
}
__global__ void k_warp(Ctx c, const float* __restrict__ frame, int C, float* __restrict__ warped,
                       uint8_t* __restrict__ fp) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int H = F.frame_h, W = F.frame_w;
    const long long n = (long long)H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / W), x = (int)(i % W);
        WarpTap w4;
        const bool ok = warp_tap(F, x, y, w4);
        fp[i] = ok ? 1 : 0;
        for (int ch = 0; ch < C; ++ch) warped[(size_t)ch * n + i] = ok ? warp_sample(frame + (size_t)ch * n, W, w4) : 0.0f;
    }
}

// Canvas (aligned frame, alignment.cpp:106-166) in HWC with a valid map.
// Warped pixel (cy + sy0, cx + sx0); integer path: warped = frame shifted by (idx, idy).
__global__ void k_align(Ctx c, const float* __restrict__ frame, const float* __restrict__ warped,
                        const uint8_t* __restrict__ fp, int C, float* __restrict__ aligned,
                        uint8_t* __restrict__ valid, int pitch, int T) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int ch_ = F.th * T, cw = F.tw * T;
    const long long n = (long long)ch_ * cw;
    const int H = F.frame_h, W = F.frame_w;
    const size_t plane = (size_t)H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int cy = (int)(i / cw), cx = (int)(i % cw);
        const int y = cy + F.sy0, x = cx + F.sx0;
        float* dst = aligned + ((size_t)cy * pitch + cx) * C;
        bool ok = y >= 0 && y < H && x >= 0 && x < W;
        if (ok && F.integer_path) {
            const int sy = y - F.idy, sx = x - F.idx;
            ok = sy >= 0 && sy < H && sx >= 0 && sx < W;
            if (ok)
                for (int ch = 0; ch < C; ++ch) dst[ch] = frame[(size_t)ch * plane + (size_t)sy * W + sx];
        } else if (ok) {
            ok = fp[(size_t)y * W + x] != 0;
            for (int ch = 0; ch < C; ++ch) dst[ch] = warped[(size_t)ch * plane + (size_t)y * W + x];
        }
        if (!ok && !(!F.integer_path && y >= 0 && y < H && x >= 0 && x < W))
            for (int ch = 0; ch < C; ++ch) dst[ch] = 0.0f;
        valid[(size_t)cy * pitch + cx] = ok ? 1 : 0;
    }
}

// Valid warped pixels that the crop dropped (alignment.cpp:131-164), bilinear path.
__global__ void k_count_dropped(Ctx c, const uint8_t* __restrict__ fp, int T, unsigned long long* counter) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int H = F.frame_h, W = F.frame_w;
    const long long n = (long long)H * W;
    unsigned long long local = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (!fp[i]) continue;
        const int y = (int)(i / W), x = (int)(i % W);
        const int cy = y - F.sy0, cx = x - F.sx0;
        if (cy < 0 || cy >= F.th * T || cx < 0 || cx >= F.tw * T) ++local;
    }
    if (local) atomicAdd(counter, local);
}

// roi_factor_map (alignment.cpp:228-239) via window_max (:198-224), rows pass.
__global__ void k_roi_rows(Ctx c, const float* __restrict__ roi, float* __restrict__ mid, int pitch, int T) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int eh = F.th * T, ew = F.tw * T;
    const long long n = (long long)eh * ew;
    const size_t plane = (size_t)pitch * c.rows * T;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / ew), x = (int)(i % ew);
        const int ks[3] = {10, 20, 40};
        for (int q = 0; q < 3; ++q) {
            const int lo = (ks[q] - 1) / 2, hi = ks[q] - 1 - lo;
            float m = 0.0f;
            for (int d = -lo; d <= hi; ++d) {
                const int xx = x + d;
                if (xx < 0 || xx >= ew) continue;
                m = fmaxf(m, roi[(size_t)y * pitch + xx]);
            }
            mid[q * plane + (size_t)y * pitch + x] = m;
        }
    }
}

__global__ void k_roi_cols(Ctx c, const float* __restrict__ mid, float* __restrict__ fac, int pitch, int T) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int eh = F.th * T, ew = F.tw * T;
    const long long n = (long long)eh * ew;
    const size_t plane = (size_t)pitch * c.rows * T;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / ew), x = (int)(i % ew);
        const int ks[3] = {10, 20, 40};
        float d[3];
        for (int q = 0; q < 3; ++q) {
            const int lo = (ks[q] - 1) / 2, hi = ks[q] - 1 - lo;
            float m = 0.0f;
            for (int dd = -lo; dd <= hi; ++dd) {
                const int yy = y + dd;
                if (yy < 0 || yy >= eh) continue;
                m = fmaxf(m, mid[q * plane + (size_t)yy * pitch + x]);
            }
            d[q] = m;
        }
        const float mean = __fdiv_rn(__fadd_rn(__fadd_rn(d[0], d[1]), d[2]), 3.0f);
        fac[(size_t)y * pitch + x] = __fadd_rn(0.4f, __fmul_rn(0.6f, mean));
    }
}

// Tile covered iff any valid pixel (alignment.cpp:179-183).
__global__ void k_coverage(Ctx c, const uint8_t* __restrict__ valid, int pitch, int T, uint8_t* __restrict__ cov) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int ti = blockIdx.x;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    int any = 0;
    for (int p = threadIdx.x; p < T * T && !any; p += blockDim.x) {
        const int y = tr * T + p / T, x = tc * T + p % T;
        if (valid[(size_t)y * pitch + x]) any = 1;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) cov[ti] = any ? 1 : 0;
}

// Per-pixel significance of cand = trunc + raw (engine.cpp:119-139).
__global__ void k_input_sig(Ctx c, const float* __restrict__ aligned, const uint8_t* __restrict__ cov, BufDev acc,
                            BufDev trunc, const float* __restrict__ fac, float thr, int pitch, int T,
                            uint8_t* __restrict__ sig) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int eh = F.th * T, ew = F.tw * T;
    const long long n = (long long)eh * ew;
    const int C = acc.C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / ew), x = (int)(i % ew);
        const int tr = y / T, tc = x / T;
        const bool covered = cov[tr * F.tw + tc] != 0;
        const size_t off = ((size_t)(y - tr * T) * T + (x - tc * T)) * C;
        const float* a = tile_ptr(c, F, acc, tr, tc) + off;
        const float* t = tile_ptr(c, F, trunc, tr, tc) + off;
        const float* al = aligned + ((size_t)y * pitch + x) * C;
        float m = 0.0f;
        for (int ch = 0; ch < C; ++ch) {
            const float raw = covered ? __fsub_rn(al[ch], a[ch]) : 0.0f;
            m = fmaxf(m, fabsf(__fadd_rn(t[ch], raw)));
        }
        if (fac) m = __fmul_rn(m, fac[(size_t)y * pitch + x]);
        sig[(size_t)y * pitch + x] = m > thr ? 1 : 0;
    }
}

// Supporter rule: keep iff >= 2 significant in the clipped 3x3 (engine.cpp:142-158).
__global__ void k_noise(Ctx c, const uint8_t* __restrict__ sig, uint8_t* __restrict__ out, int pitch, int T) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int eh = F.th * T, ew = F.tw * T;
    const long long n = (long long)eh * ew;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / ew), x = (int)(i % ew);
        uint8_t keep = 0;
        if (sig[(size_t)y * pitch + x]) {
            int sup = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= eh || xx < 0 || xx >= ew) continue;
                    sup += sig[(size_t)yy * pitch + xx] ? 1 : 0;
                }
            keep = sup >= 2;
        }
        out[(size_t)y * pitch + x] = keep;
    }
}

// Gate bit per tile (engine.cpp:160-180): covered and any significant pixel
// within the (2r+1) max-filter reach of the tile (== tile OR of the dilated
// map, window_max is a binary max filter), or fresh and covered.
__global__ void k_gate(Ctx c, const uint8_t* __restrict__ sig, const uint8_t* __restrict__ cov,
                       const uint8_t* __restrict__ fresh, int r, int pitch, int T, uint8_t* __restrict__ gate) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int ti = blockIdx.x;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    const int eh = F.th * T, ew = F.tw * T;
    if (!cov[ti]) {
        if (threadIdx.x == 0) gate[ti] = 0;
        return;
    }
    const int y0 = max(tr * T - r, 0), y1 = min((tr + 1) * T + r, eh);
    const int x0 = max(tc * T - r, 0), x1 = min((tc + 1) * T + r, ew);
    const int w = x1 - x0, n = (y1 - y0) * w;
    int any = fresh[ti] != 0;
    for (int p = threadIdx.x; p < n && !any; p += blockDim.x)
        if (sig[(size_t)(y0 + p / w) * pitch + x0 + p % w]) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) gate[ti] = any ? 1 : 0;
}

// Number of row-chunks a tile of t rows is split into so one block moves
// about kChunk floats (t rows of t*C floats each).
constexpr int kChunk = 8192;
__host__ __device__ inline int rows_per_chunk(int t, int C) {
    const int r = kChunk / (t * C);
    return r < 1 ? 1 : (r > t ? t : r);
}
__host__ __device__ inline int chunks_per_tile(int t, int C) {
    const int r = rows_per_chunk(t, C);
    return (t + r - 1) / r;
}

// Input truncation with the gate as fire (delta_layers.cpp:203-227 with
// raw = aligned - acc, alignment.cpp:183-188): fire -> acc += trunc + raw,
// trunc = 0, out = cand; else trunc += raw (the reference's double count).
__global__ void k_input_apply(Ctx c, const float* __restrict__ aligned, const uint8_t* __restrict__ cov,
                              const uint8_t* __restrict__ gate, BufDev acc, BufDev trunc, PktDev out, int pitch) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int T = acc.t, C = acc.C;
    const int nch = chunks_per_tile(T, C), rpc = rows_per_chunk(T, C);
    const int ti = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    const bool masked = cov[ti] && holds(c, F, tr, tc);
    const bool fire = masked && gate[ti];
    if (ch == 0 && threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = fire ? 1 : 0;
    if (!masked) return;
    float* a = tile_ptr(c, F, acc, tr, tc);
    float* t = tile_ptr(c, F, trunc, tr, tc);
    const int row_len = T * C;
    const int r0 = ch * rpc, r1 = min(T, r0 + rpc);
    if ((row_len & 3) == 0) {  // 16-B vectors along the tile row (rows are contiguous in all three arrays)
        const int rl4 = row_len / 4;
        for (int e = threadIdx.x; e < (r1 - r0) * rl4; e += blockDim.x) {
            const int yy = r0 + e / rl4, q = e - (e / rl4) * rl4;
            float4* a4 = reinterpret_cast<float4*>(a + (size_t)yy * row_len) + q;
            float4* t4 = reinterpret_cast<float4*>(t + (size_t)yy * row_len) + q;
            const float4 al = reinterpret_cast<const float4*>(aligned + ((size_t)(tr * T + yy) * pitch + tc * T) * C)[q];
            const float4 av = *a4, tv = *t4;
            const float4 raw = make_float4(__fsub_rn(al.x, av.x), __fsub_rn(al.y, av.y), __fsub_rn(al.z, av.z),
                                           __fsub_rn(al.w, av.w));
            const float4 cd = make_float4(__fadd_rn(tv.x, raw.x), __fadd_rn(tv.y, raw.y), __fadd_rn(tv.z, raw.z),
                                          __fadd_rn(tv.w, raw.w));
            if (fire) {
                *a4 = make_float4(__fadd_rn(av.x, cd.x), __fadd_rn(av.y, cd.y), __fadd_rn(av.z, cd.z),
                                  __fadd_rn(av.w, cd.w));
                *t4 = make_float4(0.f, 0.f, 0.f, 0.f);
                reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + yy, tc * T))[q] = cd;
            } else {
                *t4 = cd;
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < (r1 - r0) * row_len; e += blockDim.x) {
        const int yy = r0 + e / row_len, rem = e % row_len;
        const size_t bi = (size_t)yy * row_len + rem;
        const float al = aligned[((size_t)(tr * T + yy) * pitch + tc * T) * C + rem];
        const float av = a[bi], tv = t[bi];
        const float raw = __fsub_rn(al, av);
        if (fire) {
            const float cand = __fadd_rn(tv, raw);
            a[bi] = __fadd_rn(av, cand);
            t[bi] = 0.0f;
            out.d[pkt_off(out, tr * T + yy, tc * T) + rem] = cand;
        } else {
            t[bi] = __fadd_rn(tv, raw);
        }
    }
}

// ---- fused input stage (no ROI factor, no noise filter): two launches ----
// A: per canvas tile (grid-stride, one CTA per tile): aligned pixels
// (alignment.cpp:106-166, same arithmetic as k_align), coverage (:179-183) and
// per-pixel significance (engine.cpp:119-139) in one pass: each thread keeps
// its pixels' candidate maxima for both coverage outcomes and picks one once
// the tile's coverage is known.
__global__ void k_input_tile_a(Ctx c, const float* __restrict__ frame, const float* __restrict__ warped,
                               const uint8_t* __restrict__ fp, int C, float* __restrict__ aligned, int pitch, int T,
                               BufDev acc, BufDev trunc, float thr, uint8_t* __restrict__ cov,
                               uint8_t* __restrict__ sig, int direct) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int H = F.frame_h, W = F.frame_w;
    const size_t plane = (size_t)H * W;
    const int T2 = T * T;
    for (int ti = blockIdx.x; ti < F.th * F.tw; ti += gridDim.x) {
        const int tr = ti / F.tw, tc = ti - tr * F.tw;
        const float* ab = tile_ptr(c, F, acc, tr, tc);
        const float* tb = tile_ptr(c, F, trunc, tr, tc);
        int any = 0;
        uint32_t hit_c = 0, hit_u = 0;  // per pixel slot (<= 32 pixels per thread): significant if covered / not
        for (int p = threadIdx.x, slot = 0; p < T2; p += blockDim.x, ++slot) {
            const int py = p / T, px = p - py * T;
            const int cy = tr * T + py, cx = tc * T + px;
            const int y = cy + F.sy0, x = cx + F.sx0;
            float* dst = aligned + ((size_t)cy * pitch + cx) * C;
            const bool inf = y >= 0 && y < H && x >= 0 && x < W;
            bool ok = inf;
            float mc = 0.0f, mu = 0.0f;
            const float* a = ab + (size_t)p * C;
            const float* t = tb + (size_t)p * C;
            WarpTap w4;
            bool wok = false;
            if (direct && inf) wok = warp_tap(F, x, y, w4);  // bilinear sample straight from the frame
            int sy = 0, sx = 0;
            if (inf && F.integer_path) {
                sy = y - F.idy, sx = x - F.idx;
                ok = sy >= 0 && sy < H && sx >= 0 && sx < W;
            } else if (inf && direct) {
                ok = wok;
            } else if (inf) {
                ok = fp[(size_t)y * W + x] != 0;
            }
            // 4 channels at a time: every load of the group issued before any use
            for (int c0 = 0; c0 < C; c0 += 4) {
                float v[4], av[4], tv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ch = c0 + q;
                    v[q] = 0.0f, av[q] = 0.0f, tv[q] = 0.0f;
                    if (ch >= C) continue;
                    if (inf && F.integer_path) {
                        if (ok) v[q] = frame[(size_t)ch * plane + (size_t)sy * W + sx];
                    } else if (inf && direct) {
                        if (wok) v[q] = warp_sample(frame + (size_t)ch * plane, W, w4);
                    } else if (inf) {
                        v[q] = warped[(size_t)ch * plane + (size_t)y * W + x];
                    }
                    av[q] = a[ch];
                    tv[q] = t[ch];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (c0 + q >= C) continue;
                    dst[c0 + q] = v[q];
                    mc = fmaxf(mc, fabsf(__fadd_rn(tv[q], __fsub_rn(v[q], av[q]))));
                    mu = fmaxf(mu, fabsf(__fadd_rn(tv[q], 0.0f)));
                }
            }
            any |= ok ? 1 : 0;
            if (mc > thr) hit_c |= 1u << (slot & 31);
            if (mu > thr) hit_u |= 1u << (slot & 31);
        }
        const bool covered = __syncthreads_or(any) != 0;
        if (threadIdx.x == 0) cov[ti] = covered ? 1 : 0;
        const uint32_t hit = covered ? hit_c : hit_u;
        for (int p = threadIdx.x, slot = 0; p < T2; p += blockDim.x, ++slot) {
            const int py = p / T, px = p - py * T;
            sig[(size_t)(tr * T + py) * pitch + tc * T + px] = (hit >> (slot & 31)) & 1u;
        }
    }
}

// B: per tile: gate (engine.cpp:160-180, as k_gate) and the input
// truncation (as k_input_apply) in one launch.
__global__ void k_input_tile_b(Ctx c, const float* __restrict__ aligned, const uint8_t* __restrict__ cov,
                               const uint8_t* __restrict__ sig, const uint8_t* __restrict__ fresh, int r, int pitch,
                               BufDev acc, BufDev trunc, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int T = acc.t, C = acc.C;
    const int eh = F.th * T, ew = F.tw * T;
    for (int ti = blockIdx.x; ti < F.th * F.tw; ti += gridDim.x) {
        const int tr = ti / F.tw, tc = ti - tr * F.tw;
        const bool covered = cov[ti] != 0;
        int any = 0;
        if (covered) {
            any = fresh[ti] != 0;
            const int y0 = max(tr * T - r, 0), y1 = min((tr + 1) * T + r, eh);
            const int x0 = max(tc * T - r, 0), x1 = min((tc + 1) * T + r, ew);
            const int w = x1 - x0, n = (y1 - y0) * w;
            // up to 4 window bytes per thread per round, loaded together
            for (int p0 = threadIdx.x; p0 < n; p0 += 4 * blockDim.x) {
                uint8_t sv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int p = p0 + q * blockDim.x;
                    sv[q] = p < n ? sig[(size_t)(y0 + p / w) * pitch + x0 + p % w] : 0;
                }
                any |= (sv[0] | sv[1] | sv[2] | sv[3]) != 0;
            }
        }
        any = __syncthreads_or(any);
        const bool masked = covered && holds(c, F, tr, tc);
        const bool fire = masked && any;
        if (threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = fire ? 1 : 0;
        if (!masked) continue;
        float* a = tile_ptr(c, F, acc, tr, tc);
        float* t = tile_ptr(c, F, trunc, tr, tc);
        const int row_len = T * C;
        if ((row_len & 3) == 0) {
            const int rl4 = row_len / 4;
            for (int e = threadIdx.x; e < T * rl4; e += blockDim.x) {
                const int yy = e / rl4, q = e - yy * rl4;
                float4* a4 = reinterpret_cast<float4*>(a + (size_t)yy * row_len) + q;
                float4* t4 = reinterpret_cast<float4*>(t + (size_t)yy * row_len) + q;
                const float4 al = reinterpret_cast<const float4*>(aligned + ((size_t)(tr * T + yy) * pitch + tc * T) * C)[q];
                const float4 av = *a4, tv = *t4;
                const float4 raw = make_float4(__fsub_rn(al.x, av.x), __fsub_rn(al.y, av.y), __fsub_rn(al.z, av.z),
                                               __fsub_rn(al.w, av.w));
                const float4 cd = make_float4(__fadd_rn(tv.x, raw.x), __fadd_rn(tv.y, raw.y), __fadd_rn(tv.z, raw.z),
                                              __fadd_rn(tv.w, raw.w));
                if (fire) {
                    *a4 = make_float4(__fadd_rn(av.x, cd.x), __fadd_rn(av.y, cd.y), __fadd_rn(av.z, cd.z),
                                      __fadd_rn(av.w, cd.w));
                    *t4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + yy, tc * T))[q] = cd;
                } else {
                    *t4 = cd;
                }
            }
        } else {
            for (int e = threadIdx.x; e < T * row_len; e += blockDim.x) {
                const int yy = e / row_len, rem = e - yy * row_len;
                const size_t bi = (size_t)yy * row_len + rem;
                const float al = aligned[((size_t)(tr * T + yy) * pitch + tc * T) * C + rem];
                const float av = a[bi], tv = t[bi];
                const float raw = __fsub_rn(al, av);
                if (fire) {
                    const float cand = __fadd_rn(tv, raw);
                    a[bi] = __fadd_rn(av, cand);
                    t[bi] = 0.0f;
                    out.d[pkt_off(out, tr * T + yy, tc * T) + rem] = cand;
                } else {
                    t[bi] = __fadd_rn(tv, raw);
                }
            }
        }
        __syncthreads();
    }
}

// Claimed tiles of every buffer: zero, or the bias-init fill for truncated
// buffers (buffer_manager.cpp:68-89, engine.cpp:78-91; fill after zero == fill).
// Persistent grid-stride over (buffer, claim, element) with 16-byte stores.
// First kernel of every frame: the frame's parameter block is read straight
// from page-locked (mapped) host memory into its device slot, the frame's
// counters are zeroed, and the host is told the host block may be reused. No
// copy / memset node sits in the engine stream, so frames chain through
// programmatic dependent launch end to end. The parameter slot alternates per
// frame: the copy runs BEFORE the dependency wait, overlapping the previous
// frame's last kernel, which reads the other slot.
// Cross-stream handshake without stream events (which would cut the engine
// stream's programmatic-launch chain): a copy stream publishes "copy n done"
// with k_set_flag, the engine kernel that depends on it polls (bounded: traps
// after ~4 s instead of hanging the GPU).
__global__ void k_set_flag(unsigned* f, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__global__ void k_frame_begin(const uint4* __restrict__ src, uint4* __restrict__ dst, int n16,
                              uint4* __restrict__ counters, int cnt16, volatile unsigned* ack, unsigned seq,
                              const unsigned* in_flag, unsigned in_val, unsigned* done_ctr) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int i = tid; i < n16; i += nth) dst[i] = src[i];
    wait_flag(in_flag, in_val);  // host path: this frame's input copy has landed
    pdl_enter();
    for (int i = tid; i < cnt16; i += nth) counters[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        // per-engine counter (engines sharing a GPU run frame_begin concurrently)
        if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {  // every CTA has read its part of the host block
            *done_ctr = 0;
            *ack = seq;  // the host only needs to see it eventually (it spins); every read above has returned
        }
    }
}

// Frame-boundary trace (DFX_FRAME_TRACE=1, development only): [64 frames][4]
// globaltimer stamps: claims entry, claims past its dependency wait, densify end.
__device__ unsigned long long g_fstamp[64 * 4];
__device__ unsigned g_fseq;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void k_claims(Ctx c, const ClaimRec* __restrict__ recs, const int* __restrict__ plain_slots,
                         SlotDev* __restrict__ table, const ClaimBuf* __restrict__ bufs, int nbuf, int trace) {
    const unsigned long long t0 = trace ? gtimer() : 0;
    pdl_enter();
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned s = atomicAdd(&g_fseq, 1u) % 64;
        g_fstamp[s * 4 + 0] = t0;
        g_fstamp[s * 4 + 1] = gtimer();
    }
    const FrameDev& F = *c.f;
    const int nq = F.nclaims;
    if (nq == 0) return;
    // the claimed slots' new owners into the persistent slot table (TileLedger
    // apply_plan, buffer_manager.cpp:68-81): read by every later kernel of the frame
    if (table)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x)
            table[recs[i].slot] = SlotDev{recs[i].tx, recs[i].ty, 1, 0};
    // the buffer descriptors in shared memory first (one round of loads, not
    // one dependent global load per buffer in the loop below)
    constexpr int kMaxBufs = 128;
    __shared__ ClaimBuf s_bufs[kMaxBufs];
    for (int i = threadIdx.x; i < nbuf && i < kMaxBufs; i += blockDim.x) s_bufs[i] = bufs[i];
    __syncthreads();
    const long long tid0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, nthr = (long long)gridDim.x * blockDim.x;
    for (int bi = 0; bi < nbuf; ++bi) {
        const ClaimBuf b = bi < kMaxBufs ? s_bufs[bi] : bufs[bi];
        const long long n = (long long)b.t * b.t * b.C;  // floats per tile
        if ((b.C & 3) == 0 && (long long)nq * (n / 4) < (1LL << 31)) {
            // 32-bit indices; shifts when the tile's float4 count / channel count are powers of two
            const int n4 = (int)(n / 4), tot = nq * n4, c4 = b.C / 4;
            const bool p2 = (n4 & (n4 - 1)) == 0 && (c4 & (c4 - 1)) == 0;
            const int sh = p2 ? __ffs(n4) - 1 : 0;
            for (int e = (int)tid0; e < tot; e += (int)nthr) {
                const int ci = p2 ? (e >> sh) : e / n4, r = e - ci * n4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (b.fill) {
                    const int ch = 4 * (p2 ? (r & (c4 - 1)) : r % c4);
                    v = make_float4(b.fill[ch], b.fill[ch + 1], b.fill[ch + 2], b.fill[ch + 3]);
                }
                reinterpret_cast<float4*>(b.d + (size_t)(recs ? recs[ci].slot : plain_slots[ci]) * n)[r] = v;
            }
        } else if ((b.C & 3) == 0) {
            const long long n4 = n / 4;
            for (long long e = tid0; e < (long long)nq * n4; e += nthr) {
                const long long ci = e / n4, r = e - ci * n4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (b.fill) {
                    const int ch = (int)((r * 4) % b.C);
                    v = make_float4(b.fill[ch], b.fill[ch + 1], b.fill[ch + 2], b.fill[ch + 3]);
                }
                reinterpret_cast<float4*>(b.d + (size_t)(recs ? recs[ci].slot : plain_slots[ci]) * n)[r] = v;
            }
        } else {
            for (long long e = tid0; e < (long long)nq * n; e += nthr) {
                const long long ci = e / n, r = e - ci * n;
                b.d[(size_t)(recs ? recs[ci].slot : plain_slots[ci]) * n + r] = b.fill ? b.fill[r % b.C] : 0.0f;
            }
        }
    }
}

// Ring ("dilated border") pixels of a packet added into a wrapped buffer at
// owned slots (delta_layers.cpp:168-183 stash; :262-275 for maxpool acc).
__global__ void k_ring_add(Ctx c, PktDev in, BufDev dst) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int h = in.halo, t = in.t, C = in.C;
    const int eh = F.th * t, ew = F.tw * t;
    const int gw = ew + 2 * h;
    // strips: top h x gw, bottom h x gw, left eh x h, right eh x h
    const long long npx = 2LL * h * gw + 2LL * eh * h;
    const long long n = npx * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long p = i / C;
        const int ch = (int)(i % C);
        int y, x;
        if (p < (long long)h * gw) {
            y = -h + (int)(p / gw);
            x = -h + (int)(p % gw);
        } else if (p < 2LL * h * gw) {
            const long long q = p - (long long)h * gw;
            y = eh + (int)(q / gw);
            x = -h + (int)(q % gw);
        } else if (p < 2LL * h * gw + (long long)eh * h) {
            const long long q = p - 2LL * h * gw;
            y = (int)(q / h);
            x = -h + (int)(q % h);
        } else {
            const long long q = p - 2LL * h * gw - (long long)eh * h;
            y = (int)(q / h);
            x = ew + (int)(q % h);
        }
        const int qy = floor_div32(y, t), qx = floor_div32(x, t);
        if (!in.ext[ext_idx(in, qy, qx)]) continue;  // tile never written: zero
        if (!holds(c, F, qy, qx)) continue;
        float* b = buf_px(c, F, dst, y, x);
        b[ch] = __fadd_rn(b[ch], in.d[pkt_off(in, y, x) + ch]);
    }
}

// tile_max of |trunc + delta| over a masked owned tile (delta_layers.cpp:194-201).
__global__ void k_trunc_max(Ctx c, PktDev in, BufDev trunc, unsigned* __restrict__ tile_max) {
    pdl_enter();
    __shared__ float red[32];
    const FrameDev& F = *c.f;
    const int T = in.t, C = in.C;
    const int nch = chunks_per_tile(T, C), rpc = rows_per_chunk(T, C);
    const int ti = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    if (!in.ext[ext_idx(in, tr, tc)] || !holds(c, F, tr, tc)) return;
    const float* tb = tile_ptr(c, F, trunc, tr, tc);
    const int row_len = T * C;
    const int r0 = ch * rpc, r1 = min(T, r0 + rpc);
    float m = 0.0f;
    if ((C & 3) == 0) {
        const int rl4 = row_len / 4;
        for (int e = threadIdx.x; e < (r1 - r0) * rl4; e += blockDim.x) {
            const int yy = r0 + e / rl4, q = e % rl4;
            const float4 tv = reinterpret_cast<const float4*>(tb + (size_t)yy * row_len)[q];
            const float4 dv = reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * T + yy, tc * T))[q];
            m = fmaxf(m, fabsf(__fadd_rn(tv.x, dv.x)));
            m = fmaxf(m, fabsf(__fadd_rn(tv.y, dv.y)));
            m = fmaxf(m, fabsf(__fadd_rn(tv.z, dv.z)));
            m = fmaxf(m, fabsf(__fadd_rn(tv.w, dv.w)));
        }
    } else {
        for (int e = threadIdx.x; e < (r1 - r0) * row_len; e += blockDim.x) {
            const int yy = r0 + e / row_len, rem = e % row_len;
            m = fmaxf(m, fabsf(__fadd_rn(tb[(size_t)yy * row_len + rem], in.d[pkt_off(in, tr * T + yy, tc * T) + rem])));
        }
    }
    m = block_max(m, red);
    if (threadIdx.x == 0 && m > 0.0f) atomicMax(&tile_max[ti], __float_as_uint(m));
}

// Fire / fold per masked owned tile (delta_layers.cpp:203-228).
__global__ void k_trunc_apply(Ctx c, PktDev in, BufDev acc, BufDev trunc, const unsigned* __restrict__ tile_max,
                              float thr, int relu, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int T = in.t, C = in.C;
    const int nch = chunks_per_tile(T, C), rpc = rows_per_chunk(T, C);
    const int ti = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    const bool masked = in.ext[ext_idx(in, tr, tc)] && holds(c, F, tr, tc);
    const float tmax = __uint_as_float(tile_max[ti]);
    const bool fire = masked && tmax >= thr && tmax > 0.0f;
    if (ch == 0 && threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = fire ? 1 : 0;
    if (!masked) return;
    float* ab = tile_ptr(c, F, acc, tr, tc);
    float* tb = tile_ptr(c, F, trunc, tr, tc);
    const int row_len = T * C;
    const int r0 = ch * rpc, r1 = min(T, r0 + rpc);
    if ((C & 3) == 0) {
        const int rl4 = row_len / 4;
        for (int e = threadIdx.x; e < (r1 - r0) * rl4; e += blockDim.x) {
            const int yy = r0 + e / rl4, q = e % rl4;
            float4* t4 = reinterpret_cast<float4*>(tb + (size_t)yy * row_len) + q;
            const float4 dv = reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * T + yy, tc * T))[q];
            float4 tv = *t4;
            if (fire) {
                float4* a4 = reinterpret_cast<float4*>(ab + (size_t)yy * row_len) + q;
                const float4 pv = *a4;
                float4 cd, nv, o;
                cd.x = __fadd_rn(tv.x, dv.x); cd.y = __fadd_rn(tv.y, dv.y);
                cd.z = __fadd_rn(tv.z, dv.z); cd.w = __fadd_rn(tv.w, dv.w);
                nv.x = __fadd_rn(pv.x, cd.x); nv.y = __fadd_rn(pv.y, cd.y);
                nv.z = __fadd_rn(pv.z, cd.z); nv.w = __fadd_rn(pv.w, cd.w);
                if (relu) {
                    o.x = __fsub_rn(fmaxf(nv.x, 0.f), fmaxf(pv.x, 0.f));
                    o.y = __fsub_rn(fmaxf(nv.y, 0.f), fmaxf(pv.y, 0.f));
                    o.z = __fsub_rn(fmaxf(nv.z, 0.f), fmaxf(pv.z, 0.f));
                    o.w = __fsub_rn(fmaxf(nv.w, 0.f), fmaxf(pv.w, 0.f));
                } else {
                    o = cd;
                }
                *a4 = nv;
                *t4 = make_float4(0.f, 0.f, 0.f, 0.f);
                reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + yy, tc * T))[q] = o;
            } else {
                tv.x = __fadd_rn(tv.x, dv.x); tv.y = __fadd_rn(tv.y, dv.y);
                tv.z = __fadd_rn(tv.z, dv.z); tv.w = __fadd_rn(tv.w, dv.w);
                *t4 = tv;
            }
        }
    } else {
        for (int e = threadIdx.x; e < (r1 - r0) * row_len; e += blockDim.x) {
            const int yy = r0 + e / row_len, rem = e % row_len;
            const size_t bi = (size_t)yy * row_len + rem;
            const float dv = in.d[pkt_off(in, tr * T + yy, tc * T) + rem];
            const float tv = tb[bi];
            if (fire) {
                const float cand = __fadd_rn(tv, dv), prev = ab[bi], nv = __fadd_rn(prev, cand);
                ab[bi] = nv;
                tb[bi] = 0.0f;
                out.d[pkt_off(out, tr * T + yy, tc * T) + rem] =
                    relu ? __fsub_rn(fmaxf(nv, 0.f), fmaxf(prev, 0.f)) : cand;
            } else {
                tb[bi] = __fadd_rn(tv, dv);
            }
        }
    }
}

// Fused delta activation, one HBM pass per tile (delta_layers.cpp:185-228):
// a CTA (or a cluster of cs CTAs for large tiles) loads the tile's trunc and
// delta once into registers, reduces max|trunc + delta| (cross-CTA through
// DSMEM), then fires (acc += cand, trunc = 0, out = relu(acc') - relu(acc))
// or folds (trunc += delta) straight from registers. Requires C % 4 == 0 and
// t*t*C <= cs * kTruncThreads * 4 * kTruncVec.
constexpr int kTruncThreads = 512, kTruncVec = 8;
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(const float* local, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}

__global__ void __launch_bounds__(kTruncThreads, 1)
    k_trunc_fused(Ctx c, PktDev in, BufDev acc, BufDev trunc, float thr, int relu, PktDev out, int cs) {
    pdl_enter();
    __shared__ float red[32];
    __shared__ float s_blockmax;
    const FrameDev& F = *c.f;
    const int T = in.t, C = in.C;
    const int ti = blockIdx.x / cs;
    const uint32_t rank = cs > 1 ? cluster_rank() : 0;
    // uniform per cluster: every CTA of the cluster handles the same tile
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    const bool masked = in.ext[ext_idx(in, tr, tc)] && holds(c, F, tr, tc);
    if (!masked) {
        if (rank == 0 && threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = 0;
        return;
    }
    const int E4 = T * T * C / 4;              // float4s in the tile
    const int per = (E4 + cs - 1) / cs;         // float4s of this CTA
    const int q0 = rank * per, q1 = min(E4, q0 + per);
    const int row4 = T * C / 4;                 // float4s per tile row
    float4* tb = reinterpret_cast<float4*>(tile_ptr(c, F, trunc, tr, tc));
    float4 tv[kTruncVec], dv[kTruncVec];
    float m = 0.0f;
#pragma unroll
    for (int j = 0; j < kTruncVec; ++j) {
        const int q = q0 + threadIdx.x + j * kTruncThreads;
        if (q < q1) {
            const int yy = q / row4, rem = q - yy * row4;
            tv[j] = tb[q];
            dv[j] = reinterpret_cast<const float4*>(in.d + pkt_off(in, tr * T + yy, tc * T))[rem];
            m = fmaxf(m, fabsf(__fadd_rn(tv[j].x, dv[j].x)));
            m = fmaxf(m, fabsf(__fadd_rn(tv[j].y, dv[j].y)));
            m = fmaxf(m, fabsf(__fadd_rn(tv[j].z, dv[j].z)));
            m = fmaxf(m, fabsf(__fadd_rn(tv[j].w, dv[j].w)));
        }
    }
    m = block_max(m, red);
    if (cs > 1) {
        if (threadIdx.x == 0) s_blockmax = m;
        cluster_sync_all();
        float mm = 0.0f;
        for (int r = 0; r < cs; ++r) mm = fmaxf(mm, ld_dsmem_f32(&s_blockmax, r));
        m = mm;
        cluster_sync_all();  // remote reads done before any CTA of the cluster exits
    }
    const bool fire = m >= thr && m > 0.0f;
    if (rank == 0 && threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = fire ? 1 : 0;
    if (fire) {
        float4* ab = reinterpret_cast<float4*>(tile_ptr(c, F, acc, tr, tc));
#pragma unroll
        for (int j = 0; j < kTruncVec; ++j) {
            const int q = q0 + threadIdx.x + j * kTruncThreads;
            if (q < q1) {
                const int yy = q / row4, rem = q - yy * row4;
                const float4 pv = ab[q];
                float4 cd, nv, o;
                cd.x = __fadd_rn(tv[j].x, dv[j].x); cd.y = __fadd_rn(tv[j].y, dv[j].y);
                cd.z = __fadd_rn(tv[j].z, dv[j].z); cd.w = __fadd_rn(tv[j].w, dv[j].w);
                nv.x = __fadd_rn(pv.x, cd.x); nv.y = __fadd_rn(pv.y, cd.y);
                nv.z = __fadd_rn(pv.z, cd.z); nv.w = __fadd_rn(pv.w, cd.w);
                if (relu) {
                    o.x = __fsub_rn(fmaxf(nv.x, 0.f), fmaxf(pv.x, 0.f));
                    o.y = __fsub_rn(fmaxf(nv.y, 0.f), fmaxf(pv.y, 0.f));
                    o.z = __fsub_rn(fmaxf(nv.z, 0.f), fmaxf(pv.z, 0.f));
                    o.w = __fsub_rn(fmaxf(nv.w, 0.f), fmaxf(pv.w, 0.f));
                } else {
                    o = cd;
                }
                ab[q] = nv;
                tb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                reinterpret_cast<float4*>(out.d + pkt_off(out, tr * T + yy, tc * T))[rem] = o;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < kTruncVec; ++j) {
            const int q = q0 + threadIdx.x + j * kTruncThreads;
            if (q < q1) {
                float4 nt;
                nt.x = __fadd_rn(tv[j].x, dv[j].x); nt.y = __fadd_rn(tv[j].y, dv[j].y);
                nt.z = __fadd_rn(tv[j].z, dv[j].z); nt.w = __fadd_rn(tv[j].w, dv[j].w);
                tb[q] = nt;
            }
        }
    }
}

// acc += delta on masked owned tiles (delta_layers.cpp:253-261).
__global__ void k_tile_add(Ctx c, PktDev in, BufDev acc) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int T = in.t, C = in.C;
    const int nch = chunks_per_tile(T, C), rpc = rows_per_chunk(T, C);
    const int ti = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (ti >= F.th * F.tw) return;
    const int tr = ti / F.tw, tc = ti % F.tw;
    if (!in.ext[ext_idx(in, tr, tc)] || !holds(c, F, tr, tc)) return;
    float* ab = tile_ptr(c, F, acc, tr, tc);
    const int row_len = T * C;
    const int r0 = ch * rpc, r1 = min(T, r0 + rpc);
    for (int e = threadIdx.x; e < (r1 - r0) * row_len; e += blockDim.x) {
        const int yy = r0 + e / row_len, rem = e % row_len;
        const size_t bi = (size_t)yy * row_len + rem;
        ab[bi] = __fadd_rn(ab[bi], in.d[pkt_off(in, tr * T + yy, tc * T) + rem]);
    }
}

// Target test of a windowed op (delta_layers.cpp:34-70): output (oy, ox)
// whose window [o*s - back, o*s - back + span) meets a masked input tile
// grown by the input halo.
__device__ __forceinline__ bool is_target(const PktDev& in, int th, int tw, int oy, int ox, int span, int back,
                                          int s) {
    const int iy0 = oy * s - back - in.halo, iy1 = oy * s - back + span - 1 + in.halo;
    const int ix0 = ox * s - back - in.halo, ix1 = ox * s - back + span - 1 + in.halo;
    const int tr0 = max(floor_div32(iy0, in.t), 0), tr1 = min(floor_div32(iy1, in.t), th - 1);
    const int tc0 = max(floor_div32(ix0, in.t), 0), tc1 = min(floor_div32(ix1, in.t), tw - 1);
    for (int tr = tr0; tr <= tr1; ++tr)
        for (int tc = tc0; tc <= tc1; ++tc)
            if (in.ext[ext_idx(in, tr, tc)]) return true;
    return false;
}

// Block index -> extended output tile (i, j) in [-RT, th+RT) x [-RT, tw+RT).
__device__ __forceinline__ bool ext_tile(const FrameDev& F, const PktDev& out, int& i, int& j) {
    const int ew = F.tw + 2 * out.RT;
    const int b = blockIdx.x;
    if (b >= (F.th + 2 * out.RT) * ew) return false;
    i = b / ew - out.RT;
    j = b % ew - out.RT;
    return true;
}

// Pixel range of ext tile (i, j) clipped to the stored grown extent.
__device__ __forceinline__ void tile_px_range(const FrameDev& F, const PktDev& out, int i, int j, int& y0, int& y1,
                                              int& x0, int& x1) {
    const int t = out.t, h = out.halo;
    y0 = max(i * t, -h);
    y1 = min((i + 1) * t, F.th * t + h);
    x0 = max(j * t, -h);
    x1 = min((j + 1) * t, F.tw * t + h);
}

// Conv target compaction + output ext map + zero fill of non-targets.
// Iterates the GEOMETRIC grown extent (out_halo_geom) so FLOPs count ring
// targets even when the stored packet is cropped (padded_convolutions=false,
// engine.cpp:254-264). One block per extended output tile: the input-tile
// neighbourhood the tile's windows can reach is staged in shared memory, each
// pixel's target bit is computed once into a shared bitmap, the list is
// appended with one global atomic per warp (ballot + popc), and non-target
// pixels of active tiles are zeroed with 16-byte stores.
constexpr int kTgtMaxPx = 4096;  // t_out <= 64
__global__ void __launch_bounds__(256) k_conv_targets(Ctx c, PktDev in, int k, int s, int r, PktDev out, int hg,
                                                      int* __restrict__ list, int* __restrict__ count,
                                                      unsigned long long* __restrict__ flop_px,
                                                      const uint8_t* __restrict__ dense_map, int nux_max) {
    pdl_enter();
    __shared__ uint32_t s_bits[kTgtMaxPx / 32];
    __shared__ uint8_t s_nb[8][8];
    __shared__ int s_tr0, s_tc0;
    const FrameDev& F = *c.f;
    const int t = out.t;
    const int RTg = (hg + t - 1) / t;
    const int ew = F.tw + 2 * RTg;
    const int b = blockIdx.x;
    if (b >= (F.th + 2 * RTg) * ew) return;
    const int i = b / ew - RTg, j = b % ew - RTg;
    const int gy0 = max(i * t, -hg), gy1 = min((i + 1) * t, F.th * t + hg);
    const int gx0 = max(j * t, -hg), gx1 = min((j + 1) * t, F.tw * t + hg);
    const bool stored_tile = i >= -out.RT && i < F.th + out.RT && j >= -out.RT && j < F.tw + out.RT;
    // input tiles reachable from this output tile's windows
    const int ry0 = gy0 * s - r - in.halo, ry1 = (gy1 - 1) * s - r + k - 1 + in.halo;
    const int rx0 = gx0 * s - r - in.halo, rx1 = (gx1 - 1) * s - r + k - 1 + in.halo;
    const int tr0 = floor_div32(ry0, in.t), tr1 = floor_div32(ry1, in.t);
    const int tc0 = floor_div32(rx0, in.t), tc1 = floor_div32(rx1, in.t);
    const bool nb_ok = (tr1 - tr0) < 8 && (tc1 - tc0) < 8;
    if (threadIdx.x < 64) {
        const int a = threadIdx.x >> 3, bb = threadIdx.x & 7;
        const int tr = tr0 + a, tc = tc0 + bb;
        uint8_t v = 0;
        if (tr <= tr1 && tc <= tc1 && tr >= 0 && tr < F.th && tc >= 0 && tc < F.tw) v = in.ext[ext_idx(in, tr, tc)];
        s_nb[a][bb] = v;
    }
    if (threadIdx.x == 0) s_tr0 = tr0, s_tc0 = tc0;
    __syncthreads();
    const int w = gx1 - gx0, n = (gy1 - gy0) * w;
    int geo = 0, any_stored = 0;
    for (int p0 = 0; p0 < n; p0 += blockDim.x) {
        const int p = p0 + threadIdx.x;
        bool tgt = false;
        if (p < n) {
            const int oy = gy0 + p / w, ox = gx0 + p % w;
            if (nb_ok) {
                const int a0 = floor_div32(oy * s - r - in.halo, in.t) - s_tr0;
                const int a1 = floor_div32(oy * s - r + k - 1 + in.halo, in.t) - s_tr0;
                const int b0 = floor_div32(ox * s - r - in.halo, in.t) - s_tc0;
                const int b1 = floor_div32(ox * s - r + k - 1 + in.halo, in.t) - s_tc0;
                for (int a = a0; a <= a1 && !tgt; ++a)
                    for (int bb = b0; bb <= b1; ++bb)
                        if (s_nb[a][bb]) {
                            tgt = true;
                            break;
                        }
            } else {
                tgt = is_target(in, F.th, F.tw, oy, ox, k, r, s);
            }
            if (tgt) {
                ++geo;
                if (oy >= -out.halo && oy < F.th * t + out.halo && ox >= -out.halo && ox < F.tw * t + out.halo)
                    any_stored = 1;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, tgt);
        if ((threadIdx.x & 31) == 0 && p0 + (threadIdx.x & ~31) < kTgtMaxPx)
            s_bits[(p0 + (threadIdx.x & ~31)) >> 5] = m;
    }
    for (int o = 16; o > 0; o >>= 1) geo += __shfl_xor_sync(0xffffffffu, geo, o);
    if ((threadIdx.x & 31) == 0 && geo) atomicAdd(flop_px, (unsigned long long)geo);
    any_stored = __syncthreads_or(any_stored);
    if (stored_tile && threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = any_stored ? 1 : 0;
    if (!stored_tile || !any_stored) return;
    // stored pixel range of this tile
    const int y0 = max(i * t, -out.halo), y1 = min((i + 1) * t, F.th * t + out.halo);
    const int x0 = max(j * t, -out.halo), x1 = min((j + 1) * t, F.tw * t + out.halo);
    auto bit = [&](int oy, int ox) {
        const int p = (oy - gy0) * w + (ox - gx0);
        return (s_bits[p >> 5] >> (p & 31)) & 1u;
    };
    const int sw = x1 - x0, sn = (y1 - y0) * sw;
    // pixels of dense units are written whole by k_conv_dense
    const int exh = F.th * t, exw = F.tw * t;
    auto dense = [&](int oy, int ox) {
        return dense_map && oy >= 0 && oy < exh && ox >= 0 && ox < exw && dense_map[(oy >> 4) * nux_max + (ox >> 3)];
    };
    // list append: one atomic per warp
    for (int p0 = 0; p0 < sn; p0 += blockDim.x) {
        const int p = p0 + threadIdx.x;
        int oy = 0, ox = 0;
        bool tgt = false;
        if (p < sn) {
            oy = y0 + p / sw;
            ox = x0 + p % sw;
            tgt = bit(oy, ox) && !dense(oy, ox);
        }
        const unsigned m = __ballot_sync(0xffffffffu, tgt);
        int base = 0;
        if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(count, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (tgt) list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = ((oy + hg) << 16) | (ox + hg);
    }
    // zero fill non-targets
    const int C = out.C;
    if ((C & 3) == 0) {
        const int c4 = C >> 2;
        for (int e = threadIdx.x; e < sn * c4; e += blockDim.x) {
            const int p = e / c4, q = e - p * c4;
            const int oy = y0 + p / sw, ox = x0 + p % sw;
            if (!bit(oy, ox) && !dense(oy, ox))
                reinterpret_cast<float4*>(out.d + pkt_off(out, oy, ox))[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
        for (int e = threadIdx.x; e < sn * C; e += blockDim.x) {
            const int p = e / C, q = e - p * C;
            const int oy = y0 + p / sw, ox = x0 + p % sw;
            if (!bit(oy, ox) && !dense(oy, ox)) out.d[pkt_off(out, oy, ox) + q] = 0.0f;
        }
    }
}

// Max pool, halo-free input and k == stride (the engine's only pooling shape,
// network.cpp:164-166): every output pixel's window lies inside the input tile
// with the same tile coordinates, so fold (acc += delta, delta_layers.cpp:
// 253-261) and the window max / prev update (:277-317) fuse into ONE pass over
// each masked tile. Targets == all pixels of masked tiles; ownership of the
// input and output tile is the same slot.
__global__ void k_maxpool_fused(Ctx c, PktDev in, BufDev acc, BufDev prev, int k, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    const int to = out.t, ti_ = in.t, C = in.C;
    const int per_tile = to * to * C;
    const int chunk = 4096;
    const int nch = (per_tile + chunk - 1) / chunk;
    const int tix = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (tix >= F.th * F.tw) return;
    const int tr = tix / F.tw, tc = tix % F.tw;
    const bool masked = in.ext[ext_idx(in, tr, tc)] != 0;
    if (ch == 0 && threadIdx.x == 0) out.ext[ext_idx(out, tr, tc)] = masked ? 1 : 0;
    if (!masked) return;
    const bool owned = holds(c, F, tr, tc);
    const int e0 = ch * chunk, e1 = min(per_tile, e0 + chunk);
    float* ab = owned ? tile_ptr(c, F, acc, tr, tc) : nullptr;
    float* pb = owned ? tile_ptr(c, F, prev, tr, tc) : nullptr;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int px = e / C, chn = e - px * C;
        const int y = px / to, x = px - y * to;
        float* d = out.d + pkt_off(out, tr * to + y, tc * to + x) + chn;
        if (!owned) {
            *d = 0.0f;
            continue;
        }
        float m = 0.0f;
        bool first = true;
        for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
                const int iy = y * k + ky, ix = x * k + kx;
                const size_t ai = ((size_t)iy * ti_ + ix) * C + chn;
                const float v = __fadd_rn(ab[ai], in.d[pkt_off(in, tr * ti_ + iy, tc * ti_ + ix) + chn]);
                ab[ai] = v;
                m = first ? v : fmaxf(m, v);
                first = false;
            }
        float* pv = pb + ((size_t)y * to + x) * C + chn;
        *d = __fsub_rn(m, *pv);
        *pv = m;
    }
}

// Exact-order DeltaConv on CUDA cores: acc += sample * w in the reference's
// i -> ky -> kx order with separate fp32 rounding (delta_layers.cpp:121-134),
// hence bit-identical outputs. Work item = 32 target pixels x 64 couts.
constexpr int kXP = 32, kXO = 64;
__global__ void __launch_bounds__(256) k_conv_exact(Ctx c, PktDev in, const float* __restrict__ w, int cin, int cout,
                                                    int k, int s, int r, PktDev out, int hg, const int* __restrict__ list,
                                                    const int* __restrict__ count, int ci_chunk) {
    pdl_enter();
    extern __shared__ float smem[];
    __shared__ int s_y[kXP], s_x[kXP];
    const FrameDev& F = *c.f;
    const int K2 = k * k;
    float* s_in = smem;                          // [ci_chunk][K2][kXP]
    float* s_w = smem + ci_chunk * K2 * kXP;     // [kXO][ci_chunk*K2]
    const int n = *count;
    const int nob = (cout + kXO - 1) / kXO;
    const int items = ((n + kXP - 1) / kXP) * nob;
    const int p = threadIdx.x % kXP, og = threadIdx.x / kXP;  // og in [0, 8)
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int chunk = item / nob, o0 = (item % nob) * kXO;
        __syncthreads();
        if (threadIdx.x < kXP) {
            const int idx = chunk * kXP + threadIdx.x;
            if (idx < n) {
                const int v = list[idx];
                s_y[threadIdx.x] = (v >> 16) - hg;
                s_x[threadIdx.x] = (v & 0xffff) - hg;
            } else {
                s_y[threadIdx.x] = INT_MIN / 4;
                s_x[threadIdx.x] = INT_MIN / 4;
            }
        }
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int i0 = 0; i0 < cin; i0 += ci_chunk) {
            const int ci = min(ci_chunk, cin - i0);
            __syncthreads();
            for (int e = threadIdx.x; e < ci * K2 * kXP; e += blockDim.x) {
                const int pp = e % kXP, kk = (e / kXP) % K2, ii = e / (kXP * K2);
                const int iy = s_y[pp] * s - r + kk / k, ix = s_x[pp] * s - r + kk % k;
                float v = 0.0f;
                if (s_y[pp] > INT_MIN / 8 && pkt_valid(in, F.th, F.tw, iy, ix)) v = in.d[pkt_off(in, iy, ix) + i0 + ii];
                s_in[(ii * K2 + kk) * kXP + pp] = v;
            }
            for (int e = threadIdx.x; e < kXO * ci * K2; e += blockDim.x) {
                const int oo = e / (ci * K2), rem = e % (ci * K2);
                const int o = o0 + oo;
                s_w[oo * (ci_chunk * K2) + rem] = o < cout ? w[((size_t)o * cin + i0) * K2 + rem] : 0.0f;
            }
            __syncthreads();
            for (int ii = 0; ii < ci; ++ii)
                for (int kk = 0; kk < K2; ++kk) {
                    const float a = s_in[(ii * K2 + kk) * kXP + p];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        acc[q] = __fadd_rn(acc[q], __fmul_rn(a, s_w[(og + 8 * q) * (ci_chunk * K2) + ii * K2 + kk]));
                }
        }
        const int idx = chunk * kXP + p;
        if (idx < n) {
            float* d = out.d + pkt_off(out, s_y[p], s_x[p]);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int o = o0 + og + 8 * q;
                if (o < cout) d[o] = acc[q];
            }
        }
    }
}

// Max pool output (delta_layers.cpp:277-317): m over the k x k window of the
// accumulated input (first-element init, non-owned tiles read 0), out = m - prev,
// prev = m, on owned target outputs.
__global__ void k_maxpool_out(Ctx c, PktDev in, BufDev acc, BufDev prev, int k, int s, PktDev out, int hg) {
    pdl_enter();
    const FrameDev& F = *c.f;
    int i, j;
    if (!ext_tile(F, out, i, j)) return;
    int y0, y1, x0, x1;
    tile_px_range(F, out, i, j, y0, y1, x0, x1);
    const int w = x1 - x0, n = (y1 - y0) * w;
    int any = 0;
    for (int p = threadIdx.x; p < n && !any; p += blockDim.x)
        if (is_target(in, F.th, F.tw, y0 + p / w, x0 + p % w, k, 0, s)) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = any ? 1 : 0;
    if (!any) return;
    const int C = out.C;
    const bool out_owned = holds(c, F, i, j);
    for (long long e = threadIdx.x; e < (long long)n * C; e += blockDim.x) {
        const int pp = (int)(e / C), ch = (int)(e % C);
        const int oy = y0 + pp / w, ox = x0 + pp % w;
        float* d = out.d + pkt_off(out, oy, ox) + ch;
        if (!out_owned || !is_target(in, F.th, F.tw, oy, ox, k, 0, s)) {
            *d = 0.0f;
            continue;
        }
        float m = 0.0f;
        bool first = true;
        for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
                const int iy = oy * s + ky, ix = ox * s + kx;
                const int qy = floor_div32(iy, in.t), qx = floor_div32(ix, in.t);
                const float v = holds(c, F, qy, qx) ? buf_px(c, F, acc, iy, ix)[ch] : 0.0f;
                m = first ? v : fmaxf(m, v);
                first = false;
            }
        float* pv = buf_px(c, F, prev, oy, ox) + ch;
        *d = __fsub_rn(m, *pv);
        *pv = m;
    }
}

// Average pool (delta_layers.cpp:320-349): sum in (ky, kx) order times 1/k^2.
__global__ void k_avgpool(Ctx c, PktDev in, int k, int s, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    int i, j;
    if (!ext_tile(F, out, i, j)) return;
    int y0, y1, x0, x1;
    tile_px_range(F, out, i, j, y0, y1, x0, x1);
    const int w = x1 - x0, n = (y1 - y0) * w;
    int any = 0;
    for (int p = threadIdx.x; p < n && !any; p += blockDim.x)
        if (is_target(in, F.th, F.tw, y0 + p / w, x0 + p % w, k, 0, s)) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = any ? 1 : 0;
    if (!any) return;
    const int C = out.C;
    const float inv = __fdiv_rn(1.0f, (float)(k * k));
    for (long long e = threadIdx.x; e < (long long)n * C; e += blockDim.x) {
        const int pp = (int)(e / C), ch = (int)(e % C);
        const int oy = y0 + pp / w, ox = x0 + pp % w;
        float v = 0.0f;
        if (is_target(in, F.th, F.tw, oy, ox, k, 0, s)) {
            float sum = 0.0f;
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    const int iy = oy * s + ky, ix = ox * s + kx;
                    if (pkt_valid(in, F.th, F.tw, iy, ix)) sum = __fadd_rn(sum, in.d[pkt_off(in, iy, ix) + ch]);
                    else sum = __fadd_rn(sum, 0.0f);
                }
            v = __fmul_rn(sum, inv);
        }
        out.d[pkt_off(out, oy, ox) + ch] = v;
    }
}

// Nearest upsample (delta_layers.cpp:351-363).
__global__ void k_upsample(Ctx c, PktDev in, int f, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    int i, j;
    if (!ext_tile(F, out, i, j)) return;
    const bool v = in.ext[ext_idx(in, i, j)] != 0;
    if (threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = v ? 1 : 0;
    if (!v) return;
    int y0, y1, x0, x1;
    tile_px_range(F, out, i, j, y0, y1, x0, x1);
    const int w = x1 - x0, n = (y1 - y0) * w, C = out.C;
    if ((C & 3) == 0) {  // float4 columns, 32-bit index math
        const int C4 = C / 4;
        for (int e = threadIdx.x; e < n * C4; e += blockDim.x) {
            const int pp = e / C4, c4 = e - pp * C4;
            const int oy = y0 + pp / w, ox = x0 + pp % w;
            reinterpret_cast<float4*>(out.d + pkt_off(out, oy, ox))[c4] =
                reinterpret_cast<const float4*>(in.d + pkt_off(in, floor_div32(oy, f), floor_div32(ox, f)))[c4];
        }
        return;
    }
    for (long long e = threadIdx.x; e < (long long)n * C; e += blockDim.x) {
        const int pp = (int)(e / C), ch = (int)(e % C);
        const int oy = y0 + pp / w, ox = x0 + pp % w;
        out.d[pkt_off(out, oy, ox) + ch] = in.d[pkt_off(in, floor_div32(oy, f), floor_div32(ox, f)) + ch];
    }
}

// BatchNorm scale (delta_layers.cpp:365-376).
__global__ void k_bn(Ctx c, PktDev in, const float* __restrict__ scale, PktDev out) {
    pdl_enter();
    const FrameDev& F = *c.f;
    int i, j;
    if (!ext_tile(F, out, i, j)) return;
    const bool v = in.ext[ext_idx(in, i, j)] != 0;
    if (threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = v ? 1 : 0;
    if (!v) return;
    int y0, y1, x0, x1;
    tile_px_range(F, out, i, j, y0, y1, x0, x1);
    const int w = x1 - x0, n = (y1 - y0) * w, C = out.C;
    for (long long e = threadIdx.x; e < (long long)n * C; e += blockDim.x) {
        const int pp = (int)(e / C), ch = (int)(e % C);
        const int oy = y0 + pp / w, ox = x0 + pp % w;
        out.d[pkt_off(out, oy, ox) + ch] = __fmul_rn(in.d[pkt_off(in, oy, ox) + ch], scale[ch]);
    }
}

__device__ __forceinline__ bool ext_in_range(const FrameDev& F, const PktDev& p, int i, int j) {
    return i >= -p.RT && i < F.th + p.RT && j >= -p.RT && j < F.tw + p.RT;
}

// Add: zero-extended sum, mask OR (delta_layers.cpp:378-393).
// fb > 1: b is the INPUT of a nearest upsample by fb whose only consumer is
// this add (delta_layers.cpp:351-363 folded in): the upsampled packet (halo and
// tile x fb, the same tile indices and ext) is sampled on the fly.
__global__ void k_add(Ctx c, PktDev a, PktDev b, PktDev out, int fb) {
    pdl_enter();
    const FrameDev& F = *c.f;
    int i, j;
    if (!ext_tile(F, out, i, j)) return;
    const bool va = ext_in_range(F, a, i, j) && a.ext[ext_idx(a, i, j)];
    const bool vb = ext_in_range(F, b, i, j) && b.ext[ext_idx(b, i, j)];
    if (threadIdx.x == 0) out.ext[ext_idx(out, i, j)] = (va || vb) ? 1 : 0;
    if (!va && !vb) return;
    int y0, y1, x0, x1;
    tile_px_range(F, out, i, j, y0, y1, x0, x1);
    const int w = x1 - x0, n = (y1 - y0) * w, C = out.C;
    if ((C & 3) == 0) {  // float4 columns, 32-bit index math; validity per pixel
        const int C4 = C / 4;
        for (int e = threadIdx.x; e < n * C4; e += blockDim.x) {
            const int pp = e / C4, c4 = e - pp * C4;
            const int oy = y0 + pp / w, ox = x0 + pp % w;
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 sa = (va && pkt_valid(a, F.th, F.tw, oy, ox))
                                  ? reinterpret_cast<const float4*>(a.d + pkt_off(a, oy, ox))[c4] : z;
            float4 sb = z;
            if (fb == 1) {
                if (vb && pkt_valid(b, F.th, F.tw, oy, ox)) sb = reinterpret_cast<const float4*>(b.d + pkt_off(b, oy, ox))[c4];
            } else {
                const int hup = b.halo * fb, tup = b.t * fb;
                if (vb && oy >= -hup && oy < F.th * tup + hup && ox >= -hup && ox < F.tw * tup + hup &&
                    b.ext[ext_idx(b, floor_div32(oy, tup), floor_div32(ox, tup))])
                    sb = reinterpret_cast<const float4*>(b.d + pkt_off(b, floor_div32(oy, fb), floor_div32(ox, fb)))[c4];
            }
            reinterpret_cast<float4*>(out.d + pkt_off(out, oy, ox))[c4] =
                make_float4(__fadd_rn(sa.x, sb.x), __fadd_rn(sa.y, sb.y), __fadd_rn(sa.z, sb.z), __fadd_rn(sa.w, sb.w));
        }
        return;
    }
    for (long long e = threadIdx.x; e < (long long)n * C; e += blockDim.x) {
        const int pp = (int)(e / C), ch = (int)(e % C);
        const int oy = y0 + pp / w, ox = x0 + pp % w;
        const float sa = (va && pkt_valid(a, F.th, F.tw, oy, ox)) ? a.d[pkt_off(a, oy, ox) + ch] : 0.0f;
        const float sb = (vb && pkt_valid(b, F.th, F.tw, oy, ox)) ? b.d[pkt_off(b, oy, ox) + ch] : 0.0f;
        out.d[pkt_off(out, oy, ox) + ch] = __fadd_rn(sa, sb);
    }
}

// Output = acc + trunc over the placement, CHW (delta_layers.cpp:395-400).
// C % 8 == 0: a warp takes (8-channel group, output row); each lane one pixel:
// 2 x 16-B reads of acc and trunc, 8 plane writes coalesced across the warp.
__global__ void k_densify8(Ctx c, BufDev acc, BufDev trunc, float* __restrict__ out, int trace, Readback rb) {
    pdl_enter();
    wait_flag(rb.out_flag, rb.out_val);  // host path: the output slot's previous copy-out is done
    frame_readback(rb);
    densify8_body(c, acc, trunc, out, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
    if (trace) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned s = (atomicAdd(&g_fseq, 0u) + 63) % 64;
            atomicMax(&g_fstamp[s * 4 + 2], gtimer());
        }
    }
}

__global__ void k_densify(Ctx c, BufDev acc, BufDev trunc, float* __restrict__ out, Readback rb) {
    pdl_enter();
    wait_flag(rb.out_flag, rb.out_val);
    frame_readback(rb);
    const FrameDev& F = *c.f;
    const int t = acc.t, C = acc.C;
    const int oh = F.th * t, ow = F.tw * t;
    const long long n = (long long)C * oh * ow;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % ow);
        const int y = (int)((i / ow) % oh);
        const int ch = (int)(i / ((long long)ow * oh));
        const int qy = y / t, qx = x / t;
        const size_t off = (size_t)slot_of(F, c.rows, c.cols, qy, qx) * t * t * C +
                           ((size_t)(y - qy * t) * t + (x - qx * t)) * C + ch;
        out[i] = __fadd_rn(acc.d[off], trunc.d[off]);
    }
}

}  // namespace

// ------------------------------------------------------------- launchers
static int num_sms_cached() { return device_sm_count(); }
static int persistent_grid(long long work) {
    const long long cap = (long long)num_sms_cached() * 8;
    long long g = (work + kThreads - 1) / kThreads;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

unsigned long long* frame_trace_host() {
    static unsigned long long h[64 * 4];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_fstamp, sizeof h);
    return h;
}
void launch_warp(const Ctx& c, cudaStream_t s, const float* frame, int C, float* warped, uint8_t* fp) {
    // frame dims are per-frame but bounded by the staging buffer; use a persistent grid
    launch_pdl(k_warp, num_sms_cached() * 8, kThreads, 0, s, c, frame, C, warped, fp);
}
void launch_align(const Ctx& c, cudaStream_t s, const float* frame, const float* warped, const uint8_t* fp, int C,
                  float* aligned, uint8_t* valid, int pitch, int T) {
    launch_pdl(k_align, persistent_grid((long long)c.rows * T * pitch), kThreads, 0, s, c, frame, warped, fp, C, aligned,
                                                                               valid, pitch, T);
}
void launch_input_tile_a(const Ctx& c, cudaStream_t s, const float* frame, const float* warped, const uint8_t* fp,
                         int C, float* aligned, int pitch, int T, BufDev acc, BufDev trunc, float thr, uint8_t* cov,
                         uint8_t* sig, int direct) {
    // one CTA per canvas tile at most (the placement has <= rows x cols tiles)
    const int g = std::min(num_sms_cached() * 8, c.rows * c.cols);
    launch_pdl(k_input_tile_a, g, kThreads, 0, s, c, frame, warped, fp, C, aligned, pitch, T, acc, trunc, thr, cov, sig,
               direct);
}
void launch_input_tile_b(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov, const uint8_t* sig,
                         const uint8_t* fresh, int dilation, int pitch, BufDev acc, BufDev trunc, PktDev out) {
    const int g = std::min(num_sms_cached() * 8, c.rows * c.cols);
    launch_pdl(k_input_tile_b, g, kThreads, 0, s, c, aligned, cov, sig, fresh, dilation, pitch, acc, trunc, out);
}
void launch_count_dropped(const Ctx& c, cudaStream_t s, const uint8_t* fp, int T, unsigned long long* counter) {
    launch_pdl(k_count_dropped, num_sms_cached() * 4, kThreads, 0, s, c, fp, T, counter);
}
void launch_roi_factor(const Ctx& c, cudaStream_t s, const float* roi, float* tmp3, float* fac, int pitch, int T) {
    const long long n = (long long)c.rows * T * pitch;
    launch_pdl(k_roi_rows, persistent_grid(n), kThreads, 0, s, c, roi, tmp3, pitch, T);
    launch_pdl(k_roi_cols, persistent_grid(n), kThreads, 0, s, c, tmp3, fac, pitch, T);
}
void launch_coverage(const Ctx& c, cudaStream_t s, const uint8_t* valid, int pitch, int T, uint8_t* cov) {
    launch_pdl(k_coverage, c.rows * c.cols, kThreads, 0, s, c, valid, pitch, T, cov);
}
void launch_input_sig(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov, BufDev acc,
                      BufDev trunc, const float* fac, float thr, int pitch, int T, uint8_t* sig) {
    launch_pdl(k_input_sig, persistent_grid((long long)c.rows * T * pitch), kThreads, 0, s, c, aligned, cov, acc, trunc, fac,
                                                                                   thr, pitch, T, sig);
}
void launch_noise(const Ctx& c, cudaStream_t s, const uint8_t* sig, uint8_t* out, int pitch, int T) {
    launch_pdl(k_noise, persistent_grid((long long)c.rows * T * pitch), kThreads, 0, s, c, sig, out, pitch, T);
}
void launch_gate(const Ctx& c, cudaStream_t s, const uint8_t* sig, const uint8_t* cov, const uint8_t* fresh,
                 int dilation, int pitch, int T, uint8_t* gate) {
    launch_pdl(k_gate, c.rows * c.cols, kThreads, 0, s, c, sig, cov, fresh, dilation, pitch, T, gate);
}
void launch_input_apply(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov, const uint8_t* gate,
                        BufDev acc, BufDev trunc, PktDev out, int pitch) {
    const int nch = chunks_per_tile(acc.t, acc.C);
    launch_pdl(k_input_apply, c.rows * c.cols * nch, kThreads, 0, s, c, aligned, cov, gate, acc, trunc, out, pitch);
}
void launch_claims(const Ctx& c, cudaStream_t s, const ClaimRec* recs, const int* plain_slots, SlotDev* table,
                   const ClaimBuf* bufs, int nbuf, int max_claims) {
    if (nbuf <= 0 || max_claims <= 0) return;
    static const int trace = getenv("DFX_FRAME_TRACE") ? 1 : 0;
    launch_pdl(k_claims, num_sms_cached() * 8, kThreads, 0, s, c, recs, plain_slots, table, bufs, nbuf, trace);
}
void launch_ring_add(const Ctx& c, cudaStream_t s, PktDev in, BufDev dst) {
    if (in.halo <= 0) return;
    const long long n = (2LL * in.halo * (c.cols * in.t + 2 * in.halo) + 2LL * c.rows * in.t * in.halo) * in.C;
    launch_pdl(k_ring_add, persistent_grid(n), kThreads, 0, s, c, in, dst);
}
void launch_trunc_max(const Ctx& c, cudaStream_t s, PktDev in, BufDev trunc, unsigned* tile_max) {
    const int nch = chunks_per_tile(in.t, in.C);
    launch_pdl(k_trunc_max, c.rows * c.cols * nch, kThreads, 0, s, c, in, trunc, tile_max);
}
void launch_trunc_apply(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc, const unsigned* tile_max,
                        float thr, int relu, PktDev out) {
    const int nch = chunks_per_tile(in.t, in.C);
    launch_pdl(k_trunc_apply, c.rows * c.cols * nch, kThreads, 0, s, c, in, acc, trunc, tile_max, thr, relu, out);
}
bool launch_trunc_fused(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc, float thr, int relu,
                        PktDev out) {
    const long long E4 = (long long)in.t * in.t * in.C / 4;
    if ((in.C & 3) != 0) return false;
    const long long per_cta = (long long)kTruncThreads * kTruncVec;
    int cs = 1;
    while (cs * per_cta < E4) cs <<= 1;
    if (cs > 8) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.rows * c.cols * cs);
    cfg.blockDim = dim3(kTruncThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cs > 1 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_trunc_fused, c, in, acc, trunc, thr, relu, out, cs) == cudaSuccess;
}
void launch_tile_add(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc) {
    const int nch = chunks_per_tile(in.t, in.C);
    launch_pdl(k_tile_add, c.rows * c.cols * nch, kThreads, 0, s, c, in, acc);
}
static int ext_blocks(const Ctx& c, const PktDev& out) { return (c.rows + 2 * out.RT) * (c.cols + 2 * out.RT); }
void launch_maxpool_out(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, int st, PktDev out,
                        int hg) {
    launch_pdl(k_maxpool_out, ext_blocks(c, out), kThreads, 0, s, c, in, acc, prev, k, st, out, hg);
}
void launch_maxpool_fused(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, PktDev out) {
    const int nch = (out.t * out.t * in.C + 4095) / 4096;
    launch_pdl(k_maxpool_fused, c.rows * c.cols * nch, kThreads, 0, s, c, in, acc, prev, k, out);
}
void launch_avgpool(const Ctx& c, cudaStream_t s, PktDev in, int k, int st, PktDev out) {
    launch_pdl(k_avgpool, ext_blocks(c, out), kThreads, 0, s, c, in, k, st, out);
}
void launch_upsample(const Ctx& c, cudaStream_t s, PktDev in, int f, PktDev out) {
    launch_pdl(k_upsample, ext_blocks(c, out), kThreads, 0, s, c, in, f, out);
}
void launch_bn(const Ctx& c, cudaStream_t s, PktDev in, const float* scale, PktDev out) {
    launch_pdl(k_bn, ext_blocks(c, out), kThreads, 0, s, c, in, scale, out);
}
void launch_add(const Ctx& c, cudaStream_t s, PktDev a, PktDev b, PktDev out, int fb) {
    if (fb > 1 && (out.C & 3) != 0) throw std::runtime_error("add: upsample fusion needs C % 4 == 0");
    launch_pdl(k_add, ext_blocks(c, out), kThreads, 0, s, c, a, b, out, fb);
}
void launch_conv_targets(const Ctx& c, cudaStream_t s, PktDev in, int k, int st, int r, PktDev out, int hg, int* list,
                         int* count, unsigned long long* flop_px, const uint8_t* dense_map, int nux_max) {
    const int RTg = (hg + out.t - 1) / out.t;
    launch_pdl(k_conv_targets, (c.rows + 2 * RTg) * (c.cols + 2 * RTg), kThreads, 0, s, c, in, k, st, r, out, hg, list, count,
                                                                                flop_px, dense_map, nux_max);
}
void launch_conv_exact(const Ctx& c, cudaStream_t s, PktDev in, const float* w, int cin, int cout, int k, int st, int r,
                       PktDev out, int hg, const int* list, const int* count, int max_targets) {
    const int K2 = k * k;
    int ci = 40960 / (4 * K2 * (kXP + kXO));
    if (ci < 1) ci = 1;
    if (ci > cin) ci = cin;
    const size_t smem = (size_t)ci * K2 * (kXP + kXO) * sizeof(float);
    const long long items = ((long long)(max_targets + kXP - 1) / kXP) * ((cout + kXO - 1) / kXO);
    long long g = num_sms_cached() * 4;
    if (items < g) g = items;
    if (g < 1) g = 1;
    launch_pdl(k_conv_exact, (int)g, 256, smem, s, c, in, w, cin, cout, k, st, r, out, hg, list, count, ci);
}
void launch_densify(const Ctx& c, cudaStream_t s, BufDev acc, BufDev trunc, float* out, Readback rb) {
    if ((acc.C & 7) == 0) {
        static const int trace = getenv("DFX_FRAME_TRACE") ? 1 : 0;
        // one warp per (8-channel group, output row): at most (C / 8) x rows x t warps
        const long long warps = (long long)(acc.C / 8) * c.rows * acc.t;
        const int g = (int)std::min<long long>(num_sms_cached() * 8, std::max<long long>(1, (warps + 7) / 8));
        launch_pdl(k_densify8, g, kThreads, 0, s, c, acc, trunc, out, trace, rb);
        return;
    }
    launch_pdl(k_densify, persistent_grid((long long)acc.C * c.rows * acc.t * c.cols * acc.t), kThreads, 0, s, c, acc, trunc,
               out, rb);
}
void launch_frame_begin(cudaStream_t s, const void* src, void* dst, size_t bytes, void* counters, size_t cnt_bytes,
                        unsigned* ack, unsigned seq, const unsigned* in_flag, unsigned in_val, unsigned* done_ctr) {
    launch_pdl(k_frame_begin, 32, kThreads, 0, s, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst),
               (int)(bytes / 16), reinterpret_cast<uint4*>(counters), (int)(cnt_bytes / 16), (volatile unsigned*)ack,
               seq, in_flag, in_val, done_ctr);
}
// The flag write is a stream memory operation (cuStreamWriteValue32, executed
// by the stream front end after the stream's prior work, with a memory barrier):
// it needs no SM, so a kernel polling the flag can never starve it of one (with
// several engines on a GPU a flag *kernel* could wait behind polling CTAs).
// Falls back to a one-thread kernel if the driver entry point is unavailable.
void launch_set_flag(cudaStream_t s, unsigned* f, unsigned v) {
    typedef int (*WriteValue32)(cudaStream_t, unsigned long long, unsigned, unsigned);
    static WriteValue32 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        cudaGetLastError();
        return reinterpret_cast<WriteValue32>(p);
    }();
    if (fn && fn(s, (unsigned long long)(uintptr_t)f, v, 0) == 0) return;
    k_set_flag<<<1, 1, 0, s>>>(f, v);
}

DFX_KTRACE_SETTER(ktrace_set_kernels)

}  // namespace dfx
