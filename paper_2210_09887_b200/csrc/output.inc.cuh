// Output-side helpers shared by k_densify8 (kernels.cu) and the output
// layer's cooperative activation, which densifies after a grid barrier
// (kernels_hbm.cu). Textually included INSIDE the translation unit's anonymous
// namespace; the includer provides kernels.hpp / dfx_types.hpp.
#pragma once

__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned v) {
    if (!f) return;
    if (threadIdx.x == 0) {
        unsigned x;
        for (long long it = 0;; ++it) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
            if ((int)(x - v) >= 0) break;
            if (it > (1LL << 24)) __trap();
            __nanosleep(256);
        }
    }
    __syncthreads();
}

// The frame's small readback (per-layer counts, dropped pixels, fired input
// tiles) written by CTA 0 of the last kernel straight into mapped host memory.
// 16-B writes when both parts are 16-B multiples (the engine pads them): every
// PCIe write is a separate transaction, byte stores cost one each.
__device__ __forceinline__ void frame_readback(const Readback& rb) {
    if (blockIdx.x != 0 || !rb.dst) return;
    if (((rb.n1 | rb.n2) & 15) == 0) {
        uint4* d = reinterpret_cast<uint4*>(rb.dst);
        const uint4* s1 = reinterpret_cast<const uint4*>(rb.src1);
        const uint4* s2 = reinterpret_cast<const uint4*>(rb.src2);
        for (int i = threadIdx.x; i < rb.n1 / 16; i += blockDim.x) d[i] = s1[i];
        for (int i = threadIdx.x; i < rb.n2 / 16; i += blockDim.x) d[rb.n1 / 16 + i] = s2[i];
        return;
    }
    for (int i = threadIdx.x; i < rb.n1; i += blockDim.x) rb.dst[i] = rb.src1[i];
    for (int i = threadIdx.x; i < rb.n2; i += blockDim.x) rb.dst[rb.n1 + i] = rb.src2[i];
}

// The densify of the output layer (C % 8 == 0): warps take (8-channel group,
// output row) items; warp gw of nw.
__device__ __forceinline__ void densify8_body(const Ctx& c, BufDev acc, BufDev trunc, float* __restrict__ out, int gw,
                                              int nw) {
    const FrameDev& F = *c.f;
    const int t = acc.t, C = acc.C, G = C / 8;
    const int oh = F.th * t, ow = F.tw * t;
    const size_t plane = (size_t)oh * ow;
    const int lane = threadIdx.x & 31;
    for (int it = gw; it < G * oh; it += nw) {
        const int g = it / oh, y = it - g * oh;
        const int qy = y / t, yy = y - qy * t;
        // two pixels per lane per round, all 8 loads issued before any use
        for (int x0 = lane; x0 < ow; x0 += 64) {
            float4 a0[2], a1[2], t0[2], t1[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int x = x0 + 32 * u;
                if (x < ow) {
                    const int qx = x / t;
                    const size_t off = (size_t)slot_of(F, c.rows, c.cols, qy, qx) * t * t * C +
                                       ((size_t)yy * t + (x - qx * t)) * C + g * 8;
                    a0[u] = __ldcs(reinterpret_cast<const float4*>(acc.d + off));
                    a1[u] = __ldcs(reinterpret_cast<const float4*>(acc.d + off) + 1);
                    t0[u] = __ldcs(reinterpret_cast<const float4*>(trunc.d + off));
                    t1[u] = __ldcs(reinterpret_cast<const float4*>(trunc.d + off) + 1);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int x = x0 + 32 * u;
                if (x >= ow) continue;
                float* o = out + (size_t)(g * 8) * plane + (size_t)y * ow + x;
                o[0] = __fadd_rn(a0[u].x, t0[u].x);
                o[plane] = __fadd_rn(a0[u].y, t0[u].y);
                o[2 * plane] = __fadd_rn(a0[u].z, t0[u].z);
                o[3 * plane] = __fadd_rn(a0[u].w, t0[u].w);
                o[4 * plane] = __fadd_rn(a1[u].x, t1[u].x);
                o[5 * plane] = __fadd_rn(a1[u].y, t1[u].y);
                o[6 * plane] = __fadd_rn(a1[u].z, t1[u].z);
                o[7 * plane] = __fadd_rn(a1[u].w, t1[u].w);
            }
        }
    }
}
