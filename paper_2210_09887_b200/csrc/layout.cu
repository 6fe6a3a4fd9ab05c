// Layout conversions for the layer-level C-ABI (layers.cpp): the reference's
// host-side layouts <-> this library's device layouts, on the caller's stream.
//
//   DeltaPacket (delta_layers.hpp:18-46): dense grown CHW + TileMask
//     <-> PktDev: HWC at the grid pitch + ext tile map (dfx_types.hpp)
//   SphericalBuffer (tile_grid.hpp:88-128): wrapped planar CHW,
//     (c, floor_mod(gy, rows*t), floor_mod(gx, cols*t))
//     <-> slot-major [rows][cols][t][t][C]
//   aligned frame canvas CHW (alignment.cpp:106-166) -> the input stage's HWC canvas
//
// Plain grid-stride copies (these run once per layer call of a unit test or an
// integration, not on the engine's per-frame path).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.hpp"

namespace dfx {

namespace {

constexpr int kT = 256;

int grid_for(long long n) {
    long long g = (n + kT - 1) / kT;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

__global__ void k_pkt_from_chw(const float* __restrict__ chw, const uint8_t* __restrict__ mask, int th, int tw,
                               PktDev p) {
    const int gh = th * p.t + 2 * p.halo, gw = tw * p.t + 2 * p.halo;
    const long long n = (long long)p.C * gh * gw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % gw), y = (int)((i / gw) % gh), c = (int)(i / ((long long)gw * gh));
        p.d[pkt_off(p, y - p.halo, x - p.halo) + c] = chw[i];
    }
    const int eh = th + 2 * p.RT, ew = tw + 2 * p.RT;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)eh * ew;
         i += (long long)gridDim.x * blockDim.x) {
        const int ti = (int)(i / ew) - p.RT, tj = (int)(i % ew) - p.RT;
        const bool inside = ti >= 0 && ti < th && tj >= 0 && tj < tw;
        // ring tiles: the halo data is copied whole (zeros where nothing was written)
        p.ext[ext_idx(p, ti, tj)] = inside ? (mask[ti * tw + tj] ? 1 : 0) : 1;
    }
}

__global__ void k_pkt_to_chw(PktDev p, int th, int tw, float* __restrict__ chw, uint8_t* __restrict__ mask) {
    const int gh = th * p.t + 2 * p.halo, gw = tw * p.t + 2 * p.halo;
    const long long n = (long long)p.C * gh * gw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % gw) - p.halo, y = (int)((i / gw) % gh) - p.halo, c = (int)(i / ((long long)gw * gh));
        const bool v = p.ext[ext_idx(p, floor_div32(y, p.t), floor_div32(x, p.t))] != 0;
        chw[i] = v ? p.d[pkt_off(p, y, x) + c] : 0.0f;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)th * tw;
         i += (long long)gridDim.x * blockDim.x)
        mask[i] = p.ext[ext_idx(p, (int)(i / tw), (int)(i % tw))] ? 1 : 0;
}

// slot-major index of wrapped planar element (c, Y, X), Y in [0, rows*t), X in [0, cols*t)
__device__ __forceinline__ size_t slot_major(int C, int t, int cols, int c, int Y, int X) {
    const int sr = Y / t, sc = X / t;
    return ((((size_t)sr * cols + sc) * t + (Y - sr * t)) * t + (X - sc * t)) * C + c;
}

__global__ void k_state_convert(const float* __restrict__ src, float* __restrict__ dst, int C, int t, int rows,
                                int cols, int to_chw) {
    const int PH = rows * t, PW = cols * t;
    const long long n = (long long)C * PH * PW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int X = (int)(i % PW), Y = (int)((i / PW) % PH), c = (int)(i / ((long long)PW * PH));
        const size_t j = slot_major(C, t, cols, c, Y, X);
        if (to_chw) dst[i] = src[j];
        else dst[j] = src[i];
    }
}

__global__ void k_canvas_from_chw(const float* __restrict__ chw, int C, int h, int w, float* __restrict__ canvas,
                                  int pitch) {
    const long long n = (long long)C * h * w;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % w), y = (int)((i / w) % h), c = (int)(i / ((long long)w * h));
        canvas[((size_t)y * pitch + x) * C + c] = chw[i];
    }
}

}  // namespace

void launch_pkt_from_chw(cudaStream_t s, const float* chw, const uint8_t* mask_dev, int th, int tw, PktDev p) {
    const long long n = (long long)p.C * (th * p.t + 2 * p.halo) * (tw * p.t + 2 * p.halo);
    k_pkt_from_chw<<<grid_for(n), kT, 0, s>>>(chw, mask_dev, th, tw, p);
}
void launch_pkt_to_chw(cudaStream_t s, PktDev p, int th, int tw, float* chw, uint8_t* mask_dev) {
    const long long n = (long long)p.C * (th * p.t + 2 * p.halo) * (tw * p.t + 2 * p.halo);
    k_pkt_to_chw<<<grid_for(n), kT, 0, s>>>(p, th, tw, chw, mask_dev);
}
void launch_state_convert(cudaStream_t s, const float* src, float* dst, int C, int t, int rows, int cols, int to_chw) {
    const long long n = (long long)C * rows * t * cols * t;
    k_state_convert<<<grid_for(n), kT, 0, s>>>(src, dst, C, t, rows, cols, to_chw);
}
void launch_canvas_from_chw(cudaStream_t s, const float* chw, int C, int h, int w, float* canvas, int pitch) {
    k_canvas_from_chw<<<grid_for((long long)C * h * w), kT, 0, s>>>(chw, C, h, w, canvas, pitch);
}

}  // namespace dfx
