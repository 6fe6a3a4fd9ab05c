// Shared host/device definitions of the B200 delta engine.
//
// Device layout:
//  * Spherical buffer ("state", tile_grid.hpp:88-128 in the reference):
//    slot-major, channels innermost: [rows][cols][t][t][C] fp32. A global pixel
//    (gy, gx) lives in slot (floor_mod(floor_div(gy,t),rows),
//    floor_mod(floor_div(gx,t),cols)) at in-tile (floor_mod(gy,t),
//    floor_mod(gx,t)) — the same wrap as the reference's pixel-level
//    floor_mod(gy, rows*t) (tile_grid.hpp:119-123), so every tile is one
//    contiguous t*t*C block.
//  * Packet (DeltaPacket, delta_layers.hpp:18-46): dense grown extent, HWC,
//    fixed pitch (rows*t + 2*halo) x (cols*t + 2*halo) x C, plus an "ext"
//    tile-validity map over the placement tiles extended by RT = ceil(halo/t)
//    ring tiles. ext=0 means "all zero" (never read); inside the extent ext is
//    exactly the reference's TileMask.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define DFX_HD __host__ __device__ __forceinline__
#else
#define DFX_HD inline
#endif

namespace dfx {

// common.hpp:37-49 — mathematical floor div / mod.
DFX_HD int64_t floor_div64(int64_t a, int64_t n) {
    int64_t q = a / n;
    if ((a % n != 0) && ((a < 0) != (n < 0))) --q;
    return q;
}
DFX_HD int64_t floor_mod64(int64_t a, int64_t n) {
    int64_t r = a % n;
    if (r != 0 && ((r < 0) != (n < 0))) r += n;
    return r;
}
DFX_HD int64_t ceil_div64(int64_t a, int64_t n) { return -floor_div64(-a, n); }
DFX_HD int floor_div32(int a, int n) {
    int q = a / n;
    if ((a % n != 0) && ((a < 0) != (n < 0))) --q;
    return q;
}
DFX_HD int floor_mod32(int a, int n) {
    int r = a % n;
    if (r != 0 && ((r < 0) != (n < 0))) r += n;
    return r;
}

struct SlotDev {
    int64_t tx, ty;
    int used;
    int covered;
};

// One claim of the frame (buffer_manager.cpp:68-81) in the frame parameter
// block: the global tile and its slot. k_claims zeroes / bias-fills the slot's
// tiles and records the new owner in the engine's persistent device slot table.
struct ClaimRec {
    int64_t tx, ty;
    int slot;
    int pad[3];
};

// Per-frame parameters, uploaded once per frame; kernels read them from
// device memory so a frame's launch sequence is fixed (CUDA-graph friendly).
struct FrameDev {
    int64_t otx, oty;  // placement origin (tiles)
    int th, tw;        // placement tiles
    int base_sr, base_sc;  // floor_mod(oty, rows), floor_mod(otx, cols)
    int nclaims;
    int frame_h, frame_w;  // input frame size
    // canvas <- warped frame: warped (y, x) = (cy + sy0, cx + sx0)
    int sy0, sx0;
    int integer_path;  // 1: warped = frame shifted by (idx, idy)
    int idx, idy;
    int roi;           // aligned ROI present
    float inv[9];      // inverse residual homography (bilinear path)
};

// Spherical buffer (one per state array).
struct BufDev {
    float* d;
    int C, t;
};

// Delta packet storage.
struct PktDev {
    float* d;
    uint8_t* ext;
    int C, t, halo, RT;
    int pitch_w;    // pixels per stored row = cols*t + 2*halo
    int ext_pitch;  // = cols + 2*RT
};

DFX_HD size_t pkt_off(const PktDev& p, int y, int x) {
    return ((size_t)(y + p.halo) * p.pitch_w + (size_t)(x + p.halo)) * p.C;
}
DFX_HD int ext_idx(const PktDev& p, int i, int j) { return (i + p.RT) * p.ext_pitch + (j + p.RT); }

// Slot index of placement-relative tile (qy, qx) (may be negative / beyond).
// For 0 <= q < n (every placement tile) floor_mod(base + q, n) is one
// conditional subtract (base is already in [0, n)): no integer division on the
// hot path; other tiles (ring) take the general form.
DFX_HD int slot_of(const FrameDev& f, int rows, int cols, int qy, int qx) {
    int r, s;
    if ((unsigned)qy < (unsigned)rows) {
        r = f.base_sr + qy;
        r -= r >= rows ? rows : 0;
    } else {
        r = floor_mod32(f.base_sr + floor_mod32(qy, rows), rows);
    }
    if ((unsigned)qx < (unsigned)cols) {
        s = f.base_sc + qx;
        s -= s >= cols ? cols : 0;
    } else {
        s = floor_mod32(f.base_sc + floor_mod32(qx, cols), cols);
    }
    return r * cols + s;
}

}  // namespace dfx
