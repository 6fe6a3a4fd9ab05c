// Launch wrappers of the B200 delta-engine kernels (kernels.cu, conv_tc.cu).
// All take the engine's stream; all per-frame values are read on device from
// the FrameDev struct, so a frame's launch sequence has fixed shapes.
#pragma once

#include <cuda_runtime.h>

#include "dfx_types.hpp"

namespace dfx {

struct Ctx {
    const FrameDev* f;     // device
    const SlotDev* slots;  // device [rows*cols]
    int rows, cols;
    const uint8_t* own;    // device [th*tw]: placement tile owns its slot (TileLedger::holds)
};

struct ClaimBuf {
    float* d;
    const float* fill;  // per-channel fill (bias init) or nullptr for zero
    int C, t;
};

// ---- input stage (alignment.cpp:58-192, engine.cpp:110-182, 233-234) ----
void launch_align(const Ctx& c, cudaStream_t s, const float* frame, const float* warped, const uint8_t* fp,
                  int C, float* aligned, uint8_t* valid, int canvas_pitch, int T);
void launch_warp(const Ctx& c, cudaStream_t s, const float* frame, int C, float* warped, uint8_t* fp);
void launch_count_dropped(const Ctx& c, cudaStream_t s, const uint8_t* fp, int T, unsigned long long* counter);
void launch_roi_factor(const Ctx& c, cudaStream_t s, const float* roi_aligned, float* tmp3, float* fac,
                       int canvas_pitch, int T);
void launch_coverage(const Ctx& c, cudaStream_t s, const uint8_t* valid, int canvas_pitch, int T, uint8_t* cov);
void launch_input_sig(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov, BufDev acc,
                      BufDev trunc, const float* fac, float thr, int canvas_pitch, int T, uint8_t* sig);
void launch_noise(const Ctx& c, cudaStream_t s, const uint8_t* sig, uint8_t* out, int canvas_pitch, int T);
void launch_gate(const Ctx& c, cudaStream_t s, const uint8_t* sig, const uint8_t* cov, const uint8_t* fresh,
                 int dilation, int canvas_pitch, int T, uint8_t* gate);
void launch_input_apply(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov,
                        const uint8_t* gate, BufDev acc, BufDev trunc, PktDev out, int canvas_pitch);

// ---- buffer manager (buffer_manager.cpp:68-89, engine.cpp:78-91) ----
// Claims of the frame: recs (engine: ClaimRec in the parameter block; their new
// owners also go into `table`, the persistent slot table) or plain slot indices.
void launch_claims(const Ctx& c, cudaStream_t s, const ClaimRec* recs, const int* plain_slots, SlotDev* table,
                   const ClaimBuf* bufs, int nbuf, int max_claims);

// ---- truncation (delta_layers.cpp:149-232) ----
void launch_ring_add(const Ctx& c, cudaStream_t s, PktDev in, BufDev dst);
void launch_trunc_max(const Ctx& c, cudaStream_t s, PktDev in, BufDev trunc, unsigned* tile_max);
// One-pass fused truncation (register-resident tile, DSMEM max across a
// cluster); returns false when the shape needs the two-pass fallback.
bool launch_trunc_fused(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc, float thr, int relu,
                        PktDev out);
// Two streaming passes (kernels_hbm.cu): tile max, then fire / fold. Needs C % 4 == 0.
// gbar (zeroed per frame): grid-barrier counter for the single cooperative launch.
struct Readback {  // copied by the last kernel of a frame into mapped host memory
    const uint8_t* src1;
    int n1;
    const uint8_t* src2;
    int n2;
    uint8_t* dst;  // device view of the page-locked host block
    const unsigned* out_flag = nullptr;  // host path: wait until *out_flag >= out_val before writing the output
    unsigned out_val = 0;
};

// Output layer: densify (acc + trunc -> the frame's output, plus the frame's
// readback) inside the cooperative activation launch (dz_done reports it).
struct DenseOut {
    float* out;
    Readback rb;
};
// Returns the number of kernels launched (1 cooperative, 2 two-pass) or 0 when
// the packet shape needs the generic launch_trunc_max / launch_trunc_apply.
int launch_trunc_two_pass(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc, unsigned* tile_max,
                           float thr, int relu, PktDev out, unsigned* gbar, const DenseOut* dz = nullptr,
                           bool* dz_done = nullptr, BufDev pf0 = BufDev{nullptr, 0, 0},
                           BufDev pf1 = BufDev{nullptr, 0, 0});  // pf0 / pf1: consumer state prefetched per fired tile
bool launch_maxpool_vec(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, PktDev out);
void launch_trunc_apply(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                        const unsigned* tile_max, float thr, int relu, PktDev out);

// ---- pooling / linear packet ops (delta_layers.cpp:234-393) ----
void launch_tile_add(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc);
void launch_maxpool_out(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, int st,
                        PktDev out, int out_halo_geom);
// Fused fold + window max for halo-free inputs with k == stride.
void launch_maxpool_fused(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev prev, int k, PktDev out);
void launch_avgpool(const Ctx& c, cudaStream_t s, PktDev in, int k, int st, PktDev out);
void launch_upsample(const Ctx& c, cudaStream_t s, PktDev in, int f, PktDev out);
void launch_bn(const Ctx& c, cudaStream_t s, PktDev in, const float* scale, PktDev out);
// fb > 1: b is the input of an upsample-by-fb folded into the add (C % 4 == 0).
void launch_add(const Ctx& c, cudaStream_t s, PktDev a, PktDev b, PktDev out, int fb = 1);

// ---- conv (delta_layers.cpp:100-147) ----
// Target compaction: writes the compacted target list (packed (y+H)<<16 | (x+H),
// H = geometric out halo), count (targets in the stored extent) and flops
// counter (targets in the geometric grown extent), the out ext map, and
// zeros every non-target pixel of every active out tile.
// dense_map (nullable): per 16x8 output unit, 1 = computed by k_conv_dense;
// its pixels are left out of the gathered list and of the zero fill.
void launch_conv_targets(const Ctx& c, cudaStream_t s, PktDev in, int k, int st, int r, PktDev out,
                         int out_halo_geom, int* list, int* count, unsigned long long* flop_px,
                         const uint8_t* dense_map = nullptr, int nux_max = 0);
void launch_conv_exact(const Ctx& c, cudaStream_t s, PktDev in, const float* w, int cin, int cout, int k, int st,
                       int r, PktDev out, int out_halo_geom, const int* list, const int* count, int max_targets);
// tcgen05 3xTF32 conv (conv_tc.cu). wsplit: pre-split weights, see conv_tc.cu.
// splits > 1: split-K over `splits` parts into the fp32 workspace ws
// ([splits][max_targets][cout_pad]) + a fixed-order reduction (deterministic).
void launch_conv_tc(const Ctx& c, cudaStream_t s, PktDev in, const float* wsplit, int cin, int cin_pad, int cout,
                    int cout_pad, int k, int st, int r, PktDev out, int out_halo_geom, const int* list,
                    const int* count, int max_targets, int num_sms, float* ws, int splits);
// Kernel sizes the gathered-target tensor-core conv handles (k <= 7); larger
// kernels take k_conv_exact.
bool conv_tc_supported(int k);
int conv_tc_splits(int max_targets, int cin_pad, int cout_pad, int k, int num_sms);
size_t conv_tc_weight_floats(int cin_pad, int cout_pad, int k);
void conv_tc_prepare_weights(const float* w, int cin, int cout, int k, int cin_pad, int cout_pad, float* out);

// Dense-unit conv (conv_dense.cu): stride-1 convs, 16x8-pixel output units
// whose pixels are mostly targets; input patches staged once in shared memory.
struct DenseConvPlan {
    bool ok;
    int k, r, cin_pad, KC, nCB, cout_pad, NBD, nNB, nstw, smax, umax;
    int nux_max, nuy_max, units_max, nbh, nbw, t_out;
    int tpu;     // tile units: tiles of T x T px per 128-row unit (T = t_out in {2, 4, 8}); 0 = 16x8-px units
    int tsh;     // log2(t_out) in tile-unit mode
    int patch_px;
    int npb;       // patch ring depth
    int nmma;      // MMA issuer warps (1 or 2)
    int ws_units;  // max 128-row units of a frame (split-K workspace rows / 128)
    int tma;       // 16x8-px units, KC = 16: patches staged by TMA tensor-map boxes (SWIZZLE_64B)
    unsigned s_c4, patch_bytes, w_stage, acc_cols, nbuf;
    size_t smem;
};
DenseConvPlan dense_conv_plan(int cin, int cout, int k, int t_out, int rows, int cols, size_t ws_budget_bytes);
size_t dense_conv_weight_floats(const DenseConvPlan& p);
void dense_conv_prepare_weights(const DenseConvPlan& p, const float* w, int cin, int cout, float* out);
// Targets, exact out ext map, FLOP pixels, dense unit list and zero fill of a
// stride-1 conv whose every target is computed by k_conv_dense.
// Units with >= tau targets go to k_conv_dense, the targets of sparser units
// to the gathered list (list / lcount) for launch_conv_tc (tau = 1: all dense).
// tmax / tm_trunc (nullable): fused pass 1 of the consuming activation (see launch_conv_dense).
void launch_conv_plan(const Ctx& c, cudaStream_t s, const DenseConvPlan& p, PktDev in, PktDev out, int hg, int* units,
                      int* nunits, unsigned long long* flop_px, int tau, int* list, int* lcount,
                      unsigned* tmax = nullptr, BufDev tm_trunc = BufDev{nullptr, 0, 0});
long long* dense_conv_trace_buffer();
// DFX_KTRACE chain trace: per-translation-unit setters of the stamp buffer
void ktrace_set_kernels(unsigned long long* b, unsigned* c);
void ktrace_set_hbm(unsigned long long* b, unsigned* c);
void ktrace_set_dense(unsigned long long* b, unsigned* c);
void ktrace_set_tc(unsigned long long* b, unsigned* c);
unsigned long long* frame_trace_host();  // DFX_FRAME_TRACE: [64][4] frame-boundary stamps
unsigned long long* trunc_trace_buffer();  // DFX_TRUNC_TRACE: [64 launches][1024 CTAs][8] globaltimer stamps  // microbenchmark stamps (DFX_CONV_DBG & 64)
// nxt_acc / nxt_trunc: the consuming activation layer's state buffers (its tiles
// are prefetched to L2 by the conv), or {nullptr} for none.
// TMA descriptor of a conv's input packet for the patch boxes of plan p
// (cuTensorMapEncodeTiled through the runtime's driver entry point); `out` is
// a CUtensorMap (64 B, 64-B aligned). False: no TMA (the cp.async path runs).
bool dense_conv_tensor_map(const DenseConvPlan& p, PktDev in, int rows, void* out);
void launch_conv_dense(const Ctx& c, cudaStream_t s, const DenseConvPlan& p, PktDev in, PktDev out, const float* w,
                       int cin, int cout, const int* units, const int* nunits, float* ws, int* cnt, int num_sms,
                       BufDev nxt_acc = BufDev{nullptr, 0, 0}, BufDev nxt_trunc = BufDev{nullptr, 0, 0},
                       unsigned* tmax = nullptr, const void* tmap = nullptr);
// The consuming activation's pass 2 alone (its pass 1, max |trunc + delta| per
// tile, was folded into tile_max by the conv: launch_conv_plan / _dense with
// tmax), plus the halo stash pass 1 used to run. Needs C % 4 == 0.
// Upper bound on the warp work items of the activation launches that follow
// (their persistent grids shrink to it); 0 = none. Per host thread.
void set_trunc_work_hint(long long items);
// Activation pass 1 alone (tile max + halo stash; C % 4 == 0).
void launch_trunc_tilemax(const Ctx& c, cudaStream_t s, PktDev in, BufDev trunc, unsigned* tile_max);
// Activation pass 2 fused with its sole consumer, a 2x2 / stride-2 max pool
// (halo-free, C % 4 == 0): the pool layer then launches nothing.
void launch_trunc_commit_pool(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                              const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pacc, BufDev pprev,
                              PktDev pout);
// Activation pass 2 (with its fused 2x2 max pool when pacc.d != null) and the
// plan of the consuming stride-1 dense conv (plan p, input packet cin = the
// activation's / pool's output, output packet cout) in one launch.
void launch_trunc_commit_plan(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                              const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pacc, BufDev pprev,
                              PktDev pout, const DenseConvPlan& p, PktDev cin, PktDev cout, int hg, int* units,
                              int* nunits, unsigned long long* flop_px, int* list, int* lcount);
void launch_trunc_commit_stash(const Ctx& c, cudaStream_t s, PktDev in, BufDev acc, BufDev trunc,
                               const unsigned* tile_max, float thr, int relu, PktDev out, BufDev pf0, BufDev pf1);

// ---- output (delta_layers.cpp:395-400) ----
void launch_densify(const Ctx& c, cudaStream_t s, BufDev acc, BufDev trunc, float* out, Readback rb);
// Fused input stage (no ROI factor, no noise filter): A = align + coverage +
// significance per canvas tile, B = gate + input truncation per tile.
void launch_input_tile_a(const Ctx& c, cudaStream_t s, const float* frame, const float* warped, const uint8_t* fp,
                         int C, float* aligned, int pitch, int T, BufDev acc, BufDev trunc, float thr, uint8_t* cov,
                         uint8_t* sig, int direct);  // direct: bilinear samples computed from the frame (no k_warp)
void launch_input_tile_b(const Ctx& c, cudaStream_t s, const float* aligned, const uint8_t* cov, const uint8_t* sig,
                         const uint8_t* fresh, int dilation, int pitch, BufDev acc, BufDev trunc, PktDev out);
// First kernel of a frame: parameter block (mapped host -> device slot), counters zeroed, host ack.
// done_ctr: a zeroed device word private to the engine (last-CTA election for the ack)
void launch_frame_begin(cudaStream_t s, const void* src, void* dst, size_t bytes, void* counters, size_t cnt_bytes,
                        unsigned* ack, unsigned seq, const unsigned* in_flag, unsigned in_val, unsigned* done_ctr);
// copy-stream -> engine-stream handshake: *f = v (release) once the stream's prior work is done
void launch_set_flag(cudaStream_t s, unsigned* f, unsigned v);

}  // namespace dfx

namespace dfx {
// ---- layout conversions for the layer-level C-ABI (layout.cu) ----
void launch_pkt_from_chw(cudaStream_t s, const float* chw, const uint8_t* mask_dev, int th, int tw, PktDev p);
void launch_pkt_to_chw(cudaStream_t s, PktDev p, int th, int tw, float* chw, uint8_t* mask_dev);
void launch_state_convert(cudaStream_t s, const float* src, float* dst, int C, int t, int rows, int cols, int to_chw);
void launch_canvas_from_chw(cudaStream_t s, const float* chw, int C, int h, int w, float* canvas, int pitch);
}  // namespace dfx
