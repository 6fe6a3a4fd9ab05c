/*
 * dfx_b200.h — C-ABI of the B200-native MotionDeltaCNN sparse frame-difference
 * inference path (drop-in for the reference "deltaflux" engine path).
 *
 * Every entry point here replaces one piece of the reference's public surface
 * for the hot path (paths relative to /root/reference/proj):
 *
 *   dfx_engine_create        dflx::DeltaEngine::DeltaEngine(spec, cfg)   include/deltaflux/engine.hpp:47,
 *                            src/engine.cpp:7-15 (validate() at src/network.cpp:46-254)
 *   dfx_engine_create_on_stream  same, bound to a caller-supplied cudaStream_t
 *   dfx_engine_destroy       ~DeltaEngine
 *   dfx_engine_run_frame     DeltaEngine::run_frame(frame, h, roi)      engine.hpp:51, engine.cpp:184-287;
 *                            python: deltaflux._core.DeltaEngine.run_frame  bindings/py_bindings.cpp:103-121
 *   dfx_engine_run_frame_ex  run_frame with device-resident frame / output buffers
 *   dfx_engine_layer_order   ValidatedNet::topo (network.hpp:45), the FlopReport order
 *   dfx_engine_submit_frame  (async variant of run_frame for throughput; no reference counterpart)
 *   dfx_engine_submit_host_frame (pipelined host-buffer variant of run_frame; no reference counterpart)
 *   dfx_engine_sync          (completes submitted frames)
 *   dfx_engine_reset         DeltaEngine::reset()                      engine.hpp:55, engine.cpp:93-108
 *   dfx_engine_input_mask    FrameResult::input_mask                    engine.hpp:38
 *   dfx_engine_layer_flops   FrameResult::flops (FlopReport::layers)    tensor.hpp:105-123
 *   dfx_engine_read_state    truncation_state()/maxpool_state()/input_state() buffers
 *                            engine.hpp:64-67 (SphericalBuffer::storage, tile_grid.hpp:116)
 *   dfx_engine_read_packet   the per-layer DeltaPacket the observer sees  engine.hpp:69-70, engine.cpp:239,279
 *   dfx_engine_read_ledger   DeltaEngine::ledger()                     engine.hpp:64 (TileLedger, buffer_manager.hpp:13-88)
 *   dfx_wrap_tile            dflx::wrap_tile                            tile_grid.hpp:37-40
 *   dfx_validate_net         dflx::validate (host only)                 network.hpp:61-65, network.cpp:46-254
 *   dfx_ledger_*             dflx::TileLedger + plan_frame + apply_plan buffer_manager.hpp:13-126
 *   dfx_layer_ctx_*          one frame's FramePlacement + slot filter     tile_grid.hpp:43-58, delta_layers.hpp:50-57
 *   dfx_input_stage          compute_input_delta + DeltaEngine::input_gate + the gated input truncation
 *                            alignment.cpp:168-192, engine.cpp:110-182, 233-237
 *   dfx_claim_reset          apply_plan + zero_tile_everywhere + inject_bias_implicit
 *                            buffer_manager.cpp:68-89, engine.cpp:78-91
 *   dfx_delta_conv           dflx::padded_delta_conv                    delta_layers.hpp:103-104, delta_layers.cpp:100-147
 *   dfx_delta_truncate       dflx::delta_activation_truncate            delta_layers.hpp:114-116, delta_layers.cpp:149-232
 *   dfx_delta_maxpool        dflx::delta_maxpool                        delta_layers.hpp:118-119, delta_layers.cpp:234-318
 *   dfx_densify              dflx::densify                              delta_layers.hpp:127, delta_layers.cpp:395-400
 *
 * Conventions: every call returns 0 on success and a nonzero dfx_status on
 * failure; dfx_last_error() returns a thread-local message (C++ exceptions
 * cannot cross this boundary — the reference throws dflx::Error /
 * ValidationError, common.hpp:14-32; the Python mirror re-raises
 * DeltafluxError). Tensors crossing the boundary are host float32 in the
 * reference's CHW layout; spherical-buffer readbacks are in the reference's
 * wrapped CHW planar layout (c, floor_mod(gy, PH), floor_mod(gx, PW)).
 */
#ifndef DFX_B200_H
#define DFX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layer kinds, same set and meaning as dflx::LayerKind (network.hpp:11). */
typedef enum {
    DFX_CONV = 0,
    DFX_RELU = 1,
    DFX_TRUNCATE = 2,
    DFX_MAXPOOL = 3,
    DFX_AVGPOOL = 4,
    DFX_UPSAMPLE = 5,
    DFX_BATCHNORM = 6,
    DFX_ADD = 7,
    DFX_OUTPUT = 8
} dfx_layer_kind;

typedef enum {
    DFX_OK = 0,
    DFX_ERR = 1,            /* dflx::Error */
    DFX_ERR_VALIDATION = 2, /* dflx::ValidationError */
    DFX_ERR_IO = 3,         /* dflx::IoError */
    DFX_ERR_CUDA = 4        /* device failure (no reference counterpart) */
} dfx_status;

/* One layer, mirroring dflx::LayerDef (network.hpp:15-27). Pointers are only
 * read during dfx_engine_create. */
typedef struct {
    const char* name;
    int kind;               /* dfx_layer_kind */
    const char* input0;     /* "input" = network input */
    const char* input1;     /* Add only, else NULL */
    /* Conv (ConvParams, tensor.hpp:58-87): weights O-I-Kh-Kw fp32 */
    int in_channels;
    int out_channels;
    int kernel;             /* square, odd */
    int stride;
    int padding;
    const float* weights;
    const float* bias;      /* NULL = no bias */
    /* MaxPool / AvgPool */
    int pool_k;
    int pool_stride;
    /* Upsample */
    int factor;
    /* BatchNorm */
    int bn_channels;
    const float* bn_scale;
    const float* bn_shift;
    /* Relu / Truncate */
    int has_threshold;
    float threshold;
    int truncate_enabled;
} dfx_layer_desc;

typedef struct {
    int in_channels;
    int num_layers;
    const dfx_layer_desc* layers;
} dfx_net_desc;

/* Convolution arithmetic for the sparse DeltaConv kernel. */
typedef enum {
    DFX_CONV_TF32X3 = 0, /* tcgen05 kind::tf32, 3-pass split (fp32-grade), default */
    DFX_CONV_EXACT = 1   /* CUDA-core fp32, reference summation order: bit-exact */
} dfx_conv_mode;

/* dflx::EngineConfig (engine.hpp:10-21) plus the device-only knob conv_mode. */
typedef struct {
    int tile_size;
    int grid_rows;
    int grid_cols;
    float input_threshold;
    float default_threshold;
    int override_net_thresholds;
    int mask_dilation;
    int roi_enabled;
    int noise_suppression;
    int padded_convolutions;
    int conv_mode;          /* dfx_conv_mode */
} dfx_engine_config;

/* Scalar part of dflx::FrameResult / FrameEvents (engine.hpp:23-39). */
typedef struct {
    int64_t frame_index;
    int64_t origin_tx;
    int64_t origin_ty;
    int tiles_h;
    int tiles_w;
    int fresh;
    int evicted;
    int reset;
    int64_t dropped_pixels;
    double update_rate;
    uint64_t conv_flops;
    uint64_t dense_flops;
    int out_channels;
    int out_height;
    int out_width;
} dfx_frame_info;

typedef struct dfx_engine dfx_engine;

/* Buffer selectors for dfx_engine_read_state. */
enum { DFX_STATE_ACC = 0, DFX_STATE_TRUNC = 1, DFX_STATE_PREV = 2 };

const char* dfx_last_error(void);
void dfx_default_config(dfx_engine_config* cfg);

int dfx_engine_create(const dfx_net_desc* net, const dfx_engine_config* cfg, int device,
                      dfx_engine** out);
/* Same, but every kernel of the engine runs on `stream` (a cudaStream_t owned
 * by the caller; NULL = an engine-owned non-blocking stream). */
int dfx_engine_create_on_stream(const dfx_net_desc* net, const dfx_engine_config* cfg, int device, void* stream,
                                dfx_engine** out);
int dfx_engine_destroy(dfx_engine* e);

/* Synchronous frame: host CHW frame (c x h x w fp32), 3x3 row-major
 * homography, optional 1 x h x w ROI map. On return `info` is filled and the
 * densified output (out_channels x out_height x out_width, CHW) is copied to
 * `out` when out_cap (in floats) is large enough. */
int dfx_engine_run_frame(dfx_engine* e, const float* frame, int c, int h, int w, const float* h9,
                         const float* roi, dfx_frame_info* info, float* out, size_t out_cap);

/* run_frame with explicit buffer residency: frame_is_device = 1
 * when `frame` (and `roi`) are device pointers, out_is_device = 1 when `out`
 * is a device pointer (the output is copied device-to-device on the engine's
 * stream). Synchronous like dfx_engine_run_frame. */
int dfx_engine_run_frame_ex(dfx_engine* e, const float* frame, int c, int h, int w, int frame_is_device,
                            const float* h9, const float* roi, dfx_frame_info* info, float* out, size_t out_cap,
                            int out_is_device);

/* Asynchronous frame on device-resident input (frame_dev: device pointer,
 * CHW). Launches the whole frame on the engine's CUDA stream and returns
 * without waiting; results of the last frame are readable after
 * dfx_engine_sync. */
int dfx_engine_submit_frame(dfx_engine* e, const float* frame_dev, int c, int h, int w,
                            const float* h9);
/* Pipelined host-buffer frame (throughput form of dfx_engine_run_frame): the
 * frame's host->device copy and the densified output's device->host copy into
 * `out` (CHW, when out_cap is large enough) run on a copy stream overlapping
 * the compute of neighbouring frames; returns without waiting. `frame` and
 * `out` should be pinned host memory and must stay untouched until
 * dfx_engine_sync. */
int dfx_engine_submit_host_frame(dfx_engine* e, const float* frame, int c, int h, int w, const float* h9, float* out,
                                 size_t out_cap);
int dfx_engine_sync(dfx_engine* e, dfx_frame_info* info);
/* Page-locked host buffers for the pipelined host-frame path (NULL on failure). */
void* dfx_host_alloc(size_t bytes);
void dfx_host_free(void* p);

int dfx_engine_reset(dfx_engine* e);

/* Device pointer of the last densified output (CHW), valid until the next frame. */
int dfx_engine_output_device(dfx_engine* e, const float** ptr, int* c, int* h, int* w);

int dfx_engine_input_mask(dfx_engine* e, uint8_t* out, size_t cap, int* tiles_h, int* tiles_w);
int dfx_engine_num_layers(dfx_engine* e);
/* Layer indices in execution (topological) order; *n = number written. */
int dfx_engine_layer_order(dfx_engine* e, int* order, int cap, int* n);
int dfx_engine_layer_flops(dfx_engine* e, int layer, uint64_t* flops, uint64_t* dense_flops);
int dfx_engine_grid(dfx_engine* e, int* rows, int* cols);

/* Spherical buffer readback in the reference's wrapped CHW layout. layer is a
 * layer name or "input". On success *c, *h, *w give the buffer shape. */
int dfx_engine_read_state(dfx_engine* e, const char* layer, int which, float* out, size_t cap,
                          int* c, int* h, int* w);
/* Last frame's output packet of `layer` ("input" = gated input packet) as the
 * reference's dense grown CHW tensor with zeros in unmasked tiles. */
int dfx_engine_read_packet(dfx_engine* e, const char* layer, float* out, size_t cap, int* c,
                           int* gh, int* gw, int* halo, uint8_t* mask, size_t mask_cap);
int dfx_engine_read_ledger(dfx_engine* e, int* used, int64_t* ty, int64_t* tx, uint8_t* covered,
                           size_t cap);

/* Debug: per-layer gathered conv targets and dense 16x8 units of the last frame. */
int dfx_engine_debug_counts(dfx_engine* e, int* gathered, int* units, int cap);

/* Number of kernels the last frame launched. */
int dfx_engine_kernel_count(dfx_engine* e);

/* Kernel families for profiling. */
enum {
    DFX_FAM_CLAIMS = 0,       /* claim reset + bias init            (HBM)    */
    DFX_FAM_INPUT = 1,        /* input stage                        (HBM)    */
    DFX_FAM_CONV_TARGETS = 2, /* conv target compaction + zero fill (HBM)    */
    DFX_FAM_CONV_MMA = 3,     /* sparse DeltaConv                   (tensor) */
    DFX_FAM_TRUNC = 4,        /* fused delta activation / truncation (HBM)   */
    DFX_FAM_POOL = 5,         /* sparse pooling                     (HBM)    */
    DFX_FAM_LINEAR = 6,       /* upsample / batchnorm / add         (HBM)    */
    DFX_FAM_DENSIFY = 7,      /* dense output                       (HBM)    */
    DFX_FAMILIES = 8
};
/* Profiling mode: CUDA events around every launch on the engine's stream,
 * accumulated per family with the family's ALGORITHMIC work (bytes, or conv
 * FLOPs as the reference's FlopReport counts them). Frames become
 * synchronous while profiling. */
int dfx_engine_set_profiling(dfx_engine* e, int on);
int dfx_engine_reset_profile(dfx_engine* e);
int dfx_engine_profile(dfx_engine* e, int family, double* ms, uint64_t* launches, double* work);
const char* dfx_kernel_family_name(int family);
/* Device timer on the engine's stream (CUDA events): start, then stop
 * returns the elapsed milliseconds after synchronizing on the stop event. */
int dfx_engine_timer_start(dfx_engine* e);
int dfx_engine_timer_stop(dfx_engine* e, float* ms);

void dfx_wrap_tile(int64_t tx, int64_t ty, int rows, int cols, int* row, int* col);

/* Host-only network validation (dflx::validate, network.cpp:46-254): the
 * checks dfx_engine_create runs, without a device. On success `topo` holds
 * the execution order (*n entries) and *ring the stash ring width in tiles. */
int dfx_validate_net(const dfx_net_desc* net, int tile_size, int* topo, int cap, int* n, int* ring);

/* Host-only tile ledger: the TileLedger / plan_frame / apply_plan the engine
 * plans every frame with (buffer_manager.hpp:13-126, buffer_manager.cpp:7-81;
 * full reset + replan as engine.cpp:207-211). dfx_ledger_step plans and
 * applies one placement; claims are (tx, ty, victim_tx, victim_ty) with
 * victims[i] = 1 when the claim evicts; fresh tiles are (tx, ty). Slot
 * readback order is row-major over (floor_mod(ty, rows), floor_mod(tx, cols)). */
typedef struct dfx_ledger dfx_ledger;
int dfx_ledger_create(int rows, int cols, dfx_ledger** out);
int dfx_ledger_destroy(dfx_ledger* h);
int dfx_ledger_step(dfx_ledger* h, int64_t otx, int64_t oty, int th, int tw, int ring, int* full_reset,
                    int64_t* claims, int* victims, size_t claim_cap, int* nclaims, int64_t* fresh, size_t fresh_cap,
                    int* nfresh, int* evicted);
int dfx_ledger_slots(dfx_ledger* h, int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap);

/* ===================================================================== layer level
 * The reference's layer functions (delta_layers.hpp:103-127), used directly by
 * its unit tests, on DEVICE buffers in this library's native layouts:
 *
 *   dfx_packet (DeltaPacket, delta_layers.hpp:18-46): `d` = dense grown extent,
 *     HWC, (rows*tile + 2*halo) x (cols*tile + 2*halo) x channels floats (the
 *     grid's rows / cols, not the placement's); `ext` = tile validity bytes
 *     over (rows + 2*RT) x (cols + 2*RT) tiles, RT = ceil(halo / tile): inside
 *     the placement it IS the TileMask, ring tiles flag written halo data.
 *   dfx_state (SphericalBuffer, tile_grid.hpp:88-128): slot-major
 *     [rows][cols][tile][tile][channels] floats.
 *
 * A dfx_layer_ctx binds one device, one cudaStream_t and one grid; its frame
 * (dfx_layer_ctx_set_frame) is the placement plus the slot table the slot
 * filter reads (TileLedger::holds, buffer_manager.hpp:41-44). Calls are
 * stream-ordered and asynchronous except where they return host values.
 * dfx_packet_from_chw / _to_chw and dfx_state_from_chw / _to_chw convert
 * from / to the reference's layouts (dense grown CHW + TileMask; wrapped CHW
 * planar), device to device. */
typedef struct dfx_layer_ctx dfx_layer_ctx;
typedef struct {
    int64_t origin_tx, origin_ty; /* FramePlacement::origin (tiles) */
    int tiles_h, tiles_w;
} dfx_placement;
typedef struct {
    int used;
    int64_t tx, ty; /* the global tile the slot holds */
} dfx_slot;
typedef struct {
    float* d;
    uint8_t* ext;
    int channels, tile, halo;
} dfx_packet;
typedef struct {
    float* d;
    int channels, tile;
} dfx_state;

int dfx_layer_ctx_create(int rows, int cols, int device, void* stream, dfx_layer_ctx** out);
int dfx_layer_ctx_destroy(dfx_layer_ctx* c);
/* slots: rows*cols host entries in row-major (floor_mod(ty, rows), floor_mod(tx,
 * cols)) order, or NULL = every slot holds the placement tile that maps to it. */
int dfx_layer_ctx_set_frame(dfx_layer_ctx* c, const dfx_placement* place, const dfx_slot* slots);
/* Device buffer sizes of a packet / state on this grid. */
size_t dfx_packet_floats(const dfx_layer_ctx* c, int channels, int tile, int halo);
size_t dfx_packet_ext_bytes(const dfx_layer_ctx* c, int tile, int halo);
size_t dfx_state_floats(const dfx_layer_ctx* c, int channels, int tile);
/* chw: device, channels x (th*tile + 2*halo) x (tw*tile + 2*halo); mask: host th*tw bytes. */
int dfx_packet_from_chw(dfx_layer_ctx* c, const float* chw, const uint8_t* mask, dfx_packet* out);
int dfx_packet_to_chw(dfx_layer_ctx* c, const dfx_packet* p, float* chw, uint8_t* mask);
/* chw: device, channels x (rows*tile) x (cols*tile), the reference's wrapped planar layout. */
int dfx_state_from_chw(dfx_layer_ctx* c, const float* chw, dfx_state* out);
int dfx_state_to_chw(dfx_layer_ctx* c, const dfx_state* s, float* chw);

/* padded_delta_conv: out halo = windowed_out_halo(in halo, k, k/2, stride),
 * out tile = in tile / stride (dfx_delta_conv_out_halo); weights: device
 * O-I-K-K fp32 (bias is never applied here, delta_layers.hpp:100-102);
 * conv_mode DFX_CONV_TF32X3 or DFX_CONV_EXACT. *flops (host, may be NULL)
 * receives the reference's FlopReport counts (flops, dense_flops). */
int dfx_delta_conv_out_halo(int in_halo, int kernel, int stride);
int dfx_delta_conv(dfx_layer_ctx* c, const dfx_packet* in, const float* weights, int cin, int cout, int kernel,
                   int stride, int conv_mode, dfx_packet* out, uint64_t* flops);
/* delta_activation_truncate (no gate: the input stage's gate is dfx_input_stage);
 * relu = 1 for ActKind::Relu, 0 for Identity. Out packet: halo 0, in tile. */
int dfx_delta_truncate(dfx_layer_ctx* c, const dfx_packet* in, dfx_state* acc, dfx_state* trunc, float threshold,
                       int relu, dfx_packet* out);
/* delta_maxpool (k == stride): acc at the input tile, prev at the output tile;
 * out halo = windowed_out_halo(in halo, k, 0, k). */
int dfx_delta_maxpool(dfx_layer_ctx* c, const dfx_packet* in, dfx_state* acc, dfx_state* prev, int k,
                      dfx_packet* out);
/* densify: out (device, CHW channels x th*tile x tw*tile) = acc + trunc. */
int dfx_densify(dfx_layer_ctx* c, const dfx_state* acc, const dfx_state* trunc, float* out);
/* Claim reset: every claimed tile (coords: host (tx, ty) pairs) is zeroed in
 * every state, then filled with fills[b] (per-channel, device, or NULL = 0)
 * for states with a bias init (apply_plan + inject_bias_implicit). */
int dfx_claim_reset(dfx_layer_ctx* c, const int64_t* coords, int nclaims, dfx_state* const* states,
                    const float* const* fills, int nstates);
/* Input stage on an ALIGNED frame (the canvas of alignment.cpp:106-166):
 * aligned: device CHW channels x (th*T) x (tw*T); valid: device bytes (th*T) x
 * (tw*T), 1 where the pixel came from the frame; roi_factor: device floats
 * (th*T) x (tw*T) or NULL; fresh: host th*tw bytes or NULL. Computes
 * raw = aligned - acc on covered tiles, the gate (significance > threshold,
 * noise rule, dilation, fresh tiles) and the gated truncation into
 * acc / trunc; `out` (halo 0) receives the fired candidates and the gate as
 * mask; *update_rate (host, may be NULL) = fired tiles / placement tiles. */
int dfx_input_stage(dfx_layer_ctx* c, const float* aligned, const uint8_t* valid, const float* roi_factor,
                    const uint8_t* fresh, float threshold, int dilation, int noise_suppression, dfx_state* acc,
                    dfx_state* trunc, dfx_packet* out, double* update_rate);

#ifdef __cplusplus
}
#endif

#endif /* DFX_B200_H */
