// dfx_deltaflux.hpp — the reference-side drop-in: a dflx::DeltaEngine-shaped
// class over the C-ABI of libdfx_b200.so (include/dfx_b200.h).
//
// A maintainer of the reference adds this header to proj/include (next to
// deltaflux/engine.hpp) and links libdfx_b200.so; code written against
//   dflx::DeltaEngine(spec, cfg).run_frame(frame, h, roi)   engine.hpp:45-91
// switches to the B200 path by naming dflx::B200DeltaEngine instead. Every
// type in the signatures is the reference's own (NetworkSpec, EngineConfig,
// Tensor, Homography, FrameResult, TileMask, FlopReport); every failure is
// rethrown as the reference's exception hierarchy (common.hpp:14-32):
// DFX_ERR_VALIDATION -> ValidationError, DFX_ERR_IO -> IoError, anything else
// (including "no CUDA device": there is no CPU fallback) -> Error.
//
// tests/test_integration_header.py compiles this header against
// /root/reference/proj/include and links it with libdfx_b200.so.
#pragma once

#include <string>
#include <vector>

#include "deltaflux/engine.hpp"
#include "dfx_b200.h"

namespace dflx {

// dfx_status -> the reference's exceptions (common.hpp:14-32).
inline void dfx_throw(int rc) {
    if (rc == DFX_OK) return;
    const std::string msg = dfx_last_error();
    if (rc == DFX_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == DFX_ERR_IO) throw IoError(msg);
    throw Error(msg);
}

class B200DeltaEngine {
  public:
    // engine.hpp:47 — same arguments; `device` selects the GPU, `stream`
    // (a cudaStream_t, or nullptr for an engine-owned stream) the CUDA stream
    // every kernel of this engine runs on.
    B200DeltaEngine(const NetworkSpec& spec, const EngineConfig& cfg, int device = 0, void* stream = nullptr)
        : spec_(spec), cfg_(cfg) {
        std::vector<dfx_layer_desc> L;
        L.reserve(spec_.layers.size());
        for (const LayerDef& d : spec_.layers) L.push_back(to_desc(d));
        dfx_net_desc net{spec_.in_channels, (int)L.size(), L.data()};
        dfx_engine_config c;
        dfx_default_config(&c);
        c.tile_size = cfg.tile_size;
        c.grid_rows = cfg.grid_rows;
        c.grid_cols = cfg.grid_cols;
        c.input_threshold = cfg.input_threshold;
        c.default_threshold = cfg.default_threshold;
        c.override_net_thresholds = cfg.override_net_thresholds ? 1 : 0;
        c.mask_dilation = cfg.mask_dilation;
        c.roi_enabled = cfg.roi_enabled ? 1 : 0;
        c.noise_suppression = cfg.noise_suppression ? 1 : 0;
        c.padded_convolutions = cfg.padded_convolutions ? 1 : 0;
        dfx_throw(dfx_engine_create_on_stream(&net, &c, device, stream, &e_));
    }
    ~B200DeltaEngine() {
        if (e_) dfx_engine_destroy(e_);
    }
    B200DeltaEngine(const B200DeltaEngine&) = delete;
    B200DeltaEngine& operator=(const B200DeltaEngine&) = delete;

    // engine.hpp:51 — same arguments, same FrameResult (host tensors).
    FrameResult run_frame(const Tensor& frame, const Homography& h, const Tensor* roi = nullptr) {
        dfx_frame_info info{};
        size_t cap = out_capacity(frame);
        std::vector<float> out(cap);
        dfx_throw(dfx_engine_run_frame(e_, frame.data.data(), frame.channels, frame.height, frame.width, h.m.data(),
                                       roi ? roi->data.data() : nullptr, &info, out.data(), out.size()));
        FrameResult r;
        r.output = Tensor(info.out_channels, info.out_height, info.out_width);
        std::copy(out.begin(), out.begin() + (ptrdiff_t)r.output.data.size(), r.output.data.begin());
        r.place.origin = TileCoord{info.origin_tx, info.origin_ty};
        r.place.tiles_h = info.tiles_h;
        r.place.tiles_w = info.tiles_w;
        r.events.frame_index = info.frame_index;
        r.events.origin = r.place.origin;
        r.events.fresh = info.fresh;
        r.events.evicted = info.evicted;
        r.events.reset = info.reset != 0;
        r.events.dropped_pixels = info.dropped_pixels;
        r.update_rate = info.update_rate;
        // FlopReport (tensor.hpp:105-123): one entry per conv layer in execution order
        const int nl = dfx_engine_num_layers(e_);
        std::vector<int> order(nl > 0 ? nl : 1);
        int n = 0;
        dfx_throw(dfx_engine_layer_order(e_, order.data(), nl, &n));
        for (int i = 0; i < n; ++i) {
            const LayerDef& d = spec_.layers[order[i]];
            if (d.kind != LayerKind::Conv) continue;
            uint64_t f = 0, df = 0;
            dfx_throw(dfx_engine_layer_flops(e_, order[i], &f, &df));
            r.flops.add(d.name, f, df);
        }
        r.input_mask = TileMask(info.tiles_h, info.tiles_w);
        int th = 0, tw = 0;
        dfx_throw(dfx_engine_input_mask(e_, r.input_mask.bits.data(), r.input_mask.bits.size(), &th, &tw));
        ++frame_index_;
        return r;
    }

    void reset() { dfx_throw(dfx_engine_reset(e_)); }  // engine.hpp:55
    const EngineConfig& config() const { return cfg_; }
    bool initialized() const { return frame_index_ > 0; }
    int64_t frame_index() const { return frame_index_; }

    // Spherical-buffer readback in the reference's wrapped CHW layout
    // (SphericalBuffer::storage, tile_grid.hpp:116): which = DFX_STATE_*.
    Tensor read_state(const std::string& layer, int which) const {
        int c = 0, hh = 0, ww = 0;
        dfx_throw(dfx_engine_read_state(e_, layer.c_str(), which, nullptr, 0, &c, &hh, &ww));
        Tensor t(c, hh, ww);
        dfx_throw(dfx_engine_read_state(e_, layer.c_str(), which, t.data.data(), t.data.size(), &c, &hh, &ww));
        return t;
    }

  private:
    static dfx_layer_desc to_desc(const LayerDef& d) {
        dfx_layer_desc o{};
        o.name = d.name.c_str();
        o.kind = (int)d.kind;  // same enumerator order (network.hpp:11, dfx_layer_kind)
        o.input0 = d.inputs.empty() ? nullptr : d.inputs[0].c_str();
        o.input1 = d.inputs.size() > 1 ? d.inputs[1].c_str() : nullptr;
        if (d.kind == LayerKind::Conv) {
            const ConvParams& p = d.conv;
            // the C-ABI reads O*I*K*K weights behind one pointer: check the count
            // here (ConvParams::validate's message, tensor.hpp:76-86)
            if (p.weights.size() != (size_t)p.out_channels * p.in_channels * p.kernel_h * p.kernel_w)
                throw Error("conv: weight count does not match dims");
            if (!p.bias.empty() && p.bias.size() != (size_t)p.out_channels)
                throw Error("conv: bias count does not match out_channels");
            if (p.kernel_h != p.kernel_w)
                throw ValidationError("layer '" + d.name + "': the B200 path supports square kernels only");
            o.in_channels = p.in_channels;
            o.out_channels = p.out_channels;
            o.kernel = p.kernel_h;
            o.stride = p.stride;
            o.padding = p.padding;
            o.weights = p.weights.empty() ? nullptr : p.weights.data();
            o.bias = p.bias.empty() ? nullptr : p.bias.data();
        }
        o.pool_k = d.pool_k;
        o.pool_stride = d.pool_stride;
        o.factor = d.factor;
        o.bn_channels = (int)d.bn_scale.size();
        o.bn_scale = d.bn_scale.empty() ? nullptr : d.bn_scale.data();
        o.bn_shift = d.bn_shift.empty() ? nullptr : d.bn_shift.data();
        o.has_threshold = d.threshold.has_value() ? 1 : 0;
        o.threshold = d.threshold.value_or(0.0f);
        o.truncate_enabled = d.truncate_enabled ? 1 : 0;
        return o;
    }
    size_t out_capacity(const Tensor& frame) const {
        int ch = frame.channels;
        for (const LayerDef& d : spec_.layers)
            if (d.kind == LayerKind::Conv && d.conv.out_channels > ch) ch = d.conv.out_channels;
        const size_t t = (size_t)cfg_.tile_size;
        return (size_t)ch * (frame.height + 2 * t) * (frame.width + 2 * t);
    }

    NetworkSpec spec_;  // owns the strings / weights the descriptors point into during create
    EngineConfig cfg_;
    dfx_engine* e_ = nullptr;
    int64_t frame_index_ = 0;
};

}  // namespace dflx
