// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into or called by the
// product path. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load the library built from this
// file (oracle/_ref/libdfxref.so).
//
// A thin C-ABI over the UNMODIFIED reference engine (dflx::DeltaEngine,
// /root/reference/proj/src, compiled from the sources where they lie by
// oracle/Makefile). It exposes the same entry points as include/dfx_b200.h
// under the dfr_ prefix, so the parity tests drive the reference, the C
// restatement (oracle/dfx_oracle.c, dfo_ prefix) and the CUDA product
// (dfx_ prefix) through one interface.

#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "deltaflux/engine.hpp"
#include "deltaflux/synth.hpp"
#include "dfx_b200.h"

using namespace dflx;

namespace {

thread_local std::string g_err;

int fail_with(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ValidationError*>(&e)) return DFX_ERR_VALIDATION;
    if (dynamic_cast<const IoError*>(&e)) return DFX_ERR_IO;
    return DFX_ERR;
}

struct StoredPacket {
    int c = 0, gh = 0, gw = 0, halo = 0, th = 0, tw = 0;
    std::vector<float> data;
    std::vector<uint8_t> mask;
};

struct RefEngine {
    std::unique_ptr<DeltaEngine> eng;
    std::map<std::string, StoredPacket> packets;
    FrameResult last;
    bool have_last = false;
};

NetworkSpec spec_from(const dfx_net_desc* d) {
    NetworkSpec s;
    s.in_channels = d->in_channels;
    for (int i = 0; i < d->num_layers; ++i) {
        const dfx_layer_desc& L = d->layers[i];
        LayerDef l;
        l.name = L.name ? L.name : "";
        l.kind = static_cast<LayerKind>(L.kind);
        if (L.input0) l.inputs.push_back(L.input0);
        if (L.input1) l.inputs.push_back(L.input1);
        if (l.kind == LayerKind::Conv) {
            l.conv.in_channels = L.in_channels;
            l.conv.out_channels = L.out_channels;
            l.conv.kernel_h = l.conv.kernel_w = L.kernel;
            l.conv.stride = L.stride;
            l.conv.padding = L.padding;
            const size_t n = static_cast<size_t>(L.out_channels) * L.in_channels * L.kernel * L.kernel;
            l.conv.weights.assign(L.weights, L.weights + n);
            if (L.bias) l.conv.bias.assign(L.bias, L.bias + L.out_channels);
        }
        l.pool_k = L.pool_k;
        l.pool_stride = L.pool_stride;
        l.factor = L.factor;
        if (l.kind == LayerKind::BatchNorm) {
            l.bn_scale.assign(L.bn_scale, L.bn_scale + L.bn_channels);
            l.bn_shift.assign(L.bn_shift, L.bn_shift + L.bn_channels);
        }
        if (L.has_threshold) l.threshold = L.threshold;
        l.truncate_enabled = L.truncate_enabled != 0;
        s.layers.push_back(std::move(l));
    }
    return s;
}

EngineConfig cfg_from(const dfx_engine_config* c) {
    EngineConfig e;
    e.tile_size = c->tile_size;
    e.grid_rows = c->grid_rows;
    e.grid_cols = c->grid_cols;
    e.input_threshold = c->input_threshold;
    e.default_threshold = c->default_threshold;
    e.override_net_thresholds = c->override_net_thresholds != 0;
    e.mask_dilation = c->mask_dilation;
    e.roi_enabled = c->roi_enabled != 0;
    e.noise_suppression = c->noise_suppression != 0;
    e.padded_convolutions = c->padded_convolutions != 0;
    return e;
}

void fill_info(const FrameResult& r, dfx_frame_info* info) {
    info->frame_index = r.events.frame_index;
    info->origin_tx = r.place.origin.tx;
    info->origin_ty = r.place.origin.ty;
    info->tiles_h = r.place.tiles_h;
    info->tiles_w = r.place.tiles_w;
    info->fresh = r.events.fresh;
    info->evicted = r.events.evicted;
    info->reset = r.events.reset ? 1 : 0;
    info->dropped_pixels = r.events.dropped_pixels;
    info->update_rate = r.update_rate;
    info->conv_flops = r.flops.total;
    info->dense_flops = r.flops.dense_total;
    info->out_channels = r.output.channels;
    info->out_height = r.output.height;
    info->out_width = r.output.width;
}

const SphericalBuffer* pick_buffer(const DeltaEngine& e, const std::string& layer, int which) {
    if (layer == "input") {
        if (which == DFX_STATE_ACC) return &e.input_state().accumulated;
        if (which == DFX_STATE_TRUNC) return &e.input_state().truncated;
        return nullptr;
    }
    if (const TruncationState* t = e.truncation_state(layer)) {
        if (which == DFX_STATE_ACC) return &t->accumulated;
        if (which == DFX_STATE_TRUNC) return &t->truncated;
        return nullptr;
    }
    if (const MaxPoolState* p = e.maxpool_state(layer)) {
        if (which == DFX_STATE_ACC) return &p->accumulated;
        if (which == DFX_STATE_PREV) return &p->prev_out;
        return nullptr;
    }
    return nullptr;
}

}  // namespace

extern "C" {

const char* dfr_last_error(void) { return g_err.c_str(); }

int dfr_create(const dfx_net_desc* net, const dfx_engine_config* cfg, void** out) {
    try {
        auto* r = new RefEngine;
        r->eng = std::make_unique<DeltaEngine>(spec_from(net), cfg_from(cfg));
        RefEngine* rp = r;
        r->eng->set_observer([rp](const std::string& name, const DeltaPacket& p) {
            StoredPacket& s = rp->packets[name];
            s.c = p.channels();
            s.gh = p.grown_h();
            s.gw = p.grown_w();
            s.halo = p.halo;
            s.th = p.place.tiles_h;
            s.tw = p.place.tiles_w;
            s.data = p.delta.data;
            s.mask = p.mask.bits;
        });
        *out = r;
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

void dfr_destroy(void* e) { delete static_cast<RefEngine*>(e); }

int dfr_run_frame(void* ev, const float* frame, int c, int h, int w, const float* h9,
                  const float* roi, dfx_frame_info* info, float* out, size_t out_cap) {
    try {
        auto* r = static_cast<RefEngine*>(ev);
        Tensor f(c, h, w);
        std::memcpy(f.data.data(), frame, f.size() * sizeof(float));
        Homography H;
        std::memcpy(H.m.data(), h9, 9 * sizeof(float));
        Tensor roi_t;
        if (roi) {
            roi_t = Tensor(1, h, w);
            std::memcpy(roi_t.data.data(), roi, roi_t.size() * sizeof(float));
        }
        r->packets.clear();
        r->last = r->eng->run_frame(f, H, roi ? &roi_t : nullptr);
        r->have_last = true;
        fill_info(r->last, info);
        if (out && out_cap >= r->last.output.size())
            std::memcpy(out, r->last.output.data.data(), r->last.output.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

int dfr_reset(void* ev) {
    try {
        static_cast<RefEngine*>(ev)->eng->reset();
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

int dfr_input_mask(void* ev, uint8_t* out, size_t cap, int* th, int* tw) {
    auto* r = static_cast<RefEngine*>(ev);
    if (!r->have_last) {
        g_err = "no frame";
        return DFX_ERR;
    }
    const TileMask& m = r->last.input_mask;
    *th = m.tiles_h;
    *tw = m.tiles_w;
    if (cap < m.bits.size()) {
        g_err = "mask buffer too small";
        return DFX_ERR;
    }
    std::memcpy(out, m.bits.data(), m.bits.size());
    return 0;
}

int dfr_layer_flops(void* ev, const char* name, uint64_t* flops, uint64_t* dense) {
    auto* r = static_cast<RefEngine*>(ev);
    for (const auto& l : r->last.flops.layers)
        if (l.name == name) {
            *flops = l.flops;
            *dense = l.dense_flops;
            return 0;
        }
    *flops = 0;
    *dense = 0;
    return 0;
}

int dfr_grid(void* ev, int* rows, int* cols) {
    auto* r = static_cast<RefEngine*>(ev);
    const GridSpec g = r->eng->input_grid();
    *rows = g.rows;
    *cols = g.cols;
    return 0;
}

int dfr_read_state(void* ev, const char* layer, int which, float* out, size_t cap, int* c, int* h,
                   int* w) {
    auto* r = static_cast<RefEngine*>(ev);
    const SphericalBuffer* b = pick_buffer(*r->eng, layer, which);
    if (!b) {
        g_err = std::string("no state buffer for layer ") + layer;
        return DFX_ERR;
    }
    *c = b->channels();
    *h = b->spec().pixel_h();
    *w = b->spec().pixel_w();
    if (out) {
        if (cap < b->storage().size()) {
            g_err = "state buffer too small";
            return DFX_ERR;
        }
        std::memcpy(out, b->storage().data(), b->storage().size() * sizeof(float));
    }
    return 0;
}

int dfr_read_packet(void* ev, const char* layer, float* out, size_t cap, int* c, int* gh, int* gw,
                    int* halo, uint8_t* mask, size_t mask_cap) {
    auto* r = static_cast<RefEngine*>(ev);
    auto it = r->packets.find(layer);
    if (it == r->packets.end()) {
        g_err = std::string("no packet for layer ") + layer;
        return DFX_ERR;
    }
    const StoredPacket& s = it->second;
    *c = s.c;
    *gh = s.gh;
    *gw = s.gw;
    *halo = s.halo;
    if (out) {
        if (cap < s.data.size() || mask_cap < s.mask.size()) {
            g_err = "packet buffer too small";
            return DFX_ERR;
        }
        std::memcpy(out, s.data.data(), s.data.size() * sizeof(float));
        std::memcpy(mask, s.mask.data(), s.mask.size());
    }
    return 0;
}

int dfr_read_ledger(void* ev, int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) {
    auto* r = static_cast<RefEngine*>(ev);
    const TileLedger& L = r->eng->ledger();
    const size_t n = static_cast<size_t>(L.rows()) * L.cols();
    if (cap < n) {
        g_err = "ledger buffer too small";
        return DFX_ERR;
    }
    for (int rr = 0; rr < L.rows(); ++rr)
        for (int cc = 0; cc < L.cols(); ++cc) {
            const auto& s = L.slot_local(rr, cc);
            const size_t i = static_cast<size_t>(rr) * L.cols() + cc;
            used[i] = s.used ? 1 : 0;
            ty[i] = s.coord.ty;
            tx[i] = s.coord.tx;
            covered[i] = s.covered ? 1 : 0;
        }
    return 0;
}

// The reference's seeded texture generator (synth.cpp:5-30), used by the
// bench / tests to make identical inputs for every implementation.
int dfr_synth_texture(int c, int h, int w, uint32_t seed, float* out) {
    try {
        std::mt19937 rng(seed);
        const Tensor t = synth_texture(c, h, w, rng);
        std::memcpy(out, t.data.data(), t.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

// CPU baseline: `streams` independent engines (one per host thread, the
// reference's "one engine instance per video stream"), each
// running `frames` frames of its own sequence. Frame f of stream s is
// frames_data[s][f] (c x h x w) with homography h9s[s][f]. Per-frame wall
// seconds are written to secs[s * frames + f].
int dfr_run_streams(const dfx_net_desc* net, const dfx_engine_config* cfg, int streams, int frames,
                    int c, int h, int w, const float* frames_data, const float* h9s, double* secs,
                    uint64_t* flops) {
    try {
        const NetworkSpec spec = spec_from(net);
        const EngineConfig ec = cfg_from(cfg);
        std::vector<std::thread> th;
        std::vector<std::string> errs(streams);
        for (int s = 0; s < streams; ++s) {
            th.emplace_back([&, s] {
                try {
                    DeltaEngine eng(spec, ec);
                    const size_t fsz = static_cast<size_t>(c) * h * w;
                    for (int f = 0; f < frames; ++f) {
                        Tensor t(c, h, w);
                        std::memcpy(t.data.data(), frames_data + (static_cast<size_t>(s) * frames + f) * fsz,
                                    fsz * sizeof(float));
                        Homography H;
                        std::memcpy(H.m.data(), h9s + (static_cast<size_t>(s) * frames + f) * 9,
                                    9 * sizeof(float));
                        const auto t0 = std::chrono::steady_clock::now();
                        const FrameResult r = eng.run_frame(t, H);
                        const auto t1 = std::chrono::steady_clock::now();
                        secs[static_cast<size_t>(s) * frames + f] =
                            std::chrono::duration<double>(t1 - t0).count();
                        if (flops) flops[static_cast<size_t>(s) * frames + f] = r.flops.total;
                    }
                } catch (const std::exception& e) {
                    errs[s] = e.what();
                }
            });
        }
        for (auto& t : th) t.join();
        for (const auto& e : errs)
            if (!e.empty()) {
                g_err = e;
                return DFX_ERR;
            }
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

// Unmodified reference TileLedger / plan_frame / apply_plan (engine semantics
// for the full reset: engine.cpp:207-211), same signatures as dfx_ledger_*.
struct RefLedger {
    TileLedger l;
};
int dfr_ledger_create(int rows, int cols, void** out) {
    try {
        auto* h = new RefLedger;
        h->l = TileLedger(rows, cols);
        *out = h;
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}
int dfr_ledger_destroy(void* h) {
    delete static_cast<RefLedger*>(h);
    return 0;
}
int dfr_ledger_step(void* hv, int64_t otx, int64_t oty, int th, int tw, int ring, int* full_reset, int64_t* claims,
                    int* victims, size_t claim_cap, int* nclaims, int64_t* fresh, size_t fresh_cap, int* nfresh,
                    int* evicted) {
    try {
        auto* h = static_cast<RefLedger*>(hv);
        FramePlacement place;
        place.origin = TileCoord{otx, oty};
        place.tiles_h = th;
        place.tiles_w = tw;
        FramePlan plan = plan_frame(h->l, place, ring);
        *full_reset = plan.needs_full_reset ? 1 : 0;
        if (plan.needs_full_reset) {
            h->l.clear();
            plan = plan_frame(h->l, place, ring);
        }
        apply_plan(plan, h->l, [](const TileCoord&) {});
        *nclaims = (int)plan.claims.size();
        *nfresh = (int)plan.fresh_tiles.size();
        *evicted = (int)plan.evicted_tiles.size();
        for (size_t i = 0; i < plan.claims.size() && i < claim_cap; ++i) {
            claims[4 * i] = plan.claims[i].coord.tx;
            claims[4 * i + 1] = plan.claims[i].coord.ty;
            claims[4 * i + 2] = plan.claims[i].evicts ? plan.claims[i].evicts->tx : 0;
            claims[4 * i + 3] = plan.claims[i].evicts ? plan.claims[i].evicts->ty : 0;
            victims[i] = plan.claims[i].evicts ? 1 : 0;
        }
        for (size_t i = 0; i < plan.fresh_tiles.size() && i < fresh_cap; ++i) {
            fresh[2 * i] = plan.fresh_tiles[i].tx;
            fresh[2 * i + 1] = plan.fresh_tiles[i].ty;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}
int dfr_ledger_slots(void* hv, int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) {
    auto* h = static_cast<RefLedger*>(hv);
    const size_t n = (size_t)h->l.rows() * h->l.cols();
    if (cap < n) return DFX_ERR;
    for (int r = 0; r < h->l.rows(); ++r)
        for (int c = 0; c < h->l.cols(); ++c) {
            const auto& s = h->l.slot_local(r, c);
            const size_t i = (size_t)r * h->l.cols() + c;
            used[i] = s.used ? 1 : 0;
            ty[i] = s.coord.ty;
            tx[i] = s.coord.tx;
            covered[i] = s.covered ? 1 : 0;
        }
    return 0;
}

}  // extern "C"

// ---------------------------------------------------------------- layer level
// The reference's free layer functions (delta_layers.hpp:103-127) on host
// buffers in its own layouts, for tests/test_gpu_layers.py: packets as dense
// grown CHW + TileMask bytes, states as wrapped CHW planar storage, the slot
// filter from a rows*cols dfx_slot table (TileLedger::holds semantics).
namespace {

DeltaPacket packet_from(const dfx_placement* pl, int tile, int halo, int C, const float* chw, const uint8_t* mask) {
    FramePlacement p;
    p.origin = TileCoord{pl->origin_tx, pl->origin_ty};
    p.tiles_h = pl->tiles_h;
    p.tiles_w = pl->tiles_w;
    DeltaPacket k = make_packet(p, tile, tile, C, halo);
    std::memcpy(k.delta.data.data(), chw, k.delta.size() * sizeof(float));
    for (size_t i = 0; i < k.mask.bits.size(); ++i) k.mask.bits[i] = mask[i] ? 1 : 0;
    return k;
}

void packet_to(const DeltaPacket& k, float* chw, uint8_t* mask, int* halo) {
    std::memcpy(chw, k.delta.data.data(), k.delta.size() * sizeof(float));
    for (size_t i = 0; i < k.mask.bits.size(); ++i) mask[i] = k.mask.bits[i];
    if (halo) *halo = k.halo;
}

SphericalBuffer buffer_from(int rows, int cols, int tile, int C, const float* chw) {
    SphericalBuffer b(GridSpec{tile, tile, rows, cols}, C);
    const int PH = rows * tile, PW = cols * tile;
    for (int c = 0; c < C; ++c)
        for (int y = 0; y < PH; ++y)
            for (int x = 0; x < PW; ++x) b.at_global(c, y, x) = chw[((size_t)c * PH + y) * PW + x];
    return b;
}

void buffer_to(const SphericalBuffer& b, float* chw) {
    std::memcpy(chw, b.storage().data(), b.storage().size() * sizeof(float));
}

SlotFilter filter_from(const dfx_slot* slots, int rows, int cols) {
    if (!slots) return {};
    std::vector<dfx_slot> s(slots, slots + (size_t)rows * cols);
    return [s, rows, cols](const TileCoord& t) {
        const dfx_slot& q = s[(size_t)floor_mod(t.ty, rows) * cols + floor_mod(t.tx, cols)];
        return q.used && q.tx == t.tx && q.ty == t.ty;
    };
}

}  // namespace

extern "C" {

int dfr_layer_conv(const dfx_placement* pl, int tile, int halo, int C, const float* chw, const uint8_t* mask,
                   const float* w, int cout, int k, int stride, float* out_chw, uint8_t* out_mask, int* out_halo,
                   uint64_t* flops) {
    try {
        const DeltaPacket in = packet_from(pl, tile, halo, C, chw, mask);
        ConvParams p;
        p.in_channels = C;
        p.out_channels = cout;
        p.kernel_h = p.kernel_w = k;
        p.stride = stride;
        p.padding = k / 2;
        p.weights.assign(w, w + (size_t)cout * C * k * k);
        FlopReport fr;
        const DeltaPacket out = padded_delta_conv(in, p, &fr, "conv");
        packet_to(out, out_chw, out_mask, out_halo);
        flops[0] = fr.total;
        flops[1] = fr.dense_total;
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

int dfr_layer_truncate(const dfx_placement* pl, int rows, int cols, int tile, int halo, int C, const float* chw,
                       const uint8_t* mask, float* acc, float* trunc, float thr, int relu, const dfx_slot* slots,
                       float* out_chw, uint8_t* out_mask) {
    try {
        const DeltaPacket in = packet_from(pl, tile, halo, C, chw, mask);
        TruncationState st(GridSpec{tile, tile, rows, cols}, C, thr);
        st.accumulated = buffer_from(rows, cols, tile, C, acc);
        st.truncated = buffer_from(rows, cols, tile, C, trunc);
        const DeltaPacket out = delta_activation_truncate(in, st, relu ? ActKind::Relu : ActKind::Identity,
                                                          filter_from(slots, rows, cols));
        packet_to(out, out_chw, out_mask, nullptr);
        buffer_to(st.accumulated, acc);
        buffer_to(st.truncated, trunc);
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

int dfr_layer_maxpool(const dfx_placement* pl, int rows, int cols, int tile, int halo, int C, const float* chw,
                      const uint8_t* mask, float* acc, float* prev, int k, const dfx_slot* slots, float* out_chw,
                      uint8_t* out_mask, int* out_halo) {
    try {
        const DeltaPacket in = packet_from(pl, tile, halo, C, chw, mask);
        MaxPoolState st(GridSpec{tile, tile, rows, cols}, GridSpec{tile / k, tile / k, rows, cols}, C, k, k, 0);
        st.accumulated = buffer_from(rows, cols, tile, C, acc);
        st.prev_out = buffer_from(rows, cols, tile / k, C, prev);
        const DeltaPacket out = delta_maxpool(in, st, filter_from(slots, rows, cols));
        packet_to(out, out_chw, out_mask, out_halo);
        buffer_to(st.accumulated, acc);
        buffer_to(st.prev_out, prev);
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

int dfr_layer_densify(const dfx_placement* pl, int rows, int cols, int tile, int C, const float* acc,
                      const float* trunc, float* out) {
    try {
        TruncationState st(GridSpec{tile, tile, rows, cols}, C, 0.0f);
        st.accumulated = buffer_from(rows, cols, tile, C, acc);
        st.truncated = buffer_from(rows, cols, tile, C, trunc);
        FramePlacement p;
        p.origin = TileCoord{pl->origin_tx, pl->origin_ty};
        p.tiles_h = pl->tiles_h;
        p.tiles_w = pl->tiles_w;
        const Tensor t = densify(st, p);
        std::memcpy(out, t.data.data(), t.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}

}  // extern "C"

extern "C" {
// dflx::save_network (network.cpp:425-500): JSON + one DFLX file per weight
// tensor (the reference's on-disk format), for the loader tests.
int dfr_save_network(const dfx_net_desc* net, const char* path) {
    try {
        save_network(spec_from(net), path);
        return 0;
    } catch (const std::exception& e) {
        return fail_with(e);
    }
}
}  // extern "C"
