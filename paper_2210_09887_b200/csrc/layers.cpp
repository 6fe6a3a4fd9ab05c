// Layer-level C-ABI (include/dfx_b200.h, "layer level"): the reference's
// per-layer functions (delta_layers.hpp:103-127) and the input stage / claim
// reset of its engine (engine.cpp:78-182) as stream-ordered calls on device
// buffers. Each call runs the SAME kernels the engine launches for that layer
// (kernels.cu, kernels_hbm.cu, conv_tc.cu); only the per-frame parameter block
// (placement, slot table, owned map) comes from dfx_layer_ctx_set_frame instead
// of the engine's ledger. Convolutions take the gathered-target tensor-core
// kernel k_conv_tc (any stride) or k_conv_exact; the engine's dense-unit plan
// (conv_dense.cu) needs per-layer persistent plan state and stays engine-only.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "dfx_b200.h"
#include "host.hpp"
#include "kernels.hpp"

namespace dfx {
namespace {

#define LCHECK(x)                                                                                       \
    do {                                                                                                \
        cudaError_t _e = (x);                                                                           \
        if (_e != cudaSuccess) ::dfx::fail(std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x, DFX_ERR_CUDA); \
    } while (0)

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    void need(size_t count) {
        if (count <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        LCHECK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

struct LayerCtx {
    int rows = 0, cols = 0, device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool have_frame = false;
    FrameDev F{};
    DBuf<uint8_t> params;  // FrameDev | SlotDev[rows*cols] | own[rows*cols]
    size_t off_slots = 0, off_own = 0;
    DBuf<unsigned> tmax, gbar;
    DBuf<unsigned long long> counter;
    DBuf<int> list, count, claims;
    DBuf<float> wsplit, ws, canvas, fac;
    DBuf<uint8_t> bytes, canvas_valid, cov, sig, sig2, gate, fresh;
    DBuf<ClaimBuf> cbufs;

    Ctx ctx() const {
        return Ctx{reinterpret_cast<const FrameDev*>(params.p), reinterpret_cast<const SlotDev*>(params.p + off_slots),
                   rows, cols, params.p + off_own};
    }
    void use() const { LCHECK(cudaSetDevice(device)); }
    void need_frame() const { check(have_frame, "layer ctx: no frame set (dfx_layer_ctx_set_frame)"); }
    int RT(int t, int halo) const { return (halo + t - 1) / t; }
    PktDev pkt(const dfx_packet* p) const {
        check(p && p->d && p->ext && p->channels >= 1 && p->tile >= 1 && p->halo >= 0, "layer: bad packet");
        PktDev d;
        d.d = p->d;
        d.ext = p->ext;
        d.C = p->channels;
        d.t = p->tile;
        d.halo = p->halo;
        d.RT = RT(p->tile, p->halo);
        d.pitch_w = cols * p->tile + 2 * p->halo;
        d.ext_pitch = cols + 2 * d.RT;
        return d;
    }
    BufDev buf(const dfx_state* s) const {
        check(s && s->d && s->channels >= 1 && s->tile >= 1, "layer: bad state");
        return BufDev{s->d, s->channels, s->tile};
    }
    void sync() const { LCHECK(cudaStreamSynchronize(stream)); }
};

}  // namespace dfx

using dfx::LayerCtx;
struct dfx_layer_ctx {
    LayerCtx c;
};

namespace dfx {
void set_last_error(const std::string& m);  // engine.cpp: the message dfx_last_error() returns
}  // namespace dfx

namespace {
template <typename F>
int lguard(F&& f) {
    try {
        f();
        return DFX_OK;
    } catch (const dfx::Error& e) {
        dfx::set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        dfx::set_last_error(e.what());
        return DFX_ERR;
    }
}
}  // namespace

extern "C" {

int dfx_layer_ctx_create(int rows, int cols, int device, void* stream, dfx_layer_ctx** out) {
    return lguard([&] {
        dfx::check(rows >= 1 && cols >= 1, "layer ctx: bad grid dims");
        int ndev = 0;
        const cudaError_t de = cudaGetDeviceCount(&ndev);
        if (de != cudaSuccess) cudaGetLastError();
        if (de != cudaSuccess || ndev <= 0)
            dfx::fail("no CUDA device (the B200 path has no CPU fallback)", DFX_ERR_CUDA);
        auto* h = new dfx_layer_ctx;
        LayerCtx& c = h->c;
        c.rows = rows;
        c.cols = cols;
        c.device = device;
        try {
            c.use();
            if (stream) {
                c.stream = static_cast<cudaStream_t>(stream);
            } else {
                LCHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
                c.own_stream = true;
            }
            const size_t slots = (size_t)rows * cols;
            c.off_slots = (sizeof(dfx::FrameDev) + 15) / 16 * 16;
            c.off_own = c.off_slots + slots * sizeof(dfx::SlotDev);
            c.params.need(c.off_own + slots);
            c.tmax.need(slots);
            c.gbar.need(4);
            c.counter.need(1);
            c.count.need(1);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int dfx_layer_ctx_destroy(dfx_layer_ctx* h) {
    return lguard([&] {
        if (!h) return;
        cudaSetDevice(h->c.device);
        cudaStreamSynchronize(h->c.stream);
        if (h->c.own_stream) cudaStreamDestroy(h->c.stream);
        delete h;
    });
}

int dfx_layer_ctx_set_frame(dfx_layer_ctx* h, const dfx_placement* pl, const dfx_slot* slots) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        dfx::check(pl && pl->tiles_h >= 1 && pl->tiles_w >= 1, "layer ctx: bad placement");
        dfx::check(pl->tiles_h <= c.rows && pl->tiles_w <= c.cols, "plan_frame: placement larger than grid");
        dfx::FrameDev F{};
        F.otx = pl->origin_tx;
        F.oty = pl->origin_ty;
        F.th = pl->tiles_h;
        F.tw = pl->tiles_w;
        F.base_sr = (int)dfx::floor_mod64(F.oty, c.rows);
        F.base_sc = (int)dfx::floor_mod64(F.otx, c.cols);
        const size_t ns = (size_t)c.rows * c.cols;
        std::vector<uint8_t> blk(c.off_own + ns, 0);
        dfx::SlotDev* hs = reinterpret_cast<dfx::SlotDev*>(blk.data() + c.off_slots);
        if (slots) {
            for (size_t i = 0; i < ns; ++i) hs[i] = dfx::SlotDev{slots[i].tx, slots[i].ty, slots[i].used ? 1 : 0, 1};
        } else {
            // no slot filter given: the slots hold the placement grown by
            // floor((rows - th) / 2) tiles above (the rest below), likewise in x
            // (the engine's ledger on a static camera with that ring)
            const int64_t y0 = F.oty - (c.rows - F.th) / 2, x0 = F.otx - (c.cols - F.tw) / 2;
            for (int64_t ty = y0; ty < y0 + c.rows; ++ty)
                for (int64_t tx = x0; tx < x0 + c.cols; ++tx) {
                    const size_t i = (size_t)dfx::floor_mod64(ty, c.rows) * c.cols + dfx::floor_mod64(tx, c.cols);
                    hs[i] = dfx::SlotDev{tx, ty, 1, 1};
                }
        }
        uint8_t* own = blk.data() + c.off_own;
        for (int r = 0; r < F.th; ++r)
            for (int q = 0; q < F.tw; ++q) {
                const int64_t ty = F.oty + r, tx = F.otx + q;
                const dfx::SlotDev& s =
                    hs[(size_t)dfx::floor_mod64(ty, c.rows) * c.cols + dfx::floor_mod64(tx, c.cols)];
                own[r * F.tw + q] = (s.used && s.tx == tx && s.ty == ty) ? 1 : 0;
            }
        memcpy(blk.data(), &F, sizeof F);
        LCHECK(cudaMemcpyAsync(c.params.p, blk.data(), blk.size(), cudaMemcpyHostToDevice, c.stream));
        LCHECK(cudaStreamSynchronize(c.stream));  // blk is a host temporary
        c.F = F;
        c.have_frame = true;
    });
}

size_t dfx_packet_floats(const dfx_layer_ctx* h, int channels, int tile, int halo) {
    const LayerCtx& c = h->c;
    return (size_t)(c.rows * tile + 2 * halo) * (c.cols * tile + 2 * halo) * channels;
}
size_t dfx_packet_ext_bytes(const dfx_layer_ctx* h, int tile, int halo) {
    const LayerCtx& c = h->c;
    const int RT = (halo + tile - 1) / tile;
    return (size_t)(c.rows + 2 * RT) * (c.cols + 2 * RT);
}
size_t dfx_state_floats(const dfx_layer_ctx* h, int channels, int tile) {
    return (size_t)h->c.rows * tile * h->c.cols * tile * channels;
}

int dfx_packet_from_chw(dfx_layer_ctx* h, const float* chw, const uint8_t* mask, dfx_packet* out) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::PktDev p = c.pkt(out);
        const size_t nt = (size_t)c.F.th * c.F.tw;
        c.bytes.need(nt);
        LCHECK(cudaMemsetAsync(p.ext, 0, dfx_packet_ext_bytes(h, p.t, p.halo), c.stream));
        LCHECK(cudaMemcpyAsync(c.bytes.p, mask, nt, cudaMemcpyHostToDevice, c.stream));
        dfx::launch_pkt_from_chw(c.stream, chw, c.bytes.p, c.F.th, c.F.tw, p);
        LCHECK(cudaGetLastError());
        c.sync();  // `mask` is a caller host buffer
    });
}

int dfx_packet_to_chw(dfx_layer_ctx* h, const dfx_packet* in, float* chw, uint8_t* mask) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::PktDev p = c.pkt(in);
        const size_t nt = (size_t)c.F.th * c.F.tw;
        c.bytes.need(nt);
        dfx::launch_pkt_to_chw(c.stream, p, c.F.th, c.F.tw, chw, c.bytes.p);
        LCHECK(cudaGetLastError());
        if (mask) LCHECK(cudaMemcpyAsync(mask, c.bytes.p, nt, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int dfx_state_from_chw(dfx_layer_ctx* h, const float* chw, dfx_state* out) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        const dfx::BufDev b = c.buf(out);
        dfx::launch_state_convert(c.stream, chw, b.d, b.C, b.t, c.rows, c.cols, 0);
        LCHECK(cudaGetLastError());
    });
}

int dfx_state_to_chw(dfx_layer_ctx* h, const dfx_state* s, float* chw) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        const dfx::BufDev b = c.buf(s);
        dfx::launch_state_convert(c.stream, b.d, chw, b.C, b.t, c.rows, c.cols, 1);
        LCHECK(cudaGetLastError());
    });
}

int dfx_delta_conv_out_halo(int in_halo, int kernel, int stride) {
    return dfx::windowed_out_halo(in_halo, kernel, kernel / 2, stride);
}

// padded_delta_conv (delta_layers.cpp:100-147): target compaction + zero fill
// (k_conv_targets), then the gathered tensor-core conv (k_conv_tc, 3xTF32) or
// the CUDA-core conv in the reference's summation order (k_conv_exact).
int dfx_delta_conv(dfx_layer_ctx* h, const dfx_packet* in, const float* weights, int cin, int cout, int k, int stride,
                   int conv_mode, dfx_packet* out, uint64_t* flops) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::PktDev a = c.pkt(in);
        dfx::check(cin == a.C, "conv: expects " + std::to_string(cin) + " channels, gets " + std::to_string(a.C));
        dfx::check(k >= 1 && (k & 1) && stride >= 1 && cout >= 1, "conv: bad kernel / stride / channels");
        dfx::check(a.t % stride == 0, "conv: stride misaligned with tile");
        dfx::check(weights != nullptr, "conv: no weights");
        const int hg = dfx::windowed_out_halo(a.halo, k, k / 2, stride);
        dfx::check(out && out->channels == cout && out->tile == a.t / stride && out->halo == hg,
                   "conv: output packet must have cout channels, tile / stride and halo dfx_delta_conv_out_halo()");
        const dfx::PktDev o = c.pkt(out);
        const int max_targets = (c.rows * o.t + 2 * hg) * (c.cols * o.t + 2 * hg);
        c.list.need((size_t)max_targets);
        LCHECK(cudaMemsetAsync(o.ext, 0, dfx_packet_ext_bytes(h, o.t, o.halo), c.stream));
        LCHECK(cudaMemsetAsync(c.count.p, 0, sizeof(int), c.stream));
        LCHECK(cudaMemsetAsync(c.counter.p, 0, sizeof(unsigned long long), c.stream));
        const dfx::Ctx C = c.ctx();
        dfx::launch_conv_targets(C, c.stream, a, k, stride, k / 2, o, hg, c.list.p, c.count.p, c.counter.p);
        if (conv_mode == DFX_CONV_EXACT || !dfx::conv_tc_supported(k)) {
            dfx::launch_conv_exact(C, c.stream, a, weights, cin, cout, k, stride, k / 2, o, hg, c.list.p, c.count.p,
                                   max_targets);
        } else {
            const int cin_pad = (cin + 7) / 8 * 8, cout_pad = (cout + 15) / 16 * 16;
            std::vector<float> w((size_t)cout * cin * k * k);
            LCHECK(cudaMemcpyAsync(w.data(), weights, w.size() * 4, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            std::vector<float> ws(dfx::conv_tc_weight_floats(cin_pad, cout_pad, k));
            dfx::conv_tc_prepare_weights(w.data(), cin, cout, k, cin_pad, cout_pad, ws.data());
            c.wsplit.need(ws.size());
            LCHECK(cudaMemcpyAsync(c.wsplit.p, ws.data(), ws.size() * 4, cudaMemcpyHostToDevice, c.stream));
            int sms = 148;
            LCHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
            const int splits = dfx::conv_tc_splits(max_targets, cin_pad, cout_pad, k, sms);
            if (splits > 1) c.ws.need((size_t)splits * max_targets * cout_pad);
            dfx::launch_conv_tc(C, c.stream, a, c.wsplit.p, cin, cin_pad, cout, cout_pad, k, stride, k / 2, o, hg,
                                c.list.p, c.count.p, max_targets, sms, c.ws.p, splits);
            c.sync();  // `ws` (host) lives until the upload completed
        }
        LCHECK(cudaGetLastError());
        if (flops) {
            unsigned long long px = 0;
            LCHECK(cudaMemcpyAsync(&px, c.counter.p, sizeof px, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            const uint64_t per = 2ull * k * k * cin * cout;
            flops[0] = per * px;
            flops[1] = per * (uint64_t)(c.F.th * o.t) * (uint64_t)(c.F.tw * o.t);
        }
    });
}

// delta_activation_truncate (delta_layers.cpp:149-232): halo stash, tile max,
// fire / fold, exactly the engine's launch sequence for a truncation layer.
int dfx_delta_truncate(dfx_layer_ctx* h, const dfx_packet* in, dfx_state* acc, dfx_state* trunc, float thr, int relu,
                       dfx_packet* out) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::PktDev a = c.pkt(in);
        const dfx::BufDev A = c.buf(acc), T = c.buf(trunc);
        dfx::check(A.C == a.C && T.C == a.C && A.t == a.t && T.t == a.t, "truncate: state shape mismatch");
        dfx::check(out && out->channels == a.C && out->tile == a.t && out->halo == 0,
                   "truncate: output packet must have the input's channels / tile and halo 0");
        const dfx::PktDev o = c.pkt(out);
        LCHECK(cudaMemsetAsync(o.ext, 0, dfx_packet_ext_bytes(h, o.t, 0), c.stream));
        LCHECK(cudaMemsetAsync(c.tmax.p, 0, (size_t)c.rows * c.cols * sizeof(unsigned), c.stream));
        LCHECK(cudaMemsetAsync(c.gbar.p, 0, 4 * sizeof(unsigned), c.stream));
        const dfx::Ctx C = c.ctx();
        if (a.halo > 0 && (a.C & 3) != 0) dfx::launch_ring_add(C, c.stream, a, T);
        if (!dfx::launch_trunc_two_pass(C, c.stream, a, A, T, c.tmax.p, thr, relu ? 1 : 0, o, c.gbar.p)) {
            dfx::launch_trunc_max(C, c.stream, a, T, c.tmax.p);
            dfx::launch_trunc_apply(C, c.stream, a, A, T, c.tmax.p, thr, relu ? 1 : 0, o);
        }
        LCHECK(cudaGetLastError());
    });
}

// delta_maxpool (delta_layers.cpp:234-318), the engine's three launch forms.
int dfx_delta_maxpool(dfx_layer_ctx* h, const dfx_packet* in, dfx_state* acc, dfx_state* prev, int k, dfx_packet* out) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::PktDev a = c.pkt(in);
        dfx::check(k >= 1 && a.t % k == 0, "maxpool: stride misaligned with tile");
        const dfx::BufDev A = c.buf(acc), P = c.buf(prev);
        const int hg = dfx::windowed_out_halo(a.halo, k, 0, k);
        dfx::check(A.C == a.C && A.t == a.t && P.C == a.C && P.t == a.t / k, "maxpool: state shape mismatch");
        dfx::check(out && out->channels == a.C && out->tile == a.t / k && out->halo == hg,
                   "maxpool: output packet must have the input's channels, tile / k and halo "
                   "windowed_out_halo(halo, k, 0, k)");
        const dfx::PktDev o = c.pkt(out);
        LCHECK(cudaMemsetAsync(o.ext, 0, dfx_packet_ext_bytes(h, o.t, o.halo), c.stream));
        const dfx::Ctx C = c.ctx();
        if (a.halo == 0 && (a.C & 3) == 0) {
            dfx::launch_maxpool_vec(C, c.stream, a, A, P, k, o);
        } else if (a.halo == 0) {
            dfx::launch_maxpool_fused(C, c.stream, a, A, P, k, o);
        } else {
            dfx::launch_tile_add(C, c.stream, a, A);
            dfx::launch_ring_add(C, c.stream, a, A);
            dfx::launch_maxpool_out(C, c.stream, a, A, P, k, k, o, hg);
        }
        LCHECK(cudaGetLastError());
    });
}

int dfx_densify(dfx_layer_ctx* h, const dfx_state* acc, const dfx_state* trunc, float* out) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::BufDev A = c.buf(acc), T = c.buf(trunc);
        dfx::check(A.C == T.C && A.t == T.t, "densify: state shape mismatch");
        dfx::launch_densify(c.ctx(), c.stream, A, T, out, dfx::Readback{});
        LCHECK(cudaGetLastError());
    });
}

int dfx_claim_reset(dfx_layer_ctx* h, const int64_t* coords, int nclaims, dfx_state* const* states,
                    const float* const* fills, int nstates) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        dfx::check(nclaims >= 0 && nclaims <= c.rows * c.cols, "claims: bad claim count");
        if (nclaims == 0 || nstates <= 0) return;
        std::vector<int> slots(nclaims);
        for (int i = 0; i < nclaims; ++i)
            slots[i] = (int)(dfx::floor_mod64(coords[2 * i + 1], c.rows) * c.cols + dfx::floor_mod64(coords[2 * i], c.cols));
        std::vector<dfx::ClaimBuf> cb(nstates);
        for (int b = 0; b < nstates; ++b) {
            const dfx::BufDev s = c.buf(states[b]);
            cb[b] = dfx::ClaimBuf{s.d, fills ? fills[b] : nullptr, s.C, s.t};
        }
        c.claims.need((size_t)nclaims);
        c.cbufs.need((size_t)nstates);
        dfx::FrameDev F = c.F;
        F.nclaims = nclaims;
        LCHECK(cudaMemcpyAsync(c.claims.p, slots.data(), slots.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
        LCHECK(cudaMemcpyAsync(c.cbufs.p, cb.data(), cb.size() * sizeof(dfx::ClaimBuf), cudaMemcpyHostToDevice,
                               c.stream));
        LCHECK(cudaMemcpyAsync(c.params.p, &F, sizeof F, cudaMemcpyHostToDevice, c.stream));
        dfx::launch_claims(c.ctx(), c.stream, nullptr, c.claims.p, nullptr, c.cbufs.p, nstates, nclaims);
        F.nclaims = 0;
        LCHECK(cudaMemcpyAsync(c.params.p, &F, sizeof F, cudaMemcpyHostToDevice, c.stream));
        LCHECK(cudaGetLastError());
        c.sync();  // host vectors / F are temporaries
    });
}

// compute_input_delta + input_gate + gated truncation (alignment.cpp:168-192,
// engine.cpp:110-182, 233-237): the engine's unfused input kernels on a
// caller-aligned canvas.
int dfx_input_stage(dfx_layer_ctx* h, const float* aligned, const uint8_t* valid, const float* roi_factor,
                    const uint8_t* fresh, float thr, int dilation, int noise, dfx_state* acc, dfx_state* trunc,
                    dfx_packet* out, double* update_rate) {
    return lguard([&] {
        LayerCtx& c = h->c;
        c.use();
        c.need_frame();
        const dfx::BufDev A = c.buf(acc), T = c.buf(trunc);
        dfx::check(A.C == T.C && A.t == T.t, "input stage: state shape mismatch");
        dfx::check(out && out->channels == A.C && out->tile == A.t && out->halo == 0,
                   "input stage: output packet must have the state's channels / tile and halo 0");
        dfx::check(dilation >= 0 && thr >= 0.0f, "input stage: bad threshold / dilation");
        const dfx::PktDev o = c.pkt(out);
        const int Tt = A.t, C = A.C, pitch = c.cols * Tt;
        const int eh = c.F.th * Tt, ew = c.F.tw * Tt;
        const size_t canvas_px = (size_t)c.rows * Tt * pitch, nt = (size_t)c.F.th * c.F.tw;
        c.canvas.need(canvas_px * C);
        c.canvas_valid.need(canvas_px);
        c.sig.need(canvas_px);
        c.sig2.need(canvas_px);
        c.cov.need((size_t)c.rows * c.cols);
        c.gate.need((size_t)c.rows * c.cols);
        c.fresh.need((size_t)c.rows * c.cols);
        dfx::launch_canvas_from_chw(c.stream, aligned, C, eh, ew, c.canvas.p, pitch);
        LCHECK(cudaMemcpy2DAsync(c.canvas_valid.p, pitch, valid, ew, ew, eh, cudaMemcpyDeviceToDevice, c.stream));
        const float* fac = nullptr;
        if (roi_factor) {
            c.fac.need(canvas_px);
            LCHECK(cudaMemcpy2DAsync(c.fac.p, (size_t)pitch * 4, roi_factor, (size_t)ew * 4, (size_t)ew * 4, eh,
                                     cudaMemcpyDeviceToDevice, c.stream));
            fac = c.fac.p;
        }
        std::vector<uint8_t> fr(nt, 0);
        if (fresh) memcpy(fr.data(), fresh, nt);
        LCHECK(cudaMemcpyAsync(c.fresh.p, fr.data(), nt, cudaMemcpyHostToDevice, c.stream));
        LCHECK(cudaMemsetAsync(o.ext, 0, dfx_packet_ext_bytes(h, o.t, 0), c.stream));
        const dfx::Ctx X = c.ctx();
        dfx::launch_coverage(X, c.stream, c.canvas_valid.p, pitch, Tt, c.cov.p);
        dfx::launch_input_sig(X, c.stream, c.canvas.p, c.cov.p, A, T, fac, thr, pitch, Tt, c.sig.p);
        const uint8_t* sig = c.sig.p;
        if (noise) {
            dfx::launch_noise(X, c.stream, c.sig.p, c.sig2.p, pitch, Tt);
            sig = c.sig2.p;
        }
        dfx::launch_gate(X, c.stream, sig, c.cov.p, c.fresh.p, dilation, pitch, Tt, c.gate.p);
        dfx::launch_input_apply(X, c.stream, c.canvas.p, c.cov.p, c.gate.p, A, T, o, pitch);
        LCHECK(cudaGetLastError());
        std::vector<uint8_t> ext(dfx_packet_ext_bytes(h, o.t, 0));
        LCHECK(cudaMemcpyAsync(ext.data(), o.ext, ext.size(), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (update_rate) {
            int n = 0;
            for (int r = 0; r < c.F.th; ++r)
                for (int q = 0; q < c.F.tw; ++q) n += ext[(size_t)r * o.ext_pitch + q] ? 1 : 0;
            *update_rate = (double)n / ((double)c.F.th * c.F.tw);
        }
    });
}

}  // extern "C"
