// B200 delta engine: host orchestrator + C-ABI (include/dfx_b200.h).
//
// Mirrors dflx::DeltaEngine (reference include/deltaflux/engine.hpp:45-91,
// src/engine.cpp:7-287): per frame it factors the homography, snaps the frame
// to the tile grid, plans the ledger on the host (integer work), uploads one
// per-frame parameter block, and launches the device pipeline
//   claims reset/bias -> input stage -> per layer (conv | truncate | pool |
//   linear ops) -> densify
// on one CUDA stream. Every per-frame value the kernels need is read on device
// from the uploaded FrameDev block, so the launch sequence is shape-stable.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "dfx_b200.h"
#include "host.hpp"
#include "kernels.hpp"

namespace dfx {

namespace {

thread_local std::string g_err;

#define PROF(fam, call)                \
    do {                               \
        const int _pi = prof_begin(fam); \
        call;                          \
        prof_end(_pi);                 \
        ++launches_;                   \
    } while (0)

#define CUDA_CHECK(x)                                                                                  \
    do {                                                                                               \
        cudaError_t _e = (x);                                                                          \
        if (_e != cudaSuccess) fail(std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x, DFX_ERR_CUDA); \
    } while (0)

int64_t fdiv(int64_t a, int64_t n) { return floor_div64(a, n); }
int64_t cdiv(int64_t a, int64_t n) { return ceil_div64(a, n); }

template <typename T>
struct DevArr {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        release();
        n = count;
        if (count) {
            cudaError_t e = cudaMalloc(&p, count * sizeof(T));
            if (e != cudaSuccess) fail(std::string("CUDA malloc: ") + cudaGetErrorString(e), DFX_ERR_CUDA);
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevArr() { release(); }
    DevArr() = default;
    DevArr(const DevArr&) = delete;
    DevArr& operator=(const DevArr&) = delete;
    DevArr(DevArr&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DevArr& operator=(DevArr&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n, o.p = nullptr, o.n = 0;
        }
        return *this;
    }
};

// ---- homography (alignment.cpp:5-56), host double / float exactly as the reference
void hom_compose(const float* m, const float* inner, float* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += (double)m[i * 3 + k] * inner[k * 3 + j];
            r[i * 3 + j] = (float)s;
        }
    if (r[8] != 0.0f && r[8] != 1.0f) {
        const float d = r[8];
        for (int i = 0; i < 8; ++i) r[i] /= d;
        r[8] /= r[8];
    }
}
void hom_inverse(const float* a, float* r) {
    const double d = (double)a[0] * ((double)a[4] * a[8] - (double)a[5] * a[7]) -
                     (double)a[1] * ((double)a[3] * a[8] - (double)a[5] * a[6]) +
                     (double)a[2] * ((double)a[3] * a[7] - (double)a[4] * a[6]);
    check(std::fabs(d) > 1e-9, "homography: singular matrix");
    const double inv = 1.0 / d;
    r[0] = (float)(((double)a[4] * a[8] - (double)a[5] * a[7]) * inv);
    r[1] = (float)(((double)a[2] * a[7] - (double)a[1] * a[8]) * inv);
    r[2] = (float)(((double)a[1] * a[5] - (double)a[2] * a[4]) * inv);
    r[3] = (float)(((double)a[5] * a[6] - (double)a[3] * a[8]) * inv);
    r[4] = (float)(((double)a[0] * a[8] - (double)a[2] * a[6]) * inv);
    r[5] = (float)(((double)a[2] * a[3] - (double)a[0] * a[5]) * inv);
    r[6] = (float)(((double)a[3] * a[7] - (double)a[4] * a[6]) * inv);
    r[7] = (float)(((double)a[1] * a[6] - (double)a[0] * a[7]) * inv);
    r[8] = (float)(((double)a[0] * a[4] - (double)a[1] * a[3]) * inv);
}
bool hom_int_translation(const float* m, int64_t* dx, int64_t* dy) {
    auto is = [](float v, float t) { return std::fabs(v - t) < 1e-6f; };
    if (!is(m[0], 1) || !is(m[1], 0) || !is(m[3], 0) || !is(m[4], 1) || !is(m[6], 0) || !is(m[7], 0) || !is(m[8], 1))
        return false;
    const float tx = m[2], ty = m[5];
    if (std::fabs(tx - std::round(tx)) > 1e-4f || std::fabs(ty - std::round(ty)) > 1e-4f) return false;
    *dx = (int64_t)std::llround(tx);
    *dy = (int64_t)std::llround(ty);
    return true;
}

int64_t overlap(int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
    const int64_t lo = std::max(a0, b0), hi = std::min(a1, b1);
    return hi > lo ? hi - lo : 0;
}

}  // namespace

// ------------------------------------------------------------------ engine
class Engine {
  public:
    Engine(const dfx_net_desc* d, const dfx_engine_config* cfg, int device, cudaStream_t stream = nullptr);
    ~Engine();

    void run_frame(const float* frame, int c, int h, int w, const float* h9, const float* roi, dfx_frame_info* info,
                   float* out, size_t cap, bool frame_dev = false, bool out_dev = false);
    void layer_order(int* order, int cap, int* n) const {
        int k = 0;
        for (int i : net_.topo)
            if (k < cap) order[k++] = i;
        *n = k;
    }
    void submit(const float* frame_dev, int c, int h, int w, const float* h9);
    void submit_host(const float* frame, int c, int h, int w, const float* h9, float* out, size_t cap);
    void sync(dfx_frame_info* info);
    void reset();

    // readbacks
    void read_state(const std::string& layer, int which, float* out, size_t cap, int* c, int* h, int* w);
    void read_packet(const std::string& layer, float* out, size_t cap, int* c, int* gh, int* gw, int* halo,
                     uint8_t* mask, size_t mask_cap);
    void read_ledger(int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) const;
    void input_mask(uint8_t* out, size_t cap, int* th, int* tw) const;
    void layer_flops(int layer, uint64_t* f, uint64_t* d) const;
    void output_device(const float** p, int* c, int* h, int* w) const;
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    int num_layers() const { return (int)net_.layers.size(); }
    int kernel_count() const { return launches_; }
    void debug_counts(int* g, int* u, int cap) {
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        const int nl = (int)net_.layers.size();
        std::vector<int> h(2 * nl);
        CUDA_CHECK(cudaMemcpy(h.data(), counters_d_.p + off_counts_, 2 * nl * sizeof(int), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nl && i < cap; ++i) g[i] = h[i], u[i] = h[nl + i];
    }
    void set_profiling(bool on);
    void profile(int fam, double* ms, uint64_t* launches, double* work) const;
    void reset_profile();
    void timer_start();
    float timer_stop();

  private:
    struct LayerRT {
        int halo_store = 0, halo_geom = 0;  // output packet halos (runtime)
        PktDev pkt{};
        DevArr<float> pkt_d;
        DevArr<uint8_t> pkt_ext;
        // state
        BufDev acc{}, aux{};  // aux = trunc (truncation) or prev (maxpool)
        DevArr<float> acc_d, aux_d;
        float thr = 0.0f;
        bool has_bias = false;
        DevArr<float> bias_init;
        // params
        DevArr<float> w, wtc, scale;
        int cin_pad = 0, cout_pad = 0;
        DevArr<int> list;
        int max_targets = 0;
        int splits = 1;
        DevArr<float> ws;
        // dense-unit path (conv_dense.cu)
        bool dense = false;
        DenseConvPlan dp{};
        DevArr<float> wdense, wsd;
        DevArr<int> dcnt;
        DevArr<int> units;
        // fused activation pass 1: this dense conv folds max |trunc + delta| of its
        // sole consuming activation (layer tm_consumer) into that layer's tile_max;
        // the activation then runs its commit pass only (tm_fused)
        int tm_consumer = -1;
        bool tm_fused = false;
        // activation pass 2 fused with its sole consuming 2x2 max pool (layer
        // pool_consumer), which then launches nothing (pool_fused)
        int pool_consumer = -1;
        bool pool_fused = false;
        // the plan of the consuming stride-1 dense conv (layer plan_conv) runs inside
        // this activation's commit launch (plan_fused on the conv)
        int plan_conv = -1;
        bool plan_fused = false;
        // an add whose input `up_in` is a nearest upsample (sole consumer: this add)
        // samples that upsample's input itself; the upsample launches nothing
        int up_in = -1;
        bool up_fused = false;
        // branch streams (DFX_BRANCH_STREAMS=1): this layer's stream (0 = the engine
        // stream), the producer layers on other streams it waits for, and whether a
        // consumer on another stream waits for this layer's completion event
        int sid = 0;
        std::vector<int> waits;
        bool signal = false, wait_input = false;
        cudaEvent_t ev = nullptr;
        // TMA descriptor (CUtensorMap) of the input packet for the patch boxes
        alignas(64) unsigned char tmap[128];
        bool has_tmap = false;
    };

    void allocate(int th, int tw);
    void build_packet(LayerRT& rt, int C, int t, int halo);
    void enqueue(const float* frame_dev, int c, int h, int w, const float* h9, const float* roi_dev);
    void finish_info(dfx_frame_info* info);
    void ensure_staging(int c, int h, int w, bool host_frame);
    PktDev in_packet(int idx) const { return idx == -1 ? in_pkt_ : lrt_[idx].pkt; }
    Ctx ctx() const { return Ctx{d_frame_, slots_d_.p, rows_, cols_, d_own_}; }
    void wait_ack(unsigned seq);
    void set_param_slot(int i) {
        uint8_t* b = params_d_.p + (size_t)i * pstride_;
        d_frame_ = reinterpret_cast<FrameDev*>(b);
        d_claims_ = reinterpret_cast<ClaimRec*>(b + off_claims_);
        d_fresh_ = b + off_fresh_;
        d_own_ = b + off_own_;
    }

    Net net_;
    dfx_engine_config cfg_;
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    bool own_stream_ = true;
    int num_sms_ = 148;
    bool initialized_ = false;
    int64_t frame_index_ = 0;
    int rows_ = 0, cols_ = 0;
    Ledger ledger_;

    std::vector<LayerRT> lrt_;
    // input state
    BufDev in_acc_{}, in_trunc_{};
    DevArr<float> in_acc_d_, in_trunc_d_;
    PktDev in_pkt_{};
    DevArr<float> in_pkt_d_;
    DevArr<uint8_t> in_pkt_ext_;
    // input stage scratch
    int canvas_pitch_ = 0;
    DevArr<float> frame_d_, warped_d_, aligned_d_, roi_frame_d_, roi_warped_d_, roi_aligned_d_, roi_tmp_d_, fac_d_;
    DevArr<uint8_t> fp_d_, valid_d_, roi_fp_d_, roi_valid_d_, sig_d_, sig2_d_, cov_d_, gate_d_;
    // frame parameter block (device) + pinned staging
    DevArr<uint8_t> params_d_;
    uint8_t* params_hb_[2] = {nullptr, nullptr};
    cudaEvent_t params_ev_[2] = {nullptr, nullptr};
    int pslot_ = 0;
    uint8_t* params_hd_[2] = {nullptr, nullptr};  // device views of the mapped host blocks
    size_t pstride_ = 0;                           // params slot stride (16-byte multiple)
    unsigned* ack_h_ = nullptr;                    // mapped: last frame whose block k_frame_begin consumed
    unsigned* ack_d_ = nullptr;
    unsigned fseq_ = 0, pslot_seq_[2] = {0, 0};
    uint8_t* readback_d_ = nullptr;                // device view of readback_h_
    DevArr<unsigned> begin_ctr_;                   // k_frame_begin's last-CTA counter (per engine)
    // host path: copy-stream -> engine-stream flags [h2d slot 0, 1, d2h slot 0, 1]
    DevArr<unsigned> hflags_;
    const unsigned* pend_in_flag_ = nullptr;
    unsigned pend_in_val_ = 0;
    const unsigned* pend_out_flag_ = nullptr;
    unsigned pend_out_val_ = 0;
    size_t params_bytes_ = 0, off_claims_ = 0, off_fresh_ = 0, off_own_ = 0;
    // persistent device slot table (TileLedger slots: owner coord + used): full
    // upload only after allocation / reset (slots_stale_), else k_claims records
    // each frame's claims into it, so the per-frame block stays small
    DevArr<SlotDev> slots_d_;
    SlotDev* slots_h_ = nullptr;  // pinned staging of the full upload
    cudaEvent_t slots_ev_ = nullptr;
    bool slots_stale_ = true;
    FrameDev* d_frame_ = nullptr;
    ClaimRec* d_claims_ = nullptr;
    uint8_t* d_fresh_ = nullptr;
    uint8_t* d_own_ = nullptr;
    int max_claims_ = 0;
    // claims buffer table
    DevArr<ClaimBuf> claim_bufs_;
    int nclaim_bufs_ = 0;
    // per-frame counters: [nl u64 flop_px][u64 dropped][nl int counts][nl * slots u32 tile_max]
    DevArr<uint8_t> counters_d_;
    size_t cnt_bytes_ = 0, off_dropped_ = 0, off_counts_ = 0, off_ucounts_ = 0, off_gbar_ = 0, off_tmax_ = 0;
    uint8_t* readback_h_ = nullptr;  // pinned: flop_px, dropped, input mask
    int rb_n1_ = 0, rb_n2_ = 0;      // readback parts (counters, input mask), 16-B multiples
    float *in_h_ = nullptr, *out_h_ = nullptr;  // pinned staging of run_frame's caller buffers
    size_t in_h_n_ = 0, out_h_n_ = 0;
    // output (out_cur_: the buffer this frame's densify writes)
    DevArr<float> out_d_;
    float* out_cur_ = nullptr;
    // pipelined host path (submit_host): copy stream, double-buffered frame / output
    cudaStream_t cstream_ = nullptr, dstream_ = nullptr;  // host->device, device->host copies
    DevArr<float> hframe_d_[2], hout_d_[2];
    cudaEvent_t ev_h2d_[2] = {nullptr, nullptr}, ev_done_[2] = {nullptr, nullptr}, ev_d2h_[2] = {nullptr, nullptr};
    uint64_t hseq_ = 0;
    // last frame
    Placement place_{};
    dfx_frame_info pending_{};
    bool have_frame_ = false;
    int launches_ = 0;
    // ---- profiling (per kernel family CUDA events on the engine stream)
    struct ProfEv {
        cudaEvent_t a, b;
        int fam;
    };
    bool prof_ = false;
    cudaStream_t prof_s_ = nullptr;  // the stream the current launch goes to (profiling events)
    // independent branches of the network (HRNet branches, ResNet projection
    // shortcuts) on side streams joined by events (DFX_BRANCH_STREAMS=1)
    bool branch_ = false;
    bool grid_hint_ = true;  // work-proportional activation grids (DFX_GRID_HINT=0: persistent full-GPU grids)
    std::vector<cudaStream_t> bstreams_;
    bool input_signal_ = false;
    cudaEvent_t in_ev_ = nullptr;
    cudaStream_t lstream(int sid) const { return sid == 0 ? stream_ : bstreams_[sid - 1]; }
    void plan_branches();
    std::vector<ProfEv> prof_pool_;
    size_t prof_used_ = 0;
    double prof_ms_[DFX_FAMILIES] = {};
    uint64_t prof_launch_[DFX_FAMILIES] = {};
    double prof_work_[DFX_FAMILIES] = {};
    int last_nclaims_ = 0;
    cudaEvent_t timer_a_ = nullptr, timer_b_ = nullptr;
    int prof_begin(int fam);
    void prof_end(int idx);
    void prof_harvest();
};

Engine::Engine(const dfx_net_desc* d, const dfx_engine_config* cfg, int device, cudaStream_t stream)
    : cfg_(*cfg), device_(device) {
    net_ = validate_net(d, cfg->tile_size);
    check(cfg_.tile_size >= 1, "engine: tile size must be >= 1");
    check(cfg_.input_threshold >= 0.0f && cfg_.default_threshold >= 0.0f, "engine: thresholds must be >= 0");
    check(cfg_.mask_dilation >= 0, "engine: mask dilation must be >= 0");
    int ndev = 0;
    const cudaError_t de = cudaGetDeviceCount(&ndev);
    if (de != cudaSuccess) cudaGetLastError();
    if (de != cudaSuccess || ndev <= 0)
        fail(std::string("no CUDA device (the B200 path has no CPU fallback)") +
                 (de != cudaSuccess ? std::string(": ") + cudaGetErrorString(de) : std::string()),
             DFX_ERR_CUDA);
    CUDA_CHECK(cudaSetDevice(device_));
    CUDA_CHECK(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device_));
    if (stream) {
        stream_ = stream;
        own_stream_ = false;
    } else {
        CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    }
    lrt_.resize(net_.layers.size());
}

Engine::~Engine() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& e : prof_pool_) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    if (timer_a_) cudaEventDestroy(timer_a_);
    if (timer_b_) cudaEventDestroy(timer_b_);
    for (int i = 0; i < 2; ++i) {
        if (params_hb_[i]) cudaFreeHost(params_hb_[i]);
        if (params_ev_[i]) cudaEventDestroy(params_ev_[i]);
        params_hb_[i] = nullptr;
    }
    if (readback_h_) cudaFreeHost(readback_h_);
    for (cudaStream_t st : bstreams_) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    for (auto& rt : lrt_)
        if (rt.ev) cudaEventDestroy(rt.ev);
    if (in_ev_) cudaEventDestroy(in_ev_);
    if (slots_h_) cudaFreeHost(slots_h_);
    if (slots_ev_) cudaEventDestroy(slots_ev_);
    if (ack_h_) cudaFreeHost(ack_h_);
    if (in_h_) cudaFreeHost(in_h_);
    if (out_h_) cudaFreeHost(out_h_);
    if (cstream_) cudaStreamSynchronize(cstream_);
    if (dstream_) cudaStreamSynchronize(dstream_);
    for (int i = 0; i < 2; ++i) {
        if (ev_h2d_[i]) cudaEventDestroy(ev_h2d_[i]);
        if (ev_done_[i]) cudaEventDestroy(ev_done_[i]);
        if (ev_d2h_[i]) cudaEventDestroy(ev_d2h_[i]);
    }
    if (cstream_) cudaStreamDestroy(cstream_);
    if (dstream_) cudaStreamDestroy(dstream_);
    if (stream_ && own_stream_) cudaStreamDestroy(stream_);
}

void Engine::build_packet(LayerRT& rt, int C, int t, int halo) {
    PktDev& p = rt.pkt;
    p.C = C;
    p.t = t;
    p.halo = halo;
    p.RT = (halo + t - 1) / t;
    p.pitch_w = cols_ * t + 2 * halo;
    p.ext_pitch = cols_ + 2 * p.RT;
    rt.pkt_d.alloc((size_t)(rows_ * t + 2 * halo) * p.pitch_w * C);
    rt.pkt_ext.alloc(((size_t)(rows_ + 2 * p.RT) * p.ext_pitch + 15) / 16 * 16);  // 16-B readback copies
    CUDA_CHECK(cudaMemsetAsync(rt.pkt_ext.p, 0, rt.pkt_ext.n, stream_));
    p.d = rt.pkt_d.p;
    p.ext = rt.pkt_ext.p;
}

// engine.cpp:33-76: grid from the first placement, buffers per state.
void Engine::allocate(int th, int tw) {
    const int ring = cfg_.padded_convolutions ? net_.ring : 1;
    rows_ = cfg_.grid_rows > 0 ? cfg_.grid_rows : th + 2 * ring;
    cols_ = cfg_.grid_cols > 0 ? cfg_.grid_cols : tw + 2 * ring;
    check(rows_ >= 1 && cols_ >= 1, "engine: bad grid dims");
    check(rows_ * cfg_.tile_size + 64 < 32768 && cols_ * cfg_.tile_size + 64 < 32768, "engine: grid too large");
    ledger_.init(rows_, cols_);
    const int T = cfg_.tile_size, slots = rows_ * cols_;
    const size_t tile_elems_in = (size_t)T * T * net_.in_channels;

    in_acc_d_.alloc(slots * tile_elems_in);
    in_trunc_d_.alloc(slots * tile_elems_in);
    CUDA_CHECK(cudaMemsetAsync(in_acc_d_.p, 0, in_acc_d_.n * 4, stream_));
    CUDA_CHECK(cudaMemsetAsync(in_trunc_d_.p, 0, in_trunc_d_.n * 4, stream_));
    in_acc_ = {in_acc_d_.p, net_.in_channels, T};
    in_trunc_ = {in_trunc_d_.p, net_.in_channels, T};
    {
        LayerRT tmp;
        build_packet(tmp, net_.in_channels, T, 0);
        in_pkt_ = tmp.pkt;
        std::swap(in_pkt_d_.p, tmp.pkt_d.p);
        std::swap(in_pkt_d_.n, tmp.pkt_d.n);
        std::swap(in_pkt_ext_.p, tmp.pkt_ext.p);
        std::swap(in_pkt_ext_.n, tmp.pkt_ext.n);
    }
    canvas_pitch_ = cols_ * T;
    const size_t canvas_px = (size_t)rows_ * T * canvas_pitch_;
    aligned_d_.alloc(canvas_px * net_.in_channels);
    valid_d_.alloc(canvas_px);
    sig_d_.alloc(canvas_px);
    sig2_d_.alloc(canvas_px);
    cov_d_.alloc(slots);
    gate_d_.alloc(slots);
    if (cfg_.roi_enabled) {
        roi_aligned_d_.alloc(canvas_px);
        roi_valid_d_.alloc(canvas_px);
        roi_tmp_d_.alloc(canvas_px * 3);
        fac_d_.alloc(canvas_px);
    }

    // layers (runtime halos follow the actual packets, engine.cpp:247-281)
    std::vector<ClaimBuf> cbufs;
    cbufs.push_back({in_acc_d_.p, nullptr, net_.in_channels, T});
    cbufs.push_back({in_trunc_d_.p, nullptr, net_.in_channels, T});
    for (int idx : net_.topo) {
        const Layer& l = net_.layers[idx];
        LayerRT& rt = lrt_[idx];
        const int hin = l.in0 == -1 ? 0 : lrt_[l.in0].halo_store;
        switch (l.kind) {
            case DFX_CONV: {
                check(l.tile <= 64, "conv output tile larger than 64 px is not supported by the target kernel");
                rt.halo_geom = windowed_out_halo(hin, l.k, l.k / 2, l.stride);
                rt.halo_store = cfg_.padded_convolutions ? rt.halo_geom : 0;
                build_packet(rt, l.cout, l.tile, rt.halo_store);
                rt.w.alloc(l.w.size());
                CUDA_CHECK(cudaMemcpyAsync(rt.w.p, l.w.data(), l.w.size() * 4, cudaMemcpyHostToDevice, stream_));
                rt.max_targets = (rows_ * l.tile + 2 * rt.halo_geom) * (cols_ * l.tile + 2 * rt.halo_geom);
                rt.list.alloc(rt.max_targets);
                if (cfg_.conv_mode == DFX_CONV_TF32X3) {
                    rt.cin_pad = (l.cin + 7) / 8 * 8;
                    rt.cout_pad = (l.cout + 15) / 16 * 16;
                    std::vector<float> ws(conv_tc_weight_floats(rt.cin_pad, rt.cout_pad, l.k));
                    conv_tc_prepare_weights(l.w.data(), l.cin, l.cout, l.k, rt.cin_pad, rt.cout_pad, ws.data());
                    rt.wtc.alloc(ws.size());
                    CUDA_CHECK(cudaMemcpy(rt.wtc.p, ws.data(), ws.size() * 4, cudaMemcpyHostToDevice));
                    rt.splits = conv_tc_splits(rt.max_targets, rt.cin_pad, rt.cout_pad, l.k, num_sms_);
                    if (rt.splits > 1) rt.ws.alloc((size_t)rt.splits * rt.max_targets * rt.cout_pad);
                    const char* dv = getenv("DFX_DENSE");
                    // the dense-unit kernel stages a patch grown by at most 8 px of halo
                    // (launch_conv_plan); wider halos take the gathered-target kernel
                    if (l.stride == 1 && rt.halo_geom <= 8 && !(dv && dv[0] == '0')) {
                        rt.dp = dense_conv_plan(l.cin, l.cout, l.k, l.tile, rows_, cols_, (size_t)256 << 20);
                        rt.dense = rt.dp.ok;
                    }
                    if (rt.dense && rt.dp.tma)
                        rt.has_tmap = dense_conv_tensor_map(rt.dp, in_packet(l.in0), rows_, rt.tmap);
                    if (rt.dense) {
                        std::vector<float> wd(dense_conv_weight_floats(rt.dp));
                        dense_conv_prepare_weights(rt.dp, l.w.data(), l.cin, l.cout, wd.data());
                        rt.wdense.alloc(wd.size());
                        CUDA_CHECK(cudaMemcpy(rt.wdense.p, wd.data(), wd.size() * 4, cudaMemcpyHostToDevice));
                        rt.units.alloc(rt.dp.units_max);
                        if (rt.dp.smax > 1) rt.wsd.alloc((size_t)rt.dp.smax * rt.dp.ws_units * 128 * rt.dp.cout_pad);
                        rt.dcnt.alloc((size_t)rt.dp.ws_units * rt.dp.nNB);
                        CUDA_CHECK(cudaMemset(rt.dcnt.p, 0, rt.dcnt.n * sizeof(int)));
                    }
                }
                break;
            }
            case DFX_RELU:
            case DFX_TRUNCATE:
            case DFX_OUTPUT: {
                rt.halo_store = rt.halo_geom = 0;
                build_packet(rt, l.in_channels, l.in_tile, 0);
                float thr = 0.0f;
                if (l.kind != DFX_OUTPUT && l.trunc_en)
                    thr = (cfg_.override_net_thresholds || !l.has_thr) ? cfg_.default_threshold : l.thr;
                rt.thr = thr;
                const size_t n = (size_t)slots * l.in_tile * l.in_tile * l.in_channels;
                rt.acc_d.alloc(n);
                rt.aux_d.alloc(n);
                CUDA_CHECK(cudaMemsetAsync(rt.acc_d.p, 0, n * 4, stream_));
                CUDA_CHECK(cudaMemsetAsync(rt.aux_d.p, 0, n * 4, stream_));
                rt.acc = {rt.acc_d.p, l.in_channels, l.in_tile};
                rt.aux = {rt.aux_d.p, l.in_channels, l.in_tile};
                std::vector<float> bias(l.in_channels, 0.0f);
                if (l.in0 >= 0) bias = net_.layers[l.in0].beta;
                rt.has_bias = std::any_of(bias.begin(), bias.end(), [](float b) { return b != 0.0f; });
                cbufs.push_back({rt.acc_d.p, nullptr, l.in_channels, l.in_tile});
                if (rt.has_bias) {
                    rt.bias_init.alloc(bias.size());
                    CUDA_CHECK(cudaMemcpy(rt.bias_init.p, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
                    cbufs.push_back({rt.aux_d.p, rt.bias_init.p, l.in_channels, l.in_tile});
                } else {
                    cbufs.push_back({rt.aux_d.p, nullptr, l.in_channels, l.in_tile});
                }
                break;
            }
            case DFX_MAXPOOL: {
                rt.halo_store = rt.halo_geom = windowed_out_halo(hin, l.pool_k, 0, l.pool_s);
                build_packet(rt, l.in_channels, l.tile, rt.halo_store);
                const size_t na = (size_t)slots * l.in_tile * l.in_tile * l.in_channels;
                const size_t np = (size_t)slots * l.tile * l.tile * l.in_channels;
                rt.acc_d.alloc(na);
                rt.aux_d.alloc(np);
                CUDA_CHECK(cudaMemsetAsync(rt.acc_d.p, 0, na * 4, stream_));
                CUDA_CHECK(cudaMemsetAsync(rt.aux_d.p, 0, np * 4, stream_));
                rt.acc = {rt.acc_d.p, l.in_channels, l.in_tile};
                rt.aux = {rt.aux_d.p, l.in_channels, l.tile};
                cbufs.push_back({rt.acc_d.p, nullptr, l.in_channels, l.in_tile});
                cbufs.push_back({rt.aux_d.p, nullptr, l.in_channels, l.tile});
                break;
            }
            case DFX_AVGPOOL:
                rt.halo_store = rt.halo_geom = windowed_out_halo(hin, l.pool_k, 0, l.pool_s);
                build_packet(rt, l.in_channels, l.tile, rt.halo_store);
                break;
            case DFX_UPSAMPLE:
                rt.halo_store = rt.halo_geom = hin * l.factor;
                build_packet(rt, l.in_channels, l.tile, rt.halo_store);
                break;
            case DFX_BATCHNORM:
                rt.halo_store = rt.halo_geom = hin;
                build_packet(rt, l.in_channels, l.tile, rt.halo_store);
                rt.scale.alloc(l.bn_scale.size());
                CUDA_CHECK(cudaMemcpy(rt.scale.p, l.bn_scale.data(), l.bn_scale.size() * 4, cudaMemcpyHostToDevice));
                break;
            case DFX_ADD: {
                const int hb = l.in1 == -1 ? 0 : lrt_[l.in1].halo_store;
                rt.halo_store = rt.halo_geom = std::max(hin, hb);
                build_packet(rt, l.in_channels, l.tile, rt.halo_store);
                break;
            }
        }
    }
    // activation pass 1 fused into the producing dense conv (an all-thread pass at
    // the end of the kernel, and the plan's zero fill): stride-1 dense convs whose
    // sole consumer is a truncation point, 32-channel multiples
    {
        // opt-in (DFX_FUSE_TM=1): measured 3-7 % SLOWER end to end on C2 (DESIGN.md §3,
        // negative results): the conv's extra trunc reads sit on its critical tail
        const char* fe = getenv("DFX_FUSE_TM");
        const char* ce = getenv("DFX_TRUNC_COOP");
        const char* te = getenv("DFX_DENSE_TAU");
        const bool on = (fe && fe[0] == '1') && !(ce && ce[0] == '1') && !(te && atoi(te) > 1);
        for (size_t i = 0; on && i < net_.layers.size(); ++i) {
            const Layer& l = net_.layers[i];
            LayerRT& rt = lrt_[i];
            if (l.kind != DFX_CONV || !rt.dense || l.cout % 32 != 0 || rt.dp.NBD % 32 != 0) continue;
            int cj = -1, ncons = 0;
            for (size_t j = 0; j < net_.layers.size(); ++j)
                if (net_.layers[j].in0 == (int)i || net_.layers[j].in1 == (int)i) cj = (int)j, ++ncons;
            if (ncons != 1) continue;
            const int k = net_.layers[cj].kind;
            if (k != DFX_RELU && k != DFX_TRUNCATE && k != DFX_OUTPUT) continue;
            rt.tm_consumer = cj;
            lrt_[cj].tm_fused = true;
        }
    }
    // activation commit fused with its sole consuming 2x2 / stride-2 max pool
    // (tile-local; DFX_FUSE_POOL=0 keeps the separate pool launch)
    {
        const char* pe = getenv("DFX_FUSE_POOL");
        const char* ce = getenv("DFX_TRUNC_COOP");
        const bool on = !(pe && pe[0] == '0') && !(ce && ce[0] == '1');
        for (size_t i = 0; on && i < net_.layers.size(); ++i) {
            const Layer& l = net_.layers[i];
            LayerRT& rt = lrt_[i];
            if ((l.kind != DFX_RELU && l.kind != DFX_TRUNCATE) || rt.tm_fused || (l.in_channels & 3) != 0) continue;
            int pj = -1, ncons = 0;
            for (size_t j = 0; j < net_.layers.size(); ++j)
                if (net_.layers[j].in0 == (int)i || net_.layers[j].in1 == (int)i) pj = (int)j, ++ncons;
            if (ncons != 1) continue;
            const Layer& pl = net_.layers[pj];
            if (pl.kind != DFX_MAXPOOL || pl.pool_k != 2 || pl.pool_s != 2 || (l.in_tile & 1) != 0) continue;
            rt.pool_consumer = pj;
            lrt_[pj].pool_fused = true;
        }
    }
    // the next dense conv's plan inside the activation's commit launch (extra
    // blocks; the input mask comes from the activation's tile maxima);
    // DFX_FUSE_PLAN=0 keeps the standalone plan launch
    {
        const char* fe = getenv("DFX_FUSE_PLAN");
        const char* te = getenv("DFX_DENSE_TAU");
        const bool on = !(fe && fe[0] == '0') && !(te && atoi(te) > 1);
        auto sole = [&](int i) {
            int cj = -1, ncons = 0;
            for (size_t j = 0; j < net_.layers.size(); ++j)
                if (net_.layers[j].in0 == i || net_.layers[j].in1 == i) cj = (int)j, ++ncons;
            return ncons == 1 ? cj : -1;
        };
        for (size_t i = 0; on && i < net_.layers.size(); ++i) {
            const Layer& l = net_.layers[i];
            LayerRT& rt = lrt_[i];
            if ((l.kind != DFX_RELU && l.kind != DFX_TRUNCATE) || rt.tm_fused || (l.in_channels & 3) != 0) continue;
            const int src = rt.pool_consumer >= 0 ? rt.pool_consumer : (int)i;  // the conv's input layer
            const int cj = sole(src);
            if (cj < 0 || net_.layers[cj].kind != DFX_CONV || net_.layers[cj].in1 >= 0) continue;
            const LayerRT& cr = lrt_[cj];
            if (!cr.dense || net_.layers[cj].stride != 1 || cr.tm_consumer >= 0) continue;
            rt.plan_conv = cj;
            lrt_[cj].plan_fused = true;
        }
    }
    // nearest upsample folded into its sole consuming add (DFX_FUSE_UPSAMPLE=0: off)
    {
        const char* ue = getenv("DFX_FUSE_UPSAMPLE");
        const bool on = !(ue && ue[0] == '0');
        for (size_t i = 0; on && i < net_.layers.size(); ++i) {
            const Layer& l = net_.layers[i];
            if (l.kind != DFX_ADD || (l.in_channels & 3) != 0) continue;
            for (int q : {l.in1, l.in0}) {
                if (q < 0 || net_.layers[q].kind != DFX_UPSAMPLE) continue;
                int ncons = 0;
                for (const Layer& m : net_.layers) ncons += (m.in0 == q) + (m.in1 == q);
                if (ncons != 1 || l.in0 == l.in1) continue;
                lrt_[i].up_in = q;
                lrt_[q].up_fused = true;
                break;
            }
        }
    }
    nclaim_bufs_ = (int)cbufs.size();
    claim_bufs_.alloc(cbufs.size());
    CUDA_CHECK(cudaMemcpy(claim_bufs_.p, cbufs.data(), cbufs.size() * sizeof(ClaimBuf), cudaMemcpyHostToDevice));

    // frame parameter block
    max_claims_ = slots;
    // [FrameDev | fresh bytes | owned bytes | ClaimRec x max]: k_frame_begin
    // copies only the used prefix (the claims of the frame) over PCIe
    off_fresh_ = (sizeof(FrameDev) + 15) / 16 * 16;
    off_own_ = off_fresh_ + slots;
    off_claims_ = (off_own_ + slots + 15) / 16 * 16;
    params_bytes_ = off_claims_ + (size_t)max_claims_ * sizeof(ClaimRec);
    slots_d_.alloc(slots);
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&slots_h_), (size_t)slots * sizeof(SlotDev), cudaHostAllocDefault));
    CUDA_CHECK(cudaEventCreateWithFlags(&slots_ev_, cudaEventDisableTiming));
    slots_stale_ = true;
    // two device slots (alternating per frame) filled by k_frame_begin from two
    // mapped page-locked host blocks
    pstride_ = (params_bytes_ + 255) / 256 * 256;
    params_d_.alloc(2 * pstride_);
    for (int i = 0; i < 2; ++i) {
        CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&params_hb_[i]), pstride_, cudaHostAllocMapped));
        memset(params_hb_[i], 0, pstride_);
        CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&params_hd_[i]), params_hb_[i], 0));
        CUDA_CHECK(cudaEventCreateWithFlags(&params_ev_[i], cudaEventDisableTiming));
    }
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&ack_h_), 64, cudaHostAllocMapped));
    *reinterpret_cast<volatile unsigned*>(ack_h_) = 0;
    CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ack_d_), ack_h_, 0));
    begin_ctr_.alloc(1);
    CUDA_CHECK(cudaMemset(begin_ctr_.p, 0, sizeof(unsigned)));
    fseq_ = 0;
    pslot_seq_[0] = pslot_seq_[1] = 0;
    set_param_slot(0);

    const size_t nl = net_.layers.size();
    off_dropped_ = nl * 8;
    off_counts_ = off_dropped_ + 8;
    off_ucounts_ = off_counts_ + nl * 4;
    off_gbar_ = off_ucounts_ + nl * 4;
    off_tmax_ = (off_gbar_ + nl * 4 + 15) / 16 * 16;
    cnt_bytes_ = (off_tmax_ + nl * (size_t)slots * 4 + 15) / 16 * 16;
    counters_d_.alloc(cnt_bytes_);
    CUDA_CHECK(cudaMemset(counters_d_.p, 0, cnt_bytes_));
    rb_n1_ = (int)((nl * 8 + 8 + 15) / 16 * 16);
    rb_n2_ = (slots + 15) / 16 * 16;
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&readback_h_), rb_n1_ + rb_n2_, cudaHostAllocMapped));
    CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&readback_d_), readback_h_, 0));

    const int ot = net_.layers[net_.out_layer].in_tile;
    out_d_.alloc((size_t)net_.layers[net_.out_layer].in_channels * rows_ * ot * cols_ * ot);
    plan_branches();
    initialized_ = true;
}

void Engine::reset() {
    // engine.cpp:93-108
    if (!initialized_) return;
    ledger_.clear();
    slots_stale_ = true;  // the next frame uploads the whole (re-planned) slot table
    CUDA_CHECK(cudaMemsetAsync(in_acc_d_.p, 0, in_acc_d_.n * 4, stream_));
    CUDA_CHECK(cudaMemsetAsync(in_trunc_d_.p, 0, in_trunc_d_.n * 4, stream_));
    for (auto& rt : lrt_) {
        if (rt.acc_d.p) CUDA_CHECK(cudaMemsetAsync(rt.acc_d.p, 0, rt.acc_d.n * 4, stream_));
        if (rt.aux_d.p) CUDA_CHECK(cudaMemsetAsync(rt.aux_d.p, 0, rt.aux_d.n * 4, stream_));
    }
}

// Waits until k_frame_begin of frame `seq` acknowledged its parameter block.
// A fault (or a device-side trap) in an earlier frame means the ack never
// comes: the stream is polled every few thousand spins so the sticky CUDA
// error is reported, and a generous wall-clock bound turns a stuck device
// into an error instead of a hang.
void Engine::wait_ack(unsigned seq) {
    const volatile unsigned* ack = reinterpret_cast<volatile unsigned*>(ack_h_);
    if (*ack >= seq) return;
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 1;; ++spin) {
        if (*ack >= seq) return;
        if ((spin & 4095) == 0) {
            const cudaError_t q = cudaStreamQuery(stream_);
            if (q != cudaSuccess && q != cudaErrorNotReady) {
                cudaGetLastError();
                fail(std::string("CUDA: ") + cudaGetErrorString(q) + " (frame pipeline)", DFX_ERR_CUDA);
            }
            if (q == cudaSuccess && *ack < seq)  // stream drained without the ack: the frame never ran
                fail("frame pipeline: parameter block not acknowledged", DFX_ERR_CUDA);
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
                fail("frame pipeline: timed out waiting for the device", DFX_ERR_CUDA);
        }
    }
}

int Engine::prof_begin(int fam) {
    if (!prof_) return -1;
    if (prof_used_ == prof_pool_.size()) {
        ProfEv e{};
        CUDA_CHECK(cudaEventCreate(&e.a));
        CUDA_CHECK(cudaEventCreate(&e.b));
        prof_pool_.push_back(e);
    }
    ProfEv& e = prof_pool_[prof_used_];
    e.fam = fam;
    CUDA_CHECK(cudaEventRecord(e.a, prof_s_ ? prof_s_ : stream_));
    return (int)prof_used_++;
}
void Engine::prof_end(int idx) {
    if (idx >= 0) CUDA_CHECK(cudaEventRecord(prof_pool_[idx].b, prof_s_ ? prof_s_ : stream_));
}

// Branch streams (measured: C4 HRNet +64 %, C3 ResNet-18 +4 %, chains such
// as C2 unchanged): a layer continues its first input's stream when it is that
// producer's first consumer in execution order, else it opens a side stream
// (round robin over six); cross-stream inputs become event waits, and the
// output layer joins the engine stream (the frame's last kernel and the
// readback run there). Layers fused into their producer's launch (the pool /
// plan / tile-max fusions) are sole consumers, so they share its stream.
void Engine::plan_branches() {
    const char* gh = getenv("DFX_GRID_HINT");  // default on (C4 +5 %, C5 +2.6 %, C2 / C3 neutral); 0 disables
    grid_hint_ = !(gh && gh[0] == '0');
    const char* e = getenv("DFX_BRANCH_STREAMS");  // default on; 0 keeps one stream
    branch_ = !(e && e[0] == '0');
    if (!branch_) return;
    const int nl = (int)net_.layers.size();
    std::vector<uint8_t> claimed(nl + 1, 0);  // index nl: the network input
    int next = 0;
    int nside = 6;  // DFX_BRANCH_SIDES (1..8): side streams per engine (C4: 3 -> 6 measured +6 %, 8 = 6)
    if (const char* ns = getenv("DFX_BRANCH_SIDES")) nside = std::min(8, std::max(1, atoi(ns)));
    auto sid_of = [&](int p) { return p < 0 ? 0 : lrt_[p].sid; };
    for (int idx : net_.topo) {
        const Layer& l = net_.layers[idx];
        LayerRT& rt = lrt_[idx];
        const int p = l.in0, key = p < 0 ? nl : p;
        if (!claimed[key]) {
            rt.sid = sid_of(p);
            claimed[key] = 1;
        } else {
            rt.sid = 1 + (next++ % nside);
        }
        for (int q : {l.in0, l.in1}) {
            if (q == -2 || sid_of(q) == rt.sid) continue;
            if (q == -1) {  // the input packet: the input stage's event on the engine stream
                rt.wait_input = true;
                input_signal_ = true;
                continue;
            }
            rt.waits.push_back(q);
            lrt_[q].signal = true;
        }
    }
    if (lrt_[net_.out_layer].sid != 0) lrt_[net_.out_layer].signal = true;
    for (int i = 0; i < nside; ++i) {
        cudaStream_t st = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        bstreams_.push_back(st);
    }
    for (auto& rt : lrt_)
        if (rt.signal) CUDA_CHECK(cudaEventCreateWithFlags(&rt.ev, cudaEventDisableTiming));
    if (input_signal_) CUDA_CHECK(cudaEventCreateWithFlags(&in_ev_, cudaEventDisableTiming));
}

// engine.cpp:184-287 on device.
void Engine::enqueue(const float* frame_dev, int c, int h, int w, const float* h9, const float* roi_dev) {
    check(c == net_.in_channels, "run_frame: input channel mismatch");
    const int T = cfg_.tile_size;
    // factor the integer translation out (engine.cpp:189-192)
    const int64_t offx = (int64_t)std::llround(h9[2]), offy = (int64_t)std::llround(h9[5]);
    const float tr[9] = {1, 0, (float)(-offx), 0, 1, (float)(-offy), 0, 0, 1};
    float res[9], inv[9];
    hom_compose(tr, h9, res);
    hom_inverse(res, inv);  // warp() inverts first (alignment.cpp:59) and throws if singular
    int64_t idx = 0, idy = 0;
    const bool integer = hom_int_translation(res, &idx, &idy);
    // snap_to_grid (alignment.cpp:106-166)
    const int64_t ty0 = fdiv(offy, T), tx0 = fdiv(offx, T);
    const int my = (int)(offy - ty0 * T), mx = (int)(offx - tx0 * T);
    const int th0 = (int)cdiv(my + h, T), tw0 = (int)cdiv(mx + w, T);
    const int max_r = initialized_ ? rows_ : cfg_.grid_rows, max_c = initialized_ ? cols_ : cfg_.grid_cols;
    int drop_top = 0, drop_left = 0, th = th0, tw = tw0;
    if (max_r > 0 && th0 > max_r) {
        drop_top = (th0 - max_r) / 2;
        th = max_r;
    }
    if (max_c > 0 && tw0 > max_c) {
        drop_left = (tw0 - max_c) / 2;
        tw = max_c;
    }
    const bool cropped = th != th0 || tw != tw0;
    const int sy0 = drop_top * T - my, sx0 = drop_left * T - mx;
    Placement pl;
    pl.origin = {tx0 + drop_left, ty0 + drop_top};
    pl.th = th;
    pl.tw = tw;
    if (!initialized_) allocate(th, tw);

    dfx_frame_info& info = pending_;
    memset(&info, 0, sizeof info);
    info.frame_index = frame_index_;
    info.origin_tx = pl.origin.tx;
    info.origin_ty = pl.origin.ty;
    info.tiles_h = th;
    info.tiles_w = tw;
    if (cropped && integer) {
        // valid pixels of the shifted frame outside the crop window (alignment.cpp:233-242)
        const int64_t fy = overlap(idy, idy + h, 0, h), fx = overlap(idx, idx + w, 0, w);
        const int64_t ky = overlap(std::max<int64_t>(idy, 0), std::min<int64_t>(idy + h, h), sy0, sy0 + (int64_t)th * T);
        const int64_t kx = overlap(std::max<int64_t>(idx, 0), std::min<int64_t>(idx + w, w), sx0, sx0 + (int64_t)tw * T);
        info.dropped_pixels = fy * fx - ky * kx;
    }

    // plan (engine.cpp:206-214)
    const int ring = cfg_.padded_convolutions ? net_.ring : 0;
    check(th <= rows_ && tw <= cols_, "plan_frame: placement larger than grid");
    Plan plan = ledger_.plan(pl, ring);
    if (plan.full_reset) {
        reset();
        info.reset = 1;
        plan = ledger_.plan(pl, ring);
    }
    ledger_.apply(plan, pl);
    info.fresh = (int)plan.fresh.size();
    info.evicted = plan.evicted;
    check((int)plan.claims.size() <= max_claims_, "too many claims");

    // parameter block
    FrameDev F{};
    F.otx = pl.origin.tx;
    F.oty = pl.origin.ty;
    F.th = th;
    F.tw = tw;
    F.base_sr = (int)floor_mod64(pl.origin.ty, rows_);
    F.base_sc = (int)floor_mod64(pl.origin.tx, cols_);
    F.nclaims = (int)plan.claims.size();
    last_nclaims_ = F.nclaims;
    F.frame_h = h;
    F.frame_w = w;
    F.sy0 = sy0;
    F.sx0 = sx0;
    F.integer_path = integer ? 1 : 0;
    F.idx = (int)idx;
    F.idy = (int)idy;
    F.roi = (cfg_.roi_enabled && roi_dev) ? 1 : 0;
    for (int i = 0; i < 9; ++i) F.inv[i] = inv[i];
    // the pinned block this frame writes may still feed an in-flight upload
    pslot_ ^= 1;
    uint8_t* params_h_ = params_hb_[pslot_];
    // the host block is free once k_frame_begin of the slot's previous frame consumed it
    wait_ack(pslot_seq_[pslot_]);
    memcpy(params_h_, &F, sizeof F);
    const auto& slots = ledger_.slots();
    if (slots_stale_) {
        // first frame / after a reset: the whole slot table, copied on the engine
        // stream ahead of this frame's kernels (the frame's claims re-record the
        // same owners); the staging buffer is reused only after its last copy ran
        CUDA_CHECK(cudaEventSynchronize(slots_ev_));
        for (size_t i = 0; i < slots.size(); ++i)
            slots_h_[i] = SlotDev{slots[i].coord.tx, slots[i].coord.ty, slots[i].used ? 1 : 0, 0};
        CUDA_CHECK(cudaMemcpyAsync(slots_d_.p, slots_h_, slots.size() * sizeof(SlotDev), cudaMemcpyHostToDevice,
                                   stream_));
        CUDA_CHECK(cudaEventRecord(slots_ev_, stream_));
        slots_stale_ = false;
    }
    ClaimRec* hc = reinterpret_cast<ClaimRec*>(params_h_ + off_claims_);
    for (size_t i = 0; i < plan.claims.size(); ++i)
        hc[i] = ClaimRec{plan.claims[i].coord.tx, plan.claims[i].coord.ty, ledger_.slot_index(plan.claims[i].coord),
                         {0, 0, 0}};
    uint8_t* hf = params_h_ + off_fresh_;
    memset(hf, 0, (size_t)rows_ * cols_);
    for (const Coord& t : plan.fresh) {
        const int64_t r = t.ty - pl.origin.ty, cc = t.tx - pl.origin.tx;
        if (r >= 0 && r < th && cc >= 0 && cc < tw) hf[r * tw + cc] = 1;
    }
    // owned map of the placement tiles (TileLedger::holds, buffer_manager.hpp:41-44)
    uint8_t* ho = params_h_ + off_own_;
    for (int r = 0; r < th; ++r)
        for (int cc = 0; cc < tw; ++cc) {
            const Coord t{pl.origin.tx + cc, pl.origin.ty + r};
            const auto& sl = slots[ledger_.slot_index(t)];
            ho[r * tw + cc] = (sl.used && sl.coord.tx == t.tx && sl.coord.ty == t.ty) ? 1 : 0;
        }
    pslot_seq_[pslot_] = ++fseq_;
    set_param_slot(pslot_);
    std::atomic_thread_fence(std::memory_order_release);
    launches_ = 0;
    const size_t pbytes = off_claims_ + plan.claims.size() * sizeof(ClaimRec);  // the used prefix (16-B multiple)
    launch_frame_begin(stream_, params_hd_[pslot_], params_d_.p + (size_t)pslot_ * pstride_, pbytes, counters_d_.p,
                       cnt_bytes_, ack_d_, fseq_, pend_in_flag_, pend_in_val_, begin_ctr_.p);
    ++launches_;
    const Ctx C = ctx();
    cudaStream_t s = stream_;
    auto* flop_px = reinterpret_cast<unsigned long long*>(counters_d_.p);
    auto* dropped = reinterpret_cast<unsigned long long*>(counters_d_.p + off_dropped_);
    int* counts = reinterpret_cast<int*>(counters_d_.p + off_counts_);
    int* ucounts = reinterpret_cast<int*>(counters_d_.p + off_ucounts_);
    unsigned* gbars = reinterpret_cast<unsigned*>(counters_d_.p + off_gbar_);
    unsigned* tmax = reinterpret_cast<unsigned*>(counters_d_.p + off_tmax_);
    const int nslots = rows_ * cols_;

    // claims reset + implicit bias (buffer_manager.cpp:68-89)
    // (the host knows the claim count: frames without claims skip the launch)
    if (F.nclaims > 0)
        PROF(DFX_FAM_CLAIMS,
             launch_claims(C, s, d_claims_, nullptr, slots_d_.p, claim_bufs_.p, nclaim_bufs_, max_claims_));

    // input stage
    static const bool fuse_input = !(getenv("DFX_FUSE_INPUT") && getenv("DFX_FUSE_INPUT")[0] == '0');
    const bool fused_in = fuse_input && !F.roi && !cfg_.noise_suppression;
    // the fused stage samples the frame itself unless the crop count needs k_warp's full-frame map
    const bool direct = fused_in && !integer && !cropped;
    if (!integer && !direct) PROF(DFX_FAM_INPUT, launch_warp(C, s, frame_dev, c, warped_d_.p, fp_d_.p));
    if (cropped && !integer) PROF(DFX_FAM_INPUT, launch_count_dropped(C, s, fp_d_.p, T, dropped));
    if (fused_in) {
        // two launches: align + coverage + significance, then gate + input truncation
        PROF(DFX_FAM_INPUT, launch_input_tile_a(C, s, frame_dev, warped_d_.p, fp_d_.p, c, aligned_d_.p, canvas_pitch_, T,
                                                in_acc_, in_trunc_, cfg_.input_threshold, cov_d_.p, sig_d_.p,
                                                direct ? 1 : 0));
        PROF(DFX_FAM_INPUT, launch_input_tile_b(C, s, aligned_d_.p, cov_d_.p, sig_d_.p, d_fresh_, cfg_.mask_dilation,
                                                canvas_pitch_, in_acc_, in_trunc_, in_pkt_));
    } else {
    PROF(DFX_FAM_INPUT, launch_align(C, s, frame_dev, warped_d_.p, fp_d_.p, c, aligned_d_.p, valid_d_.p, canvas_pitch_, T));
    const float* fac = nullptr;
    if (F.roi) {
        if (!integer) PROF(DFX_FAM_INPUT, launch_warp(C, s, roi_dev, 1, roi_warped_d_.p, roi_fp_d_.p));
        PROF(DFX_FAM_INPUT, launch_align(C, s, roi_dev, roi_warped_d_.p, roi_fp_d_.p, 1, roi_aligned_d_.p, roi_valid_d_.p, canvas_pitch_, T));
        PROF(DFX_FAM_INPUT, launch_roi_factor(C, s, roi_aligned_d_.p, roi_tmp_d_.p, fac_d_.p, canvas_pitch_, T));
        ++launches_;  // two kernels (rows, cols)
        fac = fac_d_.p;
    }
    PROF(DFX_FAM_INPUT, launch_coverage(C, s, valid_d_.p, canvas_pitch_, T, cov_d_.p));
    PROF(DFX_FAM_INPUT, launch_input_sig(C, s, aligned_d_.p, cov_d_.p, in_acc_, in_trunc_, fac, cfg_.input_threshold, canvas_pitch_, T,
                     sig_d_.p));
    const uint8_t* sig = sig_d_.p;
    if (cfg_.noise_suppression) {
        PROF(DFX_FAM_INPUT, launch_noise(C, s, sig_d_.p, sig2_d_.p, canvas_pitch_, T));
        sig = sig2_d_.p;
    }
    PROF(DFX_FAM_INPUT, launch_gate(C, s, sig, cov_d_.p, d_fresh_, cfg_.mask_dilation, canvas_pitch_, T, gate_d_.p));
    PROF(DFX_FAM_INPUT, launch_input_apply(C, s, aligned_d_.p, cov_d_.p, gate_d_.p, in_acc_, in_trunc_, in_pkt_, canvas_pitch_));
    }

    // layers in topological order (engine.cpp:247-281)
    if (branch_ && input_signal_) CUDA_CHECK(cudaEventRecord(in_ev_, stream_));
    bool densified = false;  // the output layer's activation launch also densified
    for (int idx2 : net_.topo) {
        const Layer& l = net_.layers[idx2];
        LayerRT& rt = lrt_[idx2];
        const PktDev a = in_packet(l.in0);
        const cudaStream_t s = branch_ ? lstream(rt.sid) : stream_;  // this layer's stream
        prof_s_ = s;
        if (grid_hint_) {  // activation launches: grids bounded by the layer's placement work
            const bool act = l.kind == DFX_RELU || l.kind == DFX_TRUNCATE || l.kind == DFX_OUTPUT;
            const long long e4 = (long long)a.t * a.t * a.C / 4, nch = (e4 + 255) / 256;
            set_trunc_work_hint(act ? (long long)th * tw * std::max<long long>(nch, a.t / 2) : 0);
        }
        if (branch_) {
            for (int q : rt.waits) CUDA_CHECK(cudaStreamWaitEvent(s, lrt_[q].ev, 0));
            if (rt.wait_input) CUDA_CHECK(cudaStreamWaitEvent(s, in_ev_, 0));
        }
        switch (l.kind) {
            case DFX_CONV:
                if (rt.dense) {
                    // stride-1 conv: units (16x8 px, or 128/t^2 active tiles) with >= tau
                    // targets computed whole by k_conv_dense; targets of sparser units go
                    // to the gathered kernel (k_conv_tc)
                    static const int tau_env = getenv("DFX_DENSE_TAU") ? atoi(getenv("DFX_DENSE_TAU")) : -1;
                    // every unit with a target is computed whole (measured on C2 at the named
                    // ~10 % update rate: +3 % over sending sparse 16-px-tile strips to the
                    // gathered kernel with tau = 48; DFX_DENSE_TAU overrides)
                    const int tau = tau_env >= 1 ? tau_env : 1;
                    unsigned* tm = rt.tm_consumer >= 0 ? tmax + (size_t)rt.tm_consumer * nslots : nullptr;
                    const BufDev tmb = rt.tm_consumer >= 0 ? lrt_[rt.tm_consumer].aux : BufDev{nullptr, 0, 0};
                    if (!rt.plan_fused)  // else it ran inside the producing activation's commit launch
                        PROF(DFX_FAM_CONV_TARGETS, launch_conv_plan(C, s, rt.dp, a, rt.pkt, rt.halo_geom, rt.units.p,
                                                                    ucounts + idx2, flop_px + idx2, tau, rt.list.p,
                                                                    counts + idx2, tau == 1 ? tm : nullptr, tmb));
                    if (tau > 1 && l.stride == 1)
                        PROF(DFX_FAM_CONV_MMA, launch_conv_tc(C, s, a, rt.wtc.p, l.cin, rt.cin_pad, l.cout, rt.cout_pad,
                                                              l.k, l.stride, l.k / 2, rt.pkt, rt.halo_geom, rt.list.p,
                                                              counts + idx2, rt.max_targets, num_sms_, rt.ws.p,
                                                              rt.splits));
                    {
                        // the sole consuming activation's state: prefetched to L2 by the conv
                        BufDev na{nullptr, 0, 0}, nt{nullptr, 0, 0};
                        int cj = -1, ncons = 0;
                        for (size_t j = 0; j < net_.layers.size(); ++j)
                            if (net_.layers[j].in0 == idx2 || net_.layers[j].in1 == idx2) cj = (int)j, ++ncons;
                        if (ncons == 1 && (net_.layers[cj].kind == DFX_RELU || net_.layers[cj].kind == DFX_TRUNCATE ||
                                           net_.layers[cj].kind == DFX_OUTPUT))
                            na = lrt_[cj].acc, nt = lrt_[cj].aux;
                        PROF(DFX_FAM_CONV_MMA, launch_conv_dense(C, s, rt.dp, a, rt.pkt, rt.wdense.p, l.cin, l.cout,
                                                                 rt.units.p, ucounts + idx2, rt.wsd.p, rt.dcnt.p,
                                                                 num_sms_, na, nt, tau == 1 ? tm : nullptr,
                                                                 rt.has_tmap ? rt.tmap : nullptr));
                    }
                    break;
                }
                PROF(DFX_FAM_CONV_TARGETS, launch_conv_targets(C, s, a, l.k, l.stride, l.k / 2, rt.pkt, rt.halo_geom, rt.list.p, counts + idx2,
                                    flop_px + idx2));
                {
                const int pi = prof_begin(DFX_FAM_CONV_MMA);
                if (cfg_.conv_mode == DFX_CONV_EXACT || !conv_tc_supported(l.k))
                    launch_conv_exact(C, s, a, rt.w.p, l.cin, l.cout, l.k, l.stride, l.k / 2, rt.pkt, rt.halo_geom,
                                      rt.list.p, counts + idx2, rt.max_targets);
                else
                    launch_conv_tc(C, s, a, rt.wtc.p, l.cin, rt.cin_pad, l.cout, rt.cout_pad, l.k, l.stride, l.k / 2,
                                   rt.pkt, rt.halo_geom, rt.list.p, counts + idx2, rt.max_targets, num_sms_, rt.ws.p,
                                   rt.splits);
                prof_end(pi);
                ++launches_;
                }
                break;
            case DFX_RELU:
            case DFX_TRUNCATE:
            case DFX_OUTPUT:
                if (rt.tm_fused) {
                    // pass 1 ran in the producing conv: commit (+ halo stash) only
                    BufDev pf0{nullptr, 0, 0}, pf1{nullptr, 0, 0};
                    int pj = -1, ncons = 0;
                    for (size_t j = 0; j < net_.layers.size(); ++j)
                        if (net_.layers[j].in0 == idx2 || net_.layers[j].in1 == idx2) pj = (int)j, ++ncons;
                    if (ncons == 1 && net_.layers[pj].kind == DFX_MAXPOOL) pf0 = lrt_[pj].acc, pf1 = lrt_[pj].aux;
                    PROF(DFX_FAM_TRUNC, launch_trunc_commit_stash(C, s, a, rt.acc, rt.aux, tmax + (size_t)idx2 * nslots,
                                                                  rt.thr, l.kind == DFX_RELU ? 1 : 0, rt.pkt, pf0, pf1));
                    break;
                }
                if (rt.plan_conv >= 0) {
                    // pass 1 (tile max + stash), then pass 2 (with the fused max pool, if
                    // any) and the next conv's plan in one launch
                    const int cj = rt.plan_conv;
                    LayerRT& cr = lrt_[cj];
                    const bool pool = rt.pool_consumer >= 0;
                    LayerRT* pr = pool ? &lrt_[rt.pool_consumer] : nullptr;
                    unsigned* tm = tmax + (size_t)idx2 * nslots;
                    PROF(DFX_FAM_TRUNC, launch_trunc_tilemax(C, s, a, rt.aux, tm));
                    PROF(DFX_FAM_TRUNC,
                         launch_trunc_commit_plan(C, s, a, rt.acc, rt.aux, tm, rt.thr, l.kind == DFX_RELU ? 1 : 0,
                                                  rt.pkt, pool ? pr->acc : BufDev{nullptr, 0, 0},
                                                  pool ? pr->aux : BufDev{nullptr, 0, 0}, pool ? pr->pkt : PktDev{},
                                                  cr.dp, in_packet(net_.layers[cj].in0), cr.pkt, cr.halo_geom,
                                                  cr.units.p, ucounts + cj, flop_px + cj, cr.list.p, counts + cj));
                    break;
                }
                if (rt.pool_consumer >= 0) {
                    // pass 1 (tile max + stash), then pass 2 fused with the consuming max pool
                    LayerRT& pr = lrt_[rt.pool_consumer];
                    unsigned* tm = tmax + (size_t)idx2 * nslots;
                    PROF(DFX_FAM_TRUNC, launch_trunc_tilemax(C, s, a, rt.aux, tm));
                    PROF(DFX_FAM_TRUNC, launch_trunc_commit_pool(C, s, a, rt.acc, rt.aux, tm, rt.thr,
                                                                 l.kind == DFX_RELU ? 1 : 0, rt.pkt, pr.acc, pr.aux,
                                                                 pr.pkt));
                    break;
                }
                if (a.halo > 0 && (a.C & 3) != 0) PROF(DFX_FAM_TRUNC, launch_ring_add(C, s, a, rt.aux));
                {
                    // two streaming passes: tile max (+ the halo stash), then fire / fold (kernels_hbm.cu)
                    const int pi = prof_begin(DFX_FAM_TRUNC);
                    // the output layer densifies inside its activation launch
                    static const bool fuse_out = !(getenv("DFX_FUSE_OUT") && getenv("DFX_FUSE_OUT")[0] == '0');
                    DenseOut dz{nullptr, Readback{}};
                    if (fuse_out && idx2 == net_.out_layer)
                        dz = DenseOut{out_cur_ ? out_cur_ : out_d_.p,
                                      Readback{counters_d_.p, rb_n1_, in_pkt_ext_.p,
                                               rb_n2_, readback_d_, pend_out_flag_, pend_out_val_}};
                    bool dzd = false;
                    // a sole consuming max pool: its acc / prev tiles of every fired tile go to L2
                    BufDev pf0{nullptr, 0, 0}, pf1{nullptr, 0, 0};
                    {
                        int pj = -1, ncons = 0;
                        for (size_t j = 0; j < net_.layers.size(); ++j)
                            if (net_.layers[j].in0 == idx2 || net_.layers[j].in1 == idx2) pj = (int)j, ++ncons;
                        if (ncons == 1 && net_.layers[pj].kind == DFX_MAXPOOL) pf0 = lrt_[pj].acc, pf1 = lrt_[pj].aux;
                    }
                    const int nk = launch_trunc_two_pass(C, s, a, rt.acc, rt.aux, tmax + (size_t)idx2 * nslots,
                                                         rt.thr, l.kind == DFX_RELU ? 1 : 0, rt.pkt, gbars + idx2,
                                                         dz.out ? &dz : nullptr, &dzd, pf0, pf1);
                    if (dzd) densified = true;
                    prof_end(pi);
                    if (nk > 0) {
                        launches_ += nk;
                    } else {
                        PROF(DFX_FAM_TRUNC, launch_trunc_max(C, s, a, rt.aux, tmax + (size_t)idx2 * nslots));
                        PROF(DFX_FAM_TRUNC, launch_trunc_apply(C, s, a, rt.acc, rt.aux, tmax + (size_t)idx2 * nslots,
                                                             rt.thr, l.kind == DFX_RELU ? 1 : 0, rt.pkt));
                    }
                }
                break;
            case DFX_MAXPOOL:
                if (rt.pool_fused) break;  // ran inside the producing activation's commit
                if (a.halo == 0 && l.pool_k == l.pool_s && (a.C & 3) == 0) {
                    PROF(DFX_FAM_POOL, launch_maxpool_vec(C, s, a, rt.acc, rt.aux, l.pool_k, rt.pkt));
                } else if (a.halo == 0 && l.pool_k == l.pool_s) {
                    PROF(DFX_FAM_POOL, launch_maxpool_fused(C, s, a, rt.acc, rt.aux, l.pool_k, rt.pkt));
                } else {
                    PROF(DFX_FAM_POOL, launch_tile_add(C, s, a, rt.acc));
                    if (a.halo > 0) PROF(DFX_FAM_POOL, launch_ring_add(C, s, a, rt.acc));
                    PROF(DFX_FAM_POOL, launch_maxpool_out(C, s, a, rt.acc, rt.aux, l.pool_k, l.pool_s, rt.pkt, rt.halo_geom));
                }
                break;
            case DFX_AVGPOOL: PROF(DFX_FAM_POOL, launch_avgpool(C, s, a, l.pool_k, l.pool_s, rt.pkt)); break;
            case DFX_UPSAMPLE:
                if (!rt.up_fused) PROF(DFX_FAM_LINEAR, launch_upsample(C, s, a, l.factor, rt.pkt));
                break;
            case DFX_BATCHNORM: PROF(DFX_FAM_LINEAR, launch_bn(C, s, a, rt.scale.p, rt.pkt)); break;
            case DFX_ADD:
                if (rt.up_in >= 0) {  // the upsample input sampled in place (addition commutes exactly)
                    const Layer& u = net_.layers[rt.up_in];
                    const int other = rt.up_in == l.in1 ? l.in0 : l.in1;
                    PROF(DFX_FAM_LINEAR, launch_add(C, s, in_packet(other), in_packet(u.in0), rt.pkt, u.factor));
                } else {
                    PROF(DFX_FAM_LINEAR, launch_add(C, s, a, in_packet(l.in1), rt.pkt));
                }
                break;
        }
        if (branch_ && rt.signal) CUDA_CHECK(cudaEventRecord(rt.ev, s));
    }
    prof_s_ = stream_;
    if (grid_hint_) set_trunc_work_hint(0);
    if (branch_ && lrt_[net_.out_layer].sid != 0) CUDA_CHECK(cudaStreamWaitEvent(stream_, lrt_[net_.out_layer].ev, 0));
    const LayerRT& ort = lrt_[net_.out_layer];
    const Readback rb{counters_d_.p, rb_n1_, in_pkt_ext_.p, rb_n2_, readback_d_,
                      pend_out_flag_, pend_out_val_};
    if (!densified) PROF(DFX_FAM_DENSIFY, launch_densify(C, s, ort.acc, ort.aux, out_cur_ ? out_cur_ : out_d_.p, rb));
    CUDA_CHECK(cudaGetLastError());

    // the small readback (per-layer target counts, dropped, fired input tiles) is
    // written into mapped host memory by the last kernel (launch_densify)
    place_ = pl;
    const Layer& ol = net_.layers[net_.out_layer];
    info.out_channels = ol.in_channels;
    info.out_height = th * ol.in_tile;
    info.out_width = tw * ol.in_tile;
    ++frame_index_;
    have_frame_ = true;
}

void Engine::set_profiling(bool on) {
    prof_ = on;
    prof_used_ = 0;
}
void Engine::reset_profile() {
    for (int i = 0; i < DFX_FAMILIES; ++i) prof_ms_[i] = 0, prof_launch_[i] = 0, prof_work_[i] = 0;
}
void Engine::profile(int fam, double* ms, uint64_t* launches, double* work) const {
    check(fam >= 0 && fam < DFX_FAMILIES, "bad kernel family");
    *ms = prof_ms_[fam];
    *launches = prof_launch_[fam];
    *work = prof_work_[fam];
}
void Engine::timer_start() {
    if (!timer_a_) {
        CUDA_CHECK(cudaEventCreate(&timer_a_));
        CUDA_CHECK(cudaEventCreate(&timer_b_));
    }
    CUDA_CHECK(cudaEventRecord(timer_a_, stream_));
}
float Engine::timer_stop() {
    check(timer_a_ != nullptr, "timer not started");
    CUDA_CHECK(cudaEventRecord(timer_b_, stream_));
    CUDA_CHECK(cudaEventSynchronize(timer_b_));
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, timer_a_, timer_b_));
    return ms;
}

// Per-family kernel time (CUDA events) and ALGORITHMIC work of the frame
// (SURVEY §8(d) formulas: bytes for the HBM-bound families, the reference's
// FlopReport for the convs). Profiling mode only; synchronous.
void Engine::prof_harvest() {
    if (!prof_ || prof_used_ == 0) return;
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    for (size_t i = 0; i < prof_used_; ++i) {
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, prof_pool_[i].a, prof_pool_[i].b));
        prof_ms_[prof_pool_[i].fam] += ms;
        prof_launch_[prof_pool_[i].fam] += 1;
    }
    prof_used_ = 0;
    const int th = place_.th, tw = place_.tw;
    std::vector<uint8_t> cnt(cnt_bytes_);
    CUDA_CHECK(cudaMemcpy(cnt.data(), counters_d_.p, cnt_bytes_, cudaMemcpyDeviceToHost));
    const uint64_t* fpx = reinterpret_cast<const uint64_t*>(cnt.data());
    const int* counts = reinterpret_cast<const int*>(cnt.data() + off_counts_);
    auto ext_of = [&](const PktDev& p) {
        std::vector<uint8_t> e((size_t)(rows_ + 2 * p.RT) * p.ext_pitch);
        CUDA_CHECK(cudaMemcpy(e.data(), p.ext, e.size(), cudaMemcpyDeviceToHost));
        return e;
    };
    auto inside = [&](const PktDev& p, const std::vector<uint8_t>& e) {
        double n = 0;
        for (int r = 0; r < th; ++r)
            for (int c = 0; c < tw; ++c) n += e[(size_t)(r + p.RT) * p.ext_pitch + c + p.RT] ? 1 : 0;
        return n;
    };
    // valid pixels of the whole grown packet (inside tiles + ring tiles clipped to the grown extent)
    auto valid_px = [&](const PktDev& p, const std::vector<uint8_t>& e, bool ring_only) {
        double n = 0;
        for (int i = -p.RT; i < th + p.RT; ++i)
            for (int j = -p.RT; j < tw + p.RT; ++j) {
                const bool in_ext = i >= 0 && i < th && j >= 0 && j < tw;
                if (ring_only && in_ext) continue;
                if (!e[(size_t)(i + p.RT) * p.ext_pitch + j + p.RT]) continue;
                const int y0 = std::max(i * p.t, -p.halo), y1 = std::min((i + 1) * p.t, th * p.t + p.halo);
                const int x0 = std::max(j * p.t, -p.halo), x1 = std::min((j + 1) * p.t, tw * p.t + p.halo);
                if (y1 > y0 && x1 > x0) n += (double)(y1 - y0) * (x1 - x0);
            }
        return n;
    };
    double claim_elems = 0;
    {
        std::vector<ClaimBuf> cb(nclaim_bufs_);
        CUDA_CHECK(cudaMemcpy(cb.data(), claim_bufs_.p, cb.size() * sizeof(ClaimBuf), cudaMemcpyDeviceToHost));
        for (const auto& b : cb) claim_elems += (double)b.C * b.t * b.t;
    }
    prof_work_[DFX_FAM_CLAIMS] += 4.0 * claim_elems * last_nclaims_;
    {
        std::vector<uint8_t> cov((size_t)rows_ * cols_);
        CUDA_CHECK(cudaMemcpy(cov.data(), cov_d_.p, cov.size(), cudaMemcpyDeviceToHost));
        double ncov = 0;
        for (int i = 0; i < th * tw; ++i) ncov += cov[i] ? 1 : 0;
        const double F = inside(in_pkt_, ext_of(in_pkt_));
        const double T2 = (double)cfg_.tile_size * cfg_.tile_size;
        prof_work_[DFX_FAM_INPUT] += 4.0 * net_.in_channels * T2 * (3 * ncov + 3 * F + (ncov - F));
    }
    for (int idx : net_.topo) {
        const Layer& l = net_.layers[idx];
        const LayerRT& rt = lrt_[idx];
        const PktDev a = in_packet(l.in0);
        const auto ea = ext_of(a);
        const auto eo = ext_of(rt.pkt);
        switch (l.kind) {
            case DFX_CONV: {
                const double per_px = 2.0 * l.k * l.k * l.cin * l.cout;
                prof_work_[DFX_FAM_CONV_MMA] += per_px * (double)fpx[idx];
                // a plan run inside the producing activation's launch is timed with it
                prof_work_[rt.plan_fused ? DFX_FAM_TRUNC : DFX_FAM_CONV_TARGETS] +=
                    4.0 * l.cout * std::max(0.0, valid_px(rt.pkt, eo, false) - (double)counts[idx]) + 4.0 * counts[idx];
                break;
            }
            case DFX_RELU:
            case DFX_TRUNCATE:
            case DFX_OUTPUT: {
                const double A = inside(a, ea), F = inside(rt.pkt, eo), T2 = (double)a.t * a.t;
                const double H = a.halo > 0 ? valid_px(a, ea, true) : 0.0;
                prof_work_[DFX_FAM_TRUNC] += 4.0 * a.C * (T2 * (3 * A + 3 * F) + 3 * H);
                break;
            }
            case DFX_MAXPOOL: {
                const double A = inside(a, ea), T2 = (double)a.t * a.t;
                const double H = a.halo > 0 ? valid_px(a, ea, true) : 0.0;
                // a pool fused into the activation's commit is timed with the activation
                prof_work_[rt.pool_fused ? DFX_FAM_TRUNC : DFX_FAM_POOL] +=
                    4.0 * a.C * (3 * A * T2 + 3 * H + 3 * valid_px(rt.pkt, eo, false));
                break;
            }
            case DFX_AVGPOOL:
                prof_work_[DFX_FAM_POOL] += 4.0 * a.C * (valid_px(a, ea, false) + valid_px(rt.pkt, eo, false));
                break;
            case DFX_ADD: {
                const PktDev b = in_packet(l.in1);
                prof_work_[DFX_FAM_LINEAR] +=
                    4.0 * a.C * (valid_px(a, ea, false) + valid_px(b, ext_of(b), false) + valid_px(rt.pkt, eo, false));
                break;
            }
            default:
                // a folded upsample writes nothing (its add reads the input instead)
                prof_work_[DFX_FAM_LINEAR] +=
                    4.0 * a.C * (valid_px(a, ea, false) + (rt.up_fused ? 0.0 : valid_px(rt.pkt, eo, false)));
        }
    }
    {
        const Layer& ol = net_.layers[net_.out_layer];
        prof_work_[DFX_FAM_DENSIFY] += 12.0 * ol.in_channels * (double)ol.in_tile * ol.in_tile * th * tw;
    }
}

void Engine::finish_info(dfx_frame_info* out) {
    dfx_frame_info info = pending_;
    const size_t nl = net_.layers.size();
    const uint64_t* fpx = reinterpret_cast<const uint64_t*>(readback_h_);
    for (size_t i = 0; i < nl; ++i) {
        const Layer& l = net_.layers[i];
        if (l.kind != DFX_CONV) continue;
        const uint64_t per_px = 2ull * l.k * l.k * l.cin * l.cout;
        info.conv_flops += per_px * fpx[i];
        info.dense_flops += per_px * (uint64_t)(place_.th * l.tile) * (uint64_t)(place_.tw * l.tile);
    }
    const uint64_t dropped = *reinterpret_cast<const uint64_t*>(readback_h_ + nl * 8);
    if (dropped) info.dropped_pixels = (int64_t)dropped;
    const uint8_t* mask = readback_h_ + rb_n1_;
    int cnt = 0;
    for (int i = 0; i < place_.th * place_.tw; ++i) cnt += mask[(i / place_.tw) * in_pkt_.ext_pitch + i % place_.tw] ? 1 : 0;
    info.update_rate = (double)cnt / ((double)place_.th * place_.tw);
    pending_ = info;
    if (out) *out = info;
}

void Engine::ensure_staging(int c, int h, int w, bool host_frame) {
    const size_t fsz = (size_t)c * h * w, px = (size_t)h * w;
    if (host_frame && frame_d_.n < fsz) frame_d_.alloc(fsz);
    if (warped_d_.n < fsz) warped_d_.alloc(fsz);
    if (fp_d_.n < px) fp_d_.alloc(px);
    if (cfg_.roi_enabled && roi_frame_d_.n < px) {
        roi_frame_d_.alloc(px);
        roi_warped_d_.alloc(px);
        roi_fp_d_.alloc(px);
    }
}

void Engine::run_frame(const float* frame, int c, int h, int w, const float* h9, const float* roi,
                       dfx_frame_info* info, float* out, size_t cap, bool frame_dev, bool out_dev) {
    check(c == net_.in_channels, "run_frame: input channel mismatch");
    CUDA_CHECK(cudaSetDevice(device_));
    if (frame_dev) {
        // device-resident frame / ROI: no staging copies (SURVEY §8(b) frame_is_device)
        ensure_staging(c, h, w, false);
        enqueue(frame, c, h, w, h9, cfg_.roi_enabled ? roi : nullptr);
        const size_t n = (size_t)pending_.out_channels * pending_.out_height * pending_.out_width;
        if (out && cap >= n) {
            if (out_dev) {
                CUDA_CHECK(cudaMemcpyAsync(out, out_d_.p, n * 4, cudaMemcpyDeviceToDevice, stream_));
                CUDA_CHECK(cudaStreamSynchronize(stream_));
            } else {
                CUDA_CHECK(cudaMemcpyAsync(out, out_d_.p, n * 4, cudaMemcpyDeviceToHost, stream_));
                CUDA_CHECK(cudaStreamSynchronize(stream_));
            }
        } else {
            CUDA_CHECK(cudaStreamSynchronize(stream_));
        }
        CUDA_CHECK(cudaGetLastError());
        finish_info(info);
        prof_harvest();
        return;
    }
    const size_t fsz = (size_t)c * h * w;
    ensure_staging(c, h, w, true);
    // caller buffers are ordinary (pageable) host memory: stage through pinned
    // buffers so the copies run at full PCIe rate
    if (in_h_n_ < fsz) {
        if (in_h_) cudaFreeHost(in_h_);
        CUDA_CHECK(cudaMallocHost(&in_h_, fsz * 4));
        in_h_n_ = fsz;
    }
    memcpy(in_h_, frame, fsz * 4);
    CUDA_CHECK(cudaMemcpyAsync(frame_d_.p, in_h_, fsz * 4, cudaMemcpyHostToDevice, stream_));
    const float* roi_dev = nullptr;
    if (roi && cfg_.roi_enabled) {
        CUDA_CHECK(cudaMemcpyAsync(roi_frame_d_.p, roi, (size_t)h * w * 4, cudaMemcpyHostToDevice, stream_));
        roi_dev = roi_frame_d_.p;
    }
    enqueue(frame_d_.p, c, h, w, h9, roi_dev);
    const size_t n = (size_t)pending_.out_channels * pending_.out_height * pending_.out_width;
    if (out_dev && out && cap >= n) {
        CUDA_CHECK(cudaMemcpyAsync(out, out_d_.p, n * 4, cudaMemcpyDeviceToDevice, stream_));
        out = nullptr;
    }
    const bool want = out && cap >= n;
    if (want) {
        if (out_h_n_ < n) {
            if (out_h_) cudaFreeHost(out_h_);
            CUDA_CHECK(cudaMallocHost(&out_h_, n * 4));
            out_h_n_ = n;
        }
        // out_d_ is [C][th*t][tw*t] compact (k_densify writes the placement extent)
        CUDA_CHECK(cudaMemcpyAsync(out_h_, out_d_.p, n * 4, cudaMemcpyDeviceToHost, stream_));
    }
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    CUDA_CHECK(cudaGetLastError());
    if (want) memcpy(out, out_h_, n * 4);
    finish_info(info);
    prof_harvest();
}

void Engine::submit(const float* frame_dev, int c, int h, int w, const float* h9) {
    CUDA_CHECK(cudaSetDevice(device_));
    if (prof_ && prof_used_) {
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        finish_info(nullptr);
        prof_harvest();
    }
    ensure_staging(c, h, w, false);
    enqueue(frame_dev, c, h, w, h9, nullptr);
}

// Pipelined host-buffer frame (throughput form of run_frame): frame k's H2D
// copy (copy stream 1) overlaps frame k-1's compute, its output D2H copy (copy
// stream 2) overlaps frame k+1's compute; device frame and output buffers are
// double buffered and guarded by per-slot events. `frame` and `out` should be
// pinned for the copies to be asynchronous. Results of the last frame are
// readable after sync().
void Engine::submit_host(const float* frame, int c, int h, int w, const float* h9, float* out, size_t cap) {
    CUDA_CHECK(cudaSetDevice(device_));
    check(c == net_.in_channels, "run_frame: input channel mismatch");
    if (!cstream_) {
        CUDA_CHECK(cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking));
        CUDA_CHECK(cudaStreamCreateWithFlags(&dstream_, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CUDA_CHECK(cudaEventCreateWithFlags(&ev_h2d_[i], cudaEventDisableTiming));
            CUDA_CHECK(cudaEventCreateWithFlags(&ev_done_[i], cudaEventDisableTiming));
            CUDA_CHECK(cudaEventCreateWithFlags(&ev_d2h_[i], cudaEventDisableTiming));
        }
    }
    const int slot = (int)(hseq_ & 1);
    const size_t fsz = (size_t)c * h * w;
    ensure_staging(c, h, w, false);
    if (hframe_d_[slot].n < fsz) {
        CUDA_CHECK(cudaDeviceSynchronize());
        hframe_d_[slot].alloc(fsz);
    }
    if (!hflags_.p) {
        hflags_.alloc(4);
        CUDA_CHECK(cudaMemset(hflags_.p, 0, 4 * sizeof(unsigned)));
    }
    const unsigned v = (unsigned)(hseq_ + 1);
    // frame buffer free once the slot's previous frame finished computing
    CUDA_CHECK(cudaStreamWaitEvent(cstream_, ev_done_[slot], 0));
    CUDA_CHECK(cudaMemcpyAsync(hframe_d_[slot].p, frame, fsz * 4, cudaMemcpyHostToDevice, cstream_));
    launch_set_flag(cstream_, hflags_.p + slot, v);
    // the engine stream takes no event dependency (that would cut its
    // programmatic-launch chain): k_frame_begin polls the input flag, the
    // output kernel polls the slot's previous copy-out flag
    pend_in_flag_ = hflags_.p + slot;
    pend_in_val_ = v;
    pend_out_flag_ = hseq_ >= 2 ? hflags_.p + 2 + slot : nullptr;
    pend_out_val_ = v - 2;
    if (initialized_ && hout_d_[slot].n < out_d_.n) hout_d_[slot].alloc(out_d_.n);
    out_cur_ = initialized_ ? hout_d_[slot].p : nullptr;
    enqueue(hframe_d_[slot].p, c, h, w, h9, nullptr);
    pend_in_flag_ = pend_out_flag_ = nullptr;
    const float* result = out_cur_ ? out_cur_ : out_d_.p;
    out_cur_ = nullptr;
    CUDA_CHECK(cudaEventRecord(ev_done_[slot], stream_));
    const size_t n = (size_t)pending_.out_channels * pending_.out_height * pending_.out_width;
    CUDA_CHECK(cudaStreamWaitEvent(dstream_, ev_done_[slot], 0));
    if (out && cap >= n) CUDA_CHECK(cudaMemcpyAsync(out, result, n * 4, cudaMemcpyDeviceToHost, dstream_));
    launch_set_flag(dstream_, hflags_.p + 2 + slot, v);
    ++hseq_;
}

void Engine::sync(dfx_frame_info* info) {
    CUDA_CHECK(cudaSetDevice(device_));
    if (cstream_) CUDA_CHECK(cudaStreamSynchronize(cstream_));
    if (dstream_) CUDA_CHECK(cudaStreamSynchronize(dstream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    CUDA_CHECK(cudaGetLastError());
    check(have_frame_, "no frame submitted");
    finish_info(info);
    prof_harvest();
}

void Engine::output_device(const float** p, int* c, int* h, int* w) const {
    *p = out_d_.p;
    *c = pending_.out_channels;
    *h = pending_.out_height;
    *w = pending_.out_width;
}

void Engine::input_mask(uint8_t* out, size_t cap, int* th, int* tw) const {
    check(have_frame_, "no frame");
    *th = place_.th;
    *tw = place_.tw;
    check(cap >= (size_t)place_.th * place_.tw, "mask buffer too small");
    const uint8_t* mask = readback_h_ + rb_n1_;
    for (int r = 0; r < place_.th; ++r)
        for (int c = 0; c < place_.tw; ++c) out[r * place_.tw + c] = mask[r * in_pkt_.ext_pitch + c] ? 1 : 0;
}

void Engine::layer_flops(int layer, uint64_t* f, uint64_t* d) const {
    check(layer >= 0 && layer < (int)net_.layers.size(), "bad layer index");
    const Layer& l = net_.layers[layer];
    *f = *d = 0;
    if (l.kind != DFX_CONV || !have_frame_) return;
    const uint64_t per_px = 2ull * l.k * l.k * l.cin * l.cout;
    *f = per_px * reinterpret_cast<const uint64_t*>(readback_h_)[layer];
    *d = per_px * (uint64_t)(place_.th * l.tile) * (uint64_t)(place_.tw * l.tile);
}

void Engine::read_state(const std::string& layer, int which, float* out, size_t cap, int* c, int* h, int* w) {
    check(initialized_, "no state buffer for layer " + layer);
    BufDev b{};
    if (layer == "input") {
        if (which == DFX_STATE_ACC) b = in_acc_;
        else if (which == DFX_STATE_TRUNC) b = in_trunc_;
    } else {
        const int i = net_.index_of(layer);
        check(i >= 0, "no state buffer for layer " + layer);
        const int k = net_.layers[i].kind;
        const LayerRT& rt = lrt_[i];
        if (k == DFX_RELU || k == DFX_TRUNCATE || k == DFX_OUTPUT) {
            if (which == DFX_STATE_ACC) b = rt.acc;
            else if (which == DFX_STATE_TRUNC) b = rt.aux;
        } else if (k == DFX_MAXPOOL) {
            if (which == DFX_STATE_ACC) b = rt.acc;
            else if (which == DFX_STATE_PREV) b = rt.aux;
        }
    }
    check(b.d != nullptr, "no state buffer for layer " + layer);
    *c = b.C;
    *h = rows_ * b.t;
    *w = cols_ * b.t;
    if (!out) return;
    const size_t n = (size_t)b.C * rows_ * b.t * cols_ * b.t;
    check(cap >= n, "state buffer too small");
    std::vector<float> raw(n);
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    CUDA_CHECK(cudaMemcpy(raw.data(), b.d, n * 4, cudaMemcpyDeviceToHost));
    const int t = b.t, C = b.C, PW = cols_ * t;
    for (int sr = 0; sr < rows_; ++sr)
        for (int sc = 0; sc < cols_; ++sc)
            for (int y = 0; y < t; ++y)
                for (int x = 0; x < t; ++x)
                    for (int ch = 0; ch < C; ++ch)
                        out[((size_t)ch * rows_ * t + sr * t + y) * PW + sc * t + x] =
                            raw[((((size_t)sr * cols_ + sc) * t + y) * t + x) * C + ch];
}

void Engine::read_packet(const std::string& layer, float* out, size_t cap, int* c, int* gh, int* gw, int* halo,
                         uint8_t* mask, size_t mask_cap) {
    check(have_frame_, "no packet for layer " + layer);
    PktDev p;
    int f = 1;  // an upsample folded into its add: expand its input packet here
    if (layer == "input") {
        p = in_pkt_;
    } else {
        const int i = net_.index_of(layer);
        check(i >= 0, "no packet for layer " + layer);
        p = lrt_[i].pkt;
        if (lrt_[i].up_fused) {
            f = net_.layers[i].factor;
            const PktDev src = in_packet(net_.layers[i].in0);
            PktDev v = src;  // the upsampled geometry over the input's storage
            v.t = src.t * f;
            v.halo = src.halo * f;
            p.C = v.C;
            p.t = v.t;
            p.halo = v.halo;
            p.RT = src.RT;
            p.d = src.d;
            p.ext = src.ext;
            p.pitch_w = src.pitch_w;
            p.ext_pitch = src.ext_pitch;
        }
    }
    const int th = place_.th, tw = place_.tw;
    *c = p.C;
    *gh = th * p.t + 2 * p.halo;
    *gw = tw * p.t + 2 * p.halo;
    *halo = p.halo;
    if (!out) return;
    const size_t n = (size_t)p.C * *gh * *gw;
    check(cap >= n && mask_cap >= (size_t)th * tw, "packet buffer too small");
    const int sh = p.halo / f, st = p.t / f;  // the stored packet's halo / tile (f = 1: the packet itself)
    const size_t rows_stored = (size_t)rows_ * st + 2 * sh;
    std::vector<float> raw(rows_stored * p.pitch_w * p.C);
    std::vector<uint8_t> ext((size_t)(rows_ + 2 * p.RT) * p.ext_pitch);
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    CUDA_CHECK(cudaMemcpy(raw.data(), p.d, raw.size() * 4, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(ext.data(), p.ext, ext.size(), cudaMemcpyDeviceToHost));
    for (int y = -p.halo; y < th * p.t + p.halo; ++y)
        for (int x = -p.halo; x < tw * p.t + p.halo; ++x) {
            const int i = (int)floor_div64(y, p.t), j = (int)floor_div64(x, p.t);
            const bool v = ext[(size_t)(i + p.RT) * p.ext_pitch + (j + p.RT)] != 0;
            const int sy = (int)floor_div64(y, f), sx = (int)floor_div64(x, f);  // delta_layers.cpp:351-363
            for (int ch = 0; ch < p.C; ++ch)
                out[((size_t)ch * *gh + (y + p.halo)) * *gw + (x + p.halo)] =
                    v ? raw[((size_t)(sy + sh) * p.pitch_w + (sx + sh)) * p.C + ch] : 0.0f;
        }
    for (int r = 0; r < th; ++r)
        for (int cc = 0; cc < tw; ++cc) mask[r * tw + cc] = ext[(size_t)(r + p.RT) * p.ext_pitch + (cc + p.RT)] ? 1 : 0;
}

void Engine::read_ledger(int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) const {
    check(initialized_, "engine not initialized");
    const auto& s = ledger_.slots();
    check(cap >= s.size(), "ledger buffer too small");
    for (size_t i = 0; i < s.size(); ++i) {
        used[i] = s[i].used;
        ty[i] = s[i].coord.ty;
        tx[i] = s[i].coord.tx;
        covered[i] = s[i].covered;
    }
}

}  // namespace dfx

// ===================================================================== C-ABI
using dfx::Engine;
struct dfx_engine {
    Engine* e;
};

namespace {
thread_local std::string g_last;
}  // namespace
namespace dfx {
void set_last_error(const std::string& m) { g_last = m; }
}  // namespace dfx
namespace {
template <typename F>
int guard(F&& f) {
    try {
        f();
        return DFX_OK;
    } catch (const dfx::Error& e) {
        g_last = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last = e.what();
        return DFX_ERR;
    }
}
}  // namespace

extern "C" {

const char* dfx_last_error(void) { return g_last.c_str(); }

void dfx_default_config(dfx_engine_config* c) {
    // dflx::EngineConfig defaults (engine.hpp:10-21)
    c->tile_size = 32;
    c->grid_rows = 0;
    c->grid_cols = 0;
    c->input_threshold = 0.15f;
    c->default_threshold = 0.02f;
    c->override_net_thresholds = 0;
    c->mask_dilation = 10;
    c->roi_enabled = 0;
    c->noise_suppression = 0;
    c->padded_convolutions = 1;
    c->conv_mode = DFX_CONV_TF32X3;
}

int dfx_engine_create(const dfx_net_desc* net, const dfx_engine_config* cfg, int device, dfx_engine** out) {
    return guard([&] {
        auto* h = new dfx_engine{nullptr};
        try {
            h->e = new Engine(net, cfg, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int dfx_engine_create_on_stream(const dfx_net_desc* net, const dfx_engine_config* cfg, int device, void* stream,
                                dfx_engine** out) {
    return guard([&] {
        auto* h = new dfx_engine{nullptr};
        try {
            h->e = new Engine(net, cfg, device, static_cast<cudaStream_t>(stream));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int dfx_engine_destroy(dfx_engine* e) {
    return guard([&] {
        if (!e) return;
        delete e->e;
        delete e;
    });
}

int dfx_engine_run_frame(dfx_engine* e, const float* frame, int c, int h, int w, const float* h9, const float* roi,
                         dfx_frame_info* info, float* out, size_t out_cap) {
    return guard([&] { e->e->run_frame(frame, c, h, w, h9, roi, info, out, out_cap); });
}
int dfx_engine_run_frame_ex(dfx_engine* e, const float* frame, int c, int h, int w, int frame_is_device,
                            const float* h9, const float* roi, dfx_frame_info* info, float* out, size_t out_cap,
                            int out_is_device) {
    return guard([&] {
        e->e->run_frame(frame, c, h, w, h9, roi, info, out, out_cap, frame_is_device != 0, out_is_device != 0);
    });
}
int dfx_engine_layer_order(dfx_engine* e, int* order, int cap, int* n) {
    return guard([&] { e->e->layer_order(order, cap, n); });
}
int dfx_engine_submit_frame(dfx_engine* e, const float* frame_dev, int c, int h, int w, const float* h9) {
    return guard([&] { e->e->submit(frame_dev, c, h, w, h9); });
}
// Page-locked host memory from this library's CUDA runtime (frames / outputs
// for dfx_engine_submit_host_frame).
void* dfx_host_alloc(size_t bytes) {
    void* p = nullptr;
    return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}
void dfx_host_free(void* p) {
    if (p) cudaFreeHost(p);
}
int dfx_engine_submit_host_frame(dfx_engine* e, const float* frame, int c, int h, int w, const float* h9, float* out,
                                 size_t out_cap) {
    return guard([&] { e->e->submit_host(frame, c, h, w, h9, out, out_cap); });
}
int dfx_engine_sync(dfx_engine* e, dfx_frame_info* info) {
    return guard([&] { e->e->sync(info); });
}
int dfx_engine_reset(dfx_engine* e) {
    return guard([&] { e->e->reset(); });
}
int dfx_engine_output_device(dfx_engine* e, const float** p, int* c, int* h, int* w) {
    return guard([&] { e->e->output_device(p, c, h, w); });
}
int dfx_engine_input_mask(dfx_engine* e, uint8_t* out, size_t cap, int* th, int* tw) {
    return guard([&] { e->e->input_mask(out, cap, th, tw); });
}
int dfx_engine_num_layers(dfx_engine* e) { return e->e->num_layers(); }
int dfx_engine_layer_flops(dfx_engine* e, int layer, uint64_t* f, uint64_t* d) {
    return guard([&] { e->e->layer_flops(layer, f, d); });
}
int dfx_engine_grid(dfx_engine* e, int* rows, int* cols) {
    return guard([&] {
        *rows = e->e->rows();
        *cols = e->e->cols();
    });
}
int dfx_engine_read_state(dfx_engine* e, const char* layer, int which, float* out, size_t cap, int* c, int* h, int* w) {
    return guard([&] { e->e->read_state(layer, which, out, cap, c, h, w); });
}
int dfx_engine_read_packet(dfx_engine* e, const char* layer, float* out, size_t cap, int* c, int* gh, int* gw, int* halo,
                           uint8_t* mask, size_t mask_cap) {
    return guard([&] { e->e->read_packet(layer, out, cap, c, gh, gw, halo, mask, mask_cap); });
}
int dfx_engine_read_ledger(dfx_engine* e, int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) {
    return guard([&] { e->e->read_ledger(used, ty, tx, covered, cap); });
}
// ---- host-only ledger (TileLedger + plan_frame + apply_plan, buffer_manager.cpp:7-81),
// the same object the engine plans every frame with; exposed for parity fuzzing.
struct dfx_ledger {
    dfx::Ledger l;
};
int dfx_ledger_create(int rows, int cols, dfx_ledger** out) {
    return guard([&] {
        dfx::check(rows >= 1 && cols >= 1, "ledger: bad grid dims");
        auto* h = new dfx_ledger;
        h->l.init(rows, cols);
        *out = h;
    });
}
int dfx_ledger_destroy(dfx_ledger* h) {
    return guard([&] { delete h; });
}
int dfx_ledger_step(dfx_ledger* h, int64_t otx, int64_t oty, int th, int tw, int ring, int* full_reset,
                    int64_t* claims, int* victims, size_t claim_cap, int* nclaims, int64_t* fresh, size_t fresh_cap,
                    int* nfresh, int* evicted) {
    return guard([&] {
        dfx::Placement p;
        p.origin = {otx, oty};
        p.th = th;
        p.tw = tw;
        dfx::check(th <= h->l.rows() && tw <= h->l.cols(), "plan_frame: placement larger than grid");
        dfx::Plan plan = h->l.plan(p, ring);
        *full_reset = plan.full_reset ? 1 : 0;
        if (plan.full_reset) {  // engine.cpp:207-211
            h->l.clear();
            plan = h->l.plan(p, ring);
        }
        h->l.apply(plan, p);
        *nclaims = (int)plan.claims.size();
        *nfresh = (int)plan.fresh.size();
        *evicted = plan.evicted;
        for (size_t i = 0; i < plan.claims.size() && i < claim_cap; ++i) {
            claims[4 * i] = plan.claims[i].coord.tx;
            claims[4 * i + 1] = plan.claims[i].coord.ty;
            claims[4 * i + 2] = plan.claims[i].evicts ? plan.claims[i].victim.tx : 0;
            claims[4 * i + 3] = plan.claims[i].evicts ? plan.claims[i].victim.ty : 0;
            victims[i] = plan.claims[i].evicts ? 1 : 0;
        }
        for (size_t i = 0; i < plan.fresh.size() && i < fresh_cap; ++i) {
            fresh[2 * i] = plan.fresh[i].tx;
            fresh[2 * i + 1] = plan.fresh[i].ty;
        }
    });
}
int dfx_ledger_slots(dfx_ledger* h, int* used, int64_t* ty, int64_t* tx, uint8_t* covered, size_t cap) {
    return guard([&] {
        const auto& s = h->l.slots();
        dfx::check(cap >= s.size(), "ledger slots buffer too small");
        for (size_t i = 0; i < s.size(); ++i) {
            used[i] = s[i].used ? 1 : 0;
            ty[i] = s[i].coord.ty;
            tx[i] = s[i].coord.tx;
            covered[i] = s[i].covered ? 1 : 0;
        }
    });
}

// Debug: clock64 stamps of the last dense conv launch (DFX_CONV_DBG & 64).
int dfx_debug_conv_trace(long long* out, int n) {
    return guard([&] {
        long long* t = dfx::dense_conv_trace_buffer();
        dfx::check(t != nullptr, "no trace (set DFX_CONV_DBG=64)");
        cudaDeviceSynchronize();
        dfx::check(cudaMemcpy(out, t, (size_t)(n < 4096 ? n : 4096) * 8, cudaMemcpyDeviceToHost) == cudaSuccess,
                   "trace copy failed");
    });
}
// Debug: chain trace (DFX_KTRACE): enable with a device buffer of 4096 stamps
// + counter (on = 1), or copy the stamps and the count out (on = 0).
int dfx_debug_ktrace(int on, unsigned long long* out, unsigned* count) {
    return guard([&] {
        static unsigned long long* buf = nullptr;
        static unsigned* ctr = nullptr;
        if (on) {
            if (!buf) {
                dfx::check(cudaMalloc(&buf, 4096 * 8) == cudaSuccess && cudaMalloc(&ctr, 4) == cudaSuccess, "ktrace alloc");
            }
            cudaMemset(buf, 0, 4096 * 8);
            cudaMemset(ctr, 0, 4);
            dfx::ktrace_set_kernels(buf, ctr);
            dfx::ktrace_set_hbm(buf, ctr);
            dfx::ktrace_set_dense(buf, ctr);
            dfx::ktrace_set_tc(buf, ctr);
            cudaDeviceSynchronize();
        } else {
            dfx::check(buf != nullptr, "ktrace not enabled");
            cudaDeviceSynchronize();
            cudaMemcpy(out, buf, 4096 * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(count, ctr, 4, cudaMemcpyDeviceToHost);
        }
    });
}
// Debug: frame-boundary stamps (DFX_FRAME_TRACE=1), [64][4] u64.
int dfx_debug_frame_trace(unsigned long long* out) {
    return guard([&] { memcpy(out, dfx::frame_trace_host(), 64 * 4 * 8); });
}
// Debug: truncation phase stamps (DFX_TRUNC_TRACE=1), [64][1024][8] u64.
int dfx_debug_trunc_trace(unsigned long long* out, long long n) {
    return guard([&] {
        unsigned long long* t = dfx::trunc_trace_buffer();
        dfx::check(t != nullptr, "no trace (set DFX_TRUNC_TRACE=1)");
        cudaDeviceSynchronize();
        const long long cap = 64LL * 1024 * 16;
        dfx::check(cudaMemcpy(out, t, (size_t)(n < cap ? n : cap) * 8, cudaMemcpyDeviceToHost) == cudaSuccess,
                   "trace copy failed");
    });
}
// Debug: per-layer gathered-target counts and dense-unit counts of the last frame.
int dfx_engine_debug_counts(dfx_engine* e, int* gathered, int* units, int cap) {
    return guard([&] { e->e->debug_counts(gathered, units, cap); });
}
int dfx_engine_kernel_count(dfx_engine* e) { return e->e->kernel_count(); }
int dfx_engine_set_profiling(dfx_engine* e, int on) {
    return guard([&] { e->e->set_profiling(on != 0); });
}
int dfx_engine_reset_profile(dfx_engine* e) {
    return guard([&] { e->e->reset_profile(); });
}
int dfx_engine_profile(dfx_engine* e, int family, double* ms, uint64_t* launches, double* work) {
    return guard([&] { e->e->profile(family, ms, launches, work); });
}
const char* dfx_kernel_family_name(int family) {
    static const char* names[DFX_FAMILIES] = {"claims_reset", "input_stage", "conv_targets", "conv_mma",
                                              "truncate",     "pool",        "linear_ops",   "densify"};
    return (family >= 0 && family < DFX_FAMILIES) ? names[family] : "?";
}
int dfx_engine_timer_start(dfx_engine* e) {
    return guard([&] { e->e->timer_start(); });
}
int dfx_engine_timer_stop(dfx_engine* e, float* ms) {
    return guard([&] { *ms = e->e->timer_stop(); });
}

int dfx_validate_net(const dfx_net_desc* net, int tile_size, int* topo, int cap, int* n, int* ring) {
    return guard([&] {
        const dfx::Net v = dfx::validate_net(net, tile_size);
        int k = 0;
        for (int i : v.topo)
            if (k < cap) topo[k++] = i;
        *n = k;
        if (ring) *ring = v.ring;
    });
}

void dfx_wrap_tile(int64_t tx, int64_t ty, int rows, int cols, int* row, int* col) {
    // tile_grid.hpp:37-40
    *row = (int)dfx::floor_mod64(ty, rows);
    *col = (int)dfx::floor_mod64(tx, cols);
}

}  // extern "C"
