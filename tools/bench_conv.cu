// Microbenchmark of the two tcgen05 conv kernels on synthetic fully-masked
// packets (dev tool; not part of the product). Links libdfx_b200.so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include -I paper_2210_09887_b200/csrc \
//        tools/bench_conv.cu -o tools/bench_conv -Lpaper_2210_09887_b200 -ldfx_b200 -Xlinker -rpath=$PWD/paper_2210_09887_b200
// Env DFX_CONV_DBG: 1 skip MMA, 2 skip patch loads, 4 skip weight loads (dense kernel).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "kernels.hpp"

using namespace dfx;

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

static PktDev make_pkt(int C, int t, int halo, int rows, int cols, bool fill) {
    PktDev p{};
    p.C = C;
    p.t = t;
    p.halo = halo;
    p.RT = (halo + t - 1) / t;
    p.pitch_w = cols * t + 2 * halo;
    p.ext_pitch = cols + 2 * p.RT;
    const size_t n = (size_t)(rows * t + 2 * halo) * p.pitch_w * C;
    CK(cudaMalloc(&p.d, n * 4));
    std::vector<float> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = fill ? (float)((i * 2654435761u) % 1000) / 1000.0f - 0.5f : 0.0f;
    CK(cudaMemcpy(p.d, h.data(), n * 4, cudaMemcpyHostToDevice));
    const size_t ne = (size_t)(rows + 2 * p.RT) * p.ext_pitch;
    CK(cudaMalloc(&p.ext, ne));
    CK(cudaMemset(p.ext, 1, ne));
    return p;
}

int main(int argc, char** argv) {
    const int rows = 34, th = 32;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    FrameDev F{};
    F.th = F.tw = th;
    FrameDev* dF;
    CK(cudaMalloc(&dF, sizeof F));
    CK(cudaMemcpy(dF, &F, sizeof F, cudaMemcpyHostToDevice));
    SlotDev* dS;
    CK(cudaMalloc(&dS, sizeof(SlotDev) * rows * rows));
    Ctx c{dF, dS, rows, rows};
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    struct Cfg { int cin, cout, t; };
    const Cfg cfgs[] = {{64, 64, 16}, {64, 128, 8}, {128, 128, 8}, {128, 256, 4}, {256, 256, 4}, {256, 256, 2}};
    const char* dbg = getenv("DFX_CONV_DBG");
    printf("dbg=%s\n", dbg ? dbg : "0");
    const char* only = getenv("BENCH_CFG");
    int ci = -1;
    for (const Cfg& g : cfgs) {
        ++ci;
        if (only && atoi(only) != ci) continue;
        PktDev in = make_pkt(g.cin, g.t, 0, rows, rows, true);
        PktDev out = make_pkt(g.cout, g.t, 1, rows, rows, false);
        DenseConvPlan p = dense_conv_plan(g.cin, g.cout, 3, g.t, rows, rows, (size_t)256 << 20);
        std::vector<float> w((size_t)g.cout * g.cin * 9);
        for (size_t i = 0; i < w.size(); ++i) w[i] = (float)((i * 40503u) % 997) / 997.0f - 0.5f;
        std::vector<float> wd(dense_conv_weight_floats(p));
        dense_conv_prepare_weights(p, w.data(), g.cin, g.cout, wd.data());
        float* dw;
        CK(cudaMalloc(&dw, wd.size() * 4));
        CK(cudaMemcpy(dw, wd.data(), wd.size() * 4, cudaMemcpyHostToDevice));
        float* ws = nullptr;
        if (p.smax > 1) CK(cudaMalloc(&ws, (size_t)p.smax * p.units_max * 128 * p.cout_pad * 4));
        int* dcnt;
        CK(cudaMalloc(&dcnt, (size_t)p.units_max * p.nNB * 4));
        CK(cudaMemset(dcnt, 0, (size_t)p.units_max * p.nNB * 4));
        const int eh = th * g.t;
        const int nuy = eh / 16, nux = eh / 8;
        std::vector<int> units;
        for (int y = 0; y < nuy; ++y)
            for (int x = 0; x < nux; ++x) units.push_back((y << 16) | x);
        int* du;
        int* dn;
        CK(cudaMalloc(&du, units.size() * 4));
        CK(cudaMalloc(&dn, 4));
        CK(cudaMemcpy(du, units.data(), units.size() * 4, cudaMemcpyHostToDevice));
        // gather kernel inputs: targets = the same pixels
        const int cin_pad = (g.cin + 7) / 8 * 8, cout_pad = (g.cout + 15) / 16 * 16;
        std::vector<float> wt(conv_tc_weight_floats(cin_pad, cout_pad, 3));
        conv_tc_prepare_weights(w.data(), g.cin, g.cout, 3, cin_pad, cout_pad, wt.data());
        float* dwt;
        CK(cudaMalloc(&dwt, wt.size() * 4));
        CK(cudaMemcpy(dwt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice));
        const int max_targets = (rows * g.t + 2) * (rows * g.t + 2);
        const int splits = conv_tc_splits(max_targets, cin_pad, cout_pad, 3, sms);
        float* wst = nullptr;
        if (splits > 1) CK(cudaMalloc(&wst, (size_t)splits * max_targets * cout_pad * 4));
        for (int frac : {1, 4, 16}) {
            if (getenv("BENCH_FRAC") && atoi(getenv("BENCH_FRAC")) != frac) continue;
            const int n = (int)units.size() / frac;
            CK(cudaMemcpy(dn, &n, 4, cudaMemcpyHostToDevice));
            std::vector<int> list;
            for (int i = 0; i < n; ++i)
                for (int m = 0; m < 128; ++m) {
                    const int y = (units[i] >> 16) * 16 + (m >> 3), x = (units[i] & 0xffff) * 8 + (m & 7);
                    list.push_back(((y + 1) << 16) | (x + 1));
                }
            int* dl;
            int* dc;
            CK(cudaMalloc(&dl, list.size() * 4 + 4));
            CK(cudaMalloc(&dc, 4));
            CK(cudaMemcpy(dl, list.data(), list.size() * 4, cudaMemcpyHostToDevice));
            const int cnt = (int)list.size();
            CK(cudaMemcpy(dc, &cnt, 4, cudaMemcpyHostToDevice));
            const double flop = 2.0 * 9 * g.cin * g.cout * 128.0 * n;
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            float ms_d = 0, ms_g = 0;
            const int it = 10;
            for (int rep = 0; rep < 2; ++rep) {
                for (int i = 0; i < 2; ++i) launch_conv_dense(c, s, p, in, out, dw, g.cin, g.cout, du, dn, ws, dcnt, sms);
                CK(cudaEventRecord(a, s));
                for (int i = 0; i < it; ++i) launch_conv_dense(c, s, p, in, out, dw, g.cin, g.cout, du, dn, ws, dcnt, sms);
                CK(cudaEventRecord(b, s));
                CK(cudaEventSynchronize(b));
                CK(cudaEventElapsedTime(&ms_d, a, b));
                for (int i = 0; i < 2; ++i)
                    launch_conv_tc(c, s, in, dwt, g.cin, cin_pad, g.cout, cout_pad, 3, 1, 1, out, 1, dl, dc, max_targets,
                                   sms, wst, splits);
                CK(cudaEventRecord(a, s));
                for (int i = 0; i < it; ++i)
                    launch_conv_tc(c, s, in, dwt, g.cin, cin_pad, g.cout, cout_pad, 3, 1, 1, out, 1, dl, dc, max_targets,
                                   sms, wst, splits);
                CK(cudaEventRecord(b, s));
                CK(cudaEventSynchronize(b));
                CK(cudaEventElapsedTime(&ms_g, a, b));
            }
            CK(cudaGetLastError());
            if (dbg && (atoi(dbg) & 64)) {
                // one more launch, then dump CTA 0's per-K-block stamps
                launch_conv_dense(c, s, p, in, out, dw, g.cin, g.cout, du, dn, ws, dcnt, sms);
                CK(cudaStreamSynchronize(s));
                long long tr[1024];
                CK(cudaMemcpy(tr, dense_conv_trace_buffer(), sizeof tr, cudaMemcpyDeviceToHost));
                const long long t0 = tr[3];
                printf("kernel start %lld end %lld | epi item0 %lld-%lld item1 %lld-%lld\n", tr[500] - t0, tr[501] - t0,
                       tr[504] - t0, tr[505] - t0, tr[506] - t0, tr[507] - t0);
                for (int w = 0; w < 22; ++w) printf("warp %d done %lld\n", w, tr[520 + w] - t0);
                for (int k = 0; k < 3; ++k)
                    printf("kb %2d prod: start %7lld empty_ok %7lld arrive %7lld | mma: wait %7lld full_ok %7lld done %7lld\n", k,
                           tr[k * 8] - t0, tr[k * 8 + 1] - t0, tr[k * 8 + 2] - t0, tr[k * 8 + 3] - t0, tr[k * 8 + 4] - t0,
                           tr[k * 8 + 5] - t0);
            }
            printf("cin=%3d cout=%3d t=%2d units=%5d (KC=%d NBD=%d nstw=%d smax=%d): dense %8.1f us %6.1f TF/s | gather(S=%d) %8.1f us %6.1f TF/s\n",
                   g.cin, g.cout, g.t, n, p.KC, p.NBD, p.nstw, p.smax, ms_d * 1e3 / it, flop / (ms_d / it * 1e-3) / 1e12,
                   splits, ms_g * 1e3 / it, flop / (ms_g / it * 1e-3) / 1e12);
            fflush(stdout);
            cudaFree(dl);
            cudaFree(dc);
        }
    }
    return 0;
}
