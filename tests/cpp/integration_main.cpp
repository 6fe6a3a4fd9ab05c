// Compiled by tests/test_integration_header.py against the reference's own
// headers (/root/reference/proj/include) and linked with libdfx_b200.so:
// the reference-side drop-in (include/dfx_deltaflux.hpp) builds and maps
// every C-ABI failure to the reference's exception types.
#include <cstdio>
#include <cstring>

#include "dfx_deltaflux.hpp"

static dflx::NetworkSpec toy(int cin_conv) {
    dflx::NetworkSpec spec;
    spec.in_channels = 1;
    dflx::LayerDef c;
    c.name = "conv1";
    c.kind = dflx::LayerKind::Conv;
    c.inputs = {"input"};
    c.conv.in_channels = cin_conv;
    c.conv.out_channels = 4;
    c.conv.kernel_h = c.conv.kernel_w = 3;
    c.conv.stride = 1;
    c.conv.padding = 1;
    c.conv.weights.assign((size_t)4 * cin_conv * 9, 0.1f);
    dflx::LayerDef r;
    r.name = "relu1";
    r.kind = dflx::LayerKind::Relu;
    r.inputs = {"conv1"};
    dflx::LayerDef o;
    o.name = "out";
    o.kind = dflx::LayerKind::Output;
    o.inputs = {"relu1"};
    spec.layers = {c, r, o};
    return spec;
}

int main(int argc, char** argv) {
    dflx::EngineConfig cfg;
    cfg.tile_size = 16;
    // 1. an invalid network is a ValidationError (network.cpp:123-126), GPU or not
    try {
        dflx::B200DeltaEngine bad(toy(2), cfg);
        std::printf("validation: no error\n");
        return 1;
    } catch (const dflx::ValidationError& e) {
        std::printf("validation: ValidationError: %s\n", e.what());
    }
    // 2. a valid network: runs on a GPU, and is a dflx::Error without one
    try {
        dflx::B200DeltaEngine eng(toy(1), cfg);
        dflx::Tensor frame(1, 32, 48);
        for (size_t i = 0; i < frame.data.size(); ++i) frame.data[i] = (float)((i * 37) % 101) / 101.0f;
        for (int k = 0; k < 3; ++k) {
            dflx::FrameResult r = eng.run_frame(frame, dflx::Homography::translation(16.0f * k, 0.0f));
            std::printf("frame %d: update_rate %.4f fresh %d conv_flops %llu layers %zu out %dx%dx%d mask %zu\n", k,
                        r.update_rate, r.events.fresh, (unsigned long long)r.flops.total, r.flops.layers.size(),
                        r.output.channels, r.output.height, r.output.width, r.input_mask.bits.size());
        }
        std::printf("engine: ok\n");
    } catch (const dflx::ValidationError& e) {
        std::printf("engine: ValidationError: %s\n", e.what());
        return 2;
    } catch (const dflx::Error& e) {
        std::printf("engine: Error: %s\n", e.what());
    }
    return 0;
}
