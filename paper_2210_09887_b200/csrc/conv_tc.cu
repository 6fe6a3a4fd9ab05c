// tcgen05 3xTF32 sparse DeltaConv — placeholder until the kernel lands.
#include <stdexcept>
#include "kernels.hpp"
namespace dfx {
size_t conv_tc_weight_floats(int cin_pad, int cout_pad, int k) { return (size_t)2 * cin_pad * cout_pad * k * k; }
void conv_tc_prepare_weights(const float*, int, int, int, int, int, float*) {}
void launch_conv_tc(const Ctx&, cudaStream_t, PktDev, const float*, int, int, int, int, int, int, int, PktDev, int,
                    const int*, const int*, int, int) {
    throw std::runtime_error("tcgen05 conv not built yet: use conv_mode=DFX_CONV_EXACT");
}
}  // namespace dfx
