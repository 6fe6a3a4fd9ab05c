// Host-side (C++) pieces of the B200 delta engine that stay on the CPU:
// network validation and the per-frame tile ledger / plan. Both are integer
// bookkeeping, O(layers) and O(placement + ring) per frame.
#pragma once

#include <stdint.h>

#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "dfx_b200.h"

namespace dfx {

struct Error : std::runtime_error {
    int code;
    Error(const std::string& m, int c = DFX_ERR) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(const std::string& m, int code = DFX_ERR) { throw Error(m, code); }
inline void check(bool cond, const std::string& m) {
    if (!cond) fail(m);
}

// One validated layer: the reference's LayerDef + LayerInfo
// (network.hpp:15-45), with resolved input indices (-1 = network input).
struct Layer {
    std::string name;
    int kind = DFX_OUTPUT;
    int in0 = -2, in1 = -2;
    int cin = 0, cout = 0, k = 1, stride = 1, pad = 0;
    std::vector<float> w, bias;
    int pool_k = 2, pool_s = 2, factor = 2;
    std::vector<float> bn_scale, bn_shift;
    bool has_thr = false;
    float thr = 0.0f;
    bool trunc_en = true;
    // validate() facts
    int in_channels = 0, channels = 0, in_cum = 1, cum = 1, in_tile = 0, tile = 0, halo_in = 0, halo_out = 0;
    std::vector<float> beta;
};

struct Net {
    int in_channels = 1;
    std::vector<Layer> layers;
    std::vector<int> topo;
    int out_layer = -1;
    int ring = 1;
    int index_of(const std::string& n) const;
};

// network.cpp:46-254 restated: Kahn order, tiles, halos, beta, ring width.
Net validate_net(const dfx_net_desc* d, int tile_size);
int windowed_out_halo(int in_halo, int span, int back, int stride);

// ---- tile ledger (buffer_manager.hpp:13-88) ----
struct Coord {
    int64_t tx = 0, ty = 0;
    bool operator==(const Coord& o) const { return tx == o.tx && ty == o.ty; }
};
struct Placement {
    Coord origin;
    int th = 0, tw = 0;
    bool covers(const Coord& c) const {
        return c.tx >= origin.tx && c.tx < origin.tx + tw && c.ty >= origin.ty && c.ty < origin.ty + th;
    }
};
struct Slot {
    bool used = false;
    Coord coord;
    bool covered = false;
};
struct Claim {
    Coord coord;
    bool evicts = false;
    Coord victim;
};
struct Plan {
    bool full_reset = false;
    std::vector<Claim> claims;
    std::vector<Coord> fresh;
    int evicted = 0;
};

class Ledger {
  public:
    void init(int rows, int cols);
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    int slot_index(const Coord& c) const;
    const Slot& slot(const Coord& c) const { return slots_[slot_index(c)]; }
    const std::vector<Slot>& slots() const { return slots_; }
    bool holds(const Coord& c) const;
    void clear();
    Plan plan(const Placement& p, int ring) const;  // buffer_manager.cpp:7-66
    void apply(const Plan& plan, const Placement& p);  // buffer_manager.cpp:68-81 (ledger part)

  private:
    int rows_ = 0, cols_ = 0;
    std::vector<Slot> slots_;
    std::optional<int64_t> left_, right_, up_, down_;
};

}  // namespace dfx
