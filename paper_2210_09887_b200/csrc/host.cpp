// Network validation and tile ledger of the B200 delta engine (host C++).
#include "host.hpp"

#include <algorithm>
#include <deque>
#include <map>

namespace dfx {

namespace {
int64_t fdiv(int64_t a, int64_t n) {
    int64_t q = a / n;
    if ((a % n != 0) && ((a < 0) != (n < 0))) --q;
    return q;
}
int64_t fmod_(int64_t a, int64_t n) {
    int64_t r = a % n;
    if (r != 0 && ((r < 0) != (n < 0))) r += n;
    return r;
}
int64_t cdiv(int64_t a, int64_t n) { return -fdiv(-a, n); }
}  // namespace

int windowed_out_halo(int in_halo, int span, int back, int stride) {
    // delta_layers.cpp:52-56 / network.cpp:17-21
    const int64_t lo = cdiv(in_halo + span - back, stride) - 1;
    const int64_t hi = cdiv(in_halo + back, stride);
    return (int)std::max<int64_t>({0, lo, hi});
}

int Net::index_of(const std::string& n) const {
    for (size_t i = 0; i < layers.size(); ++i)
        if (layers[i].name == n) return (int)i;
    return -1;
}

Net validate_net(const dfx_net_desc* d, int tile) {
    check(tile >= 1, "validate: tile size must be >= 1");
    check(d->in_channels >= 1, "validate: input channels must be >= 1");
    check(d->num_layers >= 1, "validate: network has no layers");
    Net net;
    net.in_channels = d->in_channels;
    const int n = d->num_layers;
    std::map<std::string, int> by_name;
    for (int i = 0; i < n; ++i) {
        const dfx_layer_desc& L = d->layers[i];
        Layer l;
        l.name = L.name ? L.name : "";
        check(!l.name.empty() && l.name != "input", "validate: bad layer name '" + l.name + "'");
        check(by_name.emplace(l.name, i).second, "validate: duplicate layer name '" + l.name + "'");
        l.kind = L.kind;
        const int want = L.kind == DFX_ADD ? 2 : 1;
        const int have = (L.input0 ? 1 : 0) + (L.input1 ? 1 : 0);
        if (have != want)
            fail("layer '" + l.name + "' needs " + std::to_string(want) + " input(s)", DFX_ERR_VALIDATION);
        l.cin = L.in_channels;
        l.cout = L.out_channels;
        l.k = L.kernel;
        l.stride = L.stride;
        l.pad = L.padding;
        if (L.kind == DFX_CONV) {
            check(L.weights != nullptr, "conv: weight count does not match dims");
            l.w.assign(L.weights, L.weights + (size_t)L.out_channels * L.in_channels * L.kernel * L.kernel);
            if (L.bias) l.bias.assign(L.bias, L.bias + L.out_channels);
        }
        l.pool_k = L.pool_k;
        l.pool_s = L.pool_stride;
        l.factor = L.factor;
        if (L.kind == DFX_BATCHNORM) {
            l.bn_scale.assign(L.bn_scale, L.bn_scale + L.bn_channels);
            l.bn_shift.assign(L.bn_shift, L.bn_shift + L.bn_channels);
        }
        l.has_thr = L.has_threshold != 0;
        l.thr = L.threshold;
        l.trunc_en = L.truncate_enabled != 0;
        net.layers.push_back(std::move(l));
    }
    // Kahn's algorithm, FIFO (network.cpp:68-91)
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<int>> consumers(n);
    for (int i = 0; i < n; ++i) {
        const dfx_layer_desc& L = d->layers[i];
        const char* ins[2] = {L.input0, L.input1};
        int* dst[2] = {&net.layers[i].in0, &net.layers[i].in1};
        for (int j = 0; j < 2; ++j) {
            if (!ins[j]) continue;
            if (std::string(ins[j]) == "input") {
                *dst[j] = -1;
                continue;
            }
            auto it = by_name.find(ins[j]);
            if (it == by_name.end())
                fail("layer '" + net.layers[i].name + "' references unknown '" + ins[j] + "'", DFX_ERR_VALIDATION);
            *dst[j] = it->second;
            consumers[it->second].push_back(i);
            ++indeg[i];
        }
    }
    std::deque<int> ready;
    for (int i = 0; i < n; ++i)
        if (!indeg[i]) ready.push_back(i);
    while (!ready.empty()) {
        const int i = ready.front();
        ready.pop_front();
        net.topo.push_back(i);
        for (int c : consumers[i])
            if (--indeg[c] == 0) ready.push_back(c);
    }
    if ((int)net.topo.size() != n) fail("network graph has a cycle", DFX_ERR_VALIDATION);

    const std::vector<float> zero_beta(d->in_channels, 0.0f);
    int outputs = 0;
    struct In {
        int ch, cum, tile, halo;
        const std::vector<float>* beta;
    };
    auto info_of = [&](int idx) -> In {
        if (idx == -1) return {d->in_channels, 1, tile, 0, &zero_beta};
        const Layer& a = net.layers[idx];
        return {a.channels, a.cum, a.tile, a.halo_out, &a.beta};
    };
    for (int idx : net.topo) {
        Layer& o = net.layers[idx];
        const In a = info_of(o.in0);
        o.in_channels = a.ch;
        o.in_cum = a.cum;
        o.in_tile = a.tile;
        o.halo_in = a.halo;
        auto set_cum = [&](int cum) {
            o.cum = cum;
            if (tile % cum != 0)
                fail("layer '" + o.name + "': tile size is not a multiple of the cumulative stride", DFX_ERR_VALIDATION);
            o.tile = std::max(1, tile / cum);
        };
        switch (o.kind) {
            case DFX_CONV: {
                check(o.cin >= 1 && o.cout >= 1, "conv: channel counts must be >= 1");
                check(o.k >= 1 && o.k % 2 == 1, "conv: kernel dims must be odd");
                check(o.stride >= 1, "conv: stride must be >= 1");
                check(o.pad >= 0, "conv: padding must be >= 0");
                if (o.cin != a.ch)
                    fail("layer '" + o.name + "': expects " + std::to_string(o.cin) + " channels, gets " +
                             std::to_string(a.ch), DFX_ERR_VALIDATION);
                if (o.pad != o.k / 2)
                    fail("layer '" + o.name + "': engine convolutions need same-style padding", DFX_ERR_VALIDATION);
                if (a.tile % o.stride != 0)
                    fail("layer '" + o.name + "': stride misaligned with tile", DFX_ERR_VALIDATION);
                o.channels = o.cout;
                set_cum(a.cum * o.stride);
                o.halo_out = windowed_out_halo(a.halo, o.k, o.k / 2, o.stride);
                // network.cpp:137-150 — same fp32 summation order
                o.beta.assign(o.channels, 0.0f);
                for (int oc = 0; oc < o.channels; ++oc) {
                    float v = o.bias.empty() ? 0.0f : o.bias[oc];
                    for (int ic = 0; ic < o.cin; ++ic) {
                        float ws = 0.0f;
                        for (int q = 0; q < o.k * o.k; ++q) ws += o.w[((size_t)oc * o.cin + ic) * o.k * o.k + q];
                        v += ws * (*a.beta)[ic];
                    }
                    o.beta[oc] = v;
                }
                break;
            }
            case DFX_RELU:
            case DFX_TRUNCATE:
            case DFX_OUTPUT:
                o.channels = a.ch;
                set_cum(a.cum);
                o.halo_out = 0;
                o.beta.assign(o.channels, 0.0f);
                if (o.kind == DFX_OUTPUT && ++outputs > 1) fail("network has more than one output", DFX_ERR_VALIDATION);
                break;
            case DFX_MAXPOOL:
            case DFX_AVGPOOL:
                if (o.pool_k != o.pool_s)
                    fail("layer '" + o.name + "': engine pooling requires k == stride", DFX_ERR_VALIDATION);
                if (o.pool_s < 1 || a.tile % o.pool_s != 0)
                    fail("layer '" + o.name + "': stride misaligned with tile", DFX_ERR_VALIDATION);
                o.channels = a.ch;
                set_cum(a.cum * o.pool_s);
                o.halo_out = windowed_out_halo(a.halo, o.pool_k, 0, o.pool_s);
                o.beta = *a.beta;
                break;
            case DFX_UPSAMPLE:
                if (o.factor < 1 || a.cum % o.factor != 0)
                    fail("layer '" + o.name + "': upsample factor does not divide cumulative stride", DFX_ERR_VALIDATION);
                o.channels = a.ch;
                set_cum(a.cum / o.factor);
                o.halo_out = a.halo * o.factor;
                o.beta = *a.beta;
                break;
            case DFX_BATCHNORM:
                if ((int)o.bn_scale.size() != a.ch || o.bn_shift.size() != o.bn_scale.size())
                    fail("layer '" + o.name + "': batchnorm param count", DFX_ERR_VALIDATION);
                o.channels = a.ch;
                set_cum(a.cum);
                o.halo_out = a.halo;
                o.beta.assign(o.channels, 0.0f);
                for (int c = 0; c < o.channels; ++c) o.beta[c] = o.bn_scale[c] * (*a.beta)[c] + o.bn_shift[c];
                break;
            case DFX_ADD: {
                const In b = info_of(o.in1);
                if (a.ch != b.ch) fail("layer '" + o.name + "': add channel mismatch", DFX_ERR_VALIDATION);
                if (a.cum != b.cum)
                    fail("layer '" + o.name + "': add joins branches of different cumulative stride", DFX_ERR_VALIDATION);
                o.channels = a.ch;
                set_cum(a.cum);
                o.halo_out = std::max(a.halo, b.halo);
                o.beta.assign(o.channels, 0.0f);
                for (int c = 0; c < o.channels; ++c) o.beta[c] = (*a.beta)[c] + (*b.beta)[c];
                break;
            }
            default:
                fail("layer '" + o.name + "': unknown kind", DFX_ERR_VALIDATION);
        }
    }
    if (outputs != 1) fail("network needs exactly one output layer", DFX_ERR_VALIDATION);
    std::vector<bool> consumed(n, false);
    for (const Layer& l : net.layers) {
        if (l.in0 >= 0) consumed[l.in0] = true;
        if (l.in1 >= 0) consumed[l.in1] = true;
    }
    for (int i = 0; i < n; ++i)
        if (!consumed[i] && net.layers[i].kind != DFX_OUTPUT)
            fail("layer '" + net.layers[i].name + "' is dangling", DFX_ERR_VALIDATION);
    for (int i = 0; i < n; ++i)
        if (net.layers[i].kind == DFX_OUTPUT) net.out_layer = i;
    int64_t ring = 1;
    for (int idx : net.topo) {
        const Layer& o = net.layers[idx];
        if (o.kind == DFX_RELU || o.kind == DFX_TRUNCATE || o.kind == DFX_OUTPUT) {
            ring = std::max(ring, cdiv(o.halo_in, o.in_tile));
        } else if (o.kind == DFX_MAXPOOL) {
            const int oh = windowed_out_halo(o.halo_in, o.pool_k, 0, o.pool_s);
            ring = std::max(ring, cdiv(o.halo_in, o.in_tile));
            ring = std::max(ring, cdiv(oh, o.tile));
            ring = std::max(ring, cdiv((int64_t)oh * o.pool_s + o.pool_k, o.in_tile));
        }
    }
    net.ring = (int)ring;
    return net;
}

// ------------------------------------------------------------------ ledger
void Ledger::init(int rows, int cols) {
    rows_ = rows;
    cols_ = cols;
    slots_.assign((size_t)rows * cols, Slot{});
    left_.reset();
    right_.reset();
    up_.reset();
    down_.reset();
}
int Ledger::slot_index(const Coord& c) const { return (int)(fmod_(c.ty, rows_) * cols_ + fmod_(c.tx, cols_)); }
bool Ledger::holds(const Coord& c) const {
    const Slot& s = slots_[slot_index(c)];
    return s.used && s.coord == c;
}
void Ledger::clear() { init(rows_, cols_); }

Plan Ledger::plan(const Placement& p, int ring) const {
    Plan plan;
    const int64_t min_tx = p.origin.tx, max_tx = p.origin.tx + p.tw - 1;
    const int64_t min_ty = p.origin.ty, max_ty = p.origin.ty + p.th - 1;
    if ((left_ && min_tx <= *left_) || (right_ && max_tx >= *right_) || (up_ && min_ty <= *up_) ||
        (down_ && max_ty >= *down_)) {
        plan.full_reset = true;
        return plan;
    }
    std::vector<uint8_t> planned(slots_.size(), 0);
    for (int r = 0; r < p.th; ++r)
        for (int c = 0; c < p.tw; ++c) {
            const Coord t{p.origin.tx + c, p.origin.ty + r};
            const int si = slot_index(t);
            const Slot& s = slots_[si];
            planned[si] = 1;
            if (!s.used) {
                plan.claims.push_back({t, false, {}});
                plan.fresh.push_back(t);
            } else if (s.coord == t) {
                if (!s.covered) plan.fresh.push_back(t);
            } else {
                plan.claims.push_back({t, true, s.coord});
                plan.fresh.push_back(t);
                ++plan.evicted;
            }
        }
    for (int r = -ring; r < p.th + ring; ++r)
        for (int c = -ring; c < p.tw + ring; ++c) {
            if (r >= 0 && r < p.th && c >= 0 && c < p.tw) continue;
            const Coord t{p.origin.tx + c, p.origin.ty + r};
            const int si = slot_index(t);
            if (planned[si]) continue;
            planned[si] = 1;
            const Slot& s = slots_[si];
            if (!s.used) {
                plan.claims.push_back({t, false, {}});
            } else if (!(s.coord == t)) {
                if (p.covers(s.coord)) continue;
                plan.claims.push_back({t, true, s.coord});
                ++plan.evicted;
            }
        }
    return plan;
}

void Ledger::apply(const Plan& plan, const Placement& p) {
    const int64_t min_tx = p.origin.tx, max_tx = p.origin.tx + p.tw - 1;
    const int64_t min_ty = p.origin.ty, max_ty = p.origin.ty + p.th - 1;
    for (const Claim& c : plan.claims) {
        if (c.evicts) {
            const Coord& v = c.victim;
            if (v.tx < min_tx) left_ = left_ ? std::max(*left_, v.tx) : v.tx;
            if (v.tx > max_tx) right_ = right_ ? std::min(*right_, v.tx) : v.tx;
            if (v.ty < min_ty) up_ = up_ ? std::max(*up_, v.ty) : v.ty;
            if (v.ty > max_ty) down_ = down_ ? std::min(*down_, v.ty) : v.ty;
        }
        Slot& s = slots_[slot_index(c.coord)];
        s.used = true;
        s.coord = c.coord;
        s.covered = false;
    }
    for (const Coord& t : plan.fresh) slots_[slot_index(t)].covered = true;
}

}  // namespace dfx
