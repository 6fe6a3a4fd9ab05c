"""Layer-level C-ABI (dfx_delta_conv / dfx_delta_truncate /
dfx_delta_maxpool / dfx_densify / dfx_claim_reset / dfx_input_stage) against
the reference's own free functions (padded_delta_conv,
delta_activation_truncate, delta_maxpool, densify: delta_layers.hpp:103-127,
called through oracle/ref_shim.cpp on the same inputs) on a wrapped grid with
negative tile coordinates and a slot table holding foreign tiles.

Bar: bit-exact for truncate / maxpool / densify / claims / input stage and
for the conv in exact mode; the tf32x3 conv within 1e-4 x max(1, max|ref|)
with identical masks, halos and FLOP counts."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]

ROWS, COLS, T = 6, 7, 8
OTX, OTY, TH, TW = -3, 5, 4, 5


def _ref():
    lib = C.CDLL(oracle.REF_LIB)
    lib.dfr_last_error.restype = C.c_char_p
    return lib


def slot_table(foreign=True):
    """Placement grown by one ring tile (rows 6 = 4 + 2, cols 7 = 5 + 2), with
    one placement slot and one ring slot held by foreign tiles."""
    used = np.zeros(ROWS * COLS, np.int64)
    tx = np.zeros(ROWS * COLS, np.int64)
    ty = np.zeros(ROWS * COLS, np.int64)
    for gy in range(OTY - 1, OTY - 1 + ROWS):
        for gx in range(OTX - 1, OTX - 1 + COLS):
            i = (gy % ROWS) * COLS + (gx % COLS)
            used[i], tx[i], ty[i] = 1, gx, gy
    if foreign:
        i = ((OTY + 1) % ROWS) * COLS + ((OTX + 2) % COLS)  # placement tile (1, 2)
        tx[i] += COLS
        j = ((OTY - 1) % ROWS) * COLS + ((OTX + 3) % COLS)  # ring tile (-1, 3)
        ty[j] -= ROWS
    return used, tx, ty


def slots_c(s):
    from paper_2210_09887_b200.layers import Slot
    used, tx, ty = s
    arr = (Slot * (ROWS * COLS))()
    for i in range(ROWS * COLS):
        arr[i] = Slot(int(used[i]), int(tx[i]), int(ty[i]))
    return arr


def make_packet(rng, c, t, halo, th=TH, tw=TW, p=0.55):
    """A valid DeltaPacket (delta_layers.hpp:18-46): values only in masked
    tiles and within `halo` px of one; dense grown CHW + mask."""
    mask = (rng.random((th, tw)) < p).astype(np.uint8)
    gh, gw = th * t + 2 * halo, tw * t + 2 * halo
    allowed = np.zeros((gh, gw), bool)
    for r in range(th):
        for q in range(tw):
            if mask[r, q]:
                allowed[r * t:(r + 1) * t + 2 * halo, q * t:(q + 1) * t + 2 * halo] = True
    inside = np.zeros((gh, gw), bool)
    inside[halo:halo + th * t, halo:halo + tw * t] = True
    tile_on = np.kron(mask, np.ones((t, t), np.uint8)).astype(bool)
    inside_on = np.zeros((gh, gw), bool)
    inside_on[halo:halo + th * t, halo:halo + tw * t] = tile_on
    keep = np.where(inside, inside_on, allowed)
    d = rng.uniform(-1, 1, (c, gh, gw)).astype(np.float32) * keep[None]
    return np.ascontiguousarray(d), mask


class Dev:
    """Device buffers (torch) for one packet / state shape on the ctx grid."""

    def __init__(self, torch, ctx):
        self.torch, self.ctx = torch, ctx

    def packet(self, c, t, halo):
        from paper_2210_09887_b200.layers import Packet
        d = self.torch.zeros(self.ctx.packet_floats(c, t, halo), device="cuda")
        e = self.torch.zeros(self.ctx.packet_ext_bytes(t, halo), dtype=self.torch.uint8, device="cuda")
        return Packet(d.data_ptr(), e.data_ptr(), c, t, halo), (d, e)

    def state(self, c, t, chw=None):
        from paper_2210_09887_b200.layers import State
        d = self.torch.zeros(self.ctx.state_floats(c, t), device="cuda")
        st = State(d.data_ptr(), c, t)
        if chw is not None:
            src = self.torch.from_numpy(np.ascontiguousarray(chw)).cuda()
            self.ctx.state_from_chw(src.data_ptr(), st)
        return st, d

    def read_state(self, st, c, t):
        out = self.torch.zeros((c, ROWS * t, COLS * t), device="cuda")
        self.ctx.state_to_chw(st, out.data_ptr())
        self.torch.cuda.synchronize()
        return out.cpu().numpy()

    def read_packet(self, pk, c, t, halo):
        out = self.torch.zeros((c, TH * t + 2 * halo, TW * t + 2 * halo), device="cuda")
        m = self.ctx.packet_to_chw(pk, out.data_ptr())
        return out.cpu().numpy(), m


@pytest.fixture()
def env():
    import torch
    from paper_2210_09887_b200.layers import LayerContext
    ctx = LayerContext(ROWS, COLS)
    s = slot_table()
    ctx.set_frame(OTX, OTY, TH, TW, s)
    yield torch, ctx, Dev(torch, ctx), s
    ctx.close()


def placement():
    from paper_2210_09887_b200.layers import Placement
    return Placement(OTX, OTY, TH, TW)


@pytest.mark.parametrize("c,cout,k,s,halo,mode", [(12, 20, 3, 1, 0, "tf32x3"), (12, 20, 3, 2, 2, "tf32x3"),
                                                 (6, 16, 1, 2, 0, "tf32x3"), (8, 24, 5, 1, 1, "tf32x3"),
                                                 (12, 20, 3, 1, 2, "exact"), (6, 10, 3, 2, 1, "exact")])
def test_delta_conv_matches_padded_delta_conv(env, c, cout, k, s, halo, mode):
    torch, ctx, dev, _ = env
    from paper_2210_09887_b200.layers import conv_out_halo
    rng = np.random.default_rng(c * 100 + k * 10 + s + halo)
    x, mask = make_packet(rng, c, T, halo)
    w = rng.uniform(-0.5, 0.5, (cout, c, k, k)).astype(np.float32)
    pin, keep_in = dev.packet(c, T, halo)
    xd = torch.from_numpy(x).cuda()
    ctx.packet_from_chw(xd.data_ptr(), mask, pin)
    hg = conv_out_halo(halo, k, s)
    pout, keep_out = dev.packet(cout, T // s, hg)
    wd = torch.from_numpy(w).cuda()
    fl = ctx.delta_conv(pin, wd.data_ptr(), c, cout, k, s, mode, pout)
    got, gmask = dev.read_packet(pout, cout, T // s, hg)

    lib = _ref()
    want = np.zeros_like(got)
    wmask = np.zeros(TH * TW, np.uint8)
    oh = C.c_int()
    wfl = (C.c_uint64 * 2)()
    pl = placement()
    rc = lib.dfr_layer_conv(C.byref(pl), T, halo, c, x.ctypes.data_as(C.c_void_p), mask.ctypes.data_as(C.c_void_p),
                            w.ctypes.data_as(C.c_void_p), cout, k, s, want.ctypes.data_as(C.c_void_p),
                            wmask.ctypes.data_as(C.c_void_p), C.byref(oh), wfl)
    assert rc == 0, lib.dfr_last_error()
    assert oh.value == hg
    assert np.array_equal(gmask.ravel(), wmask)
    assert fl == (wfl[0], wfl[1])
    if mode == "exact":
        assert np.array_equal(got, want), float(np.abs(got - want).max())
    else:
        assert float(np.abs(got - want).max()) <= 1e-4 * max(1.0, float(np.abs(want).max()))


@pytest.mark.parametrize("c,halo,relu,thr", [(12, 0, 1, 0.3), (12, 2, 1, 0.5), (6, 2, 0, 0.3), (6, 0, 0, 0.0),
                                             (16, 3, 1, 0.02)])
def test_delta_truncate_matches_reference(env, c, halo, relu, thr):
    torch, ctx, dev, s = env
    rng = np.random.default_rng(7 + c + halo)
    x, mask = make_packet(rng, c, T, halo)
    acc = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    tr = rng.uniform(-0.2, 0.2, (c, ROWS * T, COLS * T)).astype(np.float32)
    pin, k1 = dev.packet(c, T, halo)
    xd = torch.from_numpy(x).cuda()
    ctx.packet_from_chw(xd.data_ptr(), mask, pin)
    sa, ka = dev.state(c, T, acc)
    st, kt = dev.state(c, T, tr)
    pout, k2 = dev.packet(c, T, 0)
    ctx.delta_truncate(pin, sa, st, thr, relu, pout)
    got, gmask = dev.read_packet(pout, c, T, 0)
    g_acc, g_tr = dev.read_state(sa, c, T), dev.read_state(st, c, T)

    lib = _ref()
    want = np.zeros_like(got)
    wmask = np.zeros(TH * TW, np.uint8)
    pl = placement()
    sl = slots_c(s)
    rc = lib.dfr_layer_truncate(C.byref(pl), ROWS, COLS, T, halo, c, x.ctypes.data_as(C.c_void_p),
                                mask.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p),
                                tr.ctypes.data_as(C.c_void_p), C.c_float(thr), relu, sl,
                                want.ctypes.data_as(C.c_void_p), wmask.ctypes.data_as(C.c_void_p))
    assert rc == 0, lib.dfr_last_error()
    assert np.array_equal(gmask.ravel(), wmask)
    assert 0 < wmask.sum() or thr > 0
    assert np.array_equal(got, want), float(np.abs(got - want).max())
    assert np.array_equal(g_acc, acc)
    assert np.array_equal(g_tr, tr)


@pytest.mark.parametrize("c,halo", [(12, 0), (6, 0), (12, 1), (6, 2)])
def test_delta_maxpool_matches_reference(env, c, halo):
    torch, ctx, dev, s = env
    rng = np.random.default_rng(31 + c + halo)
    x, mask = make_packet(rng, c, T, halo)
    acc = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    prev = rng.uniform(-1, 1, (c, ROWS * T // 2, COLS * T // 2)).astype(np.float32)
    lib = _ref()
    want_h = C.c_int()
    pin, k1 = dev.packet(c, T, halo)
    xd = torch.from_numpy(x).cuda()
    ctx.packet_from_chw(xd.data_ptr(), mask, pin)
    sa, ka = dev.state(c, T, acc)
    sp, kp = dev.state(c, T // 2, prev)
    # windowed_out_halo(halo, k=2, back=0, stride=2)
    hg = max(0, -(-(halo + 2) // 2) - 1, -(-halo // 2))
    pout, k2 = dev.packet(c, T // 2, hg)
    ctx.delta_maxpool(pin, sa, sp, 2, pout)
    got, gmask = dev.read_packet(pout, c, T // 2, hg)
    g_acc, g_prev = dev.read_state(sa, c, T), dev.read_state(sp, c, T // 2)

    want = np.zeros_like(got)
    wmask = np.zeros(TH * TW, np.uint8)
    pl = placement()
    sl = slots_c(s)
    rc = lib.dfr_layer_maxpool(C.byref(pl), ROWS, COLS, T, halo, c, x.ctypes.data_as(C.c_void_p),
                               mask.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p),
                               prev.ctypes.data_as(C.c_void_p), 2, sl, want.ctypes.data_as(C.c_void_p),
                               wmask.ctypes.data_as(C.c_void_p), C.byref(want_h))
    assert rc == 0, lib.dfr_last_error()
    assert want_h.value == hg
    assert np.array_equal(gmask.ravel(), wmask)
    assert np.array_equal(got, want), float(np.abs(got - want).max())
    assert np.array_equal(g_acc, acc)
    assert np.array_equal(g_prev, prev)


def test_densify_matches_reference(env):
    torch, ctx, dev, _ = env
    rng = np.random.default_rng(5)
    c = 8
    acc = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    tr = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    sa, ka = dev.state(c, T, acc)
    st, kt = dev.state(c, T, tr)
    out = torch.zeros((c, TH * T, TW * T), device="cuda")
    ctx.densify(sa, st, out.data_ptr())
    torch.cuda.synchronize()
    want = np.zeros((c, TH * T, TW * T), np.float32)
    pl = placement()
    rc = _ref().dfr_layer_densify(C.byref(pl), ROWS, COLS, T, c, acc.ctypes.data_as(C.c_void_p),
                                  tr.ctypes.data_as(C.c_void_p), want.ctypes.data_as(C.c_void_p))
    assert rc == 0
    assert np.array_equal(out.cpu().numpy(), want)


def test_claim_reset_zeroes_and_fills(env):
    """apply_plan + inject_bias_implicit (buffer_manager.cpp:68-89): every
    claimed tile is zero in every state, then bias-filled where a fill is given."""
    torch, ctx, dev, _ = env
    rng = np.random.default_rng(9)
    c = 12
    a0 = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    b0 = rng.uniform(-1, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    sa, ka = dev.state(c, T, a0)
    sb, kb = dev.state(c, T, b0)
    fill = rng.uniform(-1, 1, c).astype(np.float32)
    fd = torch.from_numpy(fill).cuda()
    claims = [(OTX - 1, OTY + 2), (OTX + 4, OTY - 1), (OTX + 2, OTY + 3)]
    ctx.claim_reset(claims, [sa, sb], [0, fd.data_ptr()])
    ga, gb = dev.read_state(sa, c, T), dev.read_state(sb, c, T)
    wa, wb = a0.copy(), b0.copy()
    for tx, ty in claims:
        r, q = ty % ROWS, tx % COLS
        wa[:, r * T:(r + 1) * T, q * T:(q + 1) * T] = 0
        wb[:, r * T:(r + 1) * T, q * T:(q + 1) * T] = fill[:, None, None]
    assert np.array_equal(ga, wa)
    assert np.array_equal(gb, wb)


def _input_stage_numpy(aligned, valid, acc, trunc, fresh, thr, r, own):
    """compute_input_delta (alignment.cpp:168-192) + input_gate without ROI /
    noise (engine.cpp:110-182) + the gated truncation (delta_layers.cpp:
    149-232 with gate as fire) on extent-local arrays (state tiles already
    gathered to the placement). Returns out, mask, acc', trunc'."""
    c, eh, ew = aligned.shape
    cov = valid.reshape(TH, T, TW, T).any(axis=(1, 3))
    covpx = np.kron(cov, np.ones((T, T), bool))
    raw = np.where(covpx[None], aligned - acc, np.float32(0)).astype(np.float32)
    cand = (trunc + raw).astype(np.float32)
    sig = np.abs(cand).max(axis=0) > thr
    if r > 0:
        d = np.zeros_like(sig)
        for y in range(eh):
            for x in range(ew):
                d[y, x] = sig[max(0, y - r):y + r + 1, max(0, x - r):x + r + 1].any()
        sig = d
    gate = (sig.reshape(TH, T, TW, T).any(axis=(1, 3)) & cov) | (fresh.astype(bool) & cov)
    out = np.zeros_like(aligned)
    acc2, tr2 = acc.copy(), trunc.copy()
    for i in range(TH):
        for j in range(TW):
            if not (cov[i, j] and own[i, j]):
                continue
            sl = (slice(None), slice(i * T, (i + 1) * T), slice(j * T, (j + 1) * T))
            if gate[i, j]:
                acc2[sl] = (acc[sl] + cand[sl]).astype(np.float32)
                tr2[sl] = 0
                out[sl] = cand[sl]
            else:
                tr2[sl] = (trunc[sl] + raw[sl]).astype(np.float32)
    return out, (gate & cov & own).astype(np.uint8), acc2, tr2


def test_input_stage_matches_restatement(env):
    torch, ctx, dev, s = env
    rng = np.random.default_rng(12)
    c = 3
    eh, ew = TH * T, TW * T
    aligned = rng.uniform(0, 1, (c, eh, ew)).astype(np.float32)
    valid = np.ones((eh, ew), np.uint8)
    valid[:, :T + 3] = 0  # first tile column uncovered, second partly
    aligned[:, ~valid.astype(bool)] = 0
    acc_full = rng.uniform(0, 1, (c, ROWS * T, COLS * T)).astype(np.float32)
    tr_full = rng.uniform(-0.05, 0.05, (c, ROWS * T, COLS * T)).astype(np.float32)
    # make most tiles static: aligned == acc there (tiles not in `moving`)
    moving = rng.random((TH, TW)) < 0.4
    used, stx, sty = s
    own = np.zeros((TH, TW), bool)
    for i in range(TH):
        for j in range(TW):
            gy, gx = OTY + i, OTX + j
            r, q = gy % ROWS, gx % COLS
            k = r * COLS + q
            own[i, j] = used[k] and stx[k] == gx and sty[k] == gy
            if not moving[i, j]:
                acc_full[:, r * T:(r + 1) * T, q * T:(q + 1) * T] = aligned[:, i * T:(i + 1) * T, j * T:(j + 1) * T]
    fresh = np.zeros((TH, TW), np.uint8)
    fresh[3, 4] = 1

    def gather(full):
        loc = np.zeros((c, eh, ew), np.float32)
        for i in range(TH):
            for j in range(TW):
                r, q = (OTY + i) % ROWS, (OTX + j) % COLS
                loc[:, i * T:(i + 1) * T, j * T:(j + 1) * T] = full[:, r * T:(r + 1) * T, q * T:(q + 1) * T]
        return loc

    w_out, w_mask, w_acc, w_tr = _input_stage_numpy(aligned, valid, gather(acc_full), gather(tr_full), fresh, 0.15, 2,
                                                    own)
    sa, ka = dev.state(c, T, acc_full)
    st, kt = dev.state(c, T, tr_full)
    pout, kp = dev.packet(c, T, 0)
    ad = torch.from_numpy(aligned).cuda()
    vd = torch.from_numpy(valid).cuda()
    ur = ctx.input_stage(ad.data_ptr(), vd.data_ptr(), fresh, 0.15, 2, 0, sa, st, pout)
    got, gmask = dev.read_packet(pout, c, T, 0)
    assert np.array_equal(gmask, w_mask)
    assert ur == pytest.approx(w_mask.sum() / (TH * TW))
    assert np.array_equal(got, w_out)
    assert np.array_equal(gather(dev.read_state(sa, c, T)), w_acc)
    assert np.array_equal(gather(dev.read_state(st, c, T)), w_tr)
