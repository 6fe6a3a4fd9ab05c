"""Test networks and frame sequences.

Python counterparts of the reference's test builders
(/root/reference/proj/tests/support/netgen.hpp:78-213, testutil.hpp:33-55):
random DAG networks (3x3 / 1x1 convs, stride 2, pools, upsample, batchnorm,
skip-adds, relu after dilating convs) and panning / moving-object
sequences. Inputs are generated once here and fed identically to every
implementation (reference, C restatement, CUDA path).
"""

from __future__ import annotations

import numpy as np

from paper_2210_09887_b200.network import NetworkSpec


def random_conv_weights(rng, cin, cout, k, lo=-0.5, hi=0.5):
    return rng.uniform(lo, hi, size=(cout, cin, k, k)).astype(np.float32)


def random_network(rng, max_extra_blocks=6, max_channels=16, max_downsample=4, allow_pool=True,
                   allow_upsample=True, allow_add=True, allow_stride2=True, allow_batchnorm=True,
                   bias_prob=0.6, in_channels=None):
    """netgen.hpp:78-195 — a random valid DAG."""
    spec = NetworkSpec(in_channels=int(in_channels or rng.integers(1, 4)))
    state = {"id": 0, "cur": "input", "ch": spec.in_channels, "cum": 1, "pending": False}
    junctions = []

    def nm(base):
        state["id"] += 1
        return f"{base}{state['id']}"

    def relu():
        state["cur"] = spec.relu(nm("relu"), state["cur"])
        state["pending"] = False

    def conv(k, stride, out_c):
        bias = rng.uniform(-0.5, 0.5, size=out_c).astype(np.float32) if rng.random() < bias_prob else None
        w = random_conv_weights(rng, state["ch"], out_c, k)
        state["cur"] = spec.conv(nm("conv"), state["cur"], w, bias, stride)
        state["ch"] = out_c
        if bias is not None:
            state["pending"] = True

    conv(3, 1, int(rng.integers(2, max_channels + 1)))
    relu()
    junctions.append((state["cur"], state["ch"], state["cum"], state["pending"]))
    for _ in range(int(rng.integers(0, max_extra_blocks + 1))):
        choice = int(rng.integers(0, 10))
        if choice <= 3:
            one = rng.random() < 0.35
            k = 1 if one else 3
            if k == 3 and state["pending"]:
                relu()
            s2 = allow_stride2 and not one and rng.random() < 0.25 and state["cum"] * 2 <= max_downsample
            conv(k, 2 if s2 else 1, int(rng.integers(2, max_channels + 1)))
            if s2:
                state["cum"] *= 2
            if k == 3 or rng.random() < 0.3:
                relu()
        elif choice <= 5 and allow_pool and state["cum"] * 2 <= max_downsample:
            if rng.random() < 0.6:
                state["cur"] = spec.maxpool(nm("pool"), state["cur"])
            else:
                state["cur"] = spec.avgpool(nm("pool"), state["cur"])
            state["cum"] *= 2
        elif choice == 6 and allow_upsample and state["cum"] % 2 == 0:
            state["cur"] = spec.upsample(nm("up"), state["cur"])
            state["cum"] //= 2
        elif choice == 7 and allow_batchnorm:
            sc = rng.uniform(0.5, 1.5, size=state["ch"]).astype(np.float32)
            sh = rng.uniform(-0.3, 0.3, size=state["ch"]).astype(np.float32)
            state["cur"] = spec.batchnorm(nm("bn"), state["cur"], sc, sh)
            state["pending"] = True
            if rng.random() < 0.8:
                relu()
        elif allow_add:
            comp = [j for j in junctions if j[1] == state["ch"] and j[2] == state["cum"] and j[0] != state["cur"]]
            if comp:
                pick = comp[int(rng.integers(0, len(comp)))]
                state["cur"] = spec.add(nm("add"), state["cur"], pick[0])
                state["pending"] = state["pending"] or pick[3]
        junctions.append((state["cur"], state["ch"], state["cum"], state["pending"]))
    spec.output(state["cur"])
    return spec


def random_sequence(rng, channels, h, w, frames):
    """netgen.hpp:199-213: static textured base plus a moving 0.9 square."""
    base = rng.uniform(0, 1, size=(channels, h, w)).astype(np.float32)
    size = max(4, min(h, w) // 4)
    seq = []
    for f in range(frames):
        t = base.copy()
        oy = (f * 5) % max(1, h - size)
        ox = (f * 7) % max(1, w - size)
        t[:, oy:oy + size, ox:ox + size] = 0.9
        seq.append(t)
    return seq


def box_blur5(x):
    """5x5 clipped box blur (the smoothing of synth.cpp:9-27)."""
    c, h, w = x.shape
    pad = np.pad(x, ((0, 0), (2, 2), (2, 2)))
    ones = np.pad(np.ones((h, w), np.float32), 2)
    s = np.zeros_like(x)
    n = np.zeros((h, w), np.float32)
    for dy in range(5):
        for dx in range(5):
            s += pad[:, dy:dy + h, dx:dx + w]
            n += ones[dy:dy + h, dx:dx + w]
    return (s / n).astype(np.float32)


def texture(rng, c, h, w):
    """Smooth seeded texture in [0,1] (the synth_texture recipe, numpy RNG)."""
    return box_blur5(box_blur5(rng.uniform(0, 1, size=(c, h, w)).astype(np.float32)))


def translation(dx, dy):
    return np.array([1, 0, dx, 0, 1, dy, 0, 0, 1], dtype=np.float32)


def pan_sequence(rng, c, h, w, frames, pan_x, pan_y, world=None):
    """Camera window panning (pan_x, pan_y) px/frame over a textured world,
    homography = translation(window origin) (synth.cpp:32-83)."""
    sx, sy = abs(pan_x) * (frames - 1), abs(pan_y) * (frames - 1)
    if world is None:
        world = texture(rng, c, h + sy, w + sx)
    out = []
    for f in range(frames):
        wx = pan_x * f if pan_x >= 0 else sx + pan_x * f
        wy = pan_y * f if pan_y >= 0 else sy + pan_y * f
        out.append((np.ascontiguousarray(world[:, wy:wy + h, wx:wx + w]), translation(wx, wy)))
    return out


def bilinear_sample(img, xs, ys):
    """Sample CHW img at float coords (zero outside)."""
    c, h, w = img.shape
    x0 = np.floor(xs).astype(np.int64)
    y0 = np.floor(ys).astype(np.int64)
    fx = (xs - x0).astype(np.float32)
    fy = (ys - y0).astype(np.float32)
    out = np.zeros((c,) + xs.shape, np.float32)
    for dy, wy in ((0, 1 - fy), (1, fy)):
        for dx, wx in ((0, 1 - fx), (1, fx)):
            yy = np.clip(y0 + dy, 0, h - 1)
            xx = np.clip(x0 + dx, 0, w - 1)
            out += img[:, yy, xx] * (wy * wx)[None]
    return out


def pan_rotate_sequence(rng, c, h, w, frames, pan_x, pan_y, deg_per_frame, world=None, obj=True):
    """Camera pans and rotates over a textured world; frame k's homography maps
    its pixels into world (reference) coordinates: H = T(t_k) R(theta_k) about
    the frame centre. A textured object moves in world space."""
    margin = int(abs(pan_x) * frames + abs(pan_y) * frames + max(h, w)) + 8
    if world is None:
        world = texture(rng, c, h + 2 * margin, w + 2 * margin)
    obj_tex = texture(rng, c, 40, 40) if obj else None
    seq = []
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
    for f in range(frames):
        th = np.deg2rad(deg_per_frame * f)
        ct, st = np.cos(th), np.sin(th)
        tx, ty = pan_x * f, pan_y * f
        # frame -> world: R about centre then translate
        a, b, cc_ = ct, -st, cx - ct * cx + st * cy + tx
        d, e, ff = st, ct, cy - st * cx - ct * cy + ty
        H = np.array([a, b, cc_, d, e, ff, 0, 0, 1], np.float32)
        wxs = a * xx + b * yy + cc_ + margin
        wys = d * xx + e * yy + ff + margin
        frame = bilinear_sample(world, wxs, wys)
        if obj:
            ox = 30 + 3 * f
            oy = 20 + 2 * f
            # object in frame coordinates (independent motion)
            frame[:, oy:oy + 40, ox:ox + 40] = obj_tex[:, : max(0, min(40, h - oy)), : max(0, min(40, w - ox))]
        seq.append((np.ascontiguousarray(frame, np.float32), H))
    return seq


def pan_wobble_sequence(rng, c, h, w, frames, pan_x, pan_y, deg_amp, period, obj=True, obj_v=(3, 2)):
    """Stationary camera motion for benchmarks: constant pan plus a bounded
    rotation wobble theta_k = deg_amp * sin(2 pi k / period) about the frame
    centre (frame k's homography maps its pixels into world coordinates), and
    a textured object moving in frame coordinates (wrapping around), so the
    update rate does not drift with the sequence length."""
    margin = int(abs(pan_x) * frames + abs(pan_y) * frames + max(h, w)) + 8
    world = texture(rng, c, h + 2 * margin, w + 2 * margin)
    obj_tex = texture(rng, c, 40, 40) if obj else None
    seq = []
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
    for f in range(frames):
        th = np.deg2rad(deg_amp * np.sin(2.0 * np.pi * f / period))
        ct, st = np.cos(th), np.sin(th)
        tx, ty = pan_x * f, pan_y * f
        a, b, cc_ = ct, -st, cx - ct * cx + st * cy + tx
        d, e, ff = st, ct, cy - st * cx - ct * cy + ty
        H = np.array([a, b, cc_, d, e, ff, 0, 0, 1], np.float32)
        frame = bilinear_sample(world, a * xx + b * yy + cc_ + margin, d * xx + e * yy + ff + margin)
        if obj:
            ox = (30 + obj_v[0] * f) % (w - 40)
            oy = (20 + obj_v[1] * f) % (h - 40)
            frame[:, oy:oy + 40, ox:ox + 40] = obj_tex
        seq.append((np.ascontiguousarray(frame, np.float32), H))
    return seq


def toy_net3(rng=None):
    """netgen.hpp:46-56 shape: conv 3->4 (+b), relu, conv 4->2 (+b), output."""
    rng = rng or np.random.default_rng(43)
    spec = NetworkSpec(in_channels=3)
    spec.conv("conv1", "input", random_conv_weights(rng, 3, 4, 3), rng.uniform(-0.5, 0.5, 4).astype(np.float32))
    spec.relu("relu1", "conv1")
    spec.conv("conv2", "relu1", random_conv_weights(rng, 4, 2, 3), rng.uniform(-0.5, 0.5, 2).astype(np.float32))
    spec.output("conv2")
    return spec


def c1_net(rng=None, channels=64):
    """conv 64->64 3x3 (+bias) -> relu -> output."""
    rng = rng or np.random.default_rng(2210)
    spec = NetworkSpec(in_channels=channels)
    spec.conv("conv1", "input", random_conv_weights(rng, channels, channels, 3),
              rng.uniform(-0.5, 0.5, channels).astype(np.float32))
    spec.relu("relu1", "conv1")
    spec.output("relu1")
    return spec


def vgg8_net(rng=None, in_channels=3, widths=(64, 64, "P", 128, 128, "P", 256, 256, "P", 256, 256),
             threshold=None):
    """8-layer VGG-style delta CNN, He-uniform weights, each
    conv followed by relu, three 2x2 maxpools."""
    rng = rng or np.random.default_rng(2210)
    spec = NetworkSpec(in_channels=in_channels)
    cur, ch, n = "input", in_channels, 0
    for wdt in widths:
        if wdt == "P":
            n += 1
            cur = spec.maxpool(f"pool{n}", cur)
            continue
        n += 1
        lim = float(np.sqrt(6.0 / (ch * 9)))
        w = rng.uniform(-lim, lim, size=(wdt, ch, 3, 3)).astype(np.float32)
        b = rng.uniform(-0.05, 0.05, size=wdt).astype(np.float32)
        cur = spec.conv(f"conv{n}", cur, w, b)
        cur = spec.relu(f"relu{n}", cur, threshold=threshold)
        ch = wdt
    spec.output(cur)
    return spec


def _he_conv(spec, rng, name, inp, cin, cout, k, stride=1, bias=True):
    lim = float(np.sqrt(6.0 / (cin * k * k)))
    w = rng.uniform(-lim, lim, size=(cout, cin, k, k)).astype(np.float32)
    b = rng.uniform(-0.05, 0.05, size=cout).astype(np.float32) if bias else None
    return spec.conv(name, inp, w, b, stride)


def resnet18_net(rng=None, in_channels=3, widths=(64, 128, 256, 512)):
    """ResNet-18-style delta backbone. 7x7 stride-2 stem +
    relu, 2x2 max pool (the engine requires k == stride, network.cpp:164-166),
    four stages of two basic blocks (conv3x3(s) -> relu -> conv3x3 -> add
    shortcut -> relu); the first block of stages 2-4 is strided with a 1x1
    stride-2 projection shortcut. BN folded into the conv biases. He-uniform
    random weights. Tile 32 gives per-layer tiles 16 (stem), 8, 4, 2, 1."""
    rng = rng or np.random.default_rng(2210)
    spec = NetworkSpec(in_channels=in_channels)
    cur = _he_conv(spec, rng, "stem", "input", in_channels, widths[0], 7, 2)
    cur = spec.relu("stem_relu", cur)
    cur = spec.maxpool("pool", cur)
    ch = widths[0]
    for si, wd in enumerate(widths):
        for bi in range(2):
            p = f"s{si + 1}b{bi + 1}"
            stride = 2 if (si > 0 and bi == 0) else 1
            c1 = _he_conv(spec, rng, p + "_conv1", cur, ch, wd, 3, stride)
            r1 = spec.relu(p + "_relu1", c1)
            c2 = _he_conv(spec, rng, p + "_conv2", r1, wd, wd, 3, 1)
            sc = cur
            if stride != 1 or ch != wd:
                sc = _he_conv(spec, rng, p + "_proj", cur, ch, wd, 1, stride)
            a = spec.add(p + "_add", c2, sc)
            cur = spec.relu(p + "_relu2", a)
            ch = wd
    spec.output(cur)
    return spec


def hrnet_w32_net(rng=None, in_channels=3, widths=(32, 64, 128, 256), joints=17):
    """HRNet-W32-style pose network. Stem of two 3x3 stride-2
    convs (stride 4), then branches of 32 / 64 / 128 / 256 channels at stride
    4 / 8 / 16 / 32 added one per stage by a 3x3 stride-2 transition conv; each
    stage runs one basic block per branch and fuses every branch into the
    higher-resolution ones by 1x1 conv + nearest upsample + add and into the
    lower-resolution ones by 3x3 stride-2 convs + add; a 1x1 head gives
    `joints` heatmaps at stride 4. With tile 32 the stride-32 branch has 1-px
    tiles (network.cpp:113-119)."""
    rng = rng or np.random.default_rng(2210)
    spec = NetworkSpec(in_channels=in_channels)
    n = [0]

    def nm(base):
        n[0] += 1
        return f"{base}{n[0]}"

    def conv(inp, cin, cout, k, s=1):
        return _he_conv(spec, rng, nm("conv"), inp, cin, cout, k, s)

    def relu(inp):
        return spec.relu(nm("relu"), inp)

    x = relu(conv("input", in_channels, 64, 3, 2))
    x = relu(conv(x, 64, 64, 3, 2))
    branches = [relu(conv(x, 64, widths[0], 3))]
    for stage in range(1, len(widths) + 1):
        # one basic block per branch
        nb = []
        for b, cur in enumerate(branches):
            c = widths[b]
            y = relu(conv(cur, c, c, 3))
            y = conv(y, c, c, 3)
            nb.append(relu(spec.add(nm("add"), y, cur)))
        branches = nb
        if stage == len(widths):
            break
        # fusion: every branch receives the others (up: 1x1 + upsample; down: 3x3 s2 chain)
        fused = []
        for i in range(len(branches)):
            acc = branches[i]
            for j in range(len(branches)):
                if j == i:
                    continue
                if j > i:
                    y = conv(branches[j], widths[j], widths[i], 1)
                    y = spec.upsample(nm("up"), y, factor=2 ** (j - i))
                else:
                    y = branches[j]
                    cj = widths[j]
                    for step in range(i - j):
                        co = widths[i] if step == i - j - 1 else cj
                        y = conv(y, cj, co, 3, 2)
                        if step != i - j - 1:
                            y = relu(y)
                        cj = co
                acc = spec.add(nm("add"), acc, y)
            fused.append(relu(acc))
        # transition: a new lower-resolution branch from the last one
        fused.append(relu(conv(fused[-1], widths[len(branches) - 1], widths[len(branches)], 3, 2)))
        branches = fused
    # final fusion of every branch into the stride-4 one, then the heatmap head
    acc = branches[0]
    for j in range(1, len(branches)):
        y = spec.upsample(nm("up"), conv(branches[j], widths[j], widths[0], 1), factor=2 ** j)
        acc = spec.add(nm("add"), acc, y)
    head = conv(relu(acc), widths[0], joints, 1)
    spec.output(spec.truncate("head_trunc", head))
    return spec


def patch_update_sequence(rng, c, h, w, frames, frac, tile, pan_x=0, pan_y=0):
    """SURVEY §8(d) C4 update-rate sweep: a static textured scene seen through
    an integer-translation camera (pan_x, pan_y px/frame); every frame a
    fraction `frac` of the frame's tiles (tile-aligned in world coordinates)
    receives a new textured patch, so the input update rate is ~frac."""
    sx, sy = abs(pan_x) * (frames - 1), abs(pan_y) * (frames - 1)
    world = texture(rng, c, h + sy + tile, w + sx + tile)
    patches = texture(rng, c, tile * 8, tile * 8)
    out = []
    for f in range(frames):
        wx = pan_x * f if pan_x >= 0 else sx + pan_x * f
        wy = pan_y * f if pan_y >= 0 else sy + pan_y * f
        if f > 0 and frac > 0:
            ty0, tx0 = -(-wy // tile), -(-wx // tile)
            nty, ntx = (h - (ty0 * tile - wy)) // tile, (w - (tx0 * tile - wx)) // tile
            cells = nty * ntx
            pick = rng.choice(cells, size=max(1, int(round(frac * cells))), replace=False)
            for p in pick:
                y = (ty0 + p // ntx) * tile
                x = (tx0 + p % ntx) * tile
                py, px = rng.integers(0, 7) * tile, rng.integers(0, 7) * tile
                world[:, y:y + tile, x:x + tile] = patches[:, py:py + tile, px:px + tile]
        out.append((np.ascontiguousarray(world[:, wy:wy + h, wx:wx + w]), translation(wx, wy)))
    return out
