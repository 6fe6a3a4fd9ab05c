"""`deltaflux._core` (bindings/py_bindings.cpp:38-135) over the B200 build.

The hot path — DeltaEngine.run_frame — is the product
(paper_2210_09887_b200.DeltaEngine: sm_100a kernels behind the C-ABI, no CPU
path). Network loading, tensor IO and wrap_tile are the product's mirrors.
The dense ops and run_dense are the reference's *dense oracle*
(tensor.hpp:91-100, network.cpp:256-296): plain fp32 loops the reference
exposes for checking the delta path; they are not part of the sparse path
(SURVEY §2 puts them out of scope) and are provided here as plain numpy so
that code using them keeps working. Network validation for run_dense is the
product's native validator (dfx_validate_net).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2210_09887_b200 import _capi
from paper_2210_09887_b200.engine import DeltaEngine as _Engine
from paper_2210_09887_b200.engine import EngineConfig as _EngineConfig
from paper_2210_09887_b200.engine import identity_homography, translation_homography, wrap_tile  # noqa: F401
from paper_2210_09887_b200.network import (ConvParams, DeltafluxError, IoError, NetworkSpec,  # noqa: F401
                                           ValidationError, load_network, load_tensor, save_tensor)


def _chw(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if a.ndim != 3:
        raise DeltafluxError("expected a CHW float32 array")
    return a


class EngineConfig(_EngineConfig):
    """dflx::EngineConfig with pybind-style attribute access (py_bindings.cpp:83-94)."""


class DeltaEngine(_Engine):
    """deltaflux._core.DeltaEngine: run_frame(frame, homography) -> dict (py_bindings.cpp:103-121)."""

    def __init__(self, spec, cfg):
        super().__init__(spec, cfg)

    def run_frame(self, frame, homography):  # no ROI argument in the reference binding
        return super().run_frame(_chw(frame), homography)


# ------------------------------------------------------------------ dense oracle (tensor.cpp, network.cpp:256-296)
def dense_conv2d(x, p: ConvParams):
    x = _chw(x)
    c, h, w = x.shape
    if p.in_channels != c:
        raise DeltafluxError("dense_conv2d: channel mismatch")
    k, s, pad = p.kernel_h, p.stride, p.padding
    wt = np.asarray(p.weights, np.float32).reshape(p.out_channels, p.in_channels, p.kernel_h, p.kernel_w)
    oh = (h + 2 * pad - k) // s + 1
    ow = (w + 2 * pad - p.kernel_w) // s + 1
    xp = np.zeros((c, h + 2 * pad, w + 2 * pad), np.float32)
    xp[:, pad:pad + h, pad:pad + w] = x
    out = np.zeros((p.out_channels, oh, ow), np.float32)
    for i in range(c):
        for ky in range(k):
            for kx in range(p.kernel_w):
                patch = xp[i, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s]
                out += wt[:, i, ky, kx][:, None, None] * patch[None]
    if p.bias is not None and len(p.bias):
        out += np.asarray(p.bias, np.float32)[:, None, None]
    return out


def dense_relu(x):
    return np.maximum(_chw(x), 0.0).astype(np.float32)


def dense_maxpool(x, k, s):
    x = _chw(x)
    c, h, w = x.shape
    oh, ow = (h - k) // s + 1, (w - k) // s + 1
    out = np.full((c, oh, ow), -np.inf, np.float32)
    for ky in range(k):
        for kx in range(k):
            out = np.maximum(out, x[:, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s])
    return out


def dense_avgpool(x, k, s):
    x = _chw(x)
    c, h, w = x.shape
    oh, ow = (h - k) // s + 1, (w - k) // s + 1
    out = np.zeros((c, oh, ow), np.float32)
    for ky in range(k):
        for kx in range(k):
            out += x[:, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s]
    return (out * np.float32(1.0 / (k * k))).astype(np.float32)


def dense_upsample_nearest(x, f):
    return np.repeat(np.repeat(_chw(x), f, axis=1), f, axis=2)


def run_dense(spec: NetworkSpec, tile_size: int, x):
    """network.cpp:256-296 over the product's validated topological order."""
    x = _chw(x)
    _, api = _capi.load_library()
    desc, keep = spec.to_desc()
    topo = (C.c_int * max(1, len(spec.layers)))()
    n, ring = C.c_int(), C.c_int()
    rc = api["validate_net"](C.byref(desc), int(tile_size), topo, len(spec.layers), C.byref(n), C.byref(ring))
    if rc != 0:
        msg = api["last_error"]().decode()
        raise (ValidationError if rc == 2 else DeltafluxError)(msg)
    if x.shape[0] != spec.in_channels:
        raise DeltafluxError("run_dense: input channel mismatch")
    outs = {}
    result = None
    for i in list(topo)[: n.value]:
        l = spec.layers[i]
        a = x if l.inputs[0] == "input" else outs[l.inputs[0]]
        if l.kind == "conv":
            o = dense_conv2d(a, l.conv)
        elif l.kind == "relu":
            o = dense_relu(a)
        elif l.kind in ("truncate", "output"):
            o = a
        elif l.kind == "maxpool":
            o = dense_maxpool(a, l.pool_k, l.pool_stride)
        elif l.kind == "avgpool":
            o = dense_avgpool(a, l.pool_k, l.pool_stride)
        elif l.kind == "upsample":
            o = dense_upsample_nearest(a, l.factor)
        elif l.kind == "batchnorm":
            o = (a * np.asarray(l.bn_scale, np.float32)[:, None, None] +
                 np.asarray(l.bn_shift, np.float32)[:, None, None]).astype(np.float32)
        elif l.kind == "add":
            b = x if l.inputs[1] == "input" else outs[l.inputs[1]]
            o = (a + b).astype(np.float32)
        outs[l.name] = o
        if l.kind == "output":
            result = o
    return result


# ------------------------------------------------------------------ frame IO (io.cpp:70-142)
def _load_pnm(path, color):
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open: {path}") from e
    magic = b"P6" if color else b"P5"
    tok, pos = [], 0
    while len(tok) < 4:
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":
            while pos < len(data) and data[pos:pos + 1] != b"\n":
                pos += 1
            continue
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        tok.append(data[start:pos])
    if tok[0] != magic:
        raise IoError(f"not a binary {'PPM' if color else 'PGM'}: {path}")
    w, h, mx = int(tok[1]), int(tok[2]), int(tok[3])
    c = 3 if color else 1
    px = np.frombuffer(data[pos + 1:pos + 1 + w * h * c], np.uint8)
    if px.size != w * h * c or mx != 255:
        raise IoError(f"truncated or unsupported PNM: {path}")
    return (px.reshape(h, w, c).transpose(2, 0, 1).astype(np.float32) / np.float32(255.0)).astype(np.float32)


def load_frame(path: str):
    ext = path[path.rfind("."):] if "." in path else ""
    if ext == ".ppm":
        return _load_pnm(path, True)
    if ext == ".pgm":
        return _load_pnm(path, False)
    if ext == ".dflx":
        return load_tensor(path)
    raise IoError("unknown frame format (expected .ppm/.pgm/.dflx): " + path)


def save_ppm(x, path: str) -> None:
    """io.cpp:109-126 (P6, values clamped to [0, 1], lround(v * 255))."""
    x = _chw(x)
    c, h, w = x.shape
    if c != 3:
        raise DeltafluxError("save_pnm: wrong channel count")
    v = np.clip(x, np.float32(0.0), np.float32(1.0)).astype(np.float32) * np.float32(255.0)
    img = np.floor(v.astype(np.float64) + 0.5).astype(np.uint8)  # lround for v >= 0
    try:
        with open(path, "wb") as f:
            f.write(b"P6\n%d %d\n255\n" % (w, h) + img.transpose(1, 2, 0).tobytes())
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e

