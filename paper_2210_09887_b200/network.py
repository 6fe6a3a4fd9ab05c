"""Network description: the Python mirror of dflx::LayerDef / NetworkSpec
(reference include/deltaflux/network.hpp:11-32) and of its JSON loader
(src/network.cpp:350-423, schema version 1, inline or DFLX-file weights).

The description is lowered to the C-ABI `dfx_net_desc` (include/dfx_b200.h)
by `NetworkSpec.to_desc()`; validation proper (topological order, tiles,
halos, bias responses, ring width) happens natively inside
dfx_engine_create, like the reference's validate() (network.cpp:46-254).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._capi import KINDS, LayerDesc, NetDesc


class DeltafluxError(RuntimeError):
    """Mirror of the Python exception `deltaflux.DeltafluxError`
    (py_bindings.cpp:41) — raised for dflx::Error and subclasses."""


class ValidationError(DeltafluxError):
    pass


class IoError(DeltafluxError):
    pass


@dataclass
class ConvParams:
    """dflx::ConvParams (tensor.hpp:58-87); weights O-I-Kh-Kw."""

    in_channels: int = 0
    out_channels: int = 0
    kernel_h: int = 0
    kernel_w: int = 0
    stride: int = 1
    padding: int = 0
    weights: list = field(default_factory=list)
    bias: list = field(default_factory=list)


@dataclass
class LayerDef:
    name: str
    kind: str
    inputs: List[str]
    conv: Optional[ConvParams] = None
    pool_k: int = 2
    pool_stride: int = 2
    factor: int = 2
    bn_scale: Optional[list] = None
    bn_shift: Optional[list] = None
    threshold: Optional[float] = None
    truncate_enabled: bool = True


@dataclass
class NetworkSpec:
    in_channels: int = 1
    layers: List[LayerDef] = field(default_factory=list)

    # ---- builders (the shapes tests/support/netgen.hpp builds) ----
    def conv(self, name, inp, w, bias=None, stride=1):
        w = np.ascontiguousarray(w, dtype=np.float32)
        o, i, kh, kw = w.shape
        p = ConvParams(i, o, kh, kw, stride, kh // 2, w, None if bias is None else np.asarray(bias, np.float32))
        self.layers.append(LayerDef(name, "conv", [inp], conv=p))
        return name

    def relu(self, name, inp, threshold=None, truncate=True):
        self.layers.append(LayerDef(name, "relu", [inp], threshold=threshold, truncate_enabled=truncate))
        return name

    def truncate(self, name, inp, threshold=None, truncate=True):
        self.layers.append(LayerDef(name, "truncate", [inp], threshold=threshold, truncate_enabled=truncate))
        return name

    def maxpool(self, name, inp, k=2):
        self.layers.append(LayerDef(name, "maxpool", [inp], pool_k=k, pool_stride=k))
        return name

    def avgpool(self, name, inp, k=2):
        self.layers.append(LayerDef(name, "avgpool", [inp], pool_k=k, pool_stride=k))
        return name

    def upsample(self, name, inp, factor=2):
        self.layers.append(LayerDef(name, "upsample", [inp], factor=factor))
        return name

    def batchnorm(self, name, inp, scale, shift):
        self.layers.append(LayerDef(name, "batchnorm", [inp], bn_scale=np.asarray(scale, np.float32),
                                    bn_shift=np.asarray(shift, np.float32)))
        return name

    def add(self, name, a, b):
        self.layers.append(LayerDef(name, "add", [a, b]))
        return name

    def output(self, inp, name="out"):
        self.layers.append(LayerDef(name, "output", [inp]))
        return name

    def to_desc(self):
        """Lower to the C-ABI `dfx_net_desc`. Returns (desc, keepalive)."""
        keep = []

        def fptr(a):
            if a is None or (hasattr(a, "__len__") and len(a) == 0):
                return None
            arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32).ravel())
            keep.append(arr)
            return arr.ctypes.data_as(C.POINTER(C.c_float))

        def s(x):
            if x is None:
                return None
            b = x.encode()
            keep.append(b)
            return b

        arr = (LayerDesc * max(1, len(self.layers)))()
        for i, l in enumerate(self.layers):
            d = arr[i]
            if l.kind not in KINDS:
                raise ValidationError(f"unknown layer kind '{l.kind}'")
            d.name = s(l.name)
            d.kind = KINDS[l.kind]
            d.input0 = s(l.inputs[0]) if len(l.inputs) > 0 else None
            d.input1 = s(l.inputs[1]) if len(l.inputs) > 1 else None
            if l.kind == "conv":
                p = l.conv
                d.in_channels = p.in_channels
                d.out_channels = p.out_channels
                d.kernel = p.kernel_h
                d.stride = p.stride
                d.padding = p.padding
                n = p.out_channels * p.in_channels * p.kernel_h * p.kernel_w
                if np.asarray(p.weights).size != n:
                    raise DeltafluxError("conv: weight count does not match dims")
                d.weights = fptr(p.weights)
                d.bias = fptr(p.bias)
            d.pool_k = l.pool_k
            d.pool_stride = l.pool_stride
            d.factor = l.factor
            if l.kind == "batchnorm":
                d.bn_channels = len(l.bn_scale)
                d.bn_scale = fptr(l.bn_scale)
                d.bn_shift = fptr(l.bn_shift)
            d.has_threshold = 1 if l.threshold is not None else 0
            d.threshold = float(l.threshold) if l.threshold is not None else 0.0
            d.truncate_enabled = 1 if l.truncate_enabled else 0
        keep.append(arr)
        desc = NetDesc(self.in_channels, len(self.layers), arr)
        return desc, keep


# ------------------------------------------------------------------ IO
def load_tensor(path: str) -> np.ndarray:
    """DFLX tensor file (io.hpp:11-13): 'DFLX', u32 version=1, u32 c, h, w, f32 data."""
    try:
        with open(path, "rb") as f:
            head = f.read(20)
            if len(head) < 20 or head[:4] != b"DFLX":
                raise IoError(f"not a DFLX tensor file: {path}")
            ver, c, h, w = struct.unpack("<IIII", head[4:])
            if ver != 1:
                raise IoError(f"unsupported DFLX version in {path}")
            data = np.frombuffer(f.read(), dtype="<f4")
    except OSError as e:
        raise IoError(f"cannot open: {path}") from e
    if data.size != c * h * w:
        raise IoError(f"truncated DFLX tensor: {path}")
    return data.reshape(c, h, w).astype(np.float32)


def save_tensor(x, path: str) -> None:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if x.ndim != 3:
        raise DeltafluxError("expected a CHW float32 array")
    with open(path, "wb") as f:
        f.write(b"DFLX" + struct.pack("<IIII", 1, *x.shape))
        f.write(x.astype("<f4").tobytes())


def load_network(net_path: str, weights_dir: str = "") -> NetworkSpec:
    """JSON network description, schema of network.cpp:350-423."""
    try:
        with open(net_path) as f:
            root = json.load(f)
    except OSError as e:
        raise IoError(f"cannot open: {net_path}") from e
    except json.JSONDecodeError as e:
        raise IoError(f"bad JSON in {net_path}: {e}") from e
    if root.get("version", 1) != 1:
        raise IoError("unsupported network schema version")
    d = weights_dir or os.path.dirname(net_path)
    manifest = root.get("manifest", {})

    def params(jl, file_key, inline_key, expect):
        if inline_key in jl:
            v = np.asarray(jl[inline_key], dtype=np.float32)
            if v.size != expect:
                raise IoError(f"inline weights under '{inline_key}' hold {v.size} values, expected {expect}")
            return v
        if file_key in jl:
            rel = jl[file_key]
            t = load_tensor(os.path.join(d, rel))
            if rel in manifest and int(np.prod(manifest[rel])) != t.size:
                raise IoError(f"weight file {rel} does not match its manifest shape")
            if t.size != expect:
                raise IoError(f"weight file {rel} holds {t.size} values, expected {expect}")
            return t.ravel()
        raise IoError(f"layer is missing '{file_key}'")

    try:
        spec = NetworkSpec(in_channels=int(root["input"]["channels"]))
        for jl in root["layers"]:
            name = jl["name"]
            kind = jl["kind"]
            if "inputs" in jl:
                inputs = list(jl["inputs"])
            elif "input" in jl:
                inputs = [jl["input"]]
            else:
                inputs = []
            if kind == "conv":
                o, i, k = int(jl["out_channels"]), int(jl["in_channels"]), int(jl["kernel"])
                s = int(jl.get("stride", 1))
                pad = int(jl.get("padding", k // 2))
                w = params(jl, "weights", "weights_inline", o * i * k * k)
                b = None
                if "bias_file" in jl or "bias_inline" in jl:
                    b = params(jl, "bias_file", "bias_inline", o)
                spec.layers.append(LayerDef(name, "conv", inputs, conv=ConvParams(i, o, k, k, s, pad, w, b)))
            elif kind in ("relu", "truncate"):
                spec.layers.append(LayerDef(name, kind, inputs,
                                            threshold=float(jl["threshold"]) if "threshold" in jl else None,
                                            truncate_enabled=bool(jl.get("truncate", True))))
            elif kind in ("maxpool", "avgpool"):
                k = int(jl.get("k", 2))
                spec.layers.append(LayerDef(name, kind, inputs, pool_k=k, pool_stride=int(jl.get("stride", k))))
            elif kind == "upsample":
                spec.layers.append(LayerDef(name, kind, inputs, factor=int(jl.get("factor", 2))))
            elif kind == "batchnorm":
                c = int(jl["channels"])
                spec.layers.append(LayerDef(name, kind, inputs,
                                            bn_scale=params(jl, "scale_file", "scale_inline", c),
                                            bn_shift=params(jl, "shift_file", "shift_inline", c)))
            elif kind in ("add", "output"):
                spec.layers.append(LayerDef(name, kind, inputs))
            else:
                raise IoError(f"unknown layer kind '{kind}' in {net_path}")
        return spec
    except KeyError as e:
        raise IoError(f"bad network schema in {net_path}: missing {e}") from e


def spec_to_json(spec: NetworkSpec) -> dict:
    """Schema-1 JSON (network.cpp:350-423 reader) with inline weights."""
    layers = []
    for l in spec.layers:
        j = {"name": l.name, "kind": l.kind}
        if l.kind == "add":
            j["inputs"] = list(l.inputs)
        else:
            j["input"] = l.inputs[0]
        if l.kind == "conv":
            p = l.conv
            j.update(in_channels=p.in_channels, out_channels=p.out_channels, kernel=p.kernel_h, stride=p.stride,
                     weights_inline=[float(v) for v in np.asarray(p.weights, np.float32).ravel()])
            if p.bias is not None and len(p.bias):
                j["bias_inline"] = [float(v) for v in np.asarray(p.bias, np.float32).ravel()]
        elif l.kind in ("relu", "truncate"):
            if l.threshold is not None:
                j["threshold"] = float(l.threshold)
            j["truncate"] = bool(l.truncate_enabled)
        elif l.kind in ("maxpool", "avgpool"):
            j.update(k=l.pool_k, stride=l.pool_stride)
        elif l.kind == "upsample":
            j["factor"] = l.factor
        elif l.kind == "batchnorm":
            j.update(channels=len(l.bn_scale), scale_inline=[float(v) for v in l.bn_scale],
                     shift_inline=[float(v) for v in l.bn_shift])
        layers.append(j)
    return {"version": 1, "input": {"channels": spec.in_channels}, "layers": layers}


def spec_from_json(root: dict) -> NetworkSpec:
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(root, f)
        path = f.name
    try:
        return load_network(path)
    finally:
        os.unlink(path)
