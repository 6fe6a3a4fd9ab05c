"""DeltaEngine over the C-ABI — the Python drop-in for
`deltaflux._core.DeltaEngine` / `EngineConfig` (reference
bindings/py_bindings.cpp:83-121, include/deltaflux/engine.hpp:10-91).

Every frame runs on the B200 through libdfx_b200.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import EngineConfigC, FrameInfo
from .network import DeltafluxError, IoError, NetworkSpec, ValidationError

_fp = C.POINTER(C.c_float)


@dataclass
class EngineConfig:
    """dflx::EngineConfig (engine.hpp:10-21) + conv_mode (device arithmetic of
    the sparse DeltaConv: "tf32x3" tensor cores, or "exact" CUDA-core fp32 in
    the reference's summation order)."""

    tile_size: int = 32
    grid_rows: int = 0
    grid_cols: int = 0
    input_threshold: float = 0.15
    default_threshold: float = 0.02
    override_net_thresholds: bool = False
    mask_dilation: int = 10
    roi_enabled: bool = False
    noise_suppression: bool = False
    padded_convolutions: bool = True
    conv_mode: str = "tf32x3"

    def to_c(self) -> EngineConfigC:
        c = EngineConfigC()
        c.tile_size = int(self.tile_size)
        c.grid_rows = int(self.grid_rows)
        c.grid_cols = int(self.grid_cols)
        c.input_threshold = float(self.input_threshold)
        c.default_threshold = float(self.default_threshold)
        c.override_net_thresholds = int(bool(self.override_net_thresholds))
        c.mask_dilation = int(self.mask_dilation)
        c.roi_enabled = int(bool(self.roi_enabled))
        c.noise_suppression = int(bool(self.noise_suppression))
        c.padded_convolutions = int(bool(self.padded_convolutions))
        modes = {"tf32x3": _capi.CONV_TF32X3, "exact": _capi.CONV_EXACT}
        if self.conv_mode not in modes:
            raise DeltafluxError(f"unknown conv_mode {self.conv_mode!r}")
        c.conv_mode = modes[self.conv_mode]
        return c

    @classmethod
    def from_any(cls, cfg) -> "EngineConfig":
        if isinstance(cfg, EngineConfig):
            return cfg
        out = cls()
        for k in out.__dataclass_fields__:
            if isinstance(cfg, dict):
                if k in cfg:
                    setattr(out, k, cfg[k])
            elif hasattr(cfg, k):
                setattr(out, k, getattr(cfg, k))
        if isinstance(cfg, dict) and isinstance(cfg.get("conv_mode"), int):
            out.conv_mode = {0: "tf32x3", 1: "exact"}[cfg["conv_mode"]]
        return out


def _raise(api, rc):
    if rc != 0:
        msg = api["last_error"]().decode()
        raise {2: ValidationError, 3: IoError}.get(rc, DeltafluxError)(msg)


class DeltaEngine:
    """One engine per video stream, bound to one GPU."""

    def __init__(self, spec: NetworkSpec, cfg=None, device: int = 0):
        self._lib, self._api = _capi.load_library()
        self.spec = spec
        self.config = EngineConfig.from_any(cfg if cfg is not None else EngineConfig())
        self._desc, self._keep = spec.to_desc()
        self._cfg = self.config.to_c()
        h = C.c_void_p()
        _raise(self._api, self._api["create"](C.byref(self._desc), C.byref(self._cfg), int(device), C.byref(h)))
        self._h = h
        self._out = None
        self.last_info = None

    def close(self):
        if getattr(self, "_h", None):
            self._api["destroy"](self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- reference surface (py_bindings.cpp:103-121) ----
    def run_frame(self, frame, homography, roi=None) -> dict:
        info, out = self.run_frame_full(frame, homography, roi)
        return {
            "output": out,
            "origin": (info["origin_ty"], info["origin_tx"]),
            "update_rate": info["update_rate"],
            "conv_flops": info["conv_flops"],
            "dense_flops": info["dense_flops"],
            "fresh": info["fresh"],
            "evicted": info["evicted"],
            "reset": bool(info["reset"]),
        }

    def reset(self):
        _raise(self._api, self._api["reset"](self._h))

    # ---- full result (FrameResult, engine.hpp:32-39) ----
    def run_frame_full(self, frame, homography, roi=None):
        frame = np.ascontiguousarray(frame, dtype=np.float32)
        if frame.ndim != 3:
            raise DeltafluxError("expected a CHW float32 array")
        h9 = np.ascontiguousarray(np.asarray(homography, dtype=np.float32).ravel())
        if h9.size != 9:
            raise DeltafluxError("homography expects 9 values (3x3 row-major)")
        c, hh, ww = frame.shape
        roi_p = None
        if roi is not None:
            roi = np.ascontiguousarray(roi, dtype=np.float32)
            if roi.shape != (1, hh, ww):
                raise DeltafluxError("run_frame: roi mask must be single channel at frame resolution")
            roi_p = roi.ctypes.data_as(_fp)
        cap = self._out_cap(c, hh, ww)
        if self._out is None or self._out.size < cap:
            self._out = np.empty(cap, dtype=np.float32)
        info = FrameInfo()
        _raise(self._api, self._api["run_frame"](self._h, frame.ctypes.data_as(_fp), c, hh, ww,
                                                 h9.ctypes.data_as(_fp), roi_p, C.byref(info),
                                                 self._out.ctypes.data_as(_fp), self._out.size))
        d = {k: getattr(info, k) for k, _ in FrameInfo._fields_}
        n = info.out_channels * info.out_height * info.out_width
        if n > self._out.size:
            raise DeltafluxError("output buffer too small")
        self.last_info = d
        return d, self._out[:n].reshape(info.out_channels, info.out_height, info.out_width).copy()

    def _out_cap(self, c, h, w):
        ch = max([c] + [l.conv.out_channels for l in self.spec.layers if l.conv is not None])
        t = self.config.tile_size
        return ch * (h + 2 * t) * (w + 2 * t)

    # ---- device-resident throughput path ----
    def submit_frame(self, frame_dev_ptr: int, c: int, h: int, w: int, homography):
        h9 = np.ascontiguousarray(np.asarray(homography, dtype=np.float32).ravel())
        _raise(self._api, self._api["submit_frame"](self._h, C.c_void_p(frame_dev_ptr), c, h, w,
                                                    h9.ctypes.data_as(_fp)))

    def submit_host_frame(self, frame_ptr: int, c: int, h: int, w: int, homography, out_ptr: int = 0,
                          out_floats: int = 0):
        """Pipelined host-buffer frame (dfx_engine_submit_host_frame): pinned
        host frame in, densified output copied to `out_ptr` (pinned, CHW)
        asynchronously; results after sync()."""
        h9 = np.ascontiguousarray(np.asarray(homography, dtype=np.float32).ravel())
        _raise(self._api, self._api["submit_host_frame"](self._h, C.c_void_p(frame_ptr), c, h, w,
                                                         h9.ctypes.data_as(_fp), C.c_void_p(out_ptr or None),
                                                         out_floats))

    def sync(self) -> dict:
        info = FrameInfo()
        _raise(self._api, self._api["sync"](self._h, C.byref(info)))
        self.last_info = {k: getattr(info, k) for k, _ in FrameInfo._fields_}
        return self.last_info

    def output_device(self):
        p, c, h, w = C.c_void_p(), C.c_int(), C.c_int(), C.c_int()
        _raise(self._api, self._api["output_device"](self._h, C.byref(p), C.byref(c), C.byref(h), C.byref(w)))
        return p.value, (c.value, h.value, w.value)

    def kernel_count(self) -> int:
        """Kernels launched by the last frame."""
        return self._api["kernel_count"](self._h)

    # ---- device-side measurement on the engine's stream ----
    def set_profiling(self, on: bool):
        _raise(self._api, self._api["set_profiling"](self._h, int(bool(on))))

    def reset_profile(self):
        _raise(self._api, self._api["reset_profile"](self._h))

    def profile(self) -> dict:
        """Per kernel family: total ms (CUDA events), launches, algorithmic work
        (bytes, or FLOPs for conv_mma)."""
        out = {}
        for i, name in enumerate(_capi.FAMILIES):
            ms, n, w = C.c_double(), C.c_uint64(), C.c_double()
            _raise(self._api, self._api["profile"](self._h, i, C.byref(ms), C.byref(n), C.byref(w)))
            out[name] = {"ms": ms.value, "launches": n.value, "work": w.value,
                         "bound": _capi.FAMILY_BOUND.get(name, "hbm")}
        return out

    def timer_start(self):
        _raise(self._api, self._api["timer_start"](self._h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        _raise(self._api, self._api["timer_stop"](self._h, C.byref(ms)))
        return ms.value

    # ---- introspection (engine.hpp:57-72) ----
    def grid(self):
        r, c = C.c_int(), C.c_int()
        _raise(self._api, self._api["grid"](self._h, C.byref(r), C.byref(c)))
        return r.value, c.value

    def input_mask(self):
        buf = np.zeros(1 << 16, dtype=np.uint8)
        th, tw = C.c_int(), C.c_int()
        _raise(self._api, self._api["input_mask"](self._h, buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size,
                                                  C.byref(th), C.byref(tw)))
        return buf[: th.value * tw.value].reshape(th.value, tw.value).copy()

    def layer_flops(self, name):
        idx = [l.name for l in self.spec.layers].index(name)
        f, d = C.c_uint64(), C.c_uint64()
        _raise(self._api, self._api["layer_flops"](self._h, idx, C.byref(f), C.byref(d)))
        return f.value, d.value

    def read_state(self, layer, which):
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        _raise(self._api, self._api["read_state"](self._h, layer.encode(), which, None, 0, C.byref(c), C.byref(h),
                                                  C.byref(w)))
        out = np.zeros((c.value, h.value, w.value), dtype=np.float32)
        _raise(self._api, self._api["read_state"](self._h, layer.encode(), which, out.ctypes.data_as(_fp), out.size,
                                                  C.byref(c), C.byref(h), C.byref(w)))
        return out

    def read_packet(self, layer):
        c, gh, gw, halo = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        args = (C.byref(c), C.byref(gh), C.byref(gw), C.byref(halo))
        _raise(self._api, self._api["read_packet"](self._h, layer.encode(), None, 0, *args, None, 0))
        out = np.zeros((c.value, gh.value, gw.value), dtype=np.float32)
        mask = np.zeros(1 << 16, dtype=np.uint8)
        _raise(self._api, self._api["read_packet"](self._h, layer.encode(), out.ctypes.data_as(_fp), out.size, *args,
                                                   mask.ctypes.data_as(C.POINTER(C.c_uint8)), mask.size))
        return out, halo.value, mask

    def read_ledger(self):
        rows, cols = self.grid()
        n = rows * cols
        used = np.zeros(n, np.int32)
        ty = np.zeros(n, np.int64)
        tx = np.zeros(n, np.int64)
        cov = np.zeros(n, np.uint8)
        _raise(self._api, self._api["read_ledger"](self._h, used.ctypes.data_as(C.POINTER(C.c_int)),
                                                   ty.ctypes.data_as(C.POINTER(C.c_int64)),
                                                   tx.ctypes.data_as(C.POINTER(C.c_int64)),
                                                   cov.ctypes.data_as(C.POINTER(C.c_uint8)), n))
        return used.reshape(rows, cols), ty.reshape(rows, cols), tx.reshape(rows, cols), cov.reshape(rows, cols)


def identity_homography():
    return np.eye(3, dtype=np.float32)


def translation_homography(dx: float, dy: float):
    return np.array([[1, 0, dx], [0, 1, dy], [0, 0, 1]], dtype=np.float32)


def wrap_tile(tx: int, ty: int, rows: int, cols: int):
    """dflx::wrap_tile (tile_grid.hpp:37-40) through the C-ABI."""
    lib, api = _capi.load_library()
    r, c = C.c_int(), C.c_int()
    api["wrap_tile"](int(tx), int(ty), int(rows), int(cols), C.byref(r), C.byref(c))
    return (r.value, c.value)
