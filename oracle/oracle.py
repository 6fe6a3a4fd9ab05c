"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes drivers for the two CPU checkers:
  * `RefEngine`    — the unmodified reference engine (oracle/_ref/libdfxref.so,
                     built from /root/reference by oracle/Makefile);
  * `OracleEngine` — the C restatement (oracle/build/libdfxoracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module. Both classes expose the same
methods as the product's `paper_2210_09887_b200.DeltaEngine` test hooks.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2210_09887_b200._capi import (EngineConfigC, FrameInfo, declare_engine_api)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libdfxref.so")
ORACLE_LIB = os.path.join(HERE, "build", "libdfxoracle.so")
REFERENCE_SRC = "/root/reference/proj"

_fp = C.POINTER(C.c_float)


def build(ref: bool = True, quiet: bool = True) -> None:
    """Build the C restatement, and the reference shim when the reference
    sources are present (they are not on the GPU box)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    out = None if not quiet else subprocess.DEVNULL
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True, stdout=out)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


_libs = {}


def _load(path, prefix):
    key = (path, prefix)
    if key not in _libs:
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run oracle.build())")
        lib = C.CDLL(path)
        _libs[key] = (lib, declare_engine_api(lib, prefix))
    return _libs[key]


def config_struct(cfg) -> EngineConfigC:
    """Accept an EngineConfigC, a dict, or an object with EngineConfig fields."""
    if isinstance(cfg, EngineConfigC):
        return cfg
    c = EngineConfigC()
    defaults = dict(tile_size=32, grid_rows=0, grid_cols=0, input_threshold=0.15, default_threshold=0.02,
                    override_net_thresholds=0, mask_dilation=10, roi_enabled=0, noise_suppression=0,
                    padded_convolutions=1, conv_mode=0)
    for k, v in defaults.items():
        if isinstance(cfg, dict):
            val = cfg.get(k, v)
        else:
            val = getattr(cfg, k, v)
        setattr(c, k, type(v)(val) if not isinstance(v, bool) else int(val))
    return c


class _CEngine:
    PREFIX = None
    PATH = None

    def __init__(self, spec, cfg):
        self.lib, self.api = _load(self.PATH, self.PREFIX)
        self._desc, self._keep = spec.to_desc()
        self._cfg = config_struct(cfg)
        h = C.c_void_p()
        rc = self.api["create"](C.byref(self._desc), C.byref(self._cfg), C.byref(h))
        self._check(rc)
        self.h = h
        self.spec = spec

    def _check(self, rc):
        if rc != 0:
            from paper_2210_09887_b200.network import DeltafluxError, IoError, ValidationError
            msg = self.api["last_error"]().decode()
            raise {2: ValidationError, 3: IoError}.get(rc, DeltafluxError)(msg)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.api["destroy"](self.h)
                self.h = None
        except Exception:
            pass

    def run_frame(self, frame, h9, roi=None):
        frame = np.ascontiguousarray(frame, dtype=np.float32)
        h9 = np.ascontiguousarray(np.asarray(h9, dtype=np.float32).ravel())
        c, hh, ww = frame.shape
        info = FrameInfo()
        roi_p = None
        if roi is not None:
            roi = np.ascontiguousarray(roi, dtype=np.float32)
            roi_p = roi.ctypes.data_as(_fp)
        # first call with no output to learn the shape is not possible; size generously
        cap = max(1, self._out_cap_guess(c, hh, ww))
        out = np.zeros(cap, dtype=np.float32)
        rc = self.api["run_frame"](self.h, frame.ctypes.data_as(_fp), c, hh, ww, h9.ctypes.data_as(_fp),
                                   roi_p, C.byref(info), out.ctypes.data_as(_fp), cap)
        self._check(rc)
        n = info.out_channels * info.out_height * info.out_width
        if n > cap:
            raise RuntimeError("output capacity guess too small")
        return info_dict(info), out[:n].reshape(info.out_channels, info.out_height, info.out_width).copy()

    def _out_cap_guess(self, c, h, w):
        # output extent <= (h + tile) x (w + tile) at input resolution; channels <= max in the net
        ch = max([c] + [l.conv.out_channels for l in self.spec.layers if l.conv is not None])
        t = int(self._cfg.tile_size)
        return ch * (h + 2 * t) * (w + 2 * t)

    def reset(self):
        self._check(self.api["reset"](self.h))

    def grid(self):
        r, c = C.c_int(), C.c_int()
        self._check(self.api["grid"](self.h, C.byref(r), C.byref(c)))
        return r.value, c.value

    def input_mask(self):
        buf = np.zeros(1 << 16, dtype=np.uint8)
        th, tw = C.c_int(), C.c_int()
        self._check(self.api["input_mask"](self.h, buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size,
                                           C.byref(th), C.byref(tw)))
        return buf[: th.value * tw.value].reshape(th.value, tw.value).copy()

    def read_state(self, layer, which):
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        self._check(self.api["read_state"](self.h, layer.encode(), which, None, 0, C.byref(c), C.byref(h), C.byref(w)))
        out = np.zeros((c.value, h.value, w.value), dtype=np.float32)
        self._check(self.api["read_state"](self.h, layer.encode(), which, out.ctypes.data_as(_fp), out.size,
                                           C.byref(c), C.byref(h), C.byref(w)))
        return out

    def read_packet(self, layer):
        c, gh, gw, halo = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        args = (C.byref(c), C.byref(gh), C.byref(gw), C.byref(halo))
        self._check(self.api["read_packet"](self.h, layer.encode(), None, 0, *args, None, 0))
        out = np.zeros((c.value, gh.value, gw.value), dtype=np.float32)
        mask = np.zeros(1 << 16, dtype=np.uint8)
        self._check(self.api["read_packet"](self.h, layer.encode(), out.ctypes.data_as(_fp), out.size, *args,
                                            mask.ctypes.data_as(C.POINTER(C.c_uint8)), mask.size))
        return out, halo.value, mask

    def read_ledger(self):
        rows, cols = self.grid()
        n = rows * cols
        used = np.zeros(n, np.int32)
        ty = np.zeros(n, np.int64)
        tx = np.zeros(n, np.int64)
        cov = np.zeros(n, np.uint8)
        self._check(self.api["read_ledger"](self.h, used.ctypes.data_as(C.POINTER(C.c_int)),
                                            ty.ctypes.data_as(C.POINTER(C.c_int64)),
                                            tx.ctypes.data_as(C.POINTER(C.c_int64)),
                                            cov.ctypes.data_as(C.POINTER(C.c_uint8)), n))
        return used.reshape(rows, cols), ty.reshape(rows, cols), tx.reshape(rows, cols), cov.reshape(rows, cols)


class RefEngine(_CEngine):
    """The unmodified reference engine (through oracle/ref_shim.cpp)."""
    PREFIX = "dfr"
    PATH = REF_LIB


class OracleEngine(_CEngine):
    """The C restatement (oracle/dfx_oracle.c)."""
    PREFIX = "dfo"
    PATH = ORACLE_LIB


def info_dict(info: FrameInfo) -> dict:
    return {k: getattr(info, k) for k, _ in FrameInfo._fields_}


def ref_run_streams(spec, cfg, frames, h9s, threads=None):
    """CPU baseline: one reference engine per host thread / stream.

    frames: [S, F, C, H, W] float32, h9s: [S, F, 9]. Returns (secs[S,F], flops[S,F]).
    """
    lib, _ = _load(REF_LIB, "dfr")
    fn = lib.dfr_run_streams
    fn.restype = C.c_int
    from paper_2210_09887_b200._capi import NetDesc
    fn.argtypes = [C.POINTER(NetDesc), C.POINTER(EngineConfigC), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                   _fp, _fp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    frames = np.ascontiguousarray(frames, dtype=np.float32)
    h9s = np.ascontiguousarray(h9s, dtype=np.float32)
    S, F, Cc, H, W = frames.shape
    desc, keep = spec.to_desc()
    cfg = config_struct(cfg)
    secs = np.zeros((S, F), np.float64)
    flops = np.zeros((S, F), np.uint64)
    rc = fn(C.byref(desc), C.byref(cfg), S, F, Cc, H, W, frames.ctypes.data_as(_fp), h9s.ctypes.data_as(_fp),
            secs.ctypes.data_as(C.POINTER(C.c_double)), flops.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc != 0:
        raise RuntimeError(lib.dfr_last_error().decode() if hasattr(lib, "dfr_last_error") else "dfr_run_streams failed")
    return secs, flops
