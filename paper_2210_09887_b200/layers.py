"""Layer-level entry points (include/dfx_b200.h, "layer level") from Python:
the reference's per-layer functions (delta_layers.hpp:103-127) and the
engine's input stage / claim reset on DEVICE buffers (raw device pointers,
e.g. torch tensors' data_ptr()), in this library's native layouts. See the
header for the layouts; `Packet` / `State` carry pointer + shape."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .network import DeltafluxError, ValidationError


class Placement(C.Structure):
    _fields_ = [("origin_tx", C.c_int64), ("origin_ty", C.c_int64), ("tiles_h", C.c_int), ("tiles_w", C.c_int)]


class Slot(C.Structure):
    _fields_ = [("used", C.c_int), ("tx", C.c_int64), ("ty", C.c_int64)]


class _Packet(C.Structure):
    _fields_ = [("d", C.c_void_p), ("ext", C.c_void_p), ("channels", C.c_int), ("tile", C.c_int), ("halo", C.c_int)]


class _State(C.Structure):
    _fields_ = [("d", C.c_void_p), ("channels", C.c_int), ("tile", C.c_int)]


@dataclass
class Packet:
    d: int
    ext: int
    channels: int
    tile: int
    halo: int

    def c(self):
        return _Packet(self.d, self.ext, self.channels, self.tile, self.halo)


@dataclass
class State:
    d: int
    channels: int
    tile: int

    def c(self):
        return _State(self.d, self.channels, self.tile)


def _declare(lib):
    P, V, I, F = C.POINTER, C.c_void_p, C.c_int, C.c_float
    sig = {
        "dfx_layer_ctx_create": (I, [I, I, I, V, P(V)]),
        "dfx_layer_ctx_destroy": (I, [V]),
        "dfx_layer_ctx_set_frame": (I, [V, P(Placement), V]),
        "dfx_packet_floats": (C.c_size_t, [V, I, I, I]),
        "dfx_packet_ext_bytes": (C.c_size_t, [V, I, I]),
        "dfx_state_floats": (C.c_size_t, [V, I, I]),
        "dfx_packet_from_chw": (I, [V, V, V, P(_Packet)]),
        "dfx_packet_to_chw": (I, [V, P(_Packet), V, V]),
        "dfx_state_from_chw": (I, [V, V, P(_State)]),
        "dfx_state_to_chw": (I, [V, P(_State), V]),
        "dfx_delta_conv_out_halo": (I, [I, I, I]),
        "dfx_delta_conv": (I, [V, P(_Packet), V, I, I, I, I, I, P(_Packet), P(C.c_uint64)]),
        "dfx_delta_truncate": (I, [V, P(_Packet), P(_State), P(_State), F, I, P(_Packet)]),
        "dfx_delta_maxpool": (I, [V, P(_Packet), P(_State), P(_State), I, P(_Packet)]),
        "dfx_densify": (I, [V, P(_State), P(_State), V]),
        "dfx_claim_reset": (I, [V, V, I, V, V, I]),
        "dfx_input_stage": (I, [V, V, V, V, V, F, I, I, P(_State), P(_State), P(_Packet), P(C.c_double)]),
    }
    api = {}
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
        api[name[4:]] = fn
    return api


def conv_out_halo(in_halo: int, k: int, stride: int) -> int:
    lib, _ = _capi.load_library()
    return _declare(lib)["delta_conv_out_halo"](in_halo, k, stride)


class LayerContext:
    """dfx_layer_ctx: one device, one CUDA stream (0 = its own), one grid."""

    def __init__(self, rows: int, cols: int, device: int = 0, stream: int = 0):
        self._lib, self._capi = _capi.load_library()
        self.api = _declare(self._lib)
        self.rows, self.cols = rows, cols
        h = C.c_void_p()
        self._chk(self.api["layer_ctx_create"](rows, cols, device, C.c_void_p(stream or None), C.byref(h)))
        self.h = h
        self.place = None

    def _chk(self, rc):
        if rc != 0:
            msg = self._capi["last_error"]().decode()
            raise (ValidationError if rc == 2 else DeltafluxError)(msg)

    def close(self):
        if getattr(self, "h", None):
            self.api["layer_ctx_destroy"](self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_frame(self, origin_tx, origin_ty, tiles_h, tiles_w, slots=None):
        """slots: None, or (used, tx, ty) int arrays of rows*cols entries."""
        pl = Placement(origin_tx, origin_ty, tiles_h, tiles_w)
        arr = None
        if slots is not None:
            used, tx, ty = (np.asarray(a).ravel() for a in slots)
            arr = (Slot * (self.rows * self.cols))()
            for i in range(self.rows * self.cols):
                arr[i] = Slot(int(used[i]), int(tx[i]), int(ty[i]))
        self._chk(self.api["layer_ctx_set_frame"](self.h, C.byref(pl), arr))
        self.place = (origin_tx, origin_ty, tiles_h, tiles_w)

    # sizes
    def packet_floats(self, c, t, halo):
        return self.api["packet_floats"](self.h, c, t, halo)

    def packet_ext_bytes(self, t, halo):
        return self.api["packet_ext_bytes"](self.h, t, halo)

    def state_floats(self, c, t):
        return self.api["state_floats"](self.h, c, t)

    # conversions (device pointers; masks are host numpy)
    def packet_from_chw(self, chw_ptr, mask, pkt: Packet):
        m = np.ascontiguousarray(mask, np.uint8).ravel()
        p = pkt.c()
        self._chk(self.api["packet_from_chw"](self.h, C.c_void_p(chw_ptr), m.ctypes.data, C.byref(p)))

    def packet_to_chw(self, pkt: Packet, chw_ptr):
        th, tw = self.place[2], self.place[3]
        m = np.zeros(th * tw, np.uint8)
        p = pkt.c()
        self._chk(self.api["packet_to_chw"](self.h, C.byref(p), C.c_void_p(chw_ptr), m.ctypes.data))
        return m.reshape(th, tw)

    def state_from_chw(self, chw_ptr, st: State):
        s = st.c()
        self._chk(self.api["state_from_chw"](self.h, C.c_void_p(chw_ptr), C.byref(s)))

    def state_to_chw(self, st: State, chw_ptr):
        s = st.c()
        self._chk(self.api["state_to_chw"](self.h, C.byref(s), C.c_void_p(chw_ptr)))

    # layers
    def delta_conv(self, pin: Packet, w_ptr, cin, cout, k, stride, conv_mode, pout: Packet):
        fl = (C.c_uint64 * 2)()
        a, b = pin.c(), pout.c()
        mode = {"tf32x3": _capi.CONV_TF32X3, "exact": _capi.CONV_EXACT}[conv_mode]
        self._chk(self.api["delta_conv"](self.h, C.byref(a), C.c_void_p(w_ptr), cin, cout, k, stride, mode, C.byref(b),
                                         fl))
        return int(fl[0]), int(fl[1])

    def delta_truncate(self, pin: Packet, acc: State, trunc: State, thr, relu, pout: Packet):
        a, s1, s2, b = pin.c(), acc.c(), trunc.c(), pout.c()
        self._chk(self.api["delta_truncate"](self.h, C.byref(a), C.byref(s1), C.byref(s2), float(thr), int(relu),
                                             C.byref(b)))

    def delta_maxpool(self, pin: Packet, acc: State, prev: State, k, pout: Packet):
        a, s1, s2, b = pin.c(), acc.c(), prev.c(), pout.c()
        self._chk(self.api["delta_maxpool"](self.h, C.byref(a), C.byref(s1), C.byref(s2), int(k), C.byref(b)))

    def densify(self, acc: State, trunc: State, out_ptr):
        s1, s2 = acc.c(), trunc.c()
        self._chk(self.api["densify"](self.h, C.byref(s1), C.byref(s2), C.c_void_p(out_ptr)))

    def claim_reset(self, coords, states, fills=None):
        co = np.ascontiguousarray(np.asarray(coords, np.int64).reshape(-1, 2))
        sts = [s.c() for s in states]
        parr = (C.POINTER(_State) * len(sts))(*[C.pointer(s) for s in sts])
        farr = None
        if fills is not None:
            farr = (C.c_void_p * len(sts))(*[C.c_void_p(f or None) for f in fills])
        self._chk(self.api["claim_reset"](self.h, co.ctypes.data, len(co), parr, farr, len(sts)))

    def input_stage(self, aligned_ptr, valid_ptr, fresh, thr, dilation, noise, acc: State, trunc: State,
                    pout: Packet, roi_factor_ptr=0):
        fr = None if fresh is None else np.ascontiguousarray(fresh, np.uint8).ravel()
        ur = C.c_double()
        s1, s2, b = acc.c(), trunc.c(), pout.c()
        self._chk(self.api["input_stage"](self.h, C.c_void_p(aligned_ptr), C.c_void_p(valid_ptr),
                                          C.c_void_p(roi_factor_ptr or None), None if fr is None else fr.ctypes.data,
                                          float(thr), int(dilation), int(noise), C.byref(s1), C.byref(s2),
                                          C.byref(b), C.byref(ur)))
        return ur.value
