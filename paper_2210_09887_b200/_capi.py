"""ctypes mirror of include/dfx_b200.h (the C-ABI boundary of the CUDA path).

The structures here are plain type definitions; `load_library()` binds the
in-tree CUDA library `paper_2210_09887_b200/libdfx_b200.so` and fails loudly
when it is missing — there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdfx_b200.so")

# dfx_layer_kind (dflx::LayerKind, network.hpp:11)
KINDS = {
    "conv": 0,
    "relu": 1,
    "truncate": 2,
    "maxpool": 3,
    "avgpool": 4,
    "upsample": 5,
    "batchnorm": 6,
    "add": 7,
    "output": 8,
}
KIND_NAMES = {v: k for k, v in KINDS.items()}

DFX_OK, DFX_ERR, DFX_ERR_VALIDATION, DFX_ERR_IO, DFX_ERR_CUDA = range(5)
STATE_ACC, STATE_TRUNC, STATE_PREV = 0, 1, 2
CONV_TF32X3, CONV_EXACT = 0, 1
# kernel families (dfx_b200.h DFX_FAM_*); "tensor" families are FLOP-bound, others HBM-bound
FAMILIES = ["claims_reset", "input_stage", "conv_targets", "conv_mma", "truncate", "pool", "linear_ops", "densify"]
FAMILY_BOUND = {"conv_mma": "tensor"}

_fp = C.POINTER(C.c_float)


class LayerDesc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("kind", C.c_int),
        ("input0", C.c_char_p),
        ("input1", C.c_char_p),
        ("in_channels", C.c_int),
        ("out_channels", C.c_int),
        ("kernel", C.c_int),
        ("stride", C.c_int),
        ("padding", C.c_int),
        ("weights", _fp),
        ("bias", _fp),
        ("pool_k", C.c_int),
        ("pool_stride", C.c_int),
        ("factor", C.c_int),
        ("bn_channels", C.c_int),
        ("bn_scale", _fp),
        ("bn_shift", _fp),
        ("has_threshold", C.c_int),
        ("threshold", C.c_float),
        ("truncate_enabled", C.c_int),
    ]


class NetDesc(C.Structure):
    _fields_ = [
        ("in_channels", C.c_int),
        ("num_layers", C.c_int),
        ("layers", C.POINTER(LayerDesc)),
    ]


class EngineConfigC(C.Structure):
    _fields_ = [
        ("tile_size", C.c_int),
        ("grid_rows", C.c_int),
        ("grid_cols", C.c_int),
        ("input_threshold", C.c_float),
        ("default_threshold", C.c_float),
        ("override_net_thresholds", C.c_int),
        ("mask_dilation", C.c_int),
        ("roi_enabled", C.c_int),
        ("noise_suppression", C.c_int),
        ("padded_convolutions", C.c_int),
        ("conv_mode", C.c_int),
    ]


class FrameInfo(C.Structure):
    _fields_ = [
        ("frame_index", C.c_int64),
        ("origin_tx", C.c_int64),
        ("origin_ty", C.c_int64),
        ("tiles_h", C.c_int),
        ("tiles_w", C.c_int),
        ("fresh", C.c_int),
        ("evicted", C.c_int),
        ("reset", C.c_int),
        ("dropped_pixels", C.c_int64),
        ("update_rate", C.c_double),
        ("conv_flops", C.c_uint64),
        ("dense_flops", C.c_uint64),
        ("out_channels", C.c_int),
        ("out_height", C.c_int),
        ("out_width", C.c_int),
    ]


def declare_engine_api(lib, prefix: str, engine_arg=C.c_void_p):
    """Declare the common engine entry points `<prefix>_*` on a ctypes lib.

    The product (prefix "dfx_engine"), the reference shim ("dfr") and the C
    restatement ("dfo") export the same signatures.
    """
    P = engine_arg

    def f(name, restype, *args):
        fn = getattr(lib, f"{prefix}_{name}")
        fn.restype = restype
        fn.argtypes = list(args)
        return fn

    api = {}
    api["create"] = f("create", C.c_int, C.POINTER(NetDesc), C.POINTER(EngineConfigC), C.POINTER(C.c_void_p)) \
        if prefix != "dfx_engine" else f("create", C.c_int, C.POINTER(NetDesc), C.POINTER(EngineConfigC), C.c_int, C.POINTER(C.c_void_p))
    api["destroy"] = f("destroy", None if prefix != "dfx_engine" else C.c_int, P)
    api["run_frame"] = f("run_frame", C.c_int, P, _fp, C.c_int, C.c_int, C.c_int, _fp, _fp,
                         C.POINTER(FrameInfo), _fp, C.c_size_t)
    api["reset"] = f("reset", C.c_int, P)
    api["input_mask"] = f("input_mask", C.c_int, P, C.POINTER(C.c_uint8), C.c_size_t,
                          C.POINTER(C.c_int), C.POINTER(C.c_int))
    api["grid"] = f("grid", C.c_int, P, C.POINTER(C.c_int), C.POINTER(C.c_int))
    api["read_state"] = f("read_state", C.c_int, P, C.c_char_p, C.c_int, _fp, C.c_size_t,
                          C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int))
    api["read_packet"] = f("read_packet", C.c_int, P, C.c_char_p, _fp, C.c_size_t,
                           C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                           C.POINTER(C.c_int), C.POINTER(C.c_uint8), C.c_size_t)
    api["read_ledger"] = f("read_ledger", C.c_int, P, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64), C.POINTER(C.c_uint8), C.c_size_t)
    err_name = "dfx_last_error" if prefix == "dfx_engine" else f"{prefix}_last_error"
    le = getattr(lib, err_name)
    le.restype = C.c_char_p
    le.argtypes = []
    api["last_error"] = le
    return api


_LIB = None


def load_library():
    """Load the in-tree CUDA library; raise if it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    api = declare_engine_api(lib, "dfx_engine")
    extra = {
        "default_config": (None, [C.POINTER(EngineConfigC)]),
        "wrap_tile": (None, [C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    }
    for name, (res, args) in extra.items():
        fn = getattr(lib, f"dfx_{name}")
        fn.restype = res
        fn.argtypes = args
        api[name] = fn
    for name, res, args in [
        ("submit_frame", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _fp]),
        ("submit_host_frame", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _fp, C.c_void_p,
                                        C.c_size_t]),
        ("sync", C.c_int, [C.c_void_p, C.POINTER(FrameInfo)]),
        ("output_device", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        ("num_layers", C.c_int, [C.c_void_p]),
        ("layer_flops", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        ("kernel_count", C.c_int, [C.c_void_p]),
        ("set_profiling", C.c_int, [C.c_void_p, C.c_int]),
        ("reset_profile", C.c_int, [C.c_void_p]),
        ("profile", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_double)]),
        ("timer_start", C.c_int, [C.c_void_p]),
        ("timer_stop", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ]:
        fn = getattr(lib, f"dfx_engine_{name}")
        fn.restype = res
        fn.argtypes = args
        api[name] = fn
    fn = lib.dfx_validate_net
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(NetDesc), C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    api["validate_net"] = fn
    fn = lib.dfx_host_alloc
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_size_t]
    api["host_alloc"] = fn
    fn = lib.dfx_host_free
    fn.restype = None
    fn.argtypes = [C.c_void_p]
    api["host_free"] = fn
    fn = lib.dfx_kernel_family_name
    fn.restype = C.c_char_p
    fn.argtypes = [C.c_int]
    api["family_name"] = fn
    _LIB = (lib, api)
    return _LIB
