"""The C-ABI's caller-stream and device-buffer forms:
dfx_engine_create_on_stream binds the engine to a caller's cudaStream_t, and
dfx_engine_run_frame_ex takes device-resident frames and writes the output to
device memory; both give exactly the host-path results (exact mode)."""
import ctypes as C

import numpy as np
import pytest

import netgen

pytestmark = pytest.mark.gpu


def test_caller_stream_and_device_buffers_match_host_path():
    import torch
    import paper_2210_09887_b200 as dfx
    from paper_2210_09887_b200 import _capi
    lib, api = _capi.load_library()
    spec = netgen.vgg8_net(np.random.default_rng(3), widths=(16, "P", 32))
    seq = netgen.pan_rotate_sequence(np.random.default_rng(4), 3, 96, 128, 4, 3, 1, 0.4)
    cfg = dfx.EngineConfig(tile_size=16, conv_mode="exact", input_threshold=0.05)
    ref = dfx.DeltaEngine(spec, cfg)
    want = [ref.run_frame_full(f, H) for f, H in seq]

    desc, keep = spec.to_desc()
    ccfg = cfg.to_c()
    stream = torch.cuda.Stream()
    h = C.c_void_p()
    fn = lib.dfx_engine_create_on_stream
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    assert fn(C.addressof(desc), C.addressof(ccfg), 0, C.c_void_p(stream.cuda_stream), C.byref(h)) == 0
    run = lib.dfx_engine_run_frame_ex
    run.restype = C.c_int
    run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                    C.POINTER(_capi.FrameInfo), C.c_void_p, C.c_size_t, C.c_int]
    for k, (f, H) in enumerate(seq):
        dframe = torch.from_numpy(f).cuda()
        e_info, e_out = want[k]
        dout = torch.zeros(e_out.size, device="cuda")
        info = _capi.FrameInfo()
        h9 = np.ascontiguousarray(H, np.float32)
        rc = run(h, C.c_void_p(dframe.data_ptr()), *f.shape, 1, h9.ctypes.data, None, C.byref(info),
                 C.c_void_p(dout.data_ptr()), dout.numel(), 1)
        assert rc == 0, lib.dfx_last_error()
        got = {k2: getattr(info, k2) for k2, _ in _capi.FrameInfo._fields_}
        assert got == e_info, k
        assert np.array_equal(dout.cpu().numpy().reshape(e_out.shape), e_out), k
    lib.dfx_engine_destroy(h)
