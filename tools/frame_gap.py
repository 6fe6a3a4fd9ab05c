"""Inter-frame gap on the engine stream (DFX_FRAME_TRACE=1): previous frame's
last kernel end -> next frame's first kernel past its dependency wait."""
import ctypes, os, sys
os.environ["DFX_FRAME_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import bench, paper_2210_09887_b200 as dfx  # noqa: E402
from paper_2210_09887_b200 import _capi  # noqa: E402
N = 24
spec, cfg, seq = bench.make_workload(N, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
dev = [torch.from_numpy(f).cuda() for f, _ in seq]
for k in range(N):
    e.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1])
e.sync()
lib, _ = _capi.load_library()
buf = np.zeros(256, dtype=np.uint64)
lib.dfx_debug_frame_trace.argtypes = [ctypes.c_void_p]
assert lib.dfx_debug_frame_trace(buf.ctypes.data) == 0
t = buf.reshape(64, 4).astype(np.int64)[:N]
frame = np.diff(t[:, 1]) / 1e3
gap = (t[1:, 1] - t[:-1, 2]) / 1e3
print("frame period (claims wait->claims wait) us: median %.1f" % np.median(frame[4:]))
print("gap densify end -> next claims past wait us: median %.1f min %.1f max %.1f" % (np.median(gap[4:]), gap[4:].min(), gap[4:].max()))
print("claims entry -> past wait us: median %.1f" % np.median((t[:, 1] - t[:, 0])[4:] / 1e3))
