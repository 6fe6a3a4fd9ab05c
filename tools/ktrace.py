"""Per-kernel time in the real launch chain (DFX_KTRACE stamps: CTA 0 of each
kernel records when its dependency wait returned = previous kernel complete).
Prints the last frame's kernels in launch order with their chain time."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import bench, paper_2210_09887_b200 as dfx  # noqa: E402
from paper_2210_09887_b200 import _capi  # noqa: E402
N = 12
spec, cfg, seq = bench.make_workload(N, seed=1000, config=os.environ.get("KCONFIG", "c2"))
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
dev = [torch.from_numpy(f).cuda() for f, _ in seq]
for k in range(4):
    e.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1])
e.sync()
lib, _ = _capi.load_library()
f = lib.dfx_debug_ktrace
f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
buf = np.zeros(4096, dtype=np.uint64)
cnt = np.zeros(1, dtype=np.uint32)
assert f(1, None, None) == 0
for k in range(4, N):
    e.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1])
e.sync()
assert f(0, buf.ctypes.data, cnt.ctypes.data) == 0
n = int(cnt[0])
t = buf[:n].astype(np.int64)
per = n // (N - 4)
d = np.diff(t) / 1e3
print(f"{n} stamps, {per} kernels per frame; frame period {np.median(np.diff(t[::per])) / 1e3:.1f} us")
last = d[-per + 1:]
names = os.environ.get("KNAMES", "").split(",")
for i, v in enumerate(last):  # index 0 = the frame's first kernel (k_frame_begin)
    print(f"{i:3d} {v:7.1f} us  {names[i] if i < len(names) else ''}")
print(f"sum {last.sum():.1f} us (the frame's last kernel excluded)")
