"""Time the public frame APIs on the bench workload (dev tool)."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import bench, paper_2210_09887_b200 as dfx
N = 24
spec, cfg, seq = bench.make_workload(N, seed=1000)
econf = dfx.EngineConfig(**cfg, conv_mode="tf32x3")
pinned = [torch.from_numpy(f).pin_memory() for f, _ in seq]
dfr = [p.cuda() for p in pinned]
e = dfx.DeltaEngine(spec, econf)
for k in range(3): e.run_frame_full(pinned[k].numpy(), seq[k][1])
oc, oh, ow = e.last_info["out_channels"], e.last_info["out_height"], e.last_info["out_width"]
outs = [torch.empty((oc * (oh + 64) * (ow + 64),), dtype=torch.float32).pin_memory() for _ in range(2)]
def timeit(name, fn):
    torch.cuda.synchronize(); t = time.time(); fn(); torch.cuda.synchronize()
    print(f"{name}: {(time.time() - t) * 1e3 / (N - 3):.3f} ms/frame", flush=True)
timeit("run_frame_full (sync, pageable out)", lambda: [e.run_frame_full(pinned[k].numpy(), seq[k][1]) for k in range(3, N)])
def dev():
    for k in range(3, N): e.submit_frame(dfr[k].data_ptr(), *dfr[k].shape, seq[k][1])
    e.sync()
timeit("submit_frame (device frames)", dev)
def host():
    for k in range(3, N): e.submit_host_frame(pinned[k].data_ptr(), *pinned[k].shape, seq[k][1], outs[k & 1].data_ptr(), outs[k & 1].numel())
    e.sync()
timeit("submit_host_frame (pipelined)", host)
def host_noout():
    for k in range(3, N): e.submit_host_frame(pinned[k].data_ptr(), *pinned[k].shape, seq[k][1], 0, 0)
    e.sync()
timeit("submit_host_frame (no output copy)", host_noout)
def host_sync():
    for k in range(3, N):
        e.submit_host_frame(pinned[k].data_ptr(), *pinned[k].shape, seq[k][1], outs[k & 1].data_ptr(), outs[k & 1].numel()); e.sync()
timeit("submit_host_frame + sync each", host_sync)
import ctypes as C
from paper_2210_09887_b200 import _capi
lib, api = _capi.load_library()
fb = [api["host_alloc"](pinned[0].numel() * 4) for _ in range(N)]
for k in range(N): C.memmove(fb[k], pinned[k].data_ptr(), pinned[k].numel() * 4)
ob = [api["host_alloc"](outs[0].numel() * 4) for _ in range(2)]
def host_lib():
    for k in range(3, N): e.submit_host_frame(fb[k], *pinned[k].shape, seq[k][1], ob[k & 1], outs[0].numel())
    e.sync()
timeit("submit_host_frame (library-pinned buffers)", host_lib)
