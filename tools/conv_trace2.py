"""Per-CTA timeline of one dense conv launch of the C2 bench frame
(DFX_CONV_DBG=64 DFX_CONV_TRACE_IDX=i python tools/conv_trace2.py): the
launch's work split (units, split-K S, items), then per CTA (globaltimer, us
from the first CTA start): start, first accumulator ready, items done, end,
and the split-K reducers."""
import ctypes as C
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402
from paper_2210_09887_b200 import _capi  # noqa: E402
spec, cfg, seq = bench.make_workload(8, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
for f, H in seq:
    e.run_frame_full(f, H)
lib, _ = _capi.load_library()
tr = np.zeros(4096, dtype=np.int64)
assert lib.dfx_debug_conv_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)), 4096) == 0
n, S, items, upi, listed = (int(x) for x in tr[590:595])
print(f"units {n} S {S} items {items} UPI {upi} listed {listed} items/CTA {items / 148:.2f}")
st = tr[1100:1900:2][:148].astype(np.float64)
ok = (st > 0) & (np.abs(st - st[0]) < 1e8)
t0 = st[ok].min()
us = lambda v: (v.astype(np.float64) - t0) / 1e3  # noqa: E731
en = tr[1101:1900:2][:148]
acc = tr[3100:3248]
done = tr[2100:2248]
red = tr[2600:2748]
act = ok & (acc > 0)
def mmm(v):
    return f"{np.min(v):6.1f} / {np.median(v):6.1f} / {np.max(v):6.1f}"
print("CTA start          min/med/max us", mmm(us(st[ok])))
if act.any():
    print("first acc ready    min/med/max us", mmm(us(acc[act])))
    print("items done         min/med/max us", mmm(us(done[act])))
    print("end                min/med/max us", mmm(us(en[act])))
    r = act & (red == 1)
    if r.any():
        print(f"reducers {int(r.sum())}: items done {mmm(us(done[r]))}  end {mmm(us(en[r]))}")
