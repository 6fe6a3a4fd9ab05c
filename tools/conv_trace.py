"""Pipeline stamps (clock64, CTA 0) of one dense conv of the bench frame:
DFX_CONV_DBG=64 DFX_CONV_TRACE_IDX=i python tools/conv_trace.py (i = 0..7 =
conv1, conv2, conv4, conv5, conv7, conv8, conv10, conv11)."""
import ctypes as C
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402
from paper_2210_09887_b200 import _capi  # noqa: E402
spec, cfg, seq = bench.make_workload(6, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
for f, H in seq:
    e.run_frame_full(f, H)
lib, _ = _capi.load_library()
tr = np.zeros(2048, dtype=np.int64)
assert lib.dfx_debug_conv_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)), 2048) == 0
b = tr[500]
print(f"kernel (CTA 0) {tr[501] - b} cycles; epilogue items:",
      [(int(tr[504 + 2 * i] - b), int(tr[505 + 2 * i] - b)) for i in range(4)])
print("warp exits:", [int(tr[520 + w] - b) for w in range(22)])
kb = [(int(tr[8 * g] - b), int(tr[8 * g + 1] - b), int(tr[8 * g + 2] - b)) for g in range(64) if tr[8 * g + 2]]
for g, (s, w, a) in enumerate(kb[:64]):
    print(f"kb {g:2d}: start {s:7d} empty_ok {w:7d} (+{w - s:5d}) full_arrive {a:7d} (+{a - w:5d})")
arr = np.array([a for _, _, a in kb])
if len(arr) > 2:
    print("median K-block arrive interval", np.median(np.diff(arr)), "cycles")
mm = [(int(tr[600 + 3 * q] - b), int(tr[601 + 3 * q] - b), int(tr[602 + 3 * q] - b)) for q in range(100) if tr[602 + 3 * q]]
wi = [int(tr[900 + q] - b) for q in range(120) if tr[900 + q]]
for q, (s, f, i) in enumerate(mm[:30]):
    print(f"mma pair {q:2d}: wait {s:7d} full_ok {f:7d} (+{f - s:5d}) issued {i:7d} (+{i - f:4d})  weights issued kb{2*q}: {wi[2*q] if 2*q < len(wi) else -1}")
if len(mm) > 2:
    fo = np.array([f for _, f, _ in mm])
    print("median MMA pair interval", np.median(np.diff(fo)), "cycles; median full wait", np.median([f - s for s, f, _ in mm]))
seg = np.array([[tr[8 * g + j] for j in range(8)] for g in range(64) if tr[8 * g + 2]], dtype=np.int64)
if len(seg):
    names = [("empty wait", 0, 1), ("fence_after", 1, 3), ("ld+st issue", 3, 4), ("wait::st", 4, 5), ("fence+syncwarp", 5, 6), ("arrive", 6, 2)]
    print("producer K-block segments (median / max cycles):", ", ".join(f"{n} {np.median(seg[:, b] - seg[:, a]):.0f}/{(seg[:, b] - seg[:, a]).max()}" for n, a, b in names))
    wg0 = seg[0::3]
    print("WG0 arrive -> next start gaps:", [int(wg0[i + 1, 0] - wg0[i, 2]) for i in range(min(12, len(wg0) - 1))])
cta = tr[1100:1900].reshape(400, 2)
cta = cta[(cta[:, 0] > 0) & (np.abs(cta[:, 0] - tr[1100]) < 200000)]  # this launch only (stale slots from earlier launches)
if len(cta):
    t0 = cta[:, 0].min()
    st, en = (cta[:, 0] - t0) / 1e3, (cta[:, 1] - t0) / 1e3
    print(f"CTAs {len(cta)}: start spread {st.max():.1f} us; end min/median/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f} us")
    print("slowest CTAs:", [(int(i), round(float(en[i]), 1)) for i in np.argsort(-en)[:8]])
full = tr[1100:1900].reshape(400, 2)
ok = (full[:, 0] > 0) & (np.abs(full[:, 0] - tr[1100]) < 200000)
idx = np.nonzero(ok[:148])[0]
if len(idx):
    t0 = full[idx, 0].min()
    en = (full[idx, 1] - t0) / 1e3
    sm = tr[1900 + idx]
    order = np.argsort(-en)
    print("slowest (cta, smid, end us):", [(int(idx[i]), int(sm[i]), round(float(en[i]), 1)) for i in order[:12]])
    print("fastest (cta, smid, end us):", [(int(idx[i]), int(sm[i]), round(float(en[i]), 1)) for i in order[-6:]])
print("loader startup (cycles from kernel start): poff begin %d, poff done %d, bar %d, cp.async issued %d, landed %d, pe ok %d" % tuple(int(tr[560 + i] - b) for i in range(6)))
