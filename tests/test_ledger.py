"""Tile-ledger parity on CPU: the product's host ledger (dfx_ledger_*, the
object the engine plans every frame with) against the UNMODIFIED reference
TileLedger / plan_frame / apply_plan (oracle/_ref, dfr_ledger_*), step by
step: full-reset decisions, claims with their victims, fresh tiles, eviction
counts and the whole slot table must agree bit-for-bit. This is the
reference's own acceptance fuzz (acceptance.cpp:397-427, 1e4 steps against
ledgersim) re-expressed against the reference itself, plus the KATs of
test_buffer_manager.cpp:32-132."""
import ctypes as C

import numpy as np
import pytest

from paper_2210_09887_b200 import _capi

_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)


def _bind(lib, prefix, handle_t):
    f = {}
    f["create"] = getattr(lib, f"{prefix}_create")
    f["create"].argtypes = [C.c_int, C.c_int, C.POINTER(handle_t)]
    f["create"].restype = C.c_int
    f["destroy"] = getattr(lib, f"{prefix}_destroy")
    f["destroy"].argtypes = [handle_t]
    f["step"] = getattr(lib, f"{prefix}_step")
    f["step"].argtypes = [handle_t, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, _ip, _i64p, _ip, C.c_size_t,
                          _ip, _i64p, C.c_size_t, _ip, _ip]
    f["step"].restype = C.c_int
    f["slots"] = getattr(lib, f"{prefix}_slots")
    f["slots"].argtypes = [handle_t, _ip, _i64p, _i64p, C.POINTER(C.c_uint8), C.c_size_t]
    f["slots"].restype = C.c_int
    return f


class Ledger:
    def __init__(self, lib, prefix, rows, cols):
        self.f = _bind(lib, prefix, C.c_void_p)
        self.h = C.c_void_p()
        assert self.f["create"](rows, cols, C.byref(self.h)) == 0
        self.n = rows * cols

    def step(self, otx, oty, th, tw, ring):
        cap = 4 * self.n
        reset, nc, nf, ev = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        claims = np.zeros(4 * cap, np.int64)
        victims = np.zeros(cap, np.int32)
        fresh = np.zeros(2 * cap, np.int64)
        rc = self.f["step"](self.h, otx, oty, th, tw, ring, C.byref(reset), claims.ctypes.data_as(_i64p),
                            victims.ctypes.data_as(_ip), cap, C.byref(nc), fresh.ctypes.data_as(_i64p), cap,
                            C.byref(nf), C.byref(ev))
        if rc != 0:
            return ("error", rc)
        n, m = nc.value, nf.value
        return (reset.value, claims[:4 * n].tolist(), victims[:n].tolist(), fresh[:2 * m].tolist(), ev.value)

    def slots(self):
        used = np.zeros(self.n, np.int32)
        ty = np.zeros(self.n, np.int64)
        tx = np.zeros(self.n, np.int64)
        cov = np.zeros(self.n, np.uint8)
        assert self.f["slots"](self.h, used.ctypes.data_as(_ip), ty.ctypes.data_as(_i64p), tx.ctypes.data_as(_i64p),
                               cov.ctypes.data_as(C.POINTER(C.c_uint8)), self.n) == 0
        # the content of unused slots is irrelevant
        return used.tolist(), (ty * used).tolist(), (tx * used).tolist(), (cov * used).tolist()

    def close(self):
        self.f["destroy"](self.h)


def _pair(rows, cols):
    from oracle.oracle import REF_LIB, ref_available
    if not ref_available():
        pytest.skip("reference build (oracle/_ref) not present")
    lib, _ = _capi.load_library()
    ref = C.CDLL(REF_LIB)
    return Ledger(lib, "dfx_ledger", rows, cols), Ledger(ref, "dfr_ledger", rows, cols)


@pytest.mark.parametrize("seed", range(6))
def test_ledger_fuzz_matches_reference(seed):
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(2, 9)), int(rng.integers(2, 9))
    ours, ref = _pair(rows, cols)
    ox, oy = int(rng.integers(-20, 20)), int(rng.integers(-20, 20))
    resets = 0
    for step in range(1500):
        th, tw = int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1))
        r = rng.random()
        if r < 0.7:  # pan by up to a tile or two (wrap evictions, frontiers)
            ox += int(rng.integers(-2, 3))
            oy += int(rng.integers(-2, 3))
        elif r < 0.85:  # reverse direction into restricted regions
            ox -= int(rng.integers(0, cols + 2))
        elif r < 0.95:
            ox, oy = int(rng.integers(-30, 30)), int(rng.integers(-30, 30))
        ring = int(rng.integers(0, 3))
        a = ours.step(ox, oy, th, tw, ring)
        b = ref.step(ox, oy, th, tw, ring)
        assert a == b, (seed, step, a, b)
        assert ours.slots() == ref.slots(), (seed, step)
        resets += a[0] == 1
    assert resets > 0  # the fuzz does reach the full-reset path
    ours.close()
    ref.close()


def test_ledger_kats():
    """test_buffer_manager.cpp:32-61: an identical frame claims nothing; a
    wrap eviction records a frontier and re-entering it forces a reset."""
    ours, ref = _pair(4, 4)
    for L in (ours, ref):
        first = L.step(0, 0, 3, 3, 0)
        assert first[0] == 0 and len(first[1]) // 4 == 9 and len(first[3]) // 2 == 9
        again = L.step(0, 0, 3, 3, 0)
        assert again[1] == [] and again[3] == [] and again[4] == 0
        moved = L.step(2, 0, 3, 3, 0)  # columns 3, 4 wrap onto slots of columns -1, 0
        assert moved[4] > 0
        back = L.step(0, 0, 3, 3, 0)  # re-enter the evicted (restricted) left side
        assert back[0] == 1
    ours.close()
    ref.close()
