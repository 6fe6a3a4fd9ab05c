"""Stream parallelism: independent camera streams, one engine each.

The path does not shard within a stream (every frame mutates all layer state,
reference engine.cpp:212-284), so multi-GPU scaling comes from independent
streams (one engine instance per video stream): the streams of a
job are partitioned over the ranks (one process per GPU) in contiguous
blocks, and each rank runs its block on its own GPU. There is no collective on
the data path; the only cross-rank operations are the timing barrier and the
max-over-ranks reduction of the device-measured time.

`StreamPool` runs several streams on one GPU: each engine owns its CUDA
stream, frames are submitted round robin through the pipelined host-frame API
(dfx_engine_submit_host_frame), so kernels of different streams overlap.
"""

from __future__ import annotations

from typing import List, Sequence


def partition(n_streams: int, world: int, rank: int) -> List[int]:
    """Contiguous block of stream ids owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    base, extra = divmod(n_streams, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def max_over_ranks(value: float, dist=None) -> float:
    """Job time = the slowest rank's device-measured time (all_reduce MAX)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def frames_done(local_frames: int, dist=None) -> int:
    """Total frames processed by the job (all_reduce SUM)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return int(local_frames)
    import torch
    t = torch.tensor([int(local_frames)], dtype=torch.int64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


class StreamPool:
    """Several independent camera streams on one GPU (one engine each)."""

    def __init__(self, spec, cfg, n: int, device: int = 0):
        from . import _capi
        from .engine import DeltaEngine
        self.engines = [DeltaEngine(spec, cfg, device=device) for _ in range(n)]
        _, self._api = _capi.load_library()
        self._bufs = []

    def host_buffer(self, nbytes: int) -> int:
        """Page-locked host buffer owned by the pool (freed on close)."""
        p = self._api["host_alloc"](nbytes)
        if not p:
            raise MemoryError("dfx_host_alloc failed")
        self._bufs.append(p)
        return p

    def submit(self, frames: Sequence[int], shape, homographies, outs: Sequence[int], out_floats: int):
        """One frame per stream: frames[i] / outs[i] are page-locked host
        pointers of stream i's frame and output."""
        for e, f, h, o in zip(self.engines, frames, homographies, outs):
            e.submit_host_frame(f, *shape, h, o, out_floats)

    def sync(self):
        return [e.sync() for e in self.engines]

    def close(self):
        for p in self._bufs:
            self._api["host_free"](p)
        self._bufs = []
        for e in self.engines:
            e.close()
