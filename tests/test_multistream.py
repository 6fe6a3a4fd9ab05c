"""Host side of the multi-GPU path on CPU (gloo, world_size 2): stream
partitioning over ranks and the job-level reductions bench.py uses (frames
SUM, device time MAX). One stream never shards (every frame mutates the whole
state), so ranks own disjoint blocks of independent streams and exchange no
data on the hot path."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_09887_b200.streams import frames_done, max_over_ranks, partition


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 8), (0, 4)])
def test_partition_is_a_balanced_disjoint_cover(n, world):
    parts = [partition(n, world, r) for r in range(world)]
    flat = [s for p in parts for s in p]
    assert sorted(flat) == list(range(n))
    assert len(set(flat)) == len(flat)
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1
    for p in parts:  # contiguous blocks
        assert p == list(range(p[0], p[0] + len(p))) if p else True


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = partition(64, world, rank)
    got = [None] * world
    dist.all_gather_object(got, mine)
    total = frames_done(len(mine) * 10, dist)
    slowest = max_over_ranks(1.0 + rank, dist)
    q.put((rank, got, total, slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_partition_and_reductions():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, total, slowest in res:
        flat = [s for part in got for s in part]
        assert sorted(flat) == list(range(64)) and len(set(flat)) == 64
        assert total == 640
        assert slowest == 2.0


def test_bench_gpus_2_spawns_two_ranks():
    """`python bench.py --gpus 2` without a torchrun environment launches two
    ranks itself (one process per GPU; gloo in the dry run) and rank 0 prints
    the job line with n_gpus = 2 and the max-over-ranks time."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ms_max"] == 11.0
    assert d["streams_per_rank"] == [[0], [1]]
