"""Multi-rank logic of bench.py on the CPU (gloo, world size 2): pair
partitioning covers every pair exactly once and the result gather (the
benchmark's only collective) lands every rank's records in rank order; the
reference arm exits cleanly on non-zero ranks."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _R:  # stand-in for rgbid_align_result
    def __init__(self, i):
        self.T_AB = type("P", (), {"R": [float(i)] * 9, "t": [i + 0.5] * 3})()
        self.status = 0
        self.total_iterations = 10 + i
        self.cov_degenerate = 0


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base, n = bench.partition(64, world, rank)
    rec = bench.result_records([_R(base + i) for i in range(n)], n)
    out = torch.empty((world * n, 16), dtype=torch.float64)
    bench.gather_records(rec, world, out, dist)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks timing reduction
    if rank == 0:
        q.put((out.numpy().copy(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    assert out.shape == (64, 16)
    np.testing.assert_array_equal(out[:, 0], np.arange(64, dtype=float))
    np.testing.assert_array_equal(out[:, 13], 10 + np.arange(64, dtype=float))


@pytest.mark.parametrize("world", [2, 8])
def test_partition_covers_all_pairs(world):
    import bench
    seen = []
    for r in range(world):
        base, n = bench.partition(4096, world, r)
        seen.extend(range(base, base + n))
    assert seen == list(range(4096))


@pytest.mark.parametrize("world", [2, 8])
def test_weak_partition_gives_each_rank_its_own_pairs(world):
    import bench
    blocks = [bench.partition(4096, world, r, "weak") for r in range(world)]
    assert all(n == 4096 for _, n in blocks)
    seen = [i for base, n in blocks for i in range(base, base + n)]
    assert seen == list(range(4096 * world))


def test_reference_arm_nonzero_rank_exits_clean():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and p.stdout.strip() == ""
