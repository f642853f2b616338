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
    base, n = bench.partition(65, world, rank)  # uneven: rank 0 holds one pair more
    n_max = bench.partition(65, world, 0)[1]
    rec = bench.result_records([_R(base + i) for i in range(n)], n)
    out = torch.empty((world * n_max, 16), dtype=torch.float64)
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
    assert out.shape == (66, 16)  # 2 x 33 padded records, rank 1's last slot empty
    got = np.concatenate([out[:33], out[33:65]])
    np.testing.assert_array_equal(got[:, 0], np.arange(65, dtype=float))
    np.testing.assert_array_equal(got[:, 13], 10 + np.arange(65, dtype=float))
    assert not out[65].any()


@pytest.mark.parametrize("world", [2, 8])
def test_partition_covers_all_pairs(world):
    import bench
    seen = []
    for r in range(world):
        base, n = bench.partition(4096, world, r)
        seen.extend(range(base, base + n))
    assert seen == list(range(4096))


@pytest.mark.parametrize("pairs,world", [(4096, 2), (4096, 8), (4097, 8), (5, 8)])
def test_partition_uneven_blocks(pairs, world):
    import bench
    blocks = [bench.partition(pairs, world, r) for r in range(world)]
    sizes = [n for _, n in blocks]
    assert sum(sizes) == pairs and max(sizes) - min(sizes) <= 1
    assert [b for b, _ in blocks] == [sum(sizes[:r]) for r in range(world)]


def test_reference_arm_nonzero_rank_exits_clean():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_gpus_flag_relaunches_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run (--gpus was a dead flag): both ranks start,
    rank 0 alone prints one JSON line carrying n_gpus = 2, every rank exits 0."""
    import json
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR",
                        "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "1", "--warmup", "0", "--cpu-sample", "2",
                        "--cpu-latency-runs", "0"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["cpu_baseline"]["ok"] == 2
    # the reference arm never maps the CUDA library (inputs from oracle/_build/librgbid_synth.so)
    libs = line["cpu_baseline"]["libraries_loaded"]
    assert libs and all(p.startswith("oracle/") for p in libs), libs
