"""Multi-rank host logic of the sharded path on CPU (gloo, world_size 2).

The hexes are independent, so ranks never exchange data on the path
(DESIGN.md section 7); what must be right is the partition (every hex on
exactly one rank) and the bookkeeping collectives bench.py uses: the barrier,
the max over ranks of the device time and the sum of verdict counters.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1706_01613_b200 import shard  # noqa: E402


def test_strong_shard_partitions_exactly():
    for n in (0, 1, 7, 1000, 10_000_001):
        for world in (1, 2, 3, 8):
            covered = []
            sizes = []
            for r in range(world):
                s, c = shard.strong_shard(n, world, r)
                covered.extend(range(s, s + c)) if n < 100_000 else None
                sizes.append(c)
                if r:
                    ps, pc = shard.strong_shard(n, world, r - 1)
                    assert ps + pc == s                    # contiguous, in rank order
            assert sum(sizes) == n and max(sizes) - min(sizes) <= 1
            if n < 100_000:
                assert covered == list(range(n))


def test_weak_shard_offsets():
    assert shard.weak_shard(10, 0) == (0, 10)
    assert shard.weak_shard(10, 3) == (30, 10)
    with pytest.raises(ValueError):
        shard.strong_shard(5, 2, 2)


def test_collectives_without_process_group_are_identity():
    assert shard.max_over_ranks(2.5) == 2.5
    assert shard.sum_over_ranks([1, 2]) == [1, 2]
    shard.barrier()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, n_total: int, out_dir: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, count = shard.strong_shard(n_total, world, rank)
        # every rank reports its range; rank 0 checks the union is exact
        t = torch.tensor([start, count], dtype=torch.int64)
        got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, t)
        shard.barrier()
        mx = shard.max_over_ranks(1.0 + rank * 0.25)             # "device time" of each rank
        tot = shard.sum_over_ranks([count, rank, 1])
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(f"{[g.tolist() for g in got]}|{mx}|{tot}")
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_and_bookkeeping(tmp_path):
    world, n_total = 2, 1001
    mp.spawn(_worker, args=(world, _free_port(), n_total, str(tmp_path)), nprocs=world, join=True)
    outs = [open(tmp_path / f"r{r}.txt").read() for r in range(world)]
    assert outs[0] == outs[1]                                  # every rank sees the same result
    ranges, mx, tot = outs[0].split("|")
    ranges = eval(ranges)
    assert ranges == [[0, 501], [501, 500]]
    assert float(mx) == 1.25
    assert eval(tot) == [n_total, 1, world]
