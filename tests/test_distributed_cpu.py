"""Multi-process host logic of the sharded decode path on CPU (gloo, world 2):
unit sharding covers every unit exactly once and the output gather returns the
exact unit-ordered concatenation (uneven shards included)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_03482_b200.distributed import gather_units, shard_units


@pytest.mark.parametrize("total,world", [(64, 1), (64, 2), (64, 8), (7, 2), (9, 4), (1, 1)])
def test_shards_partition_units(total, world):
    covered = []
    for r in range(world):
        s = shard_units(total, world, r)
        covered.extend(range(s.start, s.stop))
        assert abs(s.count - total / world) < 1
    assert covered == list(range(total))


def test_shard_rejects_bad_args():
    with pytest.raises(ValueError):
        shard_units(0, 2, 0)
    with pytest.raises(ValueError):
        shard_units(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = shard_units(total, world, rank)
        # stand-in for this rank's decode output: [units, G, d] tagged by global unit id
        local = torch.arange(s.start, s.stop, dtype=torch.float32)[:, None, None].expand(s.count, 4, 8)
        full = gather_units(local.contiguous(), s)
        q.put((rank, full[:, 0, 0].tolist(), tuple(full.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [64, 7])
def test_gloo_gather_two_ranks(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, shape in results:
        assert ids == [float(i) for i in range(total)]
        assert shape == (total, 4, 8)
