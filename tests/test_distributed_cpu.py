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


def _bench_worker(rank, world, port, q):
    """One rank of bench.py's strong-scaled C3 layout on CPU: its KV-head shard of the 64
    units, per-global-unit seeded inputs (bench.unit_tensor), a per-unit stand-in for the
    decode, and the output gather."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench

        w = bench.WORKLOADS["c3"]
        total = w["batch"] * w["kv_heads"]
        s = shard_units(total, world, rank)
        qs = torch.stack([bench.unit_tensor((w["G"], w["d"]), 1, s.start + i, "cpu", torch.float32)
                          for i in range(s.count)])
        local = torch.tanh(qs) * (torch.arange(s.start, s.stop)[:, None, None] + 1.0)   # [count, G, d]
        full = gather_units(local.contiguous(), s)
        q.put((rank, s.start, s.count, full.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_strong_scaled_shards_equal_single_rank():
    """Shard -> per-rank inputs -> gather over two ranks equals the single-rank computation
    bit for bit (units are independent and seeded by their global index)."""
    import bench

    w = bench.WORKLOADS["c3"]
    total = w["batch"] * w["kv_heads"]
    qs = torch.stack([bench.unit_tensor((w["G"], w["d"]), 1, u, "cpu", torch.float32) for u in range(total)])
    ref = (torch.tanh(qs) * (torch.arange(total)[:, None, None] + 1.0)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    starts = sorted((r[1], r[2]) for r in results)
    assert starts == [(0, total // 2), (total // 2, total // 2)]     # a KV-head split: 4 heads x 8 batches each
    for _, _, _, full in results:
        assert full.shape == (total, w["G"], w["d"])
        assert (full == ref).all()
