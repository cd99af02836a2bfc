"""CPU tests of the multi-GPU host logic (1D core partition):
the partition rule and the rank-ordered blob exchange over torch.distributed
(gloo, world_size 2 — the same code path the NCCL/IPC launch uses)."""
import os
import socket

import numpy as np
import pytest

from paper_2009_07463_b200.multi import exchange_blobs, partition_bounds


def check_bounds(b, nc, nt, n):
    parts = b.shape[0]
    assert b[0, 0] == 0 and b[-1, 1] == nc
    for k in range(parts):
        assert b[k, 0] % 32 == 0
        if k + 1 < parts:
            assert b[k, 1] == b[k + 1, 0] and b[k, 3] == b[k + 1, 2]
    assert b[0, 2] == nc and b[-1, 3] == nc + nt
    assert b[-1, 4] == nc + nt and b[-1, 5] == n
    for k in range(parts - 1):
        assert b[k, 4] == b[k, 5] == n


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 16])
def test_partition_bounds_cover_everything(parts):
    rng = np.random.default_rng(parts)
    nc, nt, nz = 10_000, 3_000, 500
    attached = np.sort(rng.integers(0, nc, size=nt - 40)).astype(np.uint64)
    anchor = np.concatenate([attached, np.full(40, 0xFFFFFFFF, np.uint64)])
    b = partition_bounds(nc, nt, nc + nt + nz, anchor, parts)
    check_bounds(b, nc, nt, nc + nt + nz)
    # every attached tree vertex lands in the partition owning its anchor
    for t, a in enumerate(attached):
        k = int(np.searchsorted(b[:, 0], a, side="right") - 1)
        assert b[k, 2] <= nc + t < b[k, 3]


def test_partition_bounds_tiny_and_errors():
    b = partition_bounds(5, 0, 5, np.zeros(0, np.uint64), 4)
    check_bounds(b, 5, 0, 5)
    assert (b[:3, 1] == 0).all()  # 5 vertices fit one word: all owned by the last part
    with pytest.raises(ValueError):
        partition_bounds(10, 0, 10, np.zeros(0, np.uint64), 17)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blobs = exchange_blobs(bytes([rank]) * (8 + rank))
    q.put((rank, blobs))
    dist.barrier()
    dist.destroy_process_group()


def test_blob_exchange_gloo_world2():
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert got[r] == [bytes([0]) * 8, bytes([1]) * 9]


def _merge_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2009_07463_b200.multi import merge_owned

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, nc, nt = 200, 96, 60
    rng = np.random.default_rng(7)
    anchor = np.concatenate([np.sort(rng.integers(0, nc, nt - 5)), np.full(5, 0xFFFFFFFF)])
    b = partition_bounds(nc, nt, n, anchor.astype(np.uint64), world)
    truth = rng.integers(-2**62, 2**62, n, dtype=np.int64)
    truth[::7] = -1  # unreached entries are all ones
    # junk outside the owned ranges, the owner's values inside them
    mine = np.zeros(n, bool)
    for lo, hi in ((b[rank, 0], b[rank, 1]), (b[rank, 2], b[rank, 3]), (b[rank, 4], b[rank, 5])):
        mine[int(lo):int(hi)] = True
    local = torch.from_numpy(np.where(mine, truth, 999).astype(np.int64))
    full = merge_owned(local, b[rank], dist)
    q.put((rank, bool((full.numpy() == truth).all())))
    dist.barrier()
    dist.destroy_process_group()


def test_merge_owned_result_gloo_world2():
    """multi.merge_owned (bench.py's multi-GPU validation): each rank holds only
    its owned slices; summing the masked slices over ranks gives every rank the
    whole result, negative (unreached) entries included."""
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_merge_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: True, 1: True}
