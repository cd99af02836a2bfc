"""CPU tests of the multi-GPU host logic (1D core partition):
the partition rule and the rank-ordered blob exchange over torch.distributed
(gloo, world_size 2 — the same code path the NCCL/IPC launch uses)."""
import os
import socket

import numpy as np
import pytest

from paper_2009_07463_b200.multi import exchange_blobs, partition_owner


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 16])
def test_partition_owner_rule(parts):
    """Core: 32-vertex words (the 8K·G hubs), then 256-vertex blocks, dealt round
    robin; trees follow their anchor;
    component trees and isolated vertices to the last partition. Every
    partition gets a near-equal share of the core and of its degree mass."""
    rng = np.random.default_rng(parts)
    nc, nt, nz = 100_000, 3_000, 500
    attached = np.sort(rng.integers(0, nc, size=nt - 40)).astype(np.uint64)
    anchor = np.concatenate([attached, np.full(40, 0xFFFFFFFF, np.uint64)])
    n = nc + nt + nz
    own = partition_owner(nc, nt, n, anchor, parts)
    assert own.shape == (n,) and own.max() < parts
    hub = 256 * parts * 32  # hub region: 32-vertex words dealt one at a time
    for v in (0, 31, 32, min(hub, nc) - 1):
        assert own[v] == (v // 32) % parts
    for v in (hub, hub + 255, hub + 256, nc - 1):  # then 256-vertex blocks
        if hub <= v < nc:
            assert own[v] == ((v - hub) // 256) % parts
    for t, a in enumerate(attached):
        assert own[nc + t] == own[int(a)]
    assert (own[nc + nt - 40:] == parts - 1).all()
    counts = np.bincount(own[:nc], minlength=parts)
    assert counts.max() - counts.min() <= 256 + 32


def test_partition_owner_balances_kronecker_degree_mass():
    """On a Kronecker s18 degree sequence sorted descending (as relaid core ids
    are), the round-robin ownership spreads the degree mass (the top-down work)
    far more evenly than equal id ranges (Eq. 1) would."""
    import oracle as O
    from paper_2009_07463_b200.multi import core_owner
    c = O.OracleCsr(1 << 18, O.oracle_generate(18, 16, 1))
    deg = np.sort(c.degrees().astype(np.float64))[::-1]
    deg = deg[deg > 0]
    for parts, bound in ((2, 1.05), (8, 1.25)):
        mass = np.bincount(core_owner(np.arange(len(deg)), parts), weights=deg, minlength=parts)
        ranges = np.bincount(np.arange(len(deg)) * parts // len(deg), weights=deg, minlength=parts)
        assert mass.max() / mass.mean() <= bound, parts
        assert ranges.max() / ranges.mean() > 1.4, parts


def test_partition_owner_errors():
    with pytest.raises(ValueError):
        partition_owner(10, 0, 10, np.zeros(0, np.uint64), 17)


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
    n, nc, nt = 2000, 960, 600
    rng = np.random.default_rng(7)
    anchor = np.concatenate([np.sort(rng.integers(0, nc, nt - 5)), np.full(5, 0xFFFFFFFF)])
    own = partition_owner(nc, nt, n, anchor.astype(np.uint64), world)
    truth = rng.integers(-2**62, 2**62, n, dtype=np.int64)
    truth[::7] = -1  # unreached entries are all ones
    # junk outside the owned vertices, the owner's values on them
    mine = own == rank
    local = torch.from_numpy(np.where(mine, truth, 999).astype(np.int64))
    full = merge_owned(local, torch.from_numpy(mine), dist)
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
