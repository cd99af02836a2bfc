"""Host side of the 1D core partition.

* ``partition_bounds`` restates the device partition rule (bfs_part.cu
  ``part_bounds``): core V_k = [k·nc/G, (k+1)·nc/G) rounded down to 32-vertex
  bitmap words (Eq. 1 of the paper; proj/src/preprocess.cpp:77); edge trees
  follow their anchor; component trees and isolated vertices go to the last
  partition.
* ``exchange_blobs`` / ``connect`` wire one process per GPU: each rank exports
  its partition's exchange block as a CUDA IPC blob, the blobs are all-gathered
  through torch.distributed (any backend; gloo in the CPU tests), and each rank
  opens its peers' blocks. The BFS kernels then synchronise through NVLink peer
  memory — no NCCL call on the data path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

NONE32 = 0xFFFFFFFF


def partition_bounds(nc: int, nt: int, n: int, tanchor: np.ndarray, parts: int) -> np.ndarray:
    """(parts, 6) array: core lo, hi, tree lo, hi, isolated lo, hi (relaid ids)."""
    if parts < 1 or parts > 16:
        raise ValueError("etb_layout_partition: partitions must be in [1, 16]")
    out = np.zeros((parts, 6), np.uint64)
    for k in range(parts):
        lo = 0 if k == 0 else (k * nc // parts) & ~31
        hi = nc if k + 1 == parts else ((k + 1) * nc // parts) & ~31
        out[k, 0], out[k, 1] = lo, max(lo, hi)
    anc = np.asarray(tanchor, np.uint64)
    comp = np.nonzero(anc == NONE32)[0]
    first_component = int(comp[0]) if comp.size else nt
    attached = anc[:first_component]
    for k in range(parts):
        t0 = 0 if k == 0 else int(np.searchsorted(attached, out[k, 0], side="left"))
        t1 = nt if k + 1 == parts else int(np.searchsorted(attached, out[k + 1, 0], side="left"))
        out[k, 2], out[k, 3] = nc + t0, nc + t1
        out[k, 4] = out[k, 5] = n
    out[parts - 1, 4] = nc + nt
    return out


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather one opaque blob per rank, ordered by rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, blob, group=group)
    return [bytes(b) for b in gathered]


def connect(cg, rank: int, world: int, group=None) -> None:
    """Make `cg` this rank's partition of a `world`-GPU 1D partition."""
    from .etbfs import _check, lib

    L = lib()
    size = L.etb_mp_blob_size()
    buf = C.create_string_buffer(size)
    _check(L.etb_mp_export(cg.handle, world, rank, buf))
    blobs = exchange_blobs(buf.raw, group)
    joined = C.create_string_buffer(b"".join(blobs), size * world)
    _check(L.etb_mp_connect(cg.handle, joined))
