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
* ``assemble_result`` (validation only, outside any timed region): every rank
  holds the result of the vertices it owns; the owned slices are summed over
  ranks (disjoint supports, so the sum is the merge) and written back, so the
  device validator sees the whole tree on every rank.
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


def merge_owned(local, bounds_row, dist, group=None):
    """The whole result from every rank's owned slices: this rank's owned ranges
    (core, trees, isolated; bounds_row = its row of partition_bounds) of `local`
    (a 1-D int64 tensor of interleaved {depth, parent} pairs), zero elsewhere,
    summed over ranks. Supports are disjoint, so the sum reproduces each owner's
    entries exactly (negative values included)."""
    import torch

    out = torch.zeros_like(local)
    b = [int(x) for x in bounds_row]
    for lo, hi in ((b[0], b[1]), (b[2], b[3]), (b[4], b[5])):
        if hi > lo:
            out[lo:hi] = local[lo:hi]
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


class _DeviceArray:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3}


def assemble_result(cg, D) -> None:
    """Merge the ranks' owned slices of the last result into every rank's result
    buffer and mark it whole (etb_result_mark_assembled)."""
    import torch

    from .etbfs import _check, lib, partition_bounds

    ptr = C.c_void_p()
    _check(lib().etb_result_device_ptr(cg.handle, C.byref(ptr)))
    dp = torch.as_tensor(_DeviceArray(ptr.value, cg.vertex_count), device="cuda")
    full = merge_owned(dp, partition_bounds(cg, D.world)[D.rank], D.d)
    dp.copy_(full)
    torch.cuda.synchronize()
    _check(lib().etb_result_mark_assembled(cg.handle))
