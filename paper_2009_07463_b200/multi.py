"""Host side of the 1D core partition.

* ``partition_owner`` restates the device ownership rule (bfs_part.cuh): the
  degree-sorted core is dealt round robin, as the paper's static round-robin
  shuffle (SRRS, Alg. 4) balances its segments (the equal ranges of Eq. 1,
  proj/src/preprocess.cpp:77, would give one partition every hub) — the first
  256·G bitmap words (8K·G hubs) one 32-vertex word at a time, the rest in
  256-vertex blocks; a tree vertex follows its anchor; component trees and
  isolated vertices go to the last partition.
* ``exchange_blobs`` / ``connect`` wire one process per GPU: each rank exports
  its partition's exchange block as a CUDA IPC blob, the blobs are all-gathered
  through torch.distributed (any backend; gloo in the CPU tests), and each rank
  opens its peers' blocks. The BFS kernels then synchronise through NVLink peer
  memory — no NCCL call on the data path.
* ``assemble_result`` (validation only, outside any timed region): every rank
  holds the result of the vertices it owns; the owned entries are summed over
  ranks (disjoint supports, so the sum is the merge) and written back, so the
  device validator sees the whole tree on every rank.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

NONE32 = 0xFFFFFFFF
HUB_WORDS_PER = 256  # x G bitmap words dealt one at a time
BLOCK_WORDS = 8      # the rest: 256-vertex blocks


def core_owner(v, parts):
    w = np.asarray(v, np.uint64) >> np.uint64(5)
    hw = HUB_WORDS_PER * parts
    hub = w < hw
    tail = (w - np.minimum(w, hw)) // BLOCK_WORDS
    return np.where(hub, w % parts, tail % parts).astype(np.uint32)


def partition_owner(nc: int, nt: int, n: int, tanchor: np.ndarray, parts: int) -> np.ndarray:
    """The owning partition of every relaid vertex (u32[n])."""
    if parts < 1 or parts > 16:
        raise ValueError("etb_layout_partition: partitions must be in [1, 16]")
    own = np.full(n, parts - 1, np.uint32)
    own[:nc] = core_owner(np.arange(nc, dtype=np.uint64), parts)
    anc = np.asarray(tanchor, np.uint64)[:nt]
    attached = anc != NONE32
    tree_own = np.full(nt, parts - 1, np.uint32)
    tree_own[attached] = core_owner(anc[attached], parts)
    own[nc:nc + nt] = tree_own
    return own


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


def merge_owned(local, mine, dist, group=None):
    """The whole result from every rank's owned entries: `local` (a 1-D int64
    tensor of interleaved {depth, parent} pairs) where `mine` (a bool tensor on
    the same device: this rank owns the vertex), zero elsewhere, summed over
    ranks. Supports are disjoint, so the sum reproduces each owner's entries
    exactly (negative values included)."""
    import torch

    out = torch.where(mine, local, torch.zeros_like(local))
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

    from .etbfs import _check, lib, partition_owner

    # the traversal ran on the layout's own (non-blocking) stream: finish it
    # before torch's stream reads the result, and torch's writes before the
    # library's next calls (cudaDeviceSynchronize covers every stream)
    torch.cuda.synchronize()
    ptr = C.c_void_p()
    _check(lib().etb_result_device_ptr(cg.handle, C.byref(ptr)))
    dp = torch.as_tensor(_DeviceArray(ptr.value, cg.vertex_count), device="cuda")
    mine = torch.from_numpy(partition_owner(cg, D.world) == D.rank).to(dp.device)
    full = merge_owned(dp, mine, D.d)
    dp.copy_(full)
    torch.cuda.synchronize()
    _check(lib().etb_result_mark_assembled(cg.handle))
