"""Multi-process wiring of the 1D core partition on one device, without any
traversal: two ranks (gloo for the blob exchange, as multi.connect does with
NCCL ranks on a real node) each build the same graph, export their partition's
exchange block as a CUDA IPC blob, open the peer's block and finish
etb_mp_connect. No kernel waits on another rank here (the partitioned BFS
itself is exercised in one launch by tests/test_gpu_partition.py)."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import ctypes as C

    import torch.distributed as dist

    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from paper_2009_07463_b200 import multi

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = eb.generate_graph(scale=10, edgefactor=16, seed=1)
        cg = eb.relayout_csr(g, mh=-1)
        L = E.lib()
        size = L.etb_mp_blob_size()
        buf = C.create_string_buffer(size)
        E._check(L.etb_mp_export(cg.handle, world, rank, buf))
        blobs = multi.exchange_blobs(buf.raw)
        # a blob list out of rank order is refused with the reference-style error
        bad = C.create_string_buffer(b"".join(reversed(blobs)), size * world)
        rc = L.etb_mp_connect(cg.handle, bad)
        refused = rc == E.ETB_EINVAL and b"ordered by rank" in L.etb_last_error()
        joined = C.create_string_buffer(b"".join(blobs), size * world)
        E._check(L.etb_mp_connect(cg.handle, joined))
        q.put((rank, "ok", refused, [len(b) for b in blobs]))
        dist.barrier()  # keep both exports alive until the peer has opened them
    except Exception as e:  # report, do not hang the parent
        q.put((rank, repr(e), False, []))
    finally:
        dist.destroy_process_group()


def test_ipc_export_connect_two_ranks_one_device():
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, status, refused, sizes in got:
        assert status == "ok", (rank, status)
        assert refused, rank
        assert len(sizes) == 2 and sizes[0] == sizes[1]
