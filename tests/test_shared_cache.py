"""CPU (gloo, world 2) test of the shared template segment (one host copy of a
template per box, mapped by every GPU's process): two processes map the same bytes — writes of
one are visible to the other — through the handle broadcast over the process group.  libig's
part (cudaHostRegister of the mapping, ig_cache_attach) needs a GPU and is exercised by bench.py
at N > 1."""
import multiprocessing as mp
import os
import socket

import numpy as np

from paper_2505_20600_b200.shared_cache import SharedSegment, share_handle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 3 << 20
    seg = SharedSegment.create(n, "ig_test") if rank == 0 else None
    if rank == 0:
        a = np.frombuffer(seg.buffer(), dtype=np.uint8)
        a[:] = np.arange(n, dtype=np.uint64).astype(np.uint8)  # the "recorded template"
        del a
    handle = share_handle(seg, rank)
    if rank != 0:
        seg = SharedSegment.attach(handle)
    dist.barrier()
    a = np.frombuffer(seg.buffer(), dtype=np.uint8)
    same = bool(np.array_equal(a, np.arange(n, dtype=np.uint64).astype(np.uint8)))
    dist.barrier()
    if rank == 1:
        a[12345] = 7  # a write through the second mapping ...
    dist.barrier()
    seen = int(a[12345])  # ... is seen through the first
    del a
    q.put((rank, same, seen, seg.address != 0, handle[2]))
    dist.barrier()
    seg.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_map_the_same_cache_bytes():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        same, seen, mapped, nbytes = got[r]
        assert same and mapped and nbytes == 3 << 20
        assert seen == 7


def test_single_process_attach_to_own_segment():
    seg = SharedSegment.create(1 << 16)
    other = SharedSegment.attach(seg.handle)
    a = np.frombuffer(seg.buffer(), dtype=np.uint8)
    b = np.frombuffer(other.buffer(), dtype=np.uint8)
    a[100] = 42
    assert b[100] == 42 and seg.address != other.address
    del a, b
    other.close()
    seg.close()
