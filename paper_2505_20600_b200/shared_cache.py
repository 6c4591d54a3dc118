"""One host copy of a template cache per box, shared by every GPU's worker process.

SURVEY §8(e): "Template caches live once in host shared memory.  Each process maps them with
cudaHostRegister" — the paper keeps its activation caches in host memory (P:522-526,
P:622-626) and runs one worker per GPU.  A Flux template is 28 x 57 x 2 x 4096 x 3072
bf16 = 80.3 GB (K/V) or ~66 GB (the bench's hybrid split), so eight private pinned copies do
not fit a host; one shared copy does.

The segment is an anonymous shared-memory file (memfd_create): no /dev/shm size limit applies
(container default 64 MB), it is freed when the last process closes it, and sibling processes
open it through /proc/<creator pid>/fd/<fd>.  This module only allocates and maps host bytes;
libig page-locks and maps them for its GPU (ig_cache_attach) and records the template into them
(ig_cache_template_into).
"""
from __future__ import annotations

import ctypes
import mmap
import os


class SharedSegment:
    """A MAP_SHARED mapping of `nbytes` host bytes visible to several processes.

    create: SharedSegment.create(nbytes, name) in ONE process, then share `.handle` (a small
    tuple: creator pid, fd, size) with the others, which call SharedSegment.attach(handle).
    `.address` is the mapping's virtual address in this process (for ig_cache_attach)."""

    def __init__(self, fd: int, nbytes: int, owner: bool, handle):
        self.fd = fd
        self.nbytes = nbytes
        self.owner = owner
        self.handle = handle
        self.mm = mmap.mmap(fd, nbytes, flags=mmap.MAP_SHARED, prot=mmap.PROT_READ | mmap.PROT_WRITE)
        self._view = ctypes.c_char.from_buffer(self.mm)
        self.address = ctypes.addressof(self._view)

    @classmethod
    def create(cls, nbytes: int, name: str = "ig_template") -> "SharedSegment":
        fd = os.memfd_create(name, 0)
        os.ftruncate(fd, nbytes)
        return cls(fd, nbytes, True, (os.getpid(), fd, nbytes))

    @classmethod
    def attach(cls, handle) -> "SharedSegment":
        pid, fd, nbytes = handle
        if pid == os.getpid():
            fd2 = os.dup(fd)
        else:
            fd2 = os.open(f"/proc/{pid}/fd/{fd}", os.O_RDWR)
        return cls(fd2, nbytes, False, handle)

    def buffer(self) -> memoryview:
        return memoryview(self.mm)

    def close(self):
        """Unmap and close this process's handle (the memory goes when the last one closes).
        ig_cache_free must have unregistered the range first."""
        if self.mm is None:
            return
        del self._view
        self.mm.close()
        self.mm = None
        os.close(self.fd)


def share_handle(seg_or_none, rank: int, src: int = 0, group=None):
    """Broadcast the creator's handle over a torch.distributed group (control plane only:
    a few bytes once at start-up, never on the step path)."""
    import torch.distributed as dist
    obj = [seg_or_none.handle if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]
