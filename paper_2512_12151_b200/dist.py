"""Row-partitioned PCG over several GPUs (SURVEY.md §8(e), C4 multi-GPU).

The reference is single-process (`intact/sparse.py:64-73`, `:99-150` run the
whole matvec / PCG in one numpy process); this spreads one scene's linear
solve over the ranks of a job, one GPU each.  Every rank keeps the whole
(replicated) system — the assembly, CCD and line search are computed
identically everywhere — and the PCG splits its rows into contiguous chunks:
per CG iteration each rank computes H p on its own rows, the ranks allreduce
pAp and (|r|^2, r.z) and allgather their z rows (NCCL, `csrc/dist.cu`), and
every rank ends the solve with the full solution.  `Partition.local(P)` runs
P partitions in one process on one GPU (exchanges as device copies): the
single-GPU check of the partition arithmetic against the unpartitioned solve.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes)."""
    buf = (C.c_char * 128)()
    _lib.check(_lib.lib().ibf_dist_unique_id(C.cast(buf, C.c_void_p)), "ibf_dist_unique_id")
    return bytes(buf)


def broadcast_id(group=None) -> bytes:
    """Rank 0's unique id on every rank of the torch.distributed job (any
    backend: the id is a 128-byte host object)."""
    import torch.distributed as dist
    obj = [unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class Partition:
    """An ibf_dist handle: this process's part of a row partition."""

    def __init__(self, handle, rank, world, local):
        self.handle, self.rank, self.world, self.local = handle, rank, world, local

    @classmethod
    def local_parts(cls, parts: int) -> "Partition":
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_dist_create_local(int(parts), C.byref(h)), "ibf_dist_create_local")
        return cls(h, 0, int(parts), True)

    @classmethod
    def nccl(cls, rank: int, world: int, uid: bytes) -> "Partition":
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_dist_create(int(rank), int(world), C.cast(buf, C.c_void_p), C.byref(h)),
                   "ibf_dist_create")
        return cls(h, int(rank), int(world), False)

    @classmethod
    def from_torch(cls, group=None) -> "Partition":
        """One partition per rank of the initialised torch.distributed job."""
        import torch.distributed as dist
        return cls.nccl(dist.get_rank(group), dist.get_world_size(group), broadcast_id(group))

    def row_ranges(self, n: int) -> list:
        """[(r0, r1)] of every partition for an n-row system (chunks of 32-row multiples)."""
        chunk = -(-max(n, 1) // self.world)
        chunk = -(-chunk // 32) * 32
        return [(min(n, r * chunk), min(n, (r + 1) * chunk)) for r in range(self.world)]

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_dist_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass
