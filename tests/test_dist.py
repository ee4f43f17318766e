"""Host side of the row-partitioned PCG (paper_2512_12151_b200/dist.py):
partition handles, row ranges, and the NCCL unique-id exchange over a
world-size-2 gloo process group on CPU.  The partitioned solve itself runs in
tests/test_gpu_solver.py (local partitions on one GPU vs the unpartitioned
solve)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_handles_and_row_ranges():
    from paper_2512_12151_b200 import dist
    for parts, n in ((1, 10), (2, 1089), (3, 40_000), (8, 904_562)):
        p = dist.Partition.local_parts(parts)
        rr = p.row_ranges(n)
        assert len(rr) == parts and rr[0][0] == 0 and rr[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))            # contiguous, in rank order
        assert all(r0 % 32 == 0 for r0, _ in rr)                        # 32-row aligned chunks
    with pytest.raises(ValueError):
        dist.Partition.local_parts(0)
    # world 1 needs no NCCL communicator
    one = dist.Partition.nccl(0, 1, bytes(128))
    assert one.world == 1 and not one.local
    with pytest.raises(ValueError):
        dist.Partition.nccl(0, 2, b"short")


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_12151_b200 import dist as pdist
    uid = pdist.broadcast_id()
    out.put((rank, uid))
    dist.destroy_process_group()


def test_unique_id_broadcast_world2_gloo():
    """Rank 0's NCCL unique id reaches every rank unchanged (what
    Partition.from_torch feeds ncclCommInitRank)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1]
