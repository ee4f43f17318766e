"""Scene-parallel batch sharding (C5) over a world-size-2
gloo process group on CPU: every seed runs exactly once, on the rank the
round-robin assigns, and rank 0 receives all records in seed order.  The
scene runner is injected (the GPU path is exercised by bench.py --workload c5)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_runner(seed, frames):
    from paper_2512_12151_b200.batch import SceneRecord
    return SceneRecord(seed=seed, rank=-1, frames=frames, passes=seed % 3 + 1, newton=2 * seed, cg=7 * seed,
                       device_ms=1.0, checksum=float(seed) * 0.5)


def _worker(rank, world, port, seeds, frames, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_12151_b200.batch import run_batch
    res = run_batch(seeds, frames, runner=_fake_runner)
    if rank == 0:
        records, walls = res
        out.put([(r.seed, r.rank, r.frames, r.newton, r.cg, r.checksum) for r in records] + [len(walls)])
    else:
        assert res is None
    dist.destroy_process_group()


def test_shard_round_robin():
    from paper_2512_12151_b200.batch import shard
    seeds = list(range(10))
    parts = [shard(seeds, r, 4) for r in range(4)]
    assert parts[0] == [0, 4, 8] and parts[3] == [3, 7]
    assert sorted(s for p in parts for s in p) == seeds
    with pytest.raises(ValueError):
        shard(seeds, 4, 4)


def test_batch_gather_world2_gloo():
    world, seeds, frames = 2, list(range(9)), 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[-1] == world
    recs = got[:-1]
    assert [r[0] for r in recs] == seeds                    # each seed once, seed order
    assert all(r[1] == r[0] % world for r in recs)          # ran on its round-robin rank
    assert all(r[2] == frames and r[3] == 2 * r[0] and r[4] == 7 * r[0] for r in recs)
