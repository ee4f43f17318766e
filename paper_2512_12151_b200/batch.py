"""Scene-parallel batches: independent scenes
sharded across ranks, one process per GPU, no collective on the data path.

Scenes couple nothing — alpha, beta, mu and the Newton loop are per scene
(intact/stepper.py:242-371) — so a batch of S scenes over W ranks is S/W
independent `Simulation` runs per rank.  Stacking scenes into one System would
couple them through the global alpha and change every result, so each scene
keeps its own device handles.  The only communication is one gather of the
per-scene records to rank 0 at the end (`torch.distributed.gather_object`,
NCCL or gloo).
"""

from __future__ import annotations

import dataclasses
import time
from typing import Callable, Optional, Sequence


@dataclasses.dataclass
class SceneRecord:
    seed: int
    rank: int
    frames: int
    passes: int
    newton: int
    cg: int
    device_ms: float
    checksum: float          # sum of final positions, a cheap determinism probe
    aborted: bool = False


def shard(seeds: Sequence[int], rank: int, world: int) -> list:
    """Round-robin assignment: rank r runs seeds[r], seeds[r + W], ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return list(seeds)[rank::world]


def run_scene(seed: int, frames: int, make_scene: Optional[Callable] = None) -> SceneRecord:
    """Run one C5 scene for `frames` steps on the current CUDA device."""
    import torch
    from . import scenes
    from .stepper import Simulation, StepAbortError
    make_scene = make_scene or scenes.c5_scene
    system, state, params = make_scene(seed)
    sim = Simulation(system, params, state)
    passes = newton = cg = 0
    aborted = False
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(frames):
        try:
            d = sim.advance()
        except StepAbortError:
            aborted = True
            break
        passes += len(d.iterations)
        newton += sum(r.newton_iters for r in d.iterations)
        cg += sum(r.cg_iters for r in d.iterations)
    end.record()
    torch.cuda.synchronize()
    x = sim.state.x
    return SceneRecord(seed, 0, frames, passes, newton, cg, start.elapsed_time(end), float(x.sum()), aborted)


def _run_concurrent(seeds, frames, runner, concurrency):
    """Scenes of one GPU on `concurrency` host threads, each with its own CUDA
    stream: small scenes are latency-bound (a few
    hundred launches and a host sync per Newton iteration), so several in
    flight fill the GPU.  The native calls release the GIL (ctypes), handles
    are per scene, and the library's shared counters are atomic."""
    import threading
    from concurrent.futures import ThreadPoolExecutor
    import torch
    local = threading.local()

    def work(seed):
        if not hasattr(local, "stream"):
            local.stream = torch.cuda.Stream()
        with torch.cuda.stream(local.stream):
            return runner(seed, frames)

    with ThreadPoolExecutor(max_workers=concurrency) as ex:
        return list(ex.map(work, seeds))


def run_batch(seeds: Sequence[int], frames: int, runner: Optional[Callable] = None, group=None,
              concurrency: int = 1):
    """Run this rank's shard of `seeds` (`concurrency` scenes in flight per
    GPU); rank 0 returns every record sorted by seed, other ranks return
    None.  Without an initialised process group the whole batch runs here."""
    import torch.distributed as dist
    runner = runner or run_scene
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    t0 = time.perf_counter()
    mine_seeds = shard(seeds, rank, world)
    if concurrency > 1:
        mine = _run_concurrent(mine_seeds, frames, runner, concurrency)
    else:
        mine = [runner(seed, frames) for seed in mine_seeds]
    for rec in mine:
        rec.rank = rank
    wall = time.perf_counter() - t0
    if not dist_on:
        return sorted(mine, key=lambda r: r.seed), [wall]
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((mine, wall), gathered, dst=0, group=group)
    if rank != 0:
        return None
    records = [r for part, _ in gathered for r in part]
    return sorted(records, key=lambda r: r.seed), [w for _, w in gathered]
