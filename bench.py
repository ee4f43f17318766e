"""Benchmark: ms/frame on the C4 squishy-ball compression scene (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c4ball|c5] [--precompress P] [--cell 0.02] [--plate-speed 2.0]

One "step" is one frame (= one Simulation.advance, intact/cli.py:98-116) of
the C4 scene: five squishy balls (scenes.squishy_scene: 2.30M tets, 0.90M
vertices, 1.62M surface triangles — the paper's 2.25M / 0.87M / 1.59M,
PAPER.md:810) in a pinned box under gravity, pressed by a scripted plate.
The press runs --precompress untimed frames first (default 40: the stack is
in dense multi-body contact, >1e5 active constraints), then W untimed
warm-up frames, then K timed frames.  Per timed frame the inputs (x, v) are
copied host->device from pinned memory, the frame runs through the public
step path, and (x, v) are copied back; `value` is the device time of the
frame proper (inputs resident), `e2e` the whole bracket including the
copies.  The matrix alone is ~0.6 GB, far above the 126 MB L2, so no flush
is needed between frames.

--workload c4ball is the round-1 solid-ball proxy (same tet count, 0.40M
vertices, 0.11M surface triangles); --workload c5 the scene-parallel batch.

Multi-GPU (torchrun): by default one scene with its PCG rows split over the
ranks (--mode partition: NCCL allreduce / allgather inside each CG
iteration, assembly / CCD / line search replicated, "scaling": "strong",
DESIGN.md §(e)); --mode replicas runs one scene per rank instead (value = the
slowest rank's ms/frame, `replica_scene_frames_per_s` their throughput).

--impl reference times the reference's CPU path as the oracle port (oracle/,
single-threaded numpy) on bounded samples of the same scene
(oracle/stage_timing.py); see run_reference.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import threading
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/frame and ms/Newton iter (squishy balls 2.25M tets); PCG SpMV HBM GB/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
COUNTS = os.path.join(ROOT, "profiles", "c4_frame_counts.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
PAPER_COUNTS = {"newton": 30.09, "cg": 30.09 * 28.35, "passes": 30.09, "energy": 30.09 * 1.5,
                "source": "PAPER.md:694 (Newton 30.09/frame, CG 28.35/solve); passes and energy evals assumed"}


def _fp64_peak():
    """Measured FP64 FMA throughput (TFLOP/s) from MEASURED_PEAKS.json or the
    committed tools/micro/fp64_peak run, else None."""
    for path, key in ((PEAKS, "fp64_tflops"), (os.path.join(ROOT, "profiles", "fp64_peak.json"), "fp64_tflops")):
        try:
            with open(path) as f:
                return float(json.load(f)[key])
        except Exception:
            pass
    return None


def _peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Clocks and throttle reasons sampled DURING the timed region.

    Modes (IBF_BENCH_CLOCKS): "spawn" (default) runs one nvidia-smi per
    sample, 0.2 s apart; "nvml" queries NVML (the library nvidia-smi reads)
    from a thread of this process; "lms" keeps one `nvidia-smi -lms 200`
    running (the profiling recipe's clocks line); "off".  The frame's
    host-driven share ("other_ms": the GPU waiting on the Newton loop's host
    logic) is sensitive to the box: A/B on one box over 2 runs each gave
    other_ms 32/38 (spawn), 173/140 (nvml), 61/271 (off), and 40/18 (spawn)
    vs 103/262 (lms) on another; the kernel phases do not move."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, mode=None, period=0.2):
        self.index, self.samples, self.proc = index, [], None
        self.mode = mode or os.environ.get("IBF_BENCH_CLOCKS", "spawn")
        self.period = period
        self.stop = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _nvml_sample(self, nv, h):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        return [str(sm), str(smax)] + ["Active" if r & b else "Not Active" for b in bits]

    def _run(self):
        if self.mode == "nvml":
            try:
                import pynvml as nv
                nv.nvmlInit()
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            except Exception:
                return
            while not self.stop.is_set():
                try:
                    self.samples.append(self._nvml_sample(nv, h))
                except Exception:
                    pass
                self.stop.wait(self.period)
            nv.nvmlShutdown()
            return
        while not self.stop.is_set():     # "spawn"
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self.stop.wait(self.period)

    def __enter__(self):
        if self.mode == "lms":
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
        elif self.mode != "off":
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t.is_alive():
            self.t.join(timeout=10)
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=10)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in (out or "").splitlines():
            vals = [v.strip() for v in line.split(",")]
            if len(vals) == 6:
                self.samples.append(vals)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ CPU baseline

COUNT_KEYS = ("newton", "cg", "passes", "energy")


def _scene(args):
    from paper_2512_12151_b200 import scenes
    if args.workload == "c4ball":
        return scenes.c4_scene(n=args.n, plate_speed=0.5, plate_stop=0.05)
    return scenes.squishy_scene(cell=args.cell, plate_speed=args.plate_speed, numbering=args.numbering)


def workload(args):
    """The config.workload string shared by both arms (same scene, same frames)."""
    first = args.precompress + args.warmup
    frames = f"timed frames {first}..{first + args.steps - 1} after {first} untimed"
    if args.workload == "c4ball":
        return (f"C4 solid-ball proxy: five COR balls n={args.n} ({5 * 6 * args.n ** 3} ball tets) pressed by a "
                f"plate at 0.5 m/s down to 0.05 m; {frames}")
    return (f"C4 squishy balls: five COR squishy balls (hollow core + 600 strands each, scenes.squishy_scene "
            f"cell={args.cell} m: 2.30M tets, 0.90M vertices, 1.62M surface triangles; {args.numbering} vertex "
            f"numbering) in a pinned box, pressed by a plate at {args.plate_speed} m/s under gravity; {frames}")


def _oracle_counts(counts_path=None):
    """Per-frame op counts of the last committed GPU run of this workload."""
    try:
        with open(counts_path or COUNTS) as f:
            c = json.load(f)
        return {k: float(c[k]) for k in COUNT_KEYS}, f"per-frame op counts of the GPU run in {os.path.relpath(COUNTS, ROOT)}"
    except Exception:
        return ({k: float(v) for k, v in PAPER_COUNTS.items() if k in COUNT_KEYS}, PAPER_COUNTS["source"])


def cpu_sample(system, x, x_hat, x_tilde, mu, offset, h, slices, aset_state, counts, full_blocks):
    """Oracle stage times on the given ball slices (+ the full active set),
    scaled to the scene and multiplied by the per-frame op counts."""
    from oracle import stage_timing
    meas_tot, full_tot, infos = {}, {}, []
    for j, sl in enumerate(slices):
        meas, scale, full, info = stage_timing.time_sample(system, x, x_hat, x_tilde, mu, offset, h, sl,
                                                            aset_state if j == 0 else None,
                                                            full_blocks=full_blocks, contacts=(j == 0))
        for k, v in meas.items():
            meas_tot[k] = meas_tot.get(k, 0.0) + v
        for k, v in full.items():
            # slice stages: mean over slices; full-set contact stages: once
            full_tot[k] = full_tot.get(k, 0.0) + (v / len(slices) if scale[k] != 1.0 or k == "cg_setup" else v)
        infos.append(info)
    ms, parts = stage_timing.frame_ms(full_tot, counts)
    return ms, parts, meas_tot, full_tot, infos


def _oracle_c5_scene(job):
    """One C5 scene on the oracle (a pool worker): (seed, frames) -> (frames done, s)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    seed, frames = job
    from oracle import contact as ocontact, timestep
    from paper_2512_12151_b200 import scenes
    system, state, params = scenes.c5_scene(seed)
    regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
               for r in system.regions]
    scene = timestep.Scene(system.masses, regions, system.surface_triangles, system.surface_edges,
                           system.surface_vertices, [(bc.vertices, None) for bc in system.boundary])
    x, v = state.x.copy(), state.v.copy()
    aset = ocontact.ConstraintSet()
    t = time.perf_counter()
    done = 0
    for k in range(frames):
        try:
            x, v, _, _, _ = timestep.step(x, v, scene, aset, h=params.h, offset=params.offset,
                                          k_min=params.min_iterations, step_index=k)
        except timestep.Aborted:
            break
        done += 1
    return done, time.perf_counter() - t


def run_reference_c5(args):
    """--impl reference --workload c5: the oracle port of the reference on a
    process pool with one single-threaded process per host core, one scene
    per process; each step runs one frame of `cores`
    scenes (seeds dealt in order), so a step is bounded by the slowest of
    them.  value = scene-frames / wall over the timed steps."""
    import multiprocessing as mp
    ws, rank, _ = _dist()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    seeds = list(range(args.scenes))
    ctx = mp.get_context("fork")
    frames_done, walls = 0, []
    with ctx.Pool(cores) as pool:
        for k in range(args.warmup + args.steps):
            batch = [(seeds[(k * cores + j) % len(seeds)], 1) for j in range(cores)]
            t = time.perf_counter()
            res = pool.map(_oracle_c5_scene, batch)
            w = time.perf_counter() - t
            if k >= args.warmup:
                walls.append(w)
                frames_done += sum(r[0] for r in res)
    value = frames_done / max(sum(walls), 1e-9)
    sample = (f"oracle (numpy port of intact) on a {cores}-process pool (one single-threaded process per host "
              f"core); each step = frame 0 of {cores} C5 scenes (seeds dealt round-robin), {args.steps} timed steps")
    line = {"impl": "reference", "metric": "C5 scene-frames/s (64 randomized NH drops, scene-parallel)",
            "value": value, "unit": "scene-frames/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(walls)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5: {args.scenes} C1-like drops (seeded jitter)",
                       "parallelism": f"process pool x{cores} host cores"},
            "cpu_baseline": {"value": value, "unit": "scene-frames/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "scene-frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _full_size_check():
    """The committed one-off timing of the oracle's stages at the full C4
    size against the same slice extrapolation (tools/oracle_full_stages.py):
    how far the model is from a measurement, stage by stage."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_oracle_full_stages.json")) as f:
            d = json.load(f)
        return {"source": "profiles/r2_oracle_full_stages.json", "measured_full_s": d["measured_full_s"],
                "extrapolated_over_measured": d["ratio_extrapolated_over_measured"]}
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the oracle port of the reference's CPU path (oracle/,
    single-threaded numpy like the reference), no GPU.  Each step times one
    bounded sample of the same scene at its first frame (the rest state, the
    plate's first-frame Dirichlet target, gravity): a 1/8 slice of one ball
    (assembly, CG iterations, energy, CCD over the slice's surface), scaled to
    the scene and multiplied by the per-frame op counts of the committed GPU
    run of this workload (profiles/c4_frame_counts.json)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import stage_timing
    from paper_2512_12151_b200.stepper import apply_dbc
    system, state, params = _scene(args)
    counts, src = _oracle_counts()
    h = params.h
    x = state.x
    x_tilde = x + h * state.v + (h * h) * np.asarray(params.gravity, dtype=np.float64)
    x_hat = x.copy()
    apply_dbc(x_hat, system.boundary, x, 0)
    mu = params.stiffness_constant * 1.0          # any positive mu: the stage costs do not depend on it
    slices = stage_timing.ball_slices(system, 8)
    vals, walls, parts_all = [], [], []
    for k in range(args.warmup + args.steps):
        t = time.perf_counter()
        ms, parts, meas, full, infos = cpu_sample(system, x, x_hat, x_tilde, mu, params.offset, h,
                                                  [slices[k % len(slices)]], None, counts, None)
        walls.append(time.perf_counter() - t)
        if k >= args.warmup:
            vals.append(ms)
            parts_all.append(parts)
    value = float(np.mean(vals))
    parts = {k: float(np.mean([p[k] for p in parts_all])) for k in parts_all[0]}
    sample = (f"oracle (numpy port of intact, 1 thread) per step: one 1/8 slice of one ball (~57k of 2.30M tets) at "
              f"the first frame — elastic assembly, CG iterations, energy, CCD pass over the slice's surface — "
              f"scaled to the scene (tets / stored blocks / surface triangles) and to {src}; "
              f"no constraints exist at the first frame, so contact-stage costs are not in this arm")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "ms/frame", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args), "parallelism": "one host core (numpy, single-threaded like "
                                                                 "the reference, SURVEY.md §8(d))"},
            "cpu_baseline": {"value": value, "unit": "ms/frame", "cores": 1, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "ms/frame", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "phases_ms": parts, "op_counts_per_frame": counts,
            "sample_wall_s": {"mean": float(np.mean(walls)), "total": float(np.sum(walls))},
            "extrapolation": "ms/frame = sum over stages of (sample stage time x scene/sample size) x per-frame "
                             "op count; the sampled stage times are measured, the multiplication is the model",
            "full_size_check": _full_size_check(),
            "spread_ms": {"min": float(np.min(vals)), "max": float(np.max(vals))}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def _kernel_rooflines(clocks, peak_hbm, peak_fp64):
    """Per-kernel achieved algorithmic GB/s (and FP64 TFLOP/s where counted)
    over the timed region, from ibf_kernel_clocks (events on the launching
    stream around each instrumented launch)."""
    out = {}
    for name, c in clocks.items():
        if c["launches"] <= 0 or c["ms"] <= 0:
            continue
        gbs = c["bytes"] / (c["ms"] * 1e-3) / 1e9
        row = {"launches": int(c["launches"]), "ms": round(c["ms"], 3), "avg_us": 1e3 * c["ms"] / c["launches"],
               "GBps": gbs, "hbm_frac": gbs / peak_hbm, "units": c["units"]}
        if c["flops"] > 0:
            tf = c["flops"] / (c["ms"] * 1e-3) / 1e12
            row.update(TFLOPs=tf, fp64_frac=tf / peak_fp64 if peak_fp64 else None)
        out[name] = row
    return out


def _partition_probe(dev, system, state, params, part):
    """One PCG solve of the scene's rest-state system through the NCCL
    partition against the single-GPU kernel, before anything is timed: the
    two must agree to 1e-10 (tests/test_gpu_solver.py holds the same bar for
    local partitions); raises otherwise, and the caller falls back to
    replicas."""
    import torch
    from paper_2512_12151_b200.device import empty
    n, h = system.n_vertices, params.h
    x = torch.from_numpy(state.x).cuda()
    v = torch.from_numpy(state.v).cuda()
    x_tilde = x + h * v
    g = empty((n, 3))
    dev.assemble(None, x, x_tilde, 1.0, params.offset, h, True, g)
    rhs = -g
    a, b = empty((n, 3)), empty((n, 3))
    dev.set_dist(None)
    it1, _, _ = dev.pcg(rhs, a, params.cg_tol)
    dev.set_dist(part)
    it2, _, _ = dev.pcg(rhs, b, params.cg_tol)
    dev.set_dist(None)
    torch.cuda.synchronize()
    scale = float(a.abs().max()) or 1.0
    err = float((a - b).abs().max()) / scale
    if abs(it1 - it2) > 1 or not err <= 1e-10:
        raise RuntimeError(f"partition probe: CG {it2} vs {it1}, max rel diff {err:.2e}")


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2512_12151_b200 import _lib
    from paper_2512_12151_b200.stepper import step_device
    from paper_2512_12151_b200.contact import ActiveSet

    t_setup = time.perf_counter()
    system, state, params = _scene(args)
    dev = system.device
    ccd = system.ccd
    # N > 1: one scene, its PCG rows split over the ranks (NCCL allreduce /
    # allgather inside the solve, csrc/dist.cu); assembly, CCD and line search
    # run replicated on every rank (the ranks' states stay bit-identical).
    # --mode replicas runs N independent copies instead.
    mode = "single-gpu"
    part = None
    if ws > 1:
        mode = args.mode
        if mode == "partition":
            from paper_2512_12151_b200 import dist as pdist
            try:
                part = pdist.Partition.from_torch()
                _partition_probe(dev, system, state, params, part)
                dev.set_dist(part)
            except Exception as exc:      # no working NCCL partition: say so and run replicas
                dev.set_dist(None)
                part, mode = None, f"replicas (partition unavailable: {exc})"[:200]
    aset = ActiveSet()
    aset.ensure(system.n_vertices)
    n = system.n_vertices
    x = torch.from_numpy(state.x).cuda()
    v = torch.from_numpy(state.v).cuda()
    setup_s = time.perf_counter() - t_setup
    L = _lib.lib()
    k = 0
    # untimed press to the contact-heavy regime, then the warm-up frames
    t_pre = time.perf_counter()
    for _ in range(args.precompress + args.warmup):
        x, v, _ = step_device(x, v, system, aset, params, step_index=k)
        k += 1
    torch.cuda.synchronize()
    pre_s = time.perf_counter() - t_pre
    stats = np.zeros(9)
    cst = np.zeros(3)
    cnt = np.zeros(2)
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 1)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 1)
    L.ibf_system_counts(dev.handle, _lib.host_ptr(cnt), 1)
    _lib.kernel_clocks(on=1, reset=True)
    x_pin = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    v_pin = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    x_pin.copy_(x)
    v_pin.copy_(v)
    x_dev = torch.empty_like(x)
    v_dev = torch.empty_like(v)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    newton = cg = passes = 0
    n_constraints, pass_ms, triggers = [], [], 0
    cert = []
    mon_launches = 0
    launches0 = L.ibf_launch_count()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    prof_range = os.environ.get("IBF_BENCH_PROFILE_RANGE") == "1"   # ncu --profile-from-start off
    if prof_range:
        torch.cuda.profiler.start()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        for j in range(args.steps):
            e = evs[j]
            e[0].record()
            x_dev.copy_(x_pin, non_blocking=True)
            v_dev.copy_(v_pin, non_blocking=True)
            e[1].record()
            xn, vn, diag = step_device(x_dev, v_dev, system, aset, params, step_index=k)
            k += 1
            e[2].record()
            x_pin.copy_(xn, non_blocking=True)
            v_pin.copy_(vn, non_blocking=True)
            e[3].record()
            torch.cuda.synchronize()
            # penetration certificate of the accepted state, outside the timed
            # bracket (events e0..e3): nearest VF/EE pair within the contact
            # offset, and the reference's static tri-tri test (intersect.py)
            if not args.no_certify:
                l0 = L.ibf_launch_count()
                dmin, _, _ = ccd.min_distance(xn, params.offset)
                n_hits, _ = ccd.static_intersections(xn, cap=16)
                cert.append((dmin, n_hits))
                mon_launches += L.ibf_launch_count() - l0
            newton += sum(r.newton_iters for r in diag.iterations)
            cg += sum(r.cg_iters for r in diag.iterations)
            passes += len(diag.iterations)
            triggers += diag.adaptive_triggers
            n_constraints.append(max(r.n_constraints for r in diag.iterations))
            pass_ms.append(max(r.wall_ms for r in diag.iterations))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if prof_range:
        torch.cuda.profiler.stop()
    launches = L.ibf_launch_count() - launches0 - mon_launches
    kclocks = _lib.kernel_clocks(on=0)
    frame_ms = [e[1].elapsed_time(e[2]) for e in evs]
    e2e_ms = [e[0].elapsed_time(e[3]) for e in evs]
    tot_dev, tot_e2e = float(np.sum(frame_ms)), float(np.sum(e2e_ms))
    consistent = None
    if ws > 1:
        t = torch.tensor([tot_dev, tot_e2e], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_dev, tot_e2e = float(t[0]), float(t[1])
        if part is not None:
            # the partitioned solve hands every rank the same solution: the
            # ranks' final states must agree bit for bit
            ck = torch.tensor([float(xn.double().sum()), float(vn.double().sum())], dtype=torch.float64,
                              device="cuda")
            lo, hi = ck.clone(), ck.clone()
            torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
            torch.distributed.all_reduce(hi, op=torch.distributed.ReduceOp.MAX)
            consistent = bool(torch.equal(lo, hi))
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 0)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 0)
    L.ibf_system_counts(dev.handle, _lib.host_ptr(cnt), 0)
    # one scene per rank: the per-frame latency is the slowest rank's; the
    # replicas' throughput is reported apart (scene-frames/s)
    value = tot_dev / args.steps
    e2e = tot_e2e / args.steps
    # roofline of the PCG (persistent SpMV + vector kernel): algorithmic bytes
    spmv_bytes = dev.spmv_bytes()
    pcg_ms, pcg_iters, contact_iter_terms = stats[2], stats[4], stats[8]
    pcg_bytes = pcg_iters * (spmv_bytes + 288.0 * n) + 120.0 * contact_iter_terms
    achieved = pcg_bytes / (pcg_ms * 1e-3) / 1e9 if pcg_ms > 0 else 0.0
    peak, peak_kind = _peaks()
    peak_fp64 = _fp64_peak()
    traffic = None
    try:
        with open(NCU_SUMMARY) as f:
            # dram__bytes_read.sum + dram__bytes_write.sum per CG iteration of
            # k_pcg from the committed ncu capture of this workload
            traffic = json.load(f)["k_pcg"]["dram_bytes_per_cg_iter"]
    except Exception:
        pass
    phases = {"assembly_ms": stats[0] / args.steps, "pcg_ms": stats[2] / args.steps,
              "line_search_ms": stats[5] / args.steps, "inversion_cap_ms": stats[7] / args.steps,
              "ccd_ms": cst[0] / args.steps}
    phases["other_ms"] = value - sum(phases.values())
    counts = {"newton": newton / args.steps, "cg": cg / args.steps, "passes": passes / args.steps,
              "energy": cnt[1] / args.steps}
    line = {"metric": METRIC, "value": value, "unit": "ms/frame", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
            "scaling": "strong" if part is not None else "weak",
            # value / the paper's 5,367 ms/frame (RTX 4090, FP64, the authors' own mesh)
            "vs_baseline": round(value / 5367.0, 4) if value > 0 else None,
            "vs_baseline_note": "value / 5367 ms/frame (paper Table 1, RTX 4090, its own squishy-ball mesh); "
                                "lower is better; synthetic scene of the same V/F/T",
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args),
                       "system": f"{sum(len(r.tets) for r in system.regions)} tets, {n} vertices "
                                 f"({int(system.dbc_mask.sum())} pinned), {len(system.surface_triangles)} surface "
                                 f"triangles",
                       "parallelism": (f"row-partitioned PCG x{ws} (one scene; assembly, CCD and line search "
                                       f"replicated per rank)" if part is not None else
                                       f"replicas x{ws} (one scene per GPU): {mode}" if ws > 1 else "single-gpu"),
                       "l2": "inputs > L2 (matrix ~%.0f MB, no flush needed)" % (spmv_bytes / 1e6)},
            "ms_per_newton_iter": tot_dev / max(newton, 1),
            "newton_per_frame": counts["newton"], "cg_per_frame": counts["cg"], "passes_per_frame": counts["passes"],
            "cg_per_solve": cg / max(newton, 1), "stagnation_triggers": triggers,
            "constraints": {"peak": int(max(n_constraints)), "mean_of_frame_peaks": float(np.mean(n_constraints))},
            "phases_ms": phases,
            "ccd": {"candidates_per_frame": cst[2] / args.steps, "passes_per_frame": cst[1] / args.steps,
                    "candidate_pairs_per_s": cst[2] / (cst[0] * 1e-3) if cst[0] > 0 else None},
            "roofline": {"kernel": "k_pcg (symmetric BSR SpMV + block-Jacobi vector phase + matrix-free contact)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_source": peak_kind, "traffic": traffic, "traffic_unit": "bytes per CG iteration",
                         "bytes_per_cg_iter": spmv_bytes + 288.0 * n},
            "kernels": _kernel_rooflines(kclocks, peak, peak_fp64),
            "fp64_peak_tflops": peak_fp64,
            "spmv_GBps": achieved,
            "e2e": {"value": e2e, "unit": "ms/frame", "h2d_bytes_per_step": 2 * 24 * n,
                    "d2h_bytes_per_step": 2 * 24 * n},
            "gpu_launches": int(launches), "frames_ms": [round(t, 1) for t in frame_ms],
            "frames_constraints": n_constraints,
            "slowest_pass_wall_ms": [round(t, 1) for t in pass_ms], "wall_s": wall, "setup_s": setup_s,
            "precompress_s": pre_s}
    if ws > 1 and part is None:
        line["replica_scene_frames_per_s"] = ws * args.steps / (tot_dev * 1e-3)
    if consistent is not None:
        line["ranks_bit_identical"] = consistent
    if cert:
        line["penetration_free"] = {
            "frames_checked": len(cert), "min_distance": min(c[0] for c in cert),
            "intersecting_triangle_pairs": max(c[1] for c in cert),
            "how": "every timed frame: nearest non-adjacent VF/EE pair within the contact offset "
                   "(ibf_min_distance) and the reference's static tri-tri test (ibf_static_intersection), "
                   "outside the timed region"}
    if rank == 0:
        line["clocks"] = clocks.summary()
        if not args.no_cpu_baseline and args.workload == "c4":
            os.makedirs(os.path.dirname(COUNTS), exist_ok=True)
            try:
                with open(COUNTS, "w") as f:
                    json.dump(dict(counts, cell=args.cell, plate_speed=args.plate_speed, frames=workload(args),
                                   source="bench.py GPU run"), f, indent=1)
            except OSError:
                pass
            line["cpu_baseline"] = _cpu_baseline_leg(args, system, params, xn, vn, aset, counts, dev, k)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _cpu_baseline_leg(args, system, params, x, v, aset, counts, dev, step_index):
    """The oracle on a bounded sample of the state the timed frames ended at:
    the first Newton iteration of the next frame (x_hat0 with the Dirichlet
    targets), half of one ball (4 of 8 slices) for the elastic and CCD stages,
    the whole active set for the contact stages."""
    from oracle import stage_timing
    from paper_2512_12151_b200.device import to_host
    from paper_2512_12151_b200.stepper import apply_dbc
    h = params.h
    xh, vh = to_host(x), to_host(v)
    x_tilde = xh + h * vh + (h * h) * np.asarray(params.gravity, dtype=np.float64)
    mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, h)
    x_hat = xh.copy()
    apply_dbc(x_hat, system.boundary, xh, step_index)
    # a trial point the Newton step would visit: half way to the inertial target
    free = ~system.dbc_mask
    x_hat[free] = 0.5 * (xh[free] + x_tilde[free])
    slices = stage_timing.ball_slices(system, 8)[:4]
    t = time.perf_counter()
    ms, parts, meas, full, infos = cpu_sample(system, xh, x_hat, x_tilde, mu, params.offset, h, slices,
                                              aset.export_state(), counts, dev.n_blocks)
    wall = time.perf_counter() - t
    return {"value": ms, "unit": "ms/frame", "cores": 1, "kind": "port",
            "sample": (f"oracle (numpy port of intact, 1 thread) on the state the timed frames ended at: half of one "
                       f"ball ({sum(i['tets'] for i in infos)} of {infos[0]['tets_total']} tets) for assembly, CG "
                       f"iterations, energy and the CCD pass over its surface, scaled to the scene; the full active "
                       f"set ({infos[0]['constraints']} constraints) for the contact stages; times this run's "
                       f"per-frame op counts"),
            "phases_ms": parts, "stage_s_measured": meas, "stage_s_scene": full, "sample_wall_s": wall}


def run_c5(args):
    """Scene-parallel C5 batch: `--scenes` randomized
    drops sharded round-robin over the ranks, `--steps` frames each, no
    collective on the data path (batch.py).  value = scene-frames per second
    over the whole job (max-over-ranks wall of the timed region)."""
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2512_12151_b200 import _lib
    from paper_2512_12151_b200.batch import run_batch, run_scene
    for k in range(max(args.warmup, 1)):          # warm the library and allocator
        run_scene(10_000 + k, 1)
    L = _lib.lib()
    seeds = list(range(args.scenes))
    launches0 = L.ibf_launch_count()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_batch(seeds, args.steps, concurrency=args.concurrency)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    launches = L.ibf_launch_count() - launches0
    if ws > 1:
        t = torch.tensor([wall], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        wall = float(t[0])
    if rank == 0:
        records, _walls = res
        frames = sum(r.frames for r in records)
        value = frames / wall
        line = {"metric": "C5 scene-frames/s (64 randomized NH drops, scene-parallel)", "value": value,
                "unit": "scene-frames/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C5: {args.scenes} C1-like drops (seeded jitter), {args.steps} frames each, "
                                       "round-robin over ranks, no data-path collective",
                           "parallelism": f"scene-parallel x{ws}, {args.concurrency} scenes in flight per GPU"},
                "newton_per_frame": sum(r.newton for r in records) / max(frames, 1),
                "state_checksum": sum(r.checksum for r in records),
                "aborted": sum(r.aborted for r in records),
                "e2e": {"value": value, "unit": "scene-frames/s", "h2d_bytes_per_step": None,
                        "d2h_bytes_per_step": None, "note": "each scene runs through Simulation from host state"},
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cell", type=float, default=0.02, help="c4: squishy-ball cell edge (m)")
    ap.add_argument("--plate-speed", type=float, default=2.0, help="c4: plate speed (m/s)")
    ap.add_argument("--numbering", default="lattice", choices=["sell", "lattice", "morton"],
                    help="c4: squishy-ball vertex numbering (mesh.sell_numbering / lattice / Morton)")
    ap.add_argument("--n", type=int, default=42, help="c4ball: ball resolution (42 -> 2.22M tets)")
    ap.add_argument("--precompress", type=int, default=40,
                    help="untimed frames of the press before warm-up (reaches the contact-heavy regime)")
    ap.add_argument("--mode", default="partition", choices=["partition", "replicas"],
                    help="N > 1: row-partitioned PCG of one scene (strong scaling) or N independent replicas")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-certify", action="store_true", help="skip the per-frame penetration certificate")
    ap.add_argument("--workload", default="c4", choices=["c4", "c4ball", "c5"],
                    help="c4: the headline squishy-ball press (default); c4ball: the solid-ball proxy; "
                         "c5: scene-parallel batch of drops")
    ap.add_argument("--scenes", type=int, default=64, help="c5: number of scenes in the batch")
    ap.add_argument("--concurrency", type=int, default=8,
                    help="c5: scenes in flight per GPU (host threads, one CUDA stream each)")
    args = ap.parse_args()
    if args.impl == "reference":
        if args.workload == "c5":
            run_reference_c5(args)
        else:
            run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
