"""Benchmark: ms/frame on the C4 squishy-ball compression scene (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 112]

One "step" is one frame (= one Simulation.advance, intact/cli.py:98-116) of
the 2.22M-tet five-ball compression scene (solid-ball
proxy — see paper_2512_12151_b200/scenes.py and DESIGN.md).  The press runs
--precompress untimed frames first (default 50: the stack is squeezed to
~40 % of its height, 20-30k active constraints, ~20 Newton iterations per
frame), then W untimed warm-up frames, then K timed frames.  Per timed frame the inputs (x, v) are copied
host->device from pinned memory, the frame runs through the public
Simulation/step path, and (x, v) are copied back; `value` is the device time
of the frame proper (inputs resident), `e2e` the whole bracket including the
copies.  The matrix alone is ~0.5 GB, far above the 126 MB L2, so no flush
is needed between frames.

Multi-GPU (torchrun): a single scene does not shard in this round, so each
rank runs an independent replica ("replicas only"); value = max
over ranks of the timed region / (N*K) frames, scaling "weak".

--impl reference times the reference's CPU algorithm (the oracle
restatement, oracle/) on the host cores: unit costs of its hot-path stages
(assemble, PCG iteration, energy, CCD pass) measured on one reduced shell,
scaled to the C4 size and to the per-frame operation counts.
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
PLATE_SPEED = 0.5   # m/s: 5 mm per frame
PLATE_STOP = 0.05   # m: the press holds once its underside reaches this height (stack 0.345 m tall)
PAPER_COUNTS = {"newton": 30.09, "cg": 30.09 * 28.35, "passes": 30.09, "energy": 30.09 * 1.5,
                "source": "PAPER.md:694 (Newton 30.09/frame, CG 28.35/solve); passes and energy evals assumed"}


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

def reference_unit_costs(n_sample=16, seed=0):
    """Time the reference algorithm's stages (oracle restatement) on one
    ball of resolution n_sample, in a strained configuration."""
    from oracle import blocksparse, geometry, newton
    from paper_2512_12151_b200 import scenes
    ball = scenes.shell_sphere(n_sample, 0.1, layers=(n_sample + 1) // 2)
    from paper_2512_12151_b200.mesh import compute_rest_data
    rest = compute_rest_data(ball, 1e2)
    from paper_2512_12151_b200.elasticity import Material, MaterialModel
    mat = Material(MaterialModel.COR, 1e4, 0.4)
    R = [("cor", mat.mu, mat.lam, ball.tets, rest.shape_rows, rest.volumes)]
    rng = np.random.default_rng(seed)
    x = ball.rest_positions * np.array([1.0, 1.0, 0.97])          # squashed: nonzero elastic forces
    x_tilde = ball.rest_positions + 1e-4 * rng.standard_normal(x.shape)
    h = 0.01
    t = time.perf_counter()
    g, H = newton.assemble(x, x_tilde, rest.masses, R, None, 1.0, 1e-3, h)
    t_asm = time.perf_counter() - t
    t = time.perf_counter()
    _, its, _, _ = blocksparse.pcg(H, -g, 1e-12, max_iters=20)
    t_cg = (time.perf_counter() - t) / max(its, 1)
    t = time.perf_counter()
    newton.energy(x, x_tilde, rest.masses, R, None, 1.0, 1e-3, h)
    t_en = time.perf_counter() - t
    x_hat = x + 2e-3 * rng.standard_normal(x.shape)
    t = time.perf_counter()
    geometry.step_limit(x, x_hat, ball.surface_tris, ball.surface_edges, ball.surface_verts, 1e-4)
    t_ccd = time.perf_counter() - t
    return {"assemble_s": t_asm, "cg_iter_s": t_cg, "energy_s": t_en, "ccd_pass_s": t_ccd,
            "tets": int(ball.n_tets), "blocks": int(len(H.rows)), "tris": int(len(ball.surface_tris)),
            "n_sample": n_sample}


def reference_ms_per_frame(units, full, counts):
    """Scale sampled unit costs to the full scene and per-frame op counts."""
    st = units["tets"] / 1.0
    s_asm = full["tets"] / st
    s_cg = full["blocks"] / units["blocks"]
    s_ccd = full["tris"] / units["tris"]
    asm = units["assemble_s"] * s_asm * (counts["newton"] + 1.0)      # + mu-init assembly per frame
    cg = units["cg_iter_s"] * s_cg * counts["cg"]
    en = units["energy_s"] * s_asm * counts["energy"]
    ccd = units["ccd_pass_s"] * s_ccd * counts["passes"]
    return 1e3 * (asm + cg + en + ccd), {"assemble_ms": 1e3 * asm, "pcg_ms": 1e3 * cg, "energy_ms": 1e3 * en,
                                         "ccd_ms": 1e3 * ccd}


def _full_sizes(n):
    """Five solid n-balls (Kuhn grid): tets, surface tris, vertices."""
    return {"tets": 5 * 6 * n ** 3, "tris": 5 * 12 * n * n, "verts": 5 * (n + 1) ** 3}


def workload(args):
    """The config.workload string shared by both arms (same scene, same frames)."""
    full = _full_sizes(args.n)
    first = args.precompress + args.warmup
    return (f"C4 five COR balls n={args.n} ({full['tets']} ball tets, {full['verts']} ball vertices) pressed by a "
            f"plate at {PLATE_SPEED} m/s down to {PLATE_STOP} m; timed frames {first}..{first + args.steps - 1}")


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    counts, src = PAPER_COUNTS, PAPER_COUNTS["source"]
    try:
        with open(COUNTS) as f:
            c = json.load(f)
        counts = {k: float(c[k]) for k in ("newton", "cg", "passes", "energy")}
        src = f"per-frame op counts of the GPU run recorded in {os.path.relpath(COUNTS, ROOT)}"
    except Exception:
        pass
    full = _full_sizes(args.n)
    vals = []
    units = None
    for k in range(args.warmup + args.steps):
        units = reference_unit_costs(args.sample_n, seed=k)
        full["blocks"] = units["blocks"] * full["tets"] / units["tets"]
        ms, parts = reference_ms_per_frame(units, full, counts)
        if k >= args.warmup:
            vals.append(ms)
    value = float(np.mean(vals))
    sample = (f"oracle (numpy restatement of intact) stage costs on one n={args.sample_n} shell "
              f"({units['tets']} tets), scaled to C4 ({full['tets']} tets) and {src}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "ms/frame", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args), "parallelism": "one host core (numpy, single-threaded "
                                                                 "like the reference, SPEC.md:587)"},
            "cpu_baseline": {"value": value, "unit": "ms/frame", "cores": 1, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "ms/frame", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "phases_ms": parts}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2512_12151_b200 import _lib, scenes
    from paper_2512_12151_b200.device import to_host
    from paper_2512_12151_b200.stepper import step_device
    from paper_2512_12151_b200.contact import ActiveSet
    import ctypes as C

    t_setup = time.perf_counter()
    system, state, params = scenes.c4_scene(n=args.n, plate_speed=PLATE_SPEED, plate_stop=PLATE_STOP)
    dev = system.device
    ccd = system.ccd
    aset = ActiveSet()
    aset.ensure(system.n_vertices)
    n = system.n_vertices
    x = torch.from_numpy(state.x).cuda()
    v = torch.from_numpy(state.v).cuda()
    setup_s = time.perf_counter() - t_setup
    L = _lib.lib()
    k = 0
    # untimed press to the contact-heavy regime, then the warm-up frames
    for _ in range(args.precompress + args.warmup):
        x, v, _ = step_device(x, v, system, aset, params, step_index=k)
        k += 1
    torch.cuda.synchronize()
    stats = np.zeros(9)
    cst = np.zeros(3)
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 1)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 1)
    x_pin = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    v_pin = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    x_pin.copy_(x)
    v_pin.copy_(v)
    x_dev = torch.empty_like(x)
    v_dev = torch.empty_like(v)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    newton = cg = passes = 0
    n_constraints, pass_ms = [], []
    cert = []
    mon_launches = 0
    launches0 = L.ibf_launch_count()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
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
            l0 = L.ibf_launch_count()
            dmin, _, _ = ccd.min_distance(xn, params.offset)
            n_hits, _ = ccd.static_intersections(xn, cap=16)
            cert.append((dmin, n_hits))
            mon_launches += L.ibf_launch_count() - l0
            newton += sum(r.newton_iters for r in diag.iterations)
            cg += sum(r.cg_iters for r in diag.iterations)
            passes += len(diag.iterations)
            n_constraints.append(max(r.n_constraints for r in diag.iterations))
            pass_ms.append(max(r.wall_ms for r in diag.iterations))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    launches = L.ibf_launch_count() - launches0 - mon_launches
    frame_ms = [e[1].elapsed_time(e[2]) for e in evs]
    e2e_ms = [e[0].elapsed_time(e[3]) for e in evs]
    tot_dev, tot_e2e = float(np.sum(frame_ms)), float(np.sum(e2e_ms))
    if ws > 1:
        t = torch.tensor([tot_dev, tot_e2e], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_dev, tot_e2e = float(t[0]), float(t[1])
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 0)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 0)
    frames = ws * args.steps
    value = tot_dev / frames
    e2e = tot_e2e / frames
    # roofline of the PCG (persistent SpMV + vector kernel): algorithmic bytes
    spmv_bytes = dev.spmv_bytes()
    pcg_ms, pcg_iters, contact_iter_terms = stats[2], stats[4], stats[8]
    pcg_bytes = pcg_iters * (spmv_bytes + 288.0 * n) + 120.0 * contact_iter_terms
    achieved = pcg_bytes / (pcg_ms * 1e-3) / 1e9 if pcg_ms > 0 else 0.0
    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(NCU_SUMMARY) as f:
            # dram__bytes_read.sum + dram__bytes_write.sum per CG iteration of
            # k_pcg from the committed ncu capture (profiles/ncu_summary.json)
            traffic = json.load(f)["k_pcg"]["dram_bytes_per_cg_iter"]
    except Exception:
        pass
    phases = {"assembly_ms": stats[0] / args.steps, "pcg_ms": stats[2] / args.steps,
              "line_search_ms": stats[5] / args.steps, "inversion_cap_ms": stats[7] / args.steps,
              "ccd_ms": cst[0] / args.steps}
    phases["other_ms"] = value - sum(phases.values())
    counts = {"newton": newton / args.steps, "cg": cg / args.steps, "passes": passes / args.steps,
              "energy": stats[6] / args.steps}
    line = {"metric": METRIC, "value": value, "unit": "ms/frame", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False, "scaling": "weak",
            # value / the paper's 5,367 ms/frame (RTX 4090, FP64, the authors' own mesh;
            # this is the solid-ball proxy of the same 2.2M-tet press scene)
            "vs_baseline": round(value / 5367.0, 4) if value > 0 else None,
            "vs_baseline_note": "value / 5367 ms/frame (paper Table 1, RTX 4090); lower is better; proxy scene",
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args), "system": f"{sum(len(r.tets) for r in system.regions)} tets, "
                                                            f"{n} vertices incl. the two pinned plates",
                       "parallelism": "replicas" if ws > 1 else "single-gpu",
                       "l2": "inputs > L2 (matrix ~%.0f MB)" % (spmv_bytes / 1e6)},
            "ms_per_newton_iter": value * args.steps / max(newton, 1),
            "newton_per_frame": counts["newton"], "cg_per_frame": counts["cg"], "passes_per_frame": counts["passes"],
            "peak_constraints": int(max(n_constraints)), "phases_ms": phases,
            "roofline": {"kernel": "k_pcg (symmetric BSR SpMV + block-Jacobi vector phase)", "bound": "hbm",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_source": peak_kind, "traffic": traffic, "traffic_unit": "bytes per CG iteration",
                         "bytes_per_cg_iter": spmv_bytes + 288.0 * n},
            "spmv_GBps": achieved,
            "e2e": {"value": e2e, "unit": "ms/frame", "h2d_bytes_per_step": 2 * 24 * n,
                    "d2h_bytes_per_step": 2 * 24 * n},
            "gpu_launches": int(launches), "frames_ms": [round(t, 1) for t in frame_ms],
            "slowest_pass_wall_ms": [round(t, 1) for t in pass_ms], "wall_s": wall, "setup_s": setup_s,
            "penetration_free": {"frames_checked": len(cert),
                                 "min_distance": min(c[0] for c in cert) if cert else None,
                                 "intersecting_triangle_pairs": max(c[1] for c in cert) if cert else None,
                                 "how": "every timed frame: nearest non-adjacent VF/EE pair within the contact "
                                        "offset (ibf_min_distance) and the reference's static tri-tri test "
                                        "(ibf_static_intersection), outside the timed region"}}
    if rank == 0:
        line["clocks"] = clocks.summary()
        if not args.no_cpu_baseline:
            os.makedirs(os.path.dirname(COUNTS), exist_ok=True)
            try:
                with open(COUNTS, "w") as f:
                    json.dump(dict(counts, n=args.n, source="bench.py GPU run"), f, indent=1)
            except OSError:
                pass
            full = _full_sizes(args.n)
            units = reference_unit_costs(args.sample_n)
            full["blocks"] = units["blocks"] * full["tets"] / units["tets"]
            ms, parts = reference_ms_per_frame(units, full, counts)
            line["cpu_baseline"] = {"value": ms, "unit": "ms/frame", "cores": 1, "kind": "port",
                                    "sample": f"oracle stage costs on one n={args.sample_n} shell scaled to C4 and "
                                              f"to this run's per-frame op counts", "phases_ms": parts}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


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
    ap.add_argument("--n", type=int, default=42, help="ball resolution (42 -> 2.22M tets)")
    ap.add_argument("--precompress", type=int, default=50,
                    help="untimed frames of the press before warm-up (reaches the contact-heavy regime)")
    ap.add_argument("--sample-n", type=int, default=24,
                    help="ball resolution of the CPU baseline sample (24: 83k tets, ~10 s of numpy per sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c4", choices=["c4", "c5"],
                    help="c4: the headline press scene (default); c5: scene-parallel batch of drops")
    ap.add_argument("--scenes", type=int, default=64, help="c5: number of scenes in the batch")
    ap.add_argument("--concurrency", type=int, default=8,
                    help="c5: scenes in flight per GPU (host threads, one CUDA stream each)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
