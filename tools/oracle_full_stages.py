"""Dev tool: the oracle's hot-path stages timed ONCE at the full C4 size —
the check on bench.py's reference-arm extrapolation (oracle/stage_timing.py
times 1/8 of one ball and scales by tets / stored blocks / surface
triangles).  Test infrastructure: runs the oracle (single-threaded numpy, as
the reference) on the squishy scene's first frame:

    python tools/oracle_full_stages.py [--out profiles/r2_oracle_full_stages.json]

Prints the measured full-size stage times beside the slice-extrapolated ones.
"""
import argparse
import json
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import blocksparse, geometry, newton, stage_timing
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.stepper import apply_dbc

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--cg", type=int, default=3)
args = ap.parse_args()

system, state, params = scenes.squishy_scene(cell=0.02, plate_speed=2.0)
h = params.h
x = state.x
x_tilde = x + h * state.v + (h * h) * np.asarray(params.gravity, dtype=np.float64)
x_hat = x.copy()
apply_dbc(x_hat, system.boundary, x, 0)
mu = params.stiffness_constant
regs = stage_timing.oracle_regions(system)
meas = {}
t = time.perf_counter()
g, H = newton.assemble(x_hat, x_tilde, system.masses, regs, None, mu, params.offset, h)
meas["assemble"] = time.perf_counter() - t
print(json.dumps({"assemble_s": meas["assemble"], "blocks": int(len(H.rows))}), flush=True)
t = time.perf_counter()
_, i1, _, _ = blocksparse.pcg(H, -g, 1e-30, max_iters=1)
t1 = time.perf_counter() - t
t = time.perf_counter()
_, i2, _, _ = blocksparse.pcg(H, -g, 1e-30, max_iters=1 + args.cg)
t2 = time.perf_counter() - t
meas["cg_iter"] = max(t2 - t1, 0.0) / max(i2 - i1, 1)
meas["cg_setup"] = max(t1 - meas["cg_iter"], 0.0)
print(json.dumps({"cg_iter_s": meas["cg_iter"], "cg_setup_s": meas["cg_setup"]}), flush=True)
t = time.perf_counter()
newton.energy(x_hat, x_tilde, system.masses, regs, None, mu, params.offset, h)
meas["energy"] = time.perf_counter() - t
print(json.dumps({"energy_s": meas["energy"]}), flush=True)
t = time.perf_counter()
geometry.step_limit(x, x_hat, system.surface_triangles, system.surface_edges, system.surface_vertices,
                    0.1 * params.offset)
meas["ccd"] = time.perf_counter() - t
print(json.dumps({"ccd_s": meas["ccd"]}), flush=True)
# the slice extrapolation of the same stages (what bench.py --impl reference uses)
full_blocks = len(H.rows)
ext = {}
for sl in stage_timing.ball_slices(system, 8)[:2]:
    _, _, full, info = stage_timing.time_sample(system, x, x_hat, x_tilde, mu, params.offset, h, sl,
                                                full_blocks=full_blocks)
    for k, v in full.items():
        ext.setdefault(k, []).append(v)
ext = {k: float(np.mean(v)) for k, v in ext.items()}
out = {"what": "oracle stages at the full squishy C4 size (2.30M tets, 0.90M vertices, 1.62M surface triangles), "
               "first frame, one host core (OMP/OPENBLAS threads = 1)",
       "measured_full_s": meas, "slice_extrapolated_s": ext,
       "ratio_extrapolated_over_measured": {k: ext[k] / meas[k] for k in meas if k in ext and meas[k] > 0},
       "host": os.uname().nodename, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}
print(json.dumps(out), flush=True)
if args.out:
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
