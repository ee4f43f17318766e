"""Dev tool: one CCD pass (max_step_size: LBVH broad phase + ACCD narrow
phase, intact/ccd.py:168-193) on a pressed squishy-ball state, timed per
call, with the per-kernel clocks and the candidate counts per kind.

    python tools/ccd_bench.py [--frames 45] [--load f.npz] [--reps 10] [--ncu]

The query motion is the inertial predictor x + h v (what the first pass of
the next frame asks) unless --scale is given (x + scale * h v).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_12151_b200 import _lib, scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.stepper import step_device

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=45)
ap.add_argument("--cell", type=float, default=0.02)
ap.add_argument("--numbering", default="lattice", choices=["sell", "lattice", "morton"])
ap.add_argument("--plate-speed", type=float, default=2.0)
ap.add_argument("--load", default=None)
ap.add_argument("--dump", default=None)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--ncu", action="store_true", help="profile the last call (cudaProfilerStart/Stop)")
args = ap.parse_args()

system, state, params = scenes.squishy_scene(numbering=args.numbering, cell=args.cell, plate_speed=args.plate_speed)
aset = ActiveSet()
aset.ensure(system.n_vertices)
x, v = to_dev(state.x), to_dev(state.v)
k0 = 0
if args.load:
    z = np.load(args.load)
    x, v, k0 = to_dev(z["x"]), to_dev(z["v"]), int(z["frame"])
    aset.import_state(*(z[f"a{j}"] for j in range(8)))
t = time.perf_counter()
for k in range(k0, k0 + args.frames):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
torch.cuda.synchronize()
print(json.dumps({"frames": args.frames, "press_s": time.perf_counter() - t, "constraints": len(aset)}), flush=True)
if args.dump:
    st = aset.export_state()
    np.savez(args.dump, x=x.cpu().numpy(), v=v.cpu().numpy(), frame=k0 + args.frames,
             **{f"a{j}": a for j, a in enumerate(st)})

ccd = system.ccd
L = _lib.lib()
x_hat = x + args.scale * params.h * v
x_hat[torch.from_numpy(system.dbc_mask).cuda()] = x[torch.from_numpy(system.dbc_mask).cuda()]
gap = 0.1 * params.offset
alpha = ccd.max_step_size(x, x_hat, gap, 1.0)    # warm (tree build)
torch.cuda.synchronize()
_lib.kernel_clocks(on=1, reset=True)
cst = np.zeros(3)
L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 1)
ts = []
for r in range(args.reps):
    if args.ncu and r == args.reps - 1:
        torch.cuda.profiler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    alpha = ccd.max_step_size(x, x_hat, gap, 1.0)
    e1.record()
    torch.cuda.synchronize()
    if args.ncu and r == args.reps - 1:
        torch.cuda.profiler.stop()
    ts.append(e0.elapsed_time(e1))
kc = _lib.kernel_clocks(on=0)
L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 0)
bl = ccd.blocking()
out = {"alpha": alpha, "ms_per_call": float(np.median(ts)), "ms_min": float(np.min(ts)),
       "candidates_per_call": cst[2] / args.reps, "blocking": len(bl.tois),
       "surface": {"tris": int(len(system.surface_triangles)), "edges": int(len(system.surface_edges)),
                   "verts": int(len(system.surface_vertices))},
       "kernels": {k: {"ms_per_call": c["ms"] / args.reps, "launches": c["launches"] / args.reps,
                       "units_per_call": c["units"] / args.reps} for k, c in kc.items() if c["launches"]}}
print(json.dumps(out), flush=True)
