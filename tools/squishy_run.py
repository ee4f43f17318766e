"""Dev tool: run the squishy-ball press (scenes.squishy_scene) for F frames and
print per-frame device ms / passes / Newton / CG / constraints / alpha.

    python tools/squishy_run.py --frames 40 [--cell 0.01 --n 32 --stem 23 --tip 16 --balls 5]
                                [--plate-speed 1.0] [--plate-stop 0.3] [--certify] [--every 1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.stepper import step_device

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=40)
ap.add_argument("--cell", type=float, default=0.02)
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--stem", type=int, default=23)
ap.add_argument("--tip", type=int, default=16)
ap.add_argument("--shell", type=int, default=2)
ap.add_argument("--balls", type=int, default=5)
ap.add_argument("--numbering", default="lattice", choices=["sell", "lattice", "morton"])
ap.add_argument("--plate-speed", type=float, default=1.0)
ap.add_argument("--plate-stop", type=float, default=None)
ap.add_argument("--certify", action="store_true")
ap.add_argument("--every", type=int, default=1, help="print every k-th frame")
ap.add_argument("--out", default=None)
ap.add_argument("--dump", default=None, help="save (x, v, active set, frame) after the last frame to this .npz")
ap.add_argument("--load", default=None, help="start from a --dump file instead of the scene's rest state")
ap.add_argument("--profile-frames", type=int, default=0,
                help="run the last k frames inside cudaProfilerStart/Stop (ncu --profile-from-start off)")
args = ap.parse_args()

t = time.perf_counter()
system, state, params = scenes.squishy_scene(numbering=args.numbering, cell=args.cell, n=args.n, stem=args.stem, tip=args.tip,
                                             shell=args.shell, balls=args.balls, plate_speed=args.plate_speed,
                                             plate_stop=args.plate_stop)
info = dict(system.scene_info, n_vertices=system.n_vertices, tets=int(sum(len(r.tets) for r in system.regions)),
            tris=int(len(system.surface_triangles)), build_s=time.perf_counter() - t)
print(json.dumps(info), flush=True)
aset = ActiveSet()
aset.ensure(system.n_vertices)
ccd = system.ccd
x, v = to_dev(state.x), to_dev(state.v)
k0 = 0
if args.load:
    z = np.load(args.load)
    x, v, k0 = to_dev(z["x"]), to_dev(z["v"]), int(z["frame"])
    aset.import_state(*(z[f"a{j}"] for j in range(8)))
    print(json.dumps({"loaded": args.load, "frame": k0, "constraints": len(aset)}), flush=True)
if args.certify:
    n_hits, _ = ccd.static_intersections(x, cap=16)
    dmin, _, _ = ccd.min_distance(x, params.offset)
    print(json.dumps({"frame": -1, "intersecting_pairs": int(n_hits), "min_distance": dmin}), flush=True)
rows = []
from paper_2512_12151_b200 import _lib
L = _lib.lib()
dev = system.device
free = torch.from_numpy(~system.dbc_mask).cuda()
plate = torch.from_numpy(system.boundary[-1].vertices).cuda()
for k in range(k0, k0 + args.frames):
    if args.profile_frames and k == k0 + args.frames - args.profile_frames:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    stats, cst = np.zeros(9), np.zeros(3)
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 1)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    e1.record()
    torch.cuda.synchronize()
    it = d.iterations
    row = {"frame": k, "ms": round(e0.elapsed_time(e1), 1), "passes": len(it),
           "newton": sum(r.newton_iters for r in it), "cg": sum(r.cg_iters for r in it),
           "constraints": len(aset), "triggers": d.adaptive_triggers, "mu": d.mu, "offset": d.offset,
           "min_alpha": min(r.alpha for r in it), "ball_top": round(float(x[free, 2].max()), 4),
           "plate_z": round(float(x[plate, 2].min()), 4)}
    row["cg_per_solve"] = round(row["cg"] / max(row["newton"], 1), 1)
    L.ibf_system_stats(dev.handle, _lib.host_ptr(stats), 0)
    L.ibf_ccd_stats(ccd.handle, _lib.host_ptr(cst), 0)
    row.update(asm_ms=round(stats[0], 1), pcg_ms=round(stats[2], 1), ls_ms=round(stats[5], 1),
               ccd_ms=round(cst[0], 1), cand=int(cst[2]))
    if args.certify:
        dmin, _, _ = ccd.min_distance(x, params.offset)
        n_hits, _ = ccd.static_intersections(x, cap=16)
        row.update(min_distance=dmin, intersecting_pairs=int(n_hits))
    rows.append(row)
    if k % args.every == 0 or k == args.frames - 1:
        print(json.dumps(row), flush=True)
if args.profile_frames:
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
if args.dump:
    st = aset.export_state()
    np.savez(args.dump, x=x.cpu().numpy(), v=v.cpu().numpy(), frame=k0 + args.frames,
             **{f"a{j}": a for j, a in enumerate(st)})
ms = np.array([r["ms"] for r in rows])
summary = {"frames": len(rows), "mean_ms": float(ms.mean()), "max_ms": float(ms.max()),
           "mean_newton": float(np.mean([r["newton"] for r in rows])),
           "mean_cg_per_solve": float(sum(r["cg"] for r in rows) / max(sum(r["newton"] for r in rows), 1)),
           "peak_constraints": max(r["constraints"] for r in rows), "scene": info, "args": vars(args)}
print(json.dumps(summary), flush=True)
if args.out:
    with open(args.out, "w") as f:
        json.dump(dict(summary, rows=rows), f, indent=1)
