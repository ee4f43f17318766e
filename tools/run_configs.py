"""Dev tool: run the full-size C2 (131k tets) and C3 (491k tets) scenes on
the GPU: ms/frame, Newton/frame, constraints (and how many are edge-edge),
and the penetration certificate of every frame.
At the end of each run, one CCD pass on the last state's inertial motion is
timed with its VF / EE candidate counts (EE candidate pairs/s for C3).

    python tools/run_configs.py [--c2 50] [--c3 100] [--out f.json]
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
ap.add_argument("--c2", type=int, default=50)
ap.add_argument("--c3", type=int, default=100)
ap.add_argument("--every", type=int, default=5)
ap.add_argument("--out", default=None)
args = ap.parse_args()
out = {}
for name, build, frames in (("C2", scenes.c2_scene, args.c2), ("C3", scenes.c3_scene, args.c3)):
    if frames <= 0:
        continue
    system, state, params = build()
    aset = ActiveSet()
    aset.ensure(system.n_vertices)
    x, v = to_dev(state.x), to_dev(state.v)
    recs = []
    for k in range(frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, v, d = step_device(x, v, system, aset, params, step_index=k)
        e1.record()
        torch.cuda.synchronize()
        dmin, _, _ = system.ccd.min_distance(x, params.offset)
        hits, _ = system.ccd.static_intersections(x, cap=4)
        kinds = aset.export_state()[0]
        recs.append({"frame": k, "ms": round(e0.elapsed_time(e1), 2), "passes": len(d.iterations),
                     "newton": sum(r.newton_iters for r in d.iterations), "cg": sum(r.cg_iters for r in d.iterations),
                     "constraints": len(aset), "ee_constraints": int((np.asarray(kinds) == 1).sum()),
                     "min_distance": dmin, "intersections": int(hits)})
        if k % args.every == 0 or k == frames - 1:
            print(name, json.dumps(recs[-1]), flush=True)
    # one CCD pass over the inertial motion of the last state, per kind
    x_hat = x + params.h * v
    x_hat[torch.from_numpy(system.dbc_mask).cuda()] = x[torch.from_numpy(system.dbc_mask).cuda()]
    gap = 0.1 * params.offset
    system.ccd.max_step_size(x, x_hat, gap, 1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        system.ccd.max_step_size(x, x_hat, gap, 1.0)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    vf, ee = system.ccd.candidates(x, x_hat, gap)
    ccd_ms = 1e3 * float(np.median(ts))
    out[name] = {"tets": int(sum(len(r.tets) for r in system.regions)), "vertices": int(system.n_vertices),
                 "surface_tris": int(len(system.surface_triangles)), "frames": len(recs),
                 "ms_per_frame_after_first": float(np.mean([r["ms"] for r in recs[1:]])) if len(recs) > 1 else None,
                 "max_constraints": max(r["constraints"] for r in recs),
                 "max_ee_constraints": max(r["ee_constraints"] for r in recs),
                 "first_frame_with_ee": next((r["frame"] for r in recs if r["ee_constraints"]), None),
                 "min_distance_over_frames": min(r["min_distance"] for r in recs),
                 "intersections_over_frames": max(r["intersections"] for r in recs),
                 "last_state_ccd": {"ms_per_pass": ccd_ms, "vf_candidates": int(len(vf)), "ee_candidates": int(len(ee)),
                                    "candidate_pairs_per_s": (len(vf) + len(ee)) / (ccd_ms * 1e-3),
                                    "ee_candidate_pairs_per_s": len(ee) / (ccd_ms * 1e-3)},
                 "rows": recs}
    print(name, json.dumps({k: v for k, v in out[name].items() if k != "rows"}), flush=True)
if args.out:
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
