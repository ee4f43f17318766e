"""Dev tool: the whole C4 press (plate 0.5 m/s to 5 cm, then hold), F frames,
per-frame device ms / Newton / CG / constraints, for a whole-run average
comparable to the paper's per-scene average.

    python tools/press_run.py [frames] [first_logged] [--certify]

--certify adds the penetration certificate of every accepted frame (nearest
non-adjacent VF/EE pair within the offset, static tri-tri test), outside the
timed bracket."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.stepper import step_device
certify = "--certify" in sys.argv
args = [a for a in sys.argv[1:] if not a.startswith("--")]
frames = int(args[0]) if len(args) > 0 else 100
first_logged = int(args[1]) if len(args) > 1 else 0
system, state, params = scenes.c4_scene(n=42, plate_speed=bench.PLATE_SPEED, plate_stop=bench.PLATE_STOP)
aset = ActiveSet(); aset.ensure(system.n_vertices)
ccd = system.ccd
x, v = to_dev(state.x), to_dev(state.v)
rows = []
for k in range(frames):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    e1.record(); torch.cuda.synchronize()
    rows.append({"frame": k, "ms": e0.elapsed_time(e1), "passes": len(d.iterations),
                 "newton": sum(r.newton_iters for r in d.iterations), "cg": sum(r.cg_iters for r in d.iterations),
                 "constraints": len(aset), "triggers": d.adaptive_triggers, "mu": d.mu, "offset": d.offset,
                 "min_alpha": min(r.alpha for r in d.iterations),
                 "alpha_lt_1e-4": sum(r.alpha < 1e-4 for r in d.iterations)})
    if certify:
        dmin, _, _ = ccd.min_distance(x, params.offset)
        n_hits, _ = ccd.static_intersections(x, cap=16)
        rows[-1].update(min_distance=dmin, intersecting_pairs=int(n_hits))
    if k >= first_logged:
        print(json.dumps(rows[-1]), flush=True)
ms = np.array([r["ms"] for r in rows])
cert = {}
if certify:
    cert = {"certified_frames": len(rows), "min_distance": min(r["min_distance"] for r in rows),
            "intersecting_pairs_total": sum(r["intersecting_pairs"] for r in rows)}
print(json.dumps({"frames": frames, "mean_ms": float(ms.mean()), "max_ms": float(ms.max()),
                  "mean_newton": float(np.mean([r["newton"] for r in rows])),
                  "mean_cg_per_solve": float(sum(r["cg"] for r in rows) / max(sum(r["newton"] for r in rows), 1)),
                  "peak_constraints": max(r["constraints"] for r in rows), **cert, "rows": rows}))
