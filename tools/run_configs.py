"""Dev tool: run the full-size C2 (131k tets) and C3 (491k tets) scenes on
the GPU for a few frames: ms/frame, Newton/frame, constraints and the
penetration certificate of every frame."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.stepper import step_device
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 10
out = {}
for name, build in (("C2", scenes.c2_scene), ("C3", scenes.c3_scene)):
    system, state, params = build()
    aset = ActiveSet(); aset.ensure(system.n_vertices)
    x, v = to_dev(state.x), to_dev(state.v)
    recs = []
    for k in range(frames):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, v, d = step_device(x, v, system, aset, params, step_index=k)
        e1.record(); torch.cuda.synchronize()
        dmin, _, _ = system.ccd.min_distance(x, params.offset)
        hits, _ = system.ccd.static_intersections(x, cap=4)
        recs.append({"frame": k, "ms": e0.elapsed_time(e1), "passes": len(d.iterations),
                     "newton": sum(r.newton_iters for r in d.iterations), "cg": sum(r.cg_iters for r in d.iterations),
                     "constraints": len(aset), "min_distance": dmin, "intersections": hits})
        print(name, json.dumps(recs[-1]), flush=True)
    out[name] = {"tets": int(sum(len(r.tets) for r in system.regions)), "vertices": int(system.n_vertices),
                 "surface_tris": int(len(system.surface_triangles)), "frames": recs,
                 "ms_per_frame_after_first": float(np.mean([r["ms"] for r in recs[1:]])) if frames > 1 else None}
print(json.dumps(out))
