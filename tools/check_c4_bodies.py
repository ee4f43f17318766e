"""Dev tool: per-body motion of the C4 scene frame by frame (new vs base lib via IBF_LIB)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.device import to_dev, to_host
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.stepper import step_device
n = int(sys.argv[1]); frames = int(sys.argv[2])
layers = int(os.environ["LAYERS"]) if os.environ.get("LAYERS") else None
speed = float(os.environ.get("SPEED", "0.1"))
system, state, params = scenes.c4_scene(n=n, layers=layers, plate_speed=speed)
import time
print(json.dumps({"verts": system.n_vertices, "tets": sum(len(r.tets) for r in system.regions),
                  "tris": len(system.surface_triangles)}), flush=True)
N = system.n_vertices
# body ranges from the regions' tets
ranges = []
for r in system.regions:
    ranges.append((int(r.tets.min()), int(r.tets.max()) + 1))
aset = ActiveSet(); aset.ensure(N)
xs, vs = to_dev(state.x), to_dev(state.v)
for k in range(frames):
    try:
        torch.cuda.synchronize(); t0 = time.time()
        xs, vs, diag = step_device(xs, vs, system, aset, params, step_index=k)
        torch.cuda.synchronize(); wall = time.time() - t0
    except Exception as e:
        print(json.dumps({"frame": k, "error": str(e)[:300]}), flush=True)
        break
    x, v = to_host(xs), to_host(vs)
    bodies = [{"zmin": round(float(x[a:b, 2].min()), 6), "vz": round(float(v[a:b, 2].mean()), 4),
               "vmax": round(float(np.abs(v[a:b]).max()), 4)} for a, b in ranges]
    print(json.dumps({"frame": k, "wall": round(wall, 3), "mu": diag.mu, "passes": len(diag.iterations), "newton": sum(r.newton_iters for r in diag.iterations),
                      "cg": sum(r.cg_iters for r in diag.iterations), "C": diag.iterations[-1].n_constraints,
                      "bodies": bodies}), flush=True)
