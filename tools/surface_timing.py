"""Surface extraction and OBJ export at C4 size: device / native vs numpy (dev tool)."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.mesh import extract_surface_arrays, surface_of
from paper_2512_12151_b200.io_utils import export_frame
from oracle.sceneio import obj_text

system, state, params = scenes.c4_scene()
tets = np.vstack([r.tets for r in system.regions])
out = {"tets": len(tets)}
td = torch.from_numpy(tets).cuda()
extract_surface_arrays(td)
torch.cuda.synchronize()
runs = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); t, e, v = extract_surface_arrays(td); runs.append(time.perf_counter() - t0)
out["device_s"] = min(runs)
out["device_runs_s"] = runs
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    extract_surface_arrays(td)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
t0 = time.perf_counter(); ot, oe, ov = surface_of(tets); out["numpy_s"] = time.perf_counter() - t0
out["identical"] = bool(np.array_equal(t, ot) and np.array_equal(e, oe) and np.array_equal(v, ov))
out.update(tris=len(t), edges=len(e), verts=len(v))
x = state.x
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "f.obj")
    t0 = time.perf_counter(); export_frame(x, t, p); out["export_native_s"] = time.perf_counter() - t0
    out["threads"] = os.cpu_count()
    t0 = time.perf_counter(); ref = obj_text(x, t).encode(); out["export_python_s"] = time.perf_counter() - t0
    out["obj_identical"] = open(p, "rb").read() == ref
    out["obj_mb"] = len(ref) / 1e6
print(json.dumps(out))
