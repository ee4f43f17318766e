"""Dev tool: find host-visible stalls in C4 press frames.  Every host-level
call of a pass is timed (they all end in a stream sync); passes slower than
--thresh ms are printed with the per-call split.  Also logs Python GC pauses.

    python tools/stall_hunt.py [frames=12] [pre=50]
"""
import gc, json, os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2512_12151_b200 import scenes, solver, contact, ccd as ccdmod, _lib
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.stepper import step_device

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 12
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 50
system, state, params = scenes.c4_scene(n=42, plate_speed=bench.PLATE_SPEED, plate_stop=bench.PLATE_STOP)
aset = ActiveSet(); aset.ensure(system.n_vertices)
x, v = to_dev(state.x), to_dev(state.v)
for k in range(pre):
    x, v, _ = step_device(x, v, system, aset, params, step_index=k)
torch.cuda.synchronize()

gc_pauses = []
_gc_t = {}
def _gc_cb(phase, info):
    if phase == "start":
        _gc_t["t"] = time.perf_counter()
    else:
        gc_pauses.append((info.get("generation"), 1e3 * (time.perf_counter() - _gc_t.get("t", time.perf_counter()))))
gc.callbacks.append(_gc_cb)

cur = collections.defaultdict(float)
cmax = collections.defaultdict(float)
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **kw):
        t = time.perf_counter()
        r = f(*a, **kw)
        dt = 1e3 * (time.perf_counter() - t)
        cur[name] += dt
        cmax[name] = max(cmax[name], dt)
        return r
    setattr(cls, name, g)
for cls, name in [(solver.DeviceSystem, "solve_subproblem"), (solver.DeviceSystem, "stiffness_diagonal_max"),
                  (contact.ActiveSet, "update"), (ccdmod.CCD, "max_step_size")]:
    wrap(cls, name)

slow = []
rows = []
for k in range(pre, pre + frames):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    cur.clear()
    cmax.clear()
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    e1.record(); torch.cuda.synchronize()
    walls = [r.wall_ms for r in d.iterations]
    rows.append({"frame": k, "dev_ms": e0.elapsed_time(e1), "host_ms": 1e3 * (time.perf_counter() - t0),
                 "max_pass_ms": max(walls), "calls_ms": {n: round(t, 1) for n, t in cur.items()},
                 "max_call_ms": {n: round(t, 1) for n, t in cmax.items()}})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"gc_pauses_ms": [(g, round(t, 2)) for g, t in gc_pauses if t > 1.0], "n_gc": len(gc_pauses)}))
