"""Dev tool: wall-time breakdown of C4 frames by host call (synchronised),
after the bench's pre-compression; shows where the untimed 'other' goes."""
import sys, os, json, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2512_12151_b200 import scenes, solver, contact, ccd as ccdmod, _lib
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.stepper import step_device
pre = int(sys.argv[1]) if len(sys.argv) > 1 else 50
system, state, params = scenes.c4_scene(n=42, plate_speed=bench.PLATE_SPEED, plate_stop=bench.PLATE_STOP)
aset = ActiveSet(); aset.ensure(system.n_vertices)
x, v = to_dev(state.x), to_dev(state.v)
for k in range(pre):
    x, v, _ = step_device(x, v, system, aset, params, step_index=k)
T = collections.defaultdict(float); N = collections.Counter()
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **kw):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **kw)
        torch.cuda.synchronize(); T[name] += time.perf_counter() - t; N[name] += 1
        return r
    setattr(cls, name, g)
for cls, name in [(solver.DeviceSystem, "solve_subproblem"), (solver.DeviceSystem, "stiffness_diagonal_max"),
                  (solver.DeviceSystem, "inversion_safe_step"), (contact.ActiveSet, "update"),
                  (ccdmod.CCD, "max_step_size")]:
    wrap(cls, name)
F = 3
torch.cuda.synchronize(); t0 = time.perf_counter()
st = np.zeros(9); _lib.lib().ibf_system_stats(system.device.handle, _lib.host_ptr(st), 1)
passes = 0
for k in range(pre, pre + F):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    passes += len(d.iterations)
torch.cuda.synchronize(); wall = time.perf_counter() - t0
_lib.lib().ibf_system_stats(system.device.handle, _lib.host_ptr(st), 1)
out = {"frames": F, "passes": passes, "frame_ms": 1e3 * wall / F,
       "per_frame_ms": {k: 1e3 * t / F for k, t in T.items()}, "calls_per_frame": {k: c / F for k, c in N.items()},
       "inside_subproblem_ms_per_frame": {"assembly": st[0] / F, "pcg": st[2] / F, "ls": st[5] / F, "cap": st[7] / F},
       "constraints": len(aset)}
out["unaccounted_ms"] = out["frame_ms"] - sum(out["per_frame_ms"].values())
print(json.dumps(out, indent=1))
