"""Dev tool: where one C5 scene-frame goes (host-call split, one stream)."""
import collections, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_12151_b200 import scenes, solver, contact, ccd as ccdmod, _lib
from paper_2512_12151_b200.stepper import Simulation

system, state, params = scenes.c5_scene(0)
sim = Simulation(system, params, state)
for _ in range(3):
    sim.advance()
T = collections.defaultdict(float); N = collections.Counter()
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **kw):
        t = time.perf_counter()
        r = f(*a, **kw)
        T[name] += time.perf_counter() - t; N[name] += 1
        return r
    setattr(cls, name, g)
for cls, name in [(solver.DeviceSystem, "solve_subproblem"), (solver.DeviceSystem, "stiffness_diagonal_max"),
                  (solver.DeviceSystem, "inversion_safe_step"), (contact.ActiveSet, "update"),
                  (ccdmod.CCD, "max_step_size")]:
    wrap(cls, name)
F = 20
L = _lib.lib()
l0 = L.ibf_launch_count()
import numpy as np
st = np.zeros(9)
L.ibf_system_stats(system.device.handle, _lib.host_ptr(st), 1)
torch.cuda.synchronize(); t0 = time.perf_counter()
passes = newton = 0
for _ in range(F):
    d = sim.advance()
    passes += len(d.iterations); newton += sum(r.newton_iters for r in d.iterations)
torch.cuda.synchronize(); wall = time.perf_counter() - t0
out = {"ms_per_frame": 1e3 * wall / F, "passes_per_frame": passes / F, "newton_per_frame": newton / F,
       "launches_per_frame": (L.ibf_launch_count() - l0) / F,
       "ms_per_frame_by_call": {k: round(1e3 * v / F, 3) for k, v in T.items()},
       "calls_per_frame": {k: v / F for k, v in N.items()}}
out["unaccounted_ms"] = out["ms_per_frame"] - sum(out["ms_per_frame_by_call"].values())
L.ibf_system_stats(system.device.handle, _lib.host_ptr(st), 0)
out["pcg_ms_per_frame"] = st[2] / F
out["cg_iters_per_frame"] = st[4] / F
out["us_per_cg_iter"] = 1e3 * st[2] / max(st[4], 1)
out["n_vertices"] = system.n_vertices
print(json.dumps(out, indent=1))
