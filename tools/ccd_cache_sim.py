"""Dev tool: how often would a broad-phase candidate cache stay valid?

    IBF_PY_OUTER=1 python tools/ccd_cache_sim.py --load /tmp/sq48.npz --frames 3

Steps the C4 press from a squishy_run dump through the Python outer loop and,
at every CCD call, checks for several inflation margins m whether each
surface vertex's swept box (x -> x_hat) still lies inside the box cached at
the last rebuild, inflated by m.  If every vertex passes, a candidate list
computed with the inflated boxes would be a superset of this call's
candidates.  Prints reuse counts per policy and the per-call displacements.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IBF_PY_OUTER", "1")
import numpy as np
import torch

from paper_2512_12151_b200 import ccd as ccdmod
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_dev
from paper_2512_12151_b200.stepper import step_device

ap = argparse.ArgumentParser()
ap.add_argument("--load", required=True)
ap.add_argument("--frames", type=int, default=3)
args = ap.parse_args()

system, state, params = scenes.squishy_scene(cell=0.02, plate_speed=2.0)
aset = ActiveSet()
aset.ensure(system.n_vertices)
z = np.load(args.load)
x, v, k0 = to_dev(z["x"]), to_dev(z["v"]), int(z["frame"])
aset.import_state(*(z[f"a{j}"] for j in range(8)))
sv = torch.from_numpy(np.asarray(system.surface_vertices, dtype=np.int64)).cuda()
delta = params.offset
policies = {f"abs_{f}delta": ("abs", f * delta) for f in (0.25, 0.5, 1.0, 2.0, 4.0)}
policies.update({f"rel_{f}disp": ("rel", f) for f in (0.5, 1.0, 2.0)})
cache = {k: None for k in policies}
stats = {k: {"reuse": 0, "rebuild": 0, "margin_sum": 0.0} for k in policies}
calls = []
orig = ccdmod.CCD.max_step_size


def wrapped(self, x_dev, x_hat_dev, min_gap, cap=1.0):
    a = x_dev[sv]
    b = x_hat_dev[sv]
    lo, hi = torch.minimum(a, b), torch.maximum(a, b)
    disp = (b - a).abs().amax(dim=1)
    dmax = float(disp.max())
    calls.append({"disp_max": dmax, "disp_mean": float(disp.mean()), "disp_p99": float(torch.quantile(disp[::7], 0.99))})
    for k, (kind, f) in policies.items():
        c = cache[k]
        if c is not None and bool(((lo >= c[0]).all() & (hi <= c[1]).all()).item()):
            stats[k]["reuse"] += 1
            continue
        m = f if kind == "abs" else f * dmax
        cache[k] = (lo - m, hi + m)
        stats[k]["rebuild"] += 1
        stats[k]["margin_sum"] += m
    return orig(self, x_dev, x_hat_dev, min_gap, cap)


ccdmod.CCD.max_step_size = wrapped
for k in range(k0, k0 + args.frames):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    torch.cuda.synchronize()
    print(json.dumps({"frame": k, "calls": len(calls), "constraints": len(aset)}), flush=True)
for k in stats:
    s = stats[k]
    s["mean_margin"] = s["margin_sum"] / max(s["rebuild"], 1)
print(json.dumps({"calls": len(calls), "policies": stats,
                  "disp_max_median": float(np.median([c["disp_max"] for c in calls])),
                  "disp_mean_median": float(np.median([c["disp_mean"] for c in calls])),
                  "per_call": calls}), flush=True)
