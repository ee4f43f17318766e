"""Dev tool: long-horizon parity of a full-resolution C5 drop (C1 mesh,
4.8k tets, rotated: no exact TOI ties) or of C1 itself — GPU vs the CPU
oracle for F frames: per-frame max relative position error, pass and Newton
counts, key sets.

    python tools/long_parity.py <seed|c1> [frames] [perturbation]

With a perturbation (e.g. 1e-15) a second oracle run starts from the state
perturbed by that relative amount, and every frame also reports the GPU's
distance to it and the two oracle runs' distance to each other: the
reference's own sensitivity.  C1 is an axis-aligned cube on a slab, whose
admission filter sits on exact TOI ties (intact/contact.py:151), so there the
oracle-oracle distance is the scale the GPU can be held to.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import contact as ocontact, timestep
from paper_2512_12151_b200 import Simulation, scenes

seed = sys.argv[1] if len(sys.argv) > 1 else "0"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 30
perturb = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
system, state, params = scenes.c1_scene() if seed == "c1" else scenes.c5_scene(int(seed))
regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
           for r in system.regions]
scene = timestep.Scene(system.masses, regions, system.surface_triangles, system.surface_edges,
                       system.surface_vertices, [(bc.vertices, None) for bc in system.boundary])


class OracleRun:
    def __init__(self, x, v):
        self.x, self.v, self.aset, self.t = x, v, ocontact.ConstraintSet(), 0.0

    def step(self, k):
        t = time.perf_counter()
        self.x, self.v, self.rec, _, _ = timestep.step(self.x, self.v, scene, self.aset, h=params.h,
                                                       offset=params.offset, k_min=params.min_iterations,
                                                       step_index=k)
        self.t += time.perf_counter() - t

    def keys(self):
        return sorted(ocontact.key_of(kd, q) for kd, q in zip(self.aset.kind, self.aset.quad))


runs = [OracleRun(state.x.copy(), state.v.copy())]
if perturb:
    xp = state.x * (1.0 + perturb * np.random.default_rng(1).standard_normal(state.x.shape))
    runs.append(OracleRun(xp, state.v.copy()))
sim = Simulation(system, params, state.copy())
rows = []
t_g = 0.0
for k in range(frames):
    for r in runs:
        r.step(k)
    t = time.perf_counter()
    d = sim.advance()
    xg = sim.state.x
    t_g += time.perf_counter() - t
    kg = sorted(c.key for c in sim.active_set)
    o = runs[0]
    scale = np.abs(o.x).max()
    row = {"frame": k, "rel_err": float(np.abs(xg - o.x).max() / scale),
           "passes": [len(d.iterations), len(o.rec)],
           "newton_max_diff": int(max(abs(a.newton_iters - b[3]) for a, b in zip(d.iterations, o.rec)))
           if len(d.iterations) == len(o.rec) else None,
           "keys_equal": kg == o.keys(), "constraints": len(kg)}
    if perturb:
        p = runs[1]
        row.update(rel_err_vs_perturbed=float(np.abs(xg - p.x).max() / scale),
                   oracle_spread=float(np.abs(p.x - o.x).max() / scale),
                   keys_equal_perturbed=kg == p.keys(), oracle_keys_equal=o.keys() == p.keys())
    rows.append(row)
    print(json.dumps(row), flush=True)
summary = {"seed": seed, "perturb": perturb, "frames": frames, "tets": int(sum(len(r.tets) for r in system.regions)),
           "max_rel_err": max(r["rel_err"] for r in rows), "all_keys_equal": all(r["keys_equal"] for r in rows),
           "oracle_s": runs[0].t, "gpu_s": t_g}
if perturb:
    summary.update(max_rel_err_vs_perturbed=max(r["rel_err_vs_perturbed"] for r in rows),
                   max_oracle_spread=max(r["oracle_spread"] for r in rows),
                   frames_oracle_keys_differ=sum(not r["oracle_keys_equal"] for r in rows))
print(json.dumps(dict(summary, rows=rows)))
