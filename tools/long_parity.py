"""Dev tool: long-horizon parity of a full-resolution C5 drop (C1 mesh,
4.8k tets, rotated: no exact TOI ties) — GPU vs the CPU oracle for F frames:
per-frame max relative position error, pass and Newton counts, key sets."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import contact as ocontact, timestep
from paper_2512_12151_b200 import Simulation, scenes
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 30
system, state, params = scenes.c5_scene(seed)
regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
           for r in system.regions]
scene = timestep.Scene(system.masses, regions, system.surface_triangles, system.surface_edges,
                       system.surface_vertices, [(bc.vertices, None) for bc in system.boundary])
x, v = state.x.copy(), state.v.copy()
aset = ocontact.ConstraintSet()
sim = Simulation(system, params, state.copy())
rows = []
t_o = t_g = 0.0
for k in range(frames):
    t = time.perf_counter()
    x, v, rec, _, _ = timestep.step(x, v, scene, aset, h=params.h, offset=params.offset,
                                    k_min=params.min_iterations, step_index=k)
    t_o += time.perf_counter() - t
    t = time.perf_counter()
    d = sim.advance()
    xg = sim.state.x
    t_g += time.perf_counter() - t
    kg = sorted(c.key for c in sim.active_set)
    ko = sorted(ocontact.key_of(kd, q) for kd, q in zip(aset.kind, aset.quad))
    rows.append({"frame": k, "rel_err": float(np.abs(xg - x).max() / np.abs(x).max()),
                 "passes": [len(d.iterations), len(rec)],
                 "newton_max_diff": int(max(abs(a.newton_iters - b[3]) for a, b in zip(d.iterations, rec)))
                 if len(d.iterations) == len(rec) else None,
                 "keys_equal": kg == ko, "constraints": len(kg)})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"seed": seed, "frames": frames, "tets": int(sum(len(r.tets) for r in system.regions)),
                  "max_rel_err": max(r["rel_err"] for r in rows), "all_keys_equal": all(r["keys_equal"] for r in rows),
                  "oracle_s": t_o, "gpu_s": t_g, "rows": rows}))
