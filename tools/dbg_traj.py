"""Dev tool: golden box-on-slab trajectory through Simulation, per step: active-set key
diffs against the reference's keys and the per-pass (alpha, |C|, Newton) records."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.conftest import golden
from tests.test_gpu_solver import _traj_system
import paper_2512_12151_b200 as pkg
from paper_2512_12151_b200 import Simulation, StepParams
from paper_2512_12151_b200.mesh import SimState
g = golden("trajectory.npz")
system = _traj_system(pkg, g)
sim = Simulation(system, StepParams(h=0.01, offset=1e-3, min_iterations=2), SimState(g["x0"].copy(), g["v0"].copy()))
for k in range(len(g["xs"])):
    d = sim.advance()
    keys = sorted(c.key for c in sim.active_set)
    got = {(kk[0], *kk[1]) for kk in keys}
    exp = {tuple(r) for r in g[f"keys{k}"]}
    print(k, len(got), len(exp), "missing", sorted(exp - got)[:10], "extra", sorted(got - exp)[:10], "dup", len(keys) - len(got))
    print("   passes", [(round(r.alpha, 6), r.n_constraints, r.newton_iters) for r in d.iterations])
    print("   ref   ", [(round(a, 6), int(c), int(nw)) for a, b, c, nw, cg in g[f"rec{k}"]])
