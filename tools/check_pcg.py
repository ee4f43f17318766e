"""Dev tool: PCG on the C4 matrix — true residual check and first frames' pass log."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.device import to_dev, empty, to_host
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.stepper import step_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 42
system, state, params = scenes.c4_scene(n=n)
dev = system.device
N = system.n_vertices
x = to_dev(state.x)
rng = np.random.default_rng(0)
xt = to_dev(state.x + 1e-4 * rng.standard_normal(state.x.shape))
g = empty((N, 3))
dev.assemble(None, x, xt, 1.0, 1e-3, 0.01, True, g)
rhs = -g
for tol in (1e-4, 1e-8):
    xo = empty((N, 3))
    it, conv, rel = dev.pcg(rhs, xo, tol, 0)
    y = empty((N, 3))
    dev.matvec(xo, y)
    true_rel = float(torch.linalg.norm(y - rhs) / torch.linalg.norm(rhs))
    print(json.dumps({"tol": tol, "iters": it, "conv": conv, "rel": rel, "true_rel": true_rel}), flush=True)
aset = ActiveSet(); aset.ensure(N)
xs, vs = to_dev(state.x), to_dev(state.v)
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    xs, vs, diag = step_device(xs, vs, system, aset, params, step_index=k)
    print(json.dumps({"frame": k, "passes": [(r.alpha, r.newton_iters, r.cg_iters, r.n_constraints) for r in diag.iterations],
                      "vmax": float(vs.abs().max())}), flush=True)
