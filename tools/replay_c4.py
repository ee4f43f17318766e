"""Dev tool: run C4 frames; on a failing frame, replay it from the saved
state with a logged Python Newton loop over the device primitives."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes, solver
from paper_2512_12151_b200.device import to_dev, to_host, empty
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.stepper import step_device
n = int(sys.argv[1]); frames = int(sys.argv[2])
system, state, params = scenes.c4_scene(n=n)
N = system.n_vertices
dev = system.device
aset = ActiveSet(); aset.ensure(N)
xs, vs = to_dev(state.x), to_dev(state.v)
LOG = []

def solve_logged(self, aset, x_tilde, x, x_hat, mu, offset, h, cg_tol, decay):
    aset.refresh_anchors(x)
    g = empty((N, 3)); p = empty((N, 3))
    nw = cg = 0
    for it in range(64):
        self.assemble(aset, x_hat, x_tilde, mu, offset, h, True, g)
        if not bool(g.abs().max() > 0):
            break
        iters, conv, rel = self.pcg(-g, p, cg_tol, 0)
        cg += iters
        gp = float((g * p).sum())
        y = empty((N, 3)); self.matvec(p, y)
        true_rel = float(torch.linalg.norm(y + g) / torch.linalg.norm(g))
        base = float(self.energy(aset, x_hat, x_tilde, mu, offset, h)[0])
        rs = [0.5 ** k for k in range(8)]
        es = self.energy(aset, x_hat, x_tilde, mu, offset, h, p=p, rs=rs)
        r = None
        for rr, e in zip(rs, es):
            if e < base:
                r = rr; break
        rec = {"it": it, "pcg": [iters, conv, rel], "true_rel": true_rel, "gp": gp, "pmax": float(p.abs().max()),
               "gmax": float(g.abs().max()), "base": base, "trials": [float(e) for e in es[:4]], "r": r, "C": len(aset)}
        LOG.append(rec); print(json.dumps(rec), flush=True)
        if r is None:
            r = 1.0
        x_hat.add_(r * p)
        nw += 1
        if r == 1.0:
            break
    worst = aset.dual_update_sweep(x_hat, offset, mu, decay)
    print(json.dumps({"subproblem": nw, "move": float((x_hat - x).abs().max())}), flush=True)
    return nw, cg, False, worst

for k in range(frames):
    saved = (xs.clone(), vs.clone(), aset.export_state())
    try:
        xs, vs, diag = step_device(xs, vs, system, aset, params, step_index=k)
        print(json.dumps({"frame": k, "passes": [(r.alpha, r.newton_iters, r.cg_iters, r.n_constraints) for r in diag.iterations]}), flush=True)
    except Exception as e:
        print(json.dumps({"frame": k, "error": str(e)[:200]}), flush=True)
        xs, vs, st = saved
        aset = ActiveSet(); aset.ensure(N); aset.import_state(*st)
        solver.DeviceSystem.solve_subproblem = solve_logged
        try:
            step_device(xs, vs, system, aset, params, step_index=k)
        except Exception as e2:
            print(json.dumps({"replay_error": str(e2)[:200]}), flush=True)
        break
