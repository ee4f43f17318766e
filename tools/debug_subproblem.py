"""Evolve C4 (small n) on the GPU, then solve one subproblem from the same
state on GPU and oracle and compare (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes, _lib
from paper_2512_12151_b200.stepper import step_device, _apply_dbc_device
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_host, to_dev, empty
from oracle import contact as ocontact, newton
n = int(sys.argv[1]); frames = int(sys.argv[2]); layers = int(sys.argv[3]) if len(sys.argv) > 3 else 1
system, state, params = scenes.c4_scene(n=n, layers=layers)
aset = ActiveSet(); aset.ensure(system.n_vertices)
x = torch.from_numpy(state.x).cuda(); v = torch.from_numpy(state.v).cuda()
for k in range(frames):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
print("C =", len(aset), flush=True)
dev = system.device
N = system.n_vertices
xt = to_host(x); vt = to_host(v); h = params.h
x_tilde = xt + h * vt + (h * h) * np.array(params.gravity)
mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, h)
x_hat0 = xt.copy()
for bc in system.boundary:
    if bc.kind == "scripted": x_hat0[bc.vertices] = bc.targets(None, frames)
st = aset.export_state()
o = ocontact.ConstraintSet()
o._append(st[0], st[1], [ocontact.key_of(a, b) for a, b in zip(st[0], st[1])], lam=st[2], gamma=st[3], s=st[4],
          anchor_d=st[5], anchor_grad=st[6], anchor_x=st[7])
regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes) for r in system.regions]
t = time.time()
xo, nwo, cgo, sto, wo = newton.subproblem(x_tilde, xt, x_hat0, system.masses, regions, o, mu, params.offset, h, dbc=system.dbc_mask)
print(f"oracle {time.time()-t:.1f}s nw={nwo} cg={cgo} stalled={sto} worst={wo:.6e} max|xh-x|={np.abs(xo-xt).max():.4e}", flush=True)
xh = to_dev(x_hat0)
nw, cg, stl, w = dev.solve_subproblem(aset, to_dev(x_tilde), x, xh, mu, params.offset, h, params.cg_tol, params.decay)
xg = to_host(xh)
print(f"gpu nw={nw} cg={cg} stalled={stl} worst={w:.6e} max|xh-x|={np.abs(xg-xt).max():.4e}", flush=True)
print("x_hat rel diff", np.abs(xg - xo).max() / np.abs(xo - xt).max())
sg = aset.export_state()
print("lam max diff", np.abs(sg[2] - o.lam).max(), "gamma eq", np.array_equal(sg[3], o.gamma))
