"""Diagnose GPU vs oracle divergence on a small NH drop (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_12151_b200 import scenes, Simulation
from paper_2512_12151_b200.solver import DeviceSystem
from paper_2512_12151_b200.device import to_dev, empty, to_host
from oracle import contact as ocontact, timestep, newton, blocksparse, material

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
system, state, params = scenes.c1_scene(nx=nx, ny=nx, nz=nx, size=0.1, height=0.002, speed=0.5)
regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes) for r in system.regions]
scene = timestep.Scene(system.masses, regions, system.surface_triangles, system.surface_edges, system.surface_vertices,
                       [(bc.vertices, None) for bc in system.boundary])
x, v = state.x.copy(), state.v.copy()
# single assemble + pcg comparison at the initial state
h = params.h
x_tilde = x + h * v + (h * h) * np.array(params.gravity)
x_hat = x_tilde.copy(); x_hat[system.dbc_mask] = x[system.dbc_mask]
go, Ho = newton.assemble(x_hat, x_tilde, system.masses, regions, None, 1.0, 1e-3, h, system.dbc_mask)
po, its, conv, rel = blocksparse.pcg(Ho, -go, 1e-4)
dev = system.device
xd, xtd = to_dev(x_hat), to_dev(x_tilde)
gd = empty(x.shape)
dev.assemble(None, xd, xtd, 1.0, 1e-3, h, True, gd)
pd = empty(x.shape)
it_g, conv_g, rel_g = dev.pcg(-gd, pd, 1e-4)
print("grad rel diff", np.abs(to_host(gd) - go).max() / np.abs(go).max())
print("pcg oracle its", its, conv, rel, " gpu", it_g, conv_g, rel_g)
print("p rel diff", np.abs(to_host(pd) - po).max() / np.abs(po).max())
y = np.random.default_rng(0).standard_normal(x.shape)
yd = empty(x.shape); dev.matvec(to_dev(y), yd)
print("matvec rel diff", np.abs(to_host(yd) - Ho.matvec(y)).max() / np.abs(Ho.matvec(y)).max())
capo = min(material.inversion_cap(m, x_hat, po, t, r) for m, _, _, t, r, _ in regions)
capg = dev.inversion_safe_step(xd, to_dev(po))
print("cap oracle", capo, "gpu", capg)
# energies along p
for r in (1.0, 0.5, 0.25):
    eo = newton.energy(x_hat + r * po, x_tilde, system.masses, regions, None, 1.0, 1e-3, h)
    eg = dev.energy(None, to_dev(x_hat + r * po), xtd, 1.0, 1e-3, h)[0]
    print("energy r", r, eo, eg, (eg - eo) / abs(eo))
# full steps, per-pass records
aset = ocontact.ConstraintSet()
sim = Simulation(system, params, state.copy())
for k in range(2):
    x, v, rec, _, _ = timestep.step(x, v, scene, aset, h=params.h, offset=params.offset, k_min=params.min_iterations, step_index=k)
    d = sim.advance()
    print(f"step {k}: rel err", np.abs(sim.state.x - x).max() / np.abs(x).max())
    for a, b in zip(d.iterations, rec):
        print(f"   gpu a={a.alpha:.9f} b={a.beta:.3e} C={a.n_constraints} nw={a.newton_iters} cg={a.cg_iters} | ora a={b[0]:.9f} b={b[1]:.3e} C={b[2]} nw={b[3]} cg={b[4]}")
