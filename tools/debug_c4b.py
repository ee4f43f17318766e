"""Pass-by-pass C4 frames with diagnostics of x_hat (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes, _lib
from paper_2512_12151_b200.stepper import step_device, _apply_dbc_device, beta_update, CCD_GAP_FRACTION
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.ccd import BlockingPairs
from paper_2512_12151_b200.device import to_host, empty
n = int(sys.argv[1]); frames = int(sys.argv[2])
system, state, params = scenes.c4_scene(n=n)
aset = ActiveSet(); aset.ensure(system.n_vertices)
x = torch.from_numpy(state.x).cuda(); v = torch.from_numpy(state.v).cuda()
for k in range(frames - 1):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
    print("frame", k, "ok", len(d.iterations), flush=True)
k = frames - 1
dev, ccd, L, st = system.device, system.ccd, _lib.lib(), _lib.stream()
N = system.n_vertices
x_t, v_t = x, v
x_tilde = empty((N, 3))
g3 = np.asarray(params.gravity, dtype=np.float64)
L.ibf_inertia_target(N, _lib.dev_ptr(x_t), _lib.dev_ptr(v_t), params.h, _lib.host_ptr(g3), _lib.dev_ptr(x_tilde), st)
mu = params.stiffness_constant * dev.stiffness_diagonal_max(x_t, params.h)
xx = x_t.clone(); xh = x_t.clone(); _apply_dbc_device(xh, system.boundary, x_t, k)
print("v max", float(v_t.abs().max()), "x_tilde-x max", float((x_tilde - x_t).abs().max()), "mu", mu, flush=True)
have = False; beta = 1.0
for p in range(12):
    nit, cgit, stl, worst = dev.solve_subproblem(aset, x_tilde, xx, xh, mu, params.offset, params.h, params.cg_tol, params.decay)
    dx = (xh - xx).abs()
    print(f"pass {p}: nw={nit} cg={cgit} stalled={stl} worst={worst:.3e} max|xh-x|={float(dx.max()):.3e} nan={bool(torch.isnan(xh).any())}", flush=True)
    big = (dx.max(dim=1).values > 0.01).nonzero().flatten()
    print("   verts moving >1cm:", len(big), big[:10].tolist(), flush=True)
    aset.update(ccd if have else BlockingPairs.empty())
    try:
        a = ccd.max_step_size(xx, xh, CCD_GAP_FRACTION * params.offset, 1.0)
    except Exception as e:
        print("   ccd failed", e, flush=True); break
    have = True
    L.ibf_clamp_state(N, _lib.dev_ptr(xx), _lib.dev_ptr(xh), a, st)
    beta = beta_update(beta, a, p - 1, params.min_iterations)
    print(f"   alpha={a:.6f} beta={beta:.3e} C={len(aset)} blocking={ccd.n_blocking}", flush=True)
    if beta <= params.epsilon: break
