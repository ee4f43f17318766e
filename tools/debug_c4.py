"""Run the C4 scene at small resolution frame by frame and print per-pass records (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes, _lib
from paper_2512_12151_b200.stepper import step_device
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import to_host
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
speed = float(sys.argv[3]) if len(sys.argv) > 3 else 0.25
layers = int(os.environ.get('LAYERS', '1'))
system, state, params = scenes.c4_scene(n=n, plate_speed=speed, layers=layers)
aset = ActiveSet(); aset.ensure(system.n_vertices)
x = torch.from_numpy(state.x).cuda(); v = torch.from_numpy(state.v).cuda()
print("verts", system.n_vertices, "tets", sum(len(r.tets) for r in system.regions), "tris", len(system.surface_triangles), flush=True)
for k in range(frames):
    t = time.time()
    try:
        x, v, d = step_device(x, v, system, aset, params, step_index=k)
    except Exception as e:
        print("frame", k, "failed:", e, flush=True); break
    torch.cuda.synchronize()
    xs = to_host(x)
    print(f"frame {k}: {time.time()-t:.2f}s passes={len(d.iterations)} max|x|={np.abs(xs).max():.4f} mu={d.mu:.3e}", flush=True)
    if len(sys.argv) > 4:
        for r in d.iterations[:12]:
            print(f"   a={r.alpha:.6f} b={r.beta:.3e} C={r.n_constraints} nw={r.newton_iters} cg={r.cg_iters} ms={r.wall_ms:.1f}", flush=True)
    else:
        print(f"   newton={sum(r.newton_iters for r in d.iterations)} cg={sum(r.cg_iters for r in d.iterations)} C={d.iterations[-1].n_constraints} minalpha={min(r.alpha for r in d.iterations):.4f}", flush=True)
    st = np.zeros(3); _lib.lib().ibf_ccd_stats(system.ccd.handle, _lib.host_ptr(st), 1); print("   ccd", st, flush=True)
