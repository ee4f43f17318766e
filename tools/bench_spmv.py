"""Microbenchmark: SpMV alone and PCG per-iteration cost on the C4 matrix (dev tool)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.device import to_dev, empty
n = int(sys.argv[1]) if len(sys.argv) > 1 else 42
system, state, params = scenes.c4_scene(n=n)
dev = system.device
N = system.n_vertices
x = to_dev(state.x)
xt = to_dev(state.x + 1e-4 * np.random.default_rng(0).standard_normal(state.x.shape))
g = empty((N, 3))
dev.assemble(None, x, xt, 1.0, 1e-3, 0.01, True, g)
p = torch.randn((N, 3), dtype=torch.float64, device="cuda")
y = empty((N, 3))
for _ in range(5): dev.matvec(p, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 50
e0.record()
for _ in range(R): dev.matvec(p, y)
e1.record(); torch.cuda.synchronize()
t_spmv = e0.elapsed_time(e1) / R
b = dev.spmv_bytes()
out = {"N": N, "blocks": dev.n_blocks, "spmv_ms": t_spmv, "spmv_GBps": b / t_spmv / 1e6, "spmv_bytes": b}
for _ in range(3): dev.assemble(None, x, xt, 1.0, 1e-3, 0.01, True, g)
torch.cuda.synchronize()
e0.record()
for _ in range(10): dev.assemble(None, x, xt, 1.0, 1e-3, 0.01, True, g)
e1.record(); torch.cuda.synchronize()
out["assemble_ms"] = e0.elapsed_time(e1) / 10
rs = np.ones(2)
e0.record()
for _ in range(10): dev.energy(None, x, xt, 1.0, 1e-3, 0.01, p=g, rs=(1.0, 0.5))
e1.record(); torch.cuda.synchronize()
out["energy2_ms"] = e0.elapsed_time(e1) / 10
rhs = -g
xo = empty((N, 3))
dev.pcg(rhs, xo, 1e-30, 20)
torch.cuda.synchronize()
for its in (100, 400):
    e0.record(); it, conv, rel = dev.pcg(rhs, xo, 1e-30, its); e1.record(); torch.cuda.synchronize()
    out[f"pcg_{its}_ms_per_iter"] = e0.elapsed_time(e1) / it
    out[f"pcg_{its}_GBps"] = (b + 288 * N) / (e0.elapsed_time(e1) / it) / 1e6
print(json.dumps(out))
