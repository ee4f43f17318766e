"""Dev tool: PCG cost with the matrix-free contact terms on a pressed
squishy-ball state (scenes.squishy_scene).

    python tools/pcg_contact_bench.py [--frames 30] [--cell 0.02] [--plate-speed 2.0] [--load f.npz]

Presses the scene for --frames frames (or loads a squishy_run --dump), then
assembles at the accepted state with and without the active set and times
k_spmv and k_pcg per iteration on both operators, and prints the contact
incidence statistics (constraints per vertex) that set the row imbalance.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_12151_b200 import _lib, scenes
from paper_2512_12151_b200.contact import ActiveSet
from paper_2512_12151_b200.device import empty, to_dev
from paper_2512_12151_b200.stepper import step_device

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=30)
ap.add_argument("--cell", type=float, default=0.02)
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--stem", type=int, default=23)
ap.add_argument("--tip", type=int, default=16)
ap.add_argument("--numbering", default="lattice", choices=["sell", "lattice", "morton"])
ap.add_argument("--plate-speed", type=float, default=2.0)
ap.add_argument("--load", default=None)
ap.add_argument("--dump", default=None)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--ncu", action="store_true", help="profile one PCG launch (cudaProfilerStart/Stop)")
ap.add_argument("--reorder", action="store_true", help="Morton vertex numbering instead of the lattice's")
args = ap.parse_args()

system, state, params = scenes.squishy_scene(numbering=args.numbering, cell=args.cell, n=args.n, stem=args.stem, tip=args.tip,
                                             plate_speed=args.plate_speed, reorder=args.reorder)
aset = ActiveSet()
aset.ensure(system.n_vertices)
x, v = to_dev(state.x), to_dev(state.v)
k0 = 0
if args.load:
    z = np.load(args.load)
    x, v, k0 = to_dev(z["x"]), to_dev(z["v"]), int(z["frame"])
    aset.import_state(*(z[f"a{j}"] for j in range(8)))
t = time.perf_counter()
for k in range(k0, k0 + args.frames):
    x, v, d = step_device(x, v, system, aset, params, step_index=k)
torch.cuda.synchronize()
print(json.dumps({"frames": args.frames, "press_s": time.perf_counter() - t, "constraints": len(aset)}), flush=True)
if args.dump:
    st = aset.export_state()
    np.savez(args.dump, x=x.cpu().numpy(), v=v.cpu().numpy(), frame=k0 + args.frames,
             **{f"a{j}": a for j, a in enumerate(st)})

dev = system.device
N = system.n_vertices
st = aset.export_state()
quad = st[1]
cnt = np.bincount(quad.ravel(), minlength=N)
cnt[system.dbc_mask] = 0
nz = cnt[cnt > 0]
inc = {"constraints": int(len(quad)), "rows_with_terms": int(len(nz)), "incidences": int(nz.sum()),
       "max_per_row": int(nz.max()) if len(nz) else 0,
       "p50_per_row": float(np.percentile(nz, 50)) if len(nz) else 0,
       "p99_per_row": float(np.percentile(nz, 99)) if len(nz) else 0}
# per-warp imbalance: max over the 32 rows of a warp vs their mean
w = cnt[: (N // 32) * 32].reshape(-1, 32)
inc["warp_max_sum"] = int(w.max(axis=1).sum() * 32)
inc["warp_divergence_factor"] = float(w.max(axis=1).sum() * 32 / max(w.sum(), 1))
print(json.dumps({"incidence": inc}), flush=True)

xt = to_dev(state.x) if False else x.clone()
x_tilde = x + params.h * v
mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, params.h)
g = empty((N, 3))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
p = torch.randn((N, 3), dtype=torch.float64, device="cuda")
y = empty((N, 3))
xo = empty((N, 3))
out = {"N": N, "mu": mu}
for label, a in (("no_contacts", None), ("contacts", aset)):
    if a is not None:
        a.refresh_anchors(x)
    dev.assemble(a, x, x_tilde, mu, params.offset, params.h, True, g)
    for _ in range(3):
        dev.matvec(p, y)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        dev.matvec(p, y)
    e1.record()
    torch.cuda.synchronize()
    out[f"{label}_spmv_ms"] = e0.elapsed_time(e1) / 20
    rhs = -g
    dev.pcg(rhs, xo, 1e-30, 10)
    torch.cuda.synchronize()
    if args.ncu and a is not None:
        torch.cuda.profiler.start()
    e0.record()
    it, conv, rel = dev.pcg(rhs, xo, 1e-30, args.iters)
    e1.record()
    torch.cuda.synchronize()
    if args.ncu and a is not None:
        torch.cuda.profiler.stop()
    out[f"{label}_pcg_us_per_iter"] = 1e3 * e0.elapsed_time(e1) / max(it, 1)
    out[f"{label}_pcg_iters"] = it
# assembly with the active set: whole call and per kernel (ibf_kernel_clocks)
aset.refresh_anchors(x)
for _ in range(2):
    dev.assemble(aset, x, x_tilde, mu, params.offset, params.h, True, g)
torch.cuda.synchronize()
_lib.kernel_clocks(on=1, reset=True)
e0.record()
for _ in range(10):
    dev.assemble(aset, x, x_tilde, mu, params.offset, params.h, True, g)
e1.record()
torch.cuda.synchronize()
kc = _lib.kernel_clocks(on=0)
out["assembly_ms"] = e0.elapsed_time(e1) / 10
out["assembly_kernels_us"] = {k: round(1e3 * v["ms"] / max(v["launches"], 1), 1) for k, v in kc.items() if v["launches"]}
out["spmv_bytes"] = dev.spmv_bytes()
out["bytes_per_cg_iter"] = out["spmv_bytes"] + 288.0 * N
out["contacts_GBps"] = out["bytes_per_cg_iter"] / out["contacts_pcg_us_per_iter"] / 1e3
out["no_contacts_GBps"] = out["bytes_per_cg_iter"] / out["no_contacts_pcg_us_per_iter"] / 1e3
out["shape"] = _lib.pcg_last_shape()
print(json.dumps(out), flush=True)
