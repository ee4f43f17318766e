"""GPU parity of assembly, PCG, the Newton subproblem and whole steps against
the CPU oracle and the reference's golden trajectory (marked gpu).

Tolerances (FP64, stated per north star): gradients/matvecs 1e-9 relative
(different summation order); per-step positions 1e-5 relative; Newton counts
per outer pass within +-1; active-constraint key sets and penetration-free
states exact.
"""

import numpy as np
import pytest

from oracle import contact as ocontact, geometry, material, newton, timestep
from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_12151_b200 as p
    p._lib = __import__("paper_2512_12151_b200._lib", fromlist=["lib"])
    p._lib.lib()
    return p


def _traj_system(pkg, g):
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel, System
    from paper_2512_12151_b200.stepper import BoundaryCondition
    regions = [ElasticRegion(Material(MaterialModel.LIN, 1e7, 0.3), g["reg0_tets"], g["reg0_rows"], g["reg0_vols"]),
               ElasticRegion(Material(MaterialModel.SNH, 1e5, 0.3), g["reg1_tets"], g["reg1_rows"], g["reg1_vols"])]
    n_slab = int(g["n_slab"])
    return System(g["masses"], regions, g["tris"], g["edges"], g["verts"], [BoundaryCondition(np.arange(n_slab))])


def _oracle_regions(g):
    mu_l, lam_l = material.lame(1e7, 0.3)
    mu_s, lam_s = material.lame(1e5, 0.3)
    return [("lin", mu_l, lam_l, g["reg0_tets"], g["reg0_rows"], g["reg0_vols"]),
            ("snh", mu_s, lam_s, g["reg1_tets"], g["reg1_rows"], g["reg1_vols"])]


def _oracle_set_after(g, steps):
    scene = timestep.Scene(g["masses"], _oracle_regions(g), g["tris"], g["edges"], g["verts"],
                           [(np.arange(int(g["n_slab"])), None)])
    x, v = g["x0"].copy(), g["v0"].copy()
    aset = ocontact.ConstraintSet()
    for k in range(steps):
        x, v, _, _, _ = timestep.step(x, v, scene, aset, h=0.01, offset=1e-3, k_min=2, step_index=k)
    return x, v, aset


def test_assemble_with_contacts_matches_oracle(pkg, rng):
    from paper_2512_12151_b200.contact import ConstraintBatch
    from paper_2512_12151_b200.solver import assemble, incremental_energy
    g = golden("trajectory.npz")
    x, v, aset = _oracle_set_after(g, 2)
    aset.refresh_anchors(x)
    ob = aset.snapshot()
    assert len(ob) > 0
    x_tilde = x + 0.01 * v + 1e-4 * np.array([0, 0, -9.81])
    x_hat = x + 1e-4 * rng.standard_normal(x.shape)
    x_hat[: int(g["n_slab"])] = x[: int(g["n_slab"])]
    mu, off, h = 50.0, 1e-3, 0.01
    dbc = np.zeros(len(x), dtype=bool)
    dbc[: int(g["n_slab"])] = True
    go, Ho = newton.assemble(x_hat, x_tilde, g["masses"], _oracle_regions(g), ob, mu, off, h, dbc)
    sysm = _traj_system(pkg, g)
    batch = ConstraintBatch(ob.kind, ob.quad, ob.lam, ob.gamma, ob.anchor_d, ob.anchor_grad, ob.anchor_x)
    gg, Hg = assemble(x_hat, x_tilde, sysm.masses, sysm.regions, batch, mu, off, h, dbc)
    scale = np.abs(go).max()
    assert np.abs(gg - go).max() <= 1e-9 * scale
    for _ in range(4):
        p = rng.standard_normal(x.shape)
        yo, yg = Ho.matvec(p), Hg.matvec(p)
        assert np.abs(yg - yo).max() <= 1e-9 * np.abs(yo).max()
    eo = newton.energy(x_hat, x_tilde, g["masses"], _oracle_regions(g), ob, mu, off, h)
    eg = incremental_energy(x_hat, x_tilde, sysm.masses, sysm.regions, batch, mu, off, h)
    assert eg == pytest.approx(eo, rel=1e-12)


def test_pcg_sphere_compression(pkg):
    """Flattened sphere: PCG converges within 250 iterations and matches the
    oracle's iteration count (tests/test_solver.py:246-255)."""
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel
    from paper_2512_12151_b200.mesh import build_tet_mesh, compute_rest_data
    from paper_2512_12151_b200.scenes import cell_tets, grid_points
    from paper_2512_12151_b200.solver import DeviceSystem
    from paper_2512_12151_b200.device import to_dev, empty, to_host
    n = 6
    verts = grid_points(n, n, n, 2.0) - 1.0
    sup = np.abs(verts).max(axis=1)
    nrm = np.linalg.norm(verts, axis=1)
    verts = verts * np.where(nrm > 0.0, sup / np.maximum(nrm, 1e-300), 0.0)[:, None] * 0.5
    mesh = build_tet_mesh(verts, cell_tets(n, n, n))
    rest = compute_rest_data(mesh, 1000.0)
    x = mesh.rest_positions * np.array([1.0, 1.0, 0.72])
    mu_, lam_ = material.lame(1e5, 0.4)
    go, Ho = newton.assemble(x, x, rest.masses, [("snh", mu_, lam_, mesh.tets, rest.shape_rows, rest.volumes)],
                             None, 1.0, 0.0, 0.01)
    po, its, conv, _ = __import__("oracle.blocksparse", fromlist=["pcg"]).pcg(Ho, -go, 1e-4)
    reg = ElasticRegion(Material(MaterialModel.SNH, 1e5, 0.4), mesh.tets, rest.shape_rows, rest.volumes)
    dev = DeviceSystem(rest.masses, [reg])
    xd = to_dev(x)
    gd = empty(x.shape)
    dev.assemble(None, xd, xd, 1.0, 0.0, 0.01, False, gd)
    assert np.abs(to_host(gd) - go).max() <= 1e-9 * np.abs(go).max()
    rhs = -gd
    pd = empty(x.shape)
    it_g, conv_g, rel_g = dev.pcg(rhs, pd, 1e-4)
    assert conv and conv_g and it_g <= 250
    assert abs(it_g - its) <= 1
    np.testing.assert_allclose(to_host(pd), po, rtol=1e-6, atol=1e-9 * np.abs(po).max())


def test_pcg_large_system_matches_oracle(pkg):
    """A 19.7k-vertex compressed box: above the small-system threshold, so the
    solve takes the C4 path (one thread per row, residual carried on chip,
    split phase-B barrier) — iteration count within 1 of the oracle's and the
    same solution to 1e-6."""
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel
    from paper_2512_12151_b200.mesh import build_tet_mesh, compute_rest_data
    from paper_2512_12151_b200.scenes import cell_tets, grid_points
    from paper_2512_12151_b200.solver import DeviceSystem
    from paper_2512_12151_b200.device import to_dev, empty, to_host
    n = 26
    mesh = build_tet_mesh(grid_points(n, n, n, 0.5), cell_tets(n, n, n))
    assert mesh.n_verts > 16384
    rest = compute_rest_data(mesh, 1000.0)
    x = mesh.rest_positions * np.array([1.0, 1.0, 0.8])
    mu_, lam_ = material.lame(1e5, 0.4)
    go, Ho = newton.assemble(x, x, rest.masses, [("snh", mu_, lam_, mesh.tets, rest.shape_rows, rest.volumes)],
                             None, 1.0, 0.0, 0.01)
    po, its, conv, _ = __import__("oracle.blocksparse", fromlist=["pcg"]).pcg(Ho, -go, 1e-4)
    reg = ElasticRegion(Material(MaterialModel.SNH, 1e5, 0.4), mesh.tets, rest.shape_rows, rest.volumes)
    dev = DeviceSystem(rest.masses, [reg])
    xd = to_dev(x)
    gd = empty(x.shape)
    dev.assemble(None, xd, xd, 1.0, 0.0, 0.01, False, gd)
    assert np.abs(to_host(gd) - go).max() <= 1e-9 * np.abs(go).max()
    pd = empty(x.shape)
    it_g, conv_g, _ = dev.pcg(-gd, pd, 1e-4)
    assert conv and conv_g
    assert abs(it_g - its) <= 1
    np.testing.assert_allclose(to_host(pd), po, rtol=1e-6, atol=1e-9 * np.abs(po).max())


def test_plane_settle_kkt(pkg):
    """tests/test_solver.py:196-227: converged state one offset above the
    plane, |c| contracts geometrically, lambda = 0.3, DBC rows bit-pinned."""
    from paper_2512_12151_b200.contact import ActiveSet, Constraint
    from paper_2512_12151_b200.distance import PairKind
    from paper_2512_12151_b200.solver import solve_subproblem
    x0 = np.array([[0.4, 0.4, 0.05], [0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [0.0, 2.0, 0.0]])
    masses = np.ones(4)
    dbc = np.array([False, True, True, True])
    x_tilde = x0.copy()
    x_tilde[0, 2] = -0.2
    active = ActiveSet()
    active.ensure(4)
    active.add(Constraint(kind=PairKind.VERTEX_FACE, indices=np.array([0, 1, 2, 3])))
    mu, offset = 10.0, 0.1
    x_hat = x0.copy()
    viol = []
    for _ in range(12):
        res = solve_subproblem(x_tilde, x0, x_hat, masses, [], active, mu=mu, offset=offset, h=0.01, cg_tol=1e-12,
                               decay=0.9, dbc_mask=dbc)
        x_hat = res.x_hat
        viol.append(res.worst_violation)
        assert np.array_equal(x_hat[1:], x0[1:])
    v = np.array(viol)
    live = v > 1e-9
    assert (v[1:][live[:-1]] / v[:-1][live[:-1]] < 0.9).all()
    assert v.min() < 1e-8
    assert x_hat[0, 2] == pytest.approx(offset, abs=1e-6)
    lam = active.export_state()[2][0]
    assert lam == pytest.approx(0.3, rel=1e-5)


def _min_distance(x, tris, edges, verts):
    """Smallest VF / EE distance over all non-adjacent surface pairs (oracle)."""
    vf = np.array([[v, *t] for v in verts for t in tris if v not in t])
    ee = np.array([[*a, *b] for i, a in enumerate(edges) for b in edges[i + 1:] if not set(a) & set(b)])
    return min(geometry.pair_dist(0, x[vf]).min(), geometry.pair_dist(1, x[ee]).min())


def test_trajectory_matches_reference(pkg):
    """Six steps of the golden box-on-slab drop: positions within 1e-5
    relative, Newton counts +-1 per pass, identical active key sets,
    penetration-free states."""
    from paper_2512_12151_b200 import Simulation, StepParams
    from paper_2512_12151_b200.mesh import SimState
    g = golden("trajectory.npz")
    system = _traj_system(pkg, g)
    sim = Simulation(system, StepParams(h=0.01, offset=1e-3, min_iterations=2), SimState(g["x0"].copy(),
                                                                                         g["v0"].copy()))
    scale = np.abs(g["xs"]).max()
    for k in range(len(g["xs"])):
        d = sim.advance()
        x = sim.state.x
        assert np.abs(x - g["xs"][k]).max() <= 1e-5 * scale, k
        ref = g[f"rec{k}"]
        got = np.array([[r.alpha, r.beta, r.n_constraints, r.newton_iters, r.cg_iters] for r in d.iterations])
        assert len(got) == len(ref)
        assert np.all(np.abs(got[:, 3] - ref[:, 3]) <= 1)
        np.testing.assert_allclose(got[:, 0], ref[:, 0], rtol=1e-6, atol=1e-9)
        keys = sorted(c.key for c in sim.active_set)
        assert np.array_equal(np.array([[kk[0], *kk[1]] for kk in keys]).reshape(-1, 5), g[f"keys{k}"])
        assert _min_distance(x, g["tris"], g["edges"], g["verts"]) > 0.0


def _oracle_scene(system):
    regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
               for r in system.regions]
    return timestep.Scene(system.masses, regions, system.surface_triangles, system.surface_edges,
                          system.surface_vertices,
                          [(bc.vertices, bc.trajectory if bc.kind == "scripted" else None) for bc in system.boundary])


def test_c1_per_pass_sets_on_identical_inputs(pkg):
    """C1 (NH cube on a slab, 4.8k tets), every outer pass of two frames:
    fed the oracle's exact (x, x_hat, blocking, resident set), the GPU's
    ActiveSet.update yields the identical key list (same order) and
    max_step_size the identical alpha and blocking (kind, quad, TOI) set."""
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.ccd import BlockingPairs
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.device import to_dev
    system, state, params = scenes.c1_scene()
    scene = _oracle_scene(system)
    x, v = state.x.copy(), state.v.copy()
    aset = ocontact.ConstraintSet()
    trace = []
    for k in range(2):
        x, v, _, _, _ = timestep.step(x, v, scene, aset, h=params.h, offset=params.offset,
                                      k_min=params.min_iterations, step_index=k, trace=trace)
    n = system.n_vertices
    ccd = system.ccd
    n_block = 0
    for rec in trace:
        kind, quad, gamma = rec["resident"]
        ga = ActiveSet()
        ga.ensure(n)
        z = np.zeros(len(kind))
        ga.import_state(kind, quad, z, gamma, z, z, np.zeros((len(kind), 4, 3)), np.zeros((len(kind), 4, 3)))
        ga.update(BlockingPairs(*rec["blocking"]))
        gk, gq = ga.export_state()[:2]
        assert np.array_equal(gk, rec["updated"][0]) and np.array_equal(gq, rec["updated"][1])
        alpha = ccd.max_step_size(to_dev(rec["x"]), to_dev(rec["x_hat"]), rec["min_gap"], rec["cap"])
        assert alpha == rec["alpha"]
        bl = ccd.blocking()
        ok, oq, ot = rec["new_blocking"]
        assert {(int(a), tuple(b), c) for a, b, c in zip(bl.kinds, bl.indices.tolist(), bl.tois)} == \
            {(int(a), tuple(b), c) for a, b, c in zip(ok, oq.tolist(), ot)}
        n_block += len(ot)
    assert n_block > 0 and len(trace) >= 4


def _run_both(system, state, params, steps, perturb=0.0):
    from paper_2512_12151_b200 import Simulation
    scene = _oracle_scene(system)
    x, v = state.x.copy(), state.v.copy()
    if perturb:
        rng = np.random.default_rng(3)
        free = ~system.dbc_mask
        v[free] *= 1.0 + perturb * rng.standard_normal(v[free].shape)
    aset = ocontact.ConstraintSet()
    sim = Simulation(system, params, state.copy())
    out = []
    for k in range(steps):
        x, v, rec, _, _ = timestep.step(x, v, scene, aset, h=params.h, offset=params.offset,
                                        k_min=params.min_iterations, step_index=k)
        d = sim.advance()
        out.append((sim.state.x.copy(), x.copy(), d, rec, sorted(c.key for c in sim.active_set),
                    sorted(ocontact.key_of(kd, q) for kd, q in zip(aset.kind, aset.quad))))
    return out


@pytest.mark.parametrize("seed", [0, 1])
def test_generic_drop_trajectory_matches_oracle(pkg, seed):
    """Randomised C1-like drops (C5 generator: rotated cube, no symmetric
    TOI ties): positions within 1e-5 relative per step, same number of outer
    passes, Newton counts +-1, identical active key sets."""
    from paper_2512_12151_b200 import scenes
    system, state, params = scenes.c5_scene(seed, nx=5, ny=5, nz=4)
    for xg, xo, d, rec, kg, ko in _run_both(system, state, params, 3):
        assert np.abs(xg - xo).max() <= 1e-5 * np.abs(xo).max()
        assert len(d.iterations) == len(rec)
        assert all(abs(a.newton_iters - b[3]) <= 1 for a, b in zip(d.iterations, rec))
        assert kg == ko


def test_axis_aligned_drop_tie_sensitivity(pkg):
    """The axis-aligned drop sits on exact TOI ties (symmetric pairs tie in
    the admission filter, intact/contact.py:151).  The reference itself then
    moves ~1e-4 under a 1e-15 input perturbation; the GPU lands on that
    perturbed branch (agreeing to 1e-8), i.e. its deviation from the
    unperturbed oracle is the reference's own conditioning, not an error."""
    from paper_2512_12151_b200 import scenes
    system, state, params = scenes.c1_scene(nx=3, ny=3, nz=3, size=0.1, height=0.002, speed=0.5)
    base = _run_both(system, state, params, 2)
    pert = _run_both(system, state, params, 2, perturb=1e-15)
    for (xg, xo, _, _, kg, _), (_, xp, _, _, _, kp) in zip(base, pert):
        scale = np.abs(xo).max()
        assert np.abs(xg - xp).max() <= 1e-8 * scale
        assert kg == kp


@pytest.mark.parametrize("n,layers,frames", [(16, 1, 8), (12, None, 6)])
def test_contact_heavy_subproblem_parity(pkg, n, layers, frames):
    """Evolve a small C4 scene on the GPU until hundreds of constraints are
    active, then solve one AL subproblem from that exact state on both the
    GPU and the oracle: identical Newton counts, CG counts within the
    stopping test's rounding sensitivity, x_hat within 1e-5 relative,
    identical gamma, multipliers within the propagated position bound."""
    import torch
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.device import to_dev, to_host
    from paper_2512_12151_b200.stepper import step_device
    system, state, params = scenes.c4_scene(n=n, layers=layers, plate_speed=0.25)
    aset = ActiveSet()
    aset.ensure(system.n_vertices)
    x = torch.from_numpy(state.x).cuda()
    v = torch.from_numpy(state.v).cuda()
    for k in range(frames):
        x, v, _ = step_device(x, v, system, aset, params, step_index=k)
    assert len(aset) > 50
    dev = system.device
    xt, vt, h = to_host(x), to_host(v), params.h
    x_tilde = xt + h * vt + (h * h) * np.array(params.gravity)
    mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, h)
    x_hat0 = xt.copy()
    for bc in system.boundary:
        if bc.kind == "scripted":
            x_hat0[bc.vertices] = bc.targets(None, frames)
    st = aset.export_state()
    o = ocontact.ConstraintSet()
    o._append(st[0], st[1], [ocontact.key_of(a, b) for a, b in zip(st[0], st[1])], lam=st[2], gamma=st[3],
              s=st[4], anchor_d=st[5], anchor_grad=st[6], anchor_x=st[7])
    regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
               for r in system.regions]
    o2 = ocontact.ConstraintSet()
    o2._append(st[0], st[1], [ocontact.key_of(a, b) for a, b in zip(st[0], st[1])], lam=st[2].copy(),
               gamma=st[3].copy(), s=st[4].copy(), anchor_d=st[5], anchor_grad=st[6], anchor_x=st[7])
    xo, nwo, cgo, _, wo = newton.subproblem(x_tilde, xt, x_hat0, system.masses, regions, o, mu, params.offset, h,
                                            dbc=system.dbc_mask)
    # the oracle's own rounding sensitivity: same solve from x_tilde perturbed by 1e-15 relative
    pert = x_tilde * (1.0 + 1e-15 * np.random.default_rng(1).standard_normal(x_tilde.shape))
    xo2, _, cgo2, _, _ = newton.subproblem(pert, xt, x_hat0, system.masses, regions, o2, mu, params.offset, h,
                                           dbc=system.dbc_mask)
    xh = to_dev(x_hat0)
    nw, cg, _, w = dev.solve_subproblem(aset, to_dev(x_tilde), x, xh, mu, params.offset, h, params.cg_tol,
                                        params.decay)
    xg = to_host(xh)
    assert nw == nwo
    # CG counts: the stopping test compares a slowly decaying residual (with a
    # restart every 250 iterations) against 1e-4 |b|, so its crossing point is
    # rounding-sensitive; bound by 2 % or twice the oracle's own spread.
    assert abs(cg - cgo) <= max(1, 2 * abs(cgo2 - cgo), int(0.02 * cgo)), (cg, cgo, cgo2)
    # positions: the north star's per-step bar (1e-5 relative).  Two CG runs
    # that stop on either side of the 1e-4 residual test legitimately differ
    # by up to ~cond * 1e-4 of the step, so a bound relative to the step
    # would test rounding luck, not parity.
    assert np.abs(xg - xo).max() <= 1e-5 * np.abs(xo).max()
    # ... and against the oracle's own spread: the GPU's deviation from the
    # oracle must be of the size the oracle moves by under a 1e-15 relative
    # input perturbation (its CG stops on a rounding-sensitive test too)
    err = np.abs(xg - xo).max()
    spread = np.abs(xo2 - xo).max()
    step = np.abs(xo - xt).max()
    print(f"\n[parity] n={n}: C={len(aset)} newton {nw}/{nwo} cg {cg}/{cgo} (perturbed oracle {cgo2}); "
          f"max|dx| {err:.3e} = {err / step:.3e} of the step = {err / params.offset:.3e} of delta; "
          f"oracle spread {spread:.3e}")
    assert err <= max(10.0 * spread, 1e-12 * np.abs(xo).max()), (err, spread)
    sg = aset.export_state()
    assert np.array_equal(sg[3], o.gamma)
    # lambda <- lambda - mu c with c = d + grad_d . (x_hat - anchor) - offset
    # (intact/contact.py:91-106): a position difference dx propagates as
    # |dc| <= sum_k |w_k| |dx_k|_2 <= 2 sqrt(3) max|dx| (witness weights sum
    # to 2 in absolute value), so the multipliers and the worst violation can
    # only agree to that bound — a relative bound on lambda alone is wrong
    # for constraints whose c is near zero.
    dc = 2.0 * np.sqrt(3.0) * np.abs(xg - xo).max()
    assert np.abs(sg[2] - o.lam).max() <= mu * dc + 1e-12 * np.abs(o.lam).max()
    assert abs(w - wo) <= dc + 1e-12 * abs(wo)


def _fr_system(pkg, g):
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel, System
    from paper_2512_12151_b200.stepper import BoundaryCondition
    regions = [ElasticRegion(Material(MaterialModel.LIN, 1e7, 0.3), g["s_reg0_tets"], g["s_reg0_rows"],
                             g["s_reg0_vols"]),
               ElasticRegion(Material(MaterialModel.SNH, 1e5, 0.3), g["s_reg1_tets"], g["s_reg1_rows"],
                             g["s_reg1_vols"])]
    return System(g["s_masses"], regions, g["s_tris"], g["s_edges"], g["s_verts"],
                  [BoundaryCondition(np.arange(int(g["s_n_slab"])))])


def test_friction_precompute_matches_reference(pkg):
    """friction_precompute on the device from the reference's accepted states
    and multipliers (intact/friction.py:103-151): same terms in the same
    order, witness weights bit-identical."""
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.friction import friction_precompute
    g = golden("friction.npz")
    for k in range(int(g["s_steps"])):
        kinds, quads, lam = g[f"s_akind{k}"], g[f"s_aquad{k}"], g[f"s_alam{k}"]
        n = len(kinds)
        aset = ActiveSet()
        aset.ensure(len(g["s_masses"]))
        aset.import_state(kinds, quads, lam, np.ones(n), np.zeros(n), np.zeros(n), np.zeros((n, 4, 3)),
                          np.zeros((n, 4, 3)))
        ft = friction_precompute(g[f"s_x{k}"], aset, float(g[f"s_mu{k}"]), 1e-3, 0.01, 0.5, 1e-3)
        nf = int(g[f"s_nfr{k}"])
        assert (0 if ft is None else len(ft)) == nf
        if nf:
            assert np.array_equal(ft.indices, g[f"s_fidx{k}"])
            assert np.array_equal(ft.weights, g[f"s_fw{k}"])
            np.testing.assert_allclose(ft.frames, g[f"s_ffr{k}"], rtol=0, atol=1e-14)
            np.testing.assert_allclose(ft.coeff, g[f"s_fc{k}"], rtol=1e-12)
            np.testing.assert_allclose(ft.ref, g[f"s_fref{k}"], rtol=1e-13, atol=1e-16)
            assert ft.eps == pytest.approx(1e-5)


def test_assemble_and_energy_with_friction(pkg, rng):
    """Friction terms in the gradient, the (matrix-free) Hessian and the
    incremental energy vs the oracle (FP64, 1e-9 / 1e-12 relative)."""
    from oracle import friction as ofriction
    from paper_2512_12151_b200.solver import assemble, incremental_energy
    g = golden("friction.npz")
    system = _fr_system(pkg, g)
    k = 2
    fo = ofriction.FrictionSet(g[f"s_fidx{k}"], g[f"s_fw{k}"], g[f"s_ffr{k}"], g[f"s_fc{k}"], g[f"s_fref{k}"], 1e-5)
    x = g[f"s_x{k}"]
    x_tilde = x + 1e-4 * rng.standard_normal(x.shape)
    x_hat = x + 1e-4 * rng.standard_normal(x.shape)        # slips across the eps = 1e-5 kink
    n_slab = int(g["s_n_slab"])
    x_hat[:n_slab] = x[:n_slab]
    dbc = system.dbc_mask
    mu_l, lam_l = material.lame(1e7, 0.3)
    mu_s, lam_s = material.lame(1e5, 0.3)
    oregions = [("lin", mu_l, lam_l, g["s_reg0_tets"], g["s_reg0_rows"], g["s_reg0_vols"]),
                ("snh", mu_s, lam_s, g["s_reg1_tets"], g["s_reg1_rows"], g["s_reg1_vols"])]
    go, Ho = newton.assemble(x_hat, x_tilde, system.masses, oregions, None, 1.0, 1e-3, 0.01, dbc, friction=fo)
    gg, Hg = assemble(x_hat, x_tilde, system.masses, system.regions, None, 1.0, 1e-3, 0.01, dbc, friction=fo)
    assert np.abs(gg - go).max() <= 1e-9 * np.abs(go).max()
    for _ in range(3):
        p = rng.standard_normal(x.shape)
        yo, yg = Ho.matvec(p), Hg.matvec(p)
        assert np.abs(yg - yo).max() <= 1e-9 * np.abs(yo).max()
    eo = newton.energy(x_hat, x_tilde, system.masses, oregions, None, 1.0, 1e-3, 0.01, friction=fo)
    eg = incremental_energy(x_hat, x_tilde, system.masses, system.regions, None, 1.0, 1e-3, 0.01, friction=fo)
    assert eg == pytest.approx(eo, rel=1e-12)


def test_sliding_box_with_friction_matches_reference(pkg):
    """Five steps of the box sliding on the slab with mu_f = 0.5 through
    Simulation (friction threaded step to step): positions within 1e-5
    relative of the reference, same number of friction terms per step."""
    from paper_2512_12151_b200 import Simulation, StepParams
    from paper_2512_12151_b200.mesh import SimState
    g = golden("friction.npz")
    system = _fr_system(pkg, g)
    params = StepParams(h=0.01, offset=1e-3, min_iterations=2, friction_coefficient=0.5, eps_v=1e-3)
    sim = Simulation(system, params, SimState(g["s_xinit"].copy(), g["s_vinit"].copy()))
    scale = np.abs(g["s_xinit"]).max()
    for k in range(int(g["s_steps"])):
        d = sim.advance()
        assert np.abs(sim.state.x - g[f"s_x{k}"]).max() <= 1e-5 * scale, k
        assert (0 if d.friction is None else len(d.friction)) == int(g[f"s_nfr{k}"]), k
        assert np.array_equal(np.array([r.newton_iters for r in d.iterations]), g[f"s_newton{k}"])


def _jittered(state, system, amp=1e-7, seed=5):
    """Break the exact TOI ties of axis-aligned stacks (admission compares
    TOIs for equality, intact/contact.py:151) with a sub-micron jitter of the
    free vertices."""
    from paper_2512_12151_b200.mesh import SimState
    x = state.x.copy()
    free = ~system.dbc_mask
    x[free] += amp * np.random.default_rng(seed).standard_normal(x[free].shape)
    return SimState(x, state.v.copy())


def test_c2_stack_small_matches_oracle(pkg):
    """Reduced C2 (2x2x2 cubes falling into the pinned five-slab box):
    positions 1e-5 relative per step, equal pass counts, Newton +-1,
    identical active key sets."""
    from paper_2512_12151_b200 import scenes
    system, state, params = scenes.c2_scene(grid=2, cells=(3, 3, 3), size=(0.03, 0.03, 0.03), gap=0.001)
    state = _jittered(state, system)
    out = _run_both(system, state, params, 5)
    assert max(len(kg) for *_, kg, _ in out) > 0
    for xg, xo, d, rec, kg, ko in out:
        assert np.abs(xg - xo).max() <= 1e-5 * np.abs(xo).max()
        assert len(d.iterations) == len(rec)
        assert all(abs(a.newton_iters - b[3]) <= 1 for a, b in zip(d.iterations, rec))
        assert kg == ko


def test_c3_twisted_rods_small_matches_oracle(pkg):
    """Reduced C3 (two NH rods, end layers twisted in opposite senses by
    rotational scripted Dirichlet conditions): same checks as C2."""
    from paper_2512_12151_b200 import scenes
    system, state, params = scenes.c3_scene(rows=1, cols=2, cells=(2, 2, 12), size=(0.02, 0.02, 0.12), gap=0.001,
                                            omega=6 * np.pi)
    state = _jittered(state, system)
    out = _run_both(system, state, params, 5)
    assert max(len(kg) for *_, kg, _ in out) > 0
    for xg, xo, d, rec, kg, ko in out:
        assert np.abs(xg - xo).max() <= 1e-5 * np.abs(xo).max()
        assert len(d.iterations) == len(rec)
        assert all(abs(a.newton_iters - b[3]) <= 1 for a, b in zip(d.iterations, rec))
        assert kg == ko


def test_reference_composition_through_mirror(pkg, rng):
    """The reference's own Newton-step composition (intact/solver.py:209-219)
    through the mirror: grad, H = assemble(...); p = pcg_solve(H, -grad, tol);
    descent safeguard -inv(H.diagonal_blocks()) grad.  H is a
    BlockSparseMatrix-compatible object whose explicit blocks include the
    contact cliques (intact/solver.py:144-148) and the DBC mask
    (intact/sparse.py:81-87)."""
    from paper_2512_12151_b200.contact import ConstraintBatch
    from paper_2512_12151_b200.solver import assemble
    from paper_2512_12151_b200.sparse import pcg_solve
    from oracle.blocksparse import pcg as opcg
    g = golden("trajectory.npz")
    x, v, aset = _oracle_set_after(g, 2)
    aset.refresh_anchors(x)
    ob = aset.snapshot()
    assert len(ob) > 0
    x_tilde = x + 0.01 * v + 1e-4 * np.array([0, 0, -9.81])
    x_hat = x + 1e-4 * rng.standard_normal(x.shape)
    n_slab = int(g["n_slab"])
    x_hat[:n_slab] = x[:n_slab]
    mu, off, h = 50.0, 1e-3, 0.01
    dbc = np.zeros(len(x), dtype=bool)
    dbc[:n_slab] = True
    go, Ho = newton.assemble(x_hat, x_tilde, g["masses"], _oracle_regions(g), ob, mu, off, h, dbc)
    sysm = _traj_system(pkg, g)
    batch = ConstraintBatch(ob.kind, ob.quad, ob.lam, ob.gamma, ob.anchor_d, ob.anchor_grad, ob.anchor_x)
    gg, Hg = assemble(x_hat, x_tilde, sysm.masses, sysm.regions, batch, mu, off, h, dbc)
    # explicit matrix: same coalesced (row, col) keys, blocks to 1e-10 of the largest
    assert np.array_equal(Hg.rows, Ho.rows) and np.array_equal(Hg.cols, Ho.cols)
    scale = np.abs(Ho.blocks).max()
    err_blocks = np.abs(Hg.blocks - Ho.blocks).max() / scale
    assert err_blocks <= 1e-10, err_blocks
    np.testing.assert_allclose(Hg.diagonal_blocks(), Ho.diag(), rtol=0, atol=1e-10 * scale)
    # pcg_solve on the assembled matrix (device operator, contacts matrix-free)
    p, info = pcg_solve(Hg, -gg, 1e-4)
    po, its, conv, _ = opcg(Ho, -go, 1e-4)
    assert info.converged and conv and abs(info.iterations - its) <= 1
    err_p = np.abs(p - po).max() / np.abs(po).max()
    assert err_p <= 1e-6, err_p
    # descent safeguard as the reference writes it
    pre = np.linalg.inv(Hg.diagonal_blocks())
    ps = -np.einsum("nij,nj->ni", pre, gg)
    pso = -np.einsum("nij,nj->ni", np.linalg.inv(Ho.diag()), go)
    assert np.abs(ps - pso).max() <= 1e-9 * np.abs(pso).max()
    # a second mask_dirichlet (here: also pin the top layer) detaches the explicit matrix
    top = x[:, 2] >= np.sort(x[:, 2])[-20]
    diag = g["masses"][:, None, None] * np.eye(3)
    Ho.mask(top, diag)
    Hg.mask_dirichlet(top, diag)
    q = rng.standard_normal(x.shape)
    assert np.abs(Hg.matvec(q) - Ho.matvec(q)).max() <= 1e-10 * np.abs(Ho.matvec(q)).max()
    p2, info2 = pcg_solve(Hg, -gg, 1e-4)
    po2, its2, _, _ = opcg(Ho, -go, 1e-4)
    assert abs(info2.iterations - its2) <= 1
    assert np.abs(p2 - po2).max() <= 1e-6 * np.abs(po2).max()
    print(f"explicit blocks err {err_blocks:.1e}, pcg its {info.iterations}/{its}, p err {err_p:.1e}")


def _squishy_press_state(fric, min_constraints, max_frames=120):
    """A reduced squishy-ball press (scenes.squishy_scene: five 22k-tet balls
    in the pinned box) stepped on the GPU until at least `min_constraints`
    constraints are active."""
    import torch
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.stepper import StepParams, step_device
    system, state, params = scenes.squishy_scene(cell=0.01, n=12, stem=10, tip=6, plate_speed=2.0, plate_stop=0.16)
    if fric:
        params = StepParams(h=params.h, offset=params.offset, min_iterations=2, friction_coefficient=fric,
                            eps_v=1e-3)
    aset = ActiveSet()
    aset.ensure(system.n_vertices)
    x = torch.from_numpy(state.x).cuda()
    v = torch.from_numpy(state.v).cuda()
    ft = None
    k = 0
    while len(aset) < min_constraints:
        assert k < max_frames, f"only {len(aset)} constraints after {k} frames"
        x, v, d = step_device(x, v, system, aset, params, step_index=k, friction=ft)
        ft = d.friction
        k += 1
    return system, params, aset, x, v, ft, k


@pytest.mark.parametrize("fric,pmat", [(0.0, False), (0.3, False), (0.0, True), (0.3, True)])
def test_production_pcg_path_subproblem_parity(pkg, fric, pmat, monkeypatch):
    """The PCG configuration of the C4 bench — one thread per row, several
    row sweeps per thread with the last sweep dealt out by slices, residual
    carried on chip, split phase-B barrier, contact (and friction) dots behind
    the ld.acquire ready counter — on one AL subproblem of a squishy-ball
    press state with >= 5k active constraints, vs the oracle
    (intact/solver.py:178-233, intact/sparse.py:99-150).  The grid is capped
    at 12 CTAs so each thread sweeps >= 4 rows.  Bars: equal Newton counts,
    CG counts within 2x the oracle's own spread under a 1e-15 input
    perturbation (or 2 %), positions within 4x that spread (or 1e-9 of the
    step), identical gamma, multipliers within the propagated bound.  With
    pmat the direction is materialised behind a third barrier (the C4 bench's
    configuration at >= 0.2 contact terms per row)."""
    from oracle import friction as ofriction
    monkeypatch.setenv("IBF_PCG_PMAT_RATIO", "0" if pmat else "1e9")
    from paper_2512_12151_b200 import _lib
    from paper_2512_12151_b200.device import to_dev, to_host
    system, params, aset, x, v, ft, frames = _squishy_press_state(fric, 5000)
    dev = system.device
    xt, vt, h = to_host(x), to_host(v), params.h
    x_tilde = xt + h * vt + (h * h) * np.array(params.gravity)
    mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, h)
    x_hat0 = xt.copy()
    for bc in system.boundary:
        if bc.kind == "scripted":
            x_hat0[bc.vertices] = bc.targets(None, frames)
    st = aset.export_state()
    fo = None
    if fric:
        assert ft is not None and len(ft) >= 500
        fo = ofriction.FrictionSet(ft.indices, ft.weights, ft.frames, ft.coeff, ft.ref, ft.eps)
    regions = [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes)
               for r in system.regions]

    def oracle_run(xtil):
        o = ocontact.ConstraintSet()
        o._append(st[0], st[1], [ocontact.key_of(a, b) for a, b in zip(st[0], st[1])], lam=st[2].copy(),
                  gamma=st[3].copy(), s=st[4].copy(), anchor_d=st[5], anchor_grad=st[6], anchor_x=st[7])
        out = newton.subproblem(xtil, xt, x_hat0, system.masses, regions, o, mu, params.offset, h,
                                dbc=system.dbc_mask, friction=fo)
        return out, o

    (xo, nwo, cgo, _, wo), o = oracle_run(x_tilde)
    pert = x_tilde * (1.0 + 1e-15 * np.random.default_rng(1).standard_normal(x_tilde.shape))
    (xo2, _, cgo2, _, _), _ = oracle_run(pert)
    dev.set_friction(ft if fric else None)
    xh = to_dev(x_hat0)
    try:
        with _lib.pcg_tuning(lanes_max_n=0, max_ctas=12):
            nw, cg, _, w = dev.solve_subproblem(aset, to_dev(x_tilde), x, xh, mu, params.offset, h, params.cg_tol,
                                                params.decay)
            shape = _lib.pcg_last_shape()
    finally:
        dev.set_friction(None)
    ctas, threads, sweeps, lanes, ready, terms = shape
    assert lanes == 1 and ctas == 12 and sweeps >= 2 and ready == 1, shape
    assert terms >= len(st[0]) + (len(ft) if fric else 0) >= 5000, shape
    xg = to_host(xh)
    step = np.abs(xo - x_hat0).max()
    spread = np.abs(xo2 - xo).max()
    err = np.abs(xg - xo).max()
    print(f"\n[production PCG path, fric={fric}] frames {frames}, constraints {len(st[0])}, "
          f"friction terms {len(ft) if fric else 0}, shape {shape}; Newton {nw}/{nwo}; CG {cg}/{cgo} "
          f"(oracle spread {abs(cgo2 - cgo)}); max|dx| {err:.3e} = {err / step:.2e} of the step "
          f"= {err / params.offset:.2e} of the offset; oracle spread {spread:.3e}")
    assert nw == nwo
    assert abs(cg - cgo) <= max(1, 2 * abs(cgo2 - cgo), int(0.02 * cgo)), (cg, cgo, cgo2)
    if cg == cgo:
        # same stopping iteration: the GPU must sit within the oracle's own
        # rounding spread
        assert err <= max(4.0 * spread, 1e-9 * step), (err, spread, step)
    else:
        # the stopping test (|r| <= 1e-4 |b|) fired at a different iteration:
        # the iterates differ by the last CG corrections, so the bar is the
        # north star's per-step 1e-5 relative, and at most the CG tolerance
        # times the step
        assert err <= min(1e-5 * np.abs(xo).max(), 1e-4 * step), (err, step, cg, cgo)
    sg = aset.export_state()
    assert np.array_equal(sg[3], o.gamma)
    dc = 2.0 * np.sqrt(3.0) * err
    assert np.abs(sg[2] - o.lam).max() <= mu * dc + 1e-12 * np.abs(o.lam).max()
    assert abs(w - wo) <= dc + 1e-12 * abs(wo)


def test_press_state_step_limit_and_update_on_identical_inputs(pkg):
    """One outer pass's max_step_size and ActiveSet.update on a squishy-ball
    press state with >= 5k constraints (intact/ccd.py:168-193,
    intact/contact.py:179-205): fed identical (x, x_hat, blocking, resident
    set), alpha is bit-equal, the blocking (kind, quad, TOI) sets are equal,
    and the updated key sequences are identical."""
    from paper_2512_12151_b200.ccd import BlockingPairs
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.device import to_dev, to_host
    from oracle import geometry
    system, params, aset, x, v, _, frames = _squishy_press_state(0.0, 5000)
    xt = to_host(x)
    # a trial x_hat: the inertial target, which moves every free vertex
    x_hat = xt + params.h * to_host(v) + params.h ** 2 * np.array(params.gravity)
    x_hat[system.dbc_mask] = xt[system.dbc_mask]
    gap = 0.1 * params.offset
    ccd = system.ccd
    alpha = ccd.max_step_size(x, to_dev(x_hat), gap, 1.0)
    bl = ccd.blocking()
    ao, ok, oq, ot = geometry.step_limit(xt, x_hat, system.surface_triangles, system.surface_edges,
                                         system.surface_vertices, gap)
    assert alpha == ao
    gset = {(int(a), tuple(b), c) for a, b, c in zip(bl.kinds, bl.indices.tolist(), bl.tois)}
    assert gset == {(int(a), tuple(b), c) for a, b, c in zip(ok, oq.tolist(), ot)}
    assert len(ot) > 100
    st = aset.export_state()
    o = ocontact.ConstraintSet()
    o._append(st[0], st[1], [ocontact.key_of(a, b) for a, b in zip(st[0], st[1])], lam=st[2], gamma=st[3],
              s=st[4], anchor_d=st[5], anchor_grad=st[6], anchor_x=st[7])
    ga = ActiveSet()
    ga.ensure(system.n_vertices)
    ga.import_state(*st)
    res_g = ga.update(BlockingPairs(ok, oq, ot))
    res_o = o.update(ok, oq, ot)
    gk, gq = ga.export_state()[:2]
    print(f"\n[press pass] frames {frames}, resident {len(st[0])}, alpha {alpha:.6e}, blocking {len(ot)}, "
          f"admitted/pruned GPU {res_g} oracle {res_o}, set size {len(gk)}")
    assert tuple(res_g) == tuple(res_o)
    assert np.array_equal(gk, np.asarray(o.kind)) and np.array_equal(gq, np.asarray(o.quad))


@pytest.mark.parametrize("parts", [2, 3])
def test_partitioned_pcg_matches_unpartitioned(pkg, parts):
    """The row-partitioned PCG (csrc/pcg.cu pcg_solve_dist)
    with `parts` local partitions on one GPU — each partition holds its own
    z / p / r / x vectors, computes H p on its rows only, keeps p on its
    halo, and receives the other partitions' z rows by device copies; the
    scalars are summed in partition order — against the single-GPU
    persistent kernel on the same assembled operator (reduced squishy-ball
    press, >= 5k matrix-free contact terms), then through one whole AL
    subproblem.  Only the reduction order differs, so: equal CG counts (+-1)
    and solutions within 1e-10 relative; equal Newton counts and x_hat
    within 1e-9 of the step for the subproblem (intact/sparse.py:99-150,
    intact/solver.py:178-233)."""
    from paper_2512_12151_b200 import dist
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.device import empty, to_host
    system, params, aset, x, v, _, frames = _squishy_press_state(0.0, 5000)
    dev = system.device
    n = system.n_vertices
    h = params.h
    x_tilde = x + h * v
    mu = params.stiffness_constant * dev.stiffness_diagonal_max(x, h)
    aset.refresh_anchors(x)
    g = empty((n, 3))
    dev.assemble(aset, x, x_tilde, mu, params.offset, h, True, g)
    rhs = -g
    x1, x2 = empty((n, 3)), empty((n, 3))
    it1, conv1, rel1 = dev.pcg(rhs, x1, params.cg_tol)
    part = dist.Partition.local_parts(parts)
    dev.set_dist(part)
    try:
        it2, conv2, rel2 = dev.pcg(rhs, x2, params.cg_tol)
    finally:
        dev.set_dist(None)
    a, b = to_host(x1), to_host(x2)
    err = np.abs(a - b).max() / np.abs(a).max()
    print(f"\n[partitioned PCG x{parts}] rows {n}, ranges {part.row_ranges(n)}, constraints {len(aset)}: "
          f"CG {it2} vs {it1}, rel residual {rel2:.3e} vs {rel1:.3e}, max rel diff {err:.2e}")
    assert conv1 and conv2 and abs(it1 - it2) <= 1
    assert err <= 1e-10
    # one AL subproblem (Newton loop + dual sweep) through the partition
    st = aset.export_state()
    runs = []
    for use in (None, part):
        a_set = ActiveSet()
        a_set.import_state(*st)
        a_set.ensure(n)
        xh = x.clone()
        dev.set_dist(use)
        try:
            nw, cg, _, _ = dev.solve_subproblem(a_set, x_tilde, x, xh, mu, params.offset, h, params.cg_tol,
                                                params.decay)
        finally:
            dev.set_dist(None)
        runs.append((nw, cg, to_host(xh), a_set.export_state()))
    (n1, c1, xa, sa), (n2, c2, xb, sb) = runs
    step = np.abs(xa - to_host(x)).max()
    dx = np.abs(xa - xb).max()
    print(f"[partitioned subproblem x{parts}] Newton {n2} vs {n1}, CG {c2} vs {c1}, max|dx| {dx:.2e} = "
          f"{dx / step:.2e} of the step")
    assert n1 == n2 and abs(c1 - c2) <= n1
    assert dx <= 1e-9 * step
    assert np.array_equal(sa[3], sb[3])                        # gamma: same dual branches


@pytest.mark.gpu
@pytest.mark.parametrize("scene", ["c5", "squishy"])
def test_native_outer_loop_matches_python(pkg, scene, monkeypatch):
    """Alg. 1's outer passes in native code (ibf_outer_loop) against the
    Python loop over the same native calls (stepper._outer_loop,
    intact/stepper.py:283-347): bit-identical states and identical per-pass
    records (alpha, beta, constraints, Newton and CG counts) over several
    frames of a C5 drop and of a reduced squishy-ball press."""
    import torch
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.contact import ActiveSet
    from paper_2512_12151_b200.stepper import step_device
    if scene == "c5":
        system, state, params = scenes.c5_scene(3)
        frames = 12
    else:
        system, state, params = scenes.squishy_scene(cell=0.01, n=12, stem=10, tip=6, plate_speed=2.0,
                                                     plate_stop=0.16)
        frames = 14
    runs = []
    for py in (False, True):
        if py:
            monkeypatch.setenv("IBF_PY_OUTER", "1")
        else:
            monkeypatch.delenv("IBF_PY_OUTER", raising=False)
        aset = ActiveSet()
        aset.ensure(system.n_vertices)
        x = torch.from_numpy(state.x).cuda()
        v = torch.from_numpy(state.v).cuda()
        recs = []
        for k in range(frames):
            x, v, d = step_device(x, v, system, aset, params, step_index=k)
            recs.append([(r.alpha, r.beta, r.n_constraints, r.newton_iters, r.cg_iters) for r in d.iterations])
        runs.append((x.cpu().numpy(), v.cpu().numpy(), recs, len(aset)))
    (xn, vn, rn, cn), (xp, vp, rp, cp) = runs
    print(f"\n[native outer loop, {scene}] {frames} frames, passes {sum(len(r) for r in rn)}, constraints {cn}")
    assert np.array_equal(xn, xp) and np.array_equal(vn, vp)
    assert rn == rp and cn == cp
