"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py [generator ...]   # default: all

Every output array below comes from calling `intact` functions from
/root/reference/pkg/src on seeded inputs (seed 20240611, the reference's own
fixture seed, tests/conftest.py:5-7).  The .npz files are committed; nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 20240611


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import intact  # noqa: F401
    return intact


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: " + ", ".join(f"{k}{tuple(np.shape(v))}" for k, v in arrays.items()))


def gen_distance(rng):
    from intact.distance import ee_eval, vf_eval
    n = 3000
    vf = rng.uniform(-1.0, 1.0, (n, 4, 3))
    ee = rng.uniform(-1.0, 1.0, (n, 4, 3))
    # exercise every Voronoi region: points placed around a fixed triangle
    tri = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    vf[:600, 1:] = tri
    vf[:600, 0] = rng.uniform(-0.7, 1.7, (600, 3)) * np.array([1.0, 1.0, 0.3])
    # degenerate: vertex on the triangle; coincident vertices
    vf[600:620, 0] = vf[600:620, 1]
    vf[620:640, 0] = 0.3 * vf[620:640, 1] + 0.3 * vf[620:640, 2] + 0.4 * vf[620:640, 3]
    # parallel and collinear edges, zero-length edges, crossing edges
    d = rng.standard_normal((200, 3))
    ee[:200, 1] = ee[:200, 0] + d
    ee[:200, 3] = ee[:200, 2] + 0.7 * d
    ee[200:260, 2] = ee[200:260, 0] + 0.25 * (ee[200:260, 1] - ee[200:260, 0])
    ee[200:260, 3] = ee[200:260, 0] + 1.5 * (ee[200:260, 1] - ee[200:260, 0])
    ee[260:280, 1] = ee[260:280, 0]
    ee[280:300, 3] = ee[280:300, 2]
    ee[300:330, 2] = 0.5 * (ee[300:330, 0] + ee[300:330, 1])
    out = {"vf_pts": vf, "ee_pts": ee}
    for tag, fn, pts in (("vf", vf_eval, vf), ("ee", ee_eval, ee)):
        d_, g, w, dg = fn(pts)
        out.update({f"{tag}_d": d_, f"{tag}_grad": g, f"{tag}_w": w, f"{tag}_degen": dg})
    save("distance.npz", **out)


def gen_accd(rng):
    from intact.ccd import accd_batch
    from intact.distance import PairKind
    out = {}
    for tag, kind in (("vf", PairKind.VERTEX_FACE), ("ee", PairKind.EDGE_EDGE)):
        n = 4000
        x0 = rng.uniform(-1.0, 1.0, (n, 4, 3))
        x1 = x0 + rng.uniform(-1.5, 1.5, (n, 4, 3))
        # small motions (no advancement), near-contact starts, zero motion
        x1[:500] = x0[:500] + rng.uniform(-1e-3, 1e-3, (500, 4, 3))
        x1[500:600] = x0[500:600]
        gap = np.where(np.arange(n) < 2000, 0.03, 1e-3)
        tois = np.empty(n)
        for g in np.unique(gap):
            sel = gap == g
            tois[sel] = accd_batch(kind, x0[sel], x1[sel], float(g))
        out.update({f"{tag}_x0": x0, f"{tag}_x1": x1, f"{tag}_gap": gap, f"{tag}_toi": tois})
    save("accd.npz", **out)


def _two_body_scene():
    from intact.mesh import compute_rest_data
    from intact.primitives import box_mesh, transformed
    a = box_mesh(4, 4, 2, size=(0.2, 0.2, 0.1))
    b = transformed(box_mesh(3, 3, 3, size=0.1), translate=(0.05, 0.05, 0.1015))
    return a, b, compute_rest_data(a, 1000.0), compute_rest_data(b, 1000.0)


def gen_broadphase(rng):
    from intact.ccd import candidate_pairs, max_step_size
    a, b, _, _ = _two_body_scene()
    off = a.n_verts
    x = np.vstack([a.rest_positions, b.rest_positions])
    tris = np.vstack([a.surface_tris, b.surface_tris + off])
    edges = np.vstack([a.surface_edges, b.surface_edges + off])
    verts = np.concatenate([a.surface_verts, b.surface_verts + off])
    out = {"x": x, "tris": tris, "edges": edges, "verts": verts}
    cases = []
    for c in range(4):
        x_hat = x.copy()
        x_hat[off:] += np.array([0.0, 0.0, -0.004 * (c + 1)]) + rng.uniform(-5e-4, 5e-4, (len(x) - off, 3))
        x_hat[:off] += rng.uniform(-2e-4, 2e-4, (off, 3))
        cases.append(x_hat)
    out["x_hat"] = np.stack(cases)
    gap = 1e-4
    out["min_gap"] = np.array(gap)
    for c, x_hat in enumerate(cases):
        vf, ee = candidate_pairs(x, x_hat, tris, edges, verts, gap)
        alpha, bl = max_step_size(x, x_hat, tris, edges, verts, gap, cap=1.0)
        out.update({f"vf{c}": vf, f"ee{c}": ee, f"alpha{c}": np.array(alpha),
                    f"bk{c}": bl.kinds, f"bq{c}": bl.indices, f"bt{c}": bl.tois})
    save("broadphase.npz", **out)


def gen_elastic(rng):
    from intact.elasticity import (Material, MaterialModel, element_gradients, energy_density,
                                   inversion_safe_step, pk1, psd_block_hessians)
    out = {}
    m = 200
    rows = rng.standard_normal((m, 4, 3))
    rows[:, 0] = -rows[:, 1:].sum(axis=1)
    vols = rng.uniform(0.5, 2.0, m)
    out["shape_rows"], out["volumes"] = rows, vols
    for model in MaterialModel:
        mat = Material(model, 1e5, 0.3)
        F = np.eye(3) + 0.3 * rng.standard_normal((m, 3, 3))
        if model == MaterialModel.NH:
            F[np.linalg.det(F) <= 0.05] = np.eye(3)
        else:
            F[:20, :, 2] *= -1.0   # inverted elements
        tag = model.value
        out[f"{tag}_F"] = F
        out[f"{tag}_psi"] = energy_density(mat, F)
        out[f"{tag}_P"] = pk1(mat, F)
        out[f"{tag}_grad"] = element_gradients(mat, F, rows, vols)
        out[f"{tag}_blocks"] = psd_block_hessians(mat, F, rows, vols)
    # inversion-safe step: NH unit tet squashed along -z (0.36 known answer)
    mat = Material(MaterialModel.NH, 1e5, 0.3)
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    inv = np.linalg.inv((x[1:] - x[0]).T)
    tr = np.empty((1, 4, 3))
    tr[0, 1:] = inv
    tr[0, 0] = -inv.sum(axis=0)
    tets = np.array([[0, 1, 2, 3]])
    ps = [np.zeros((4, 3)) for _ in range(3)]
    ps[0][3, 2] = -2.0
    ps[1][3] = [0.3, -0.2, -1.5]
    ps[2][1] = [-3.0, 0.1, 0.0]
    out["inv_x"], out["inv_rows"], out["inv_tets"] = x, tr, tets
    out["inv_p"] = np.stack(ps)
    out["inv_alpha"] = np.array([inversion_safe_step(mat, x, p, tets, tr) for p in ps])
    save("elastic.npz", **out)


def gen_sparse(rng):
    sys.path.insert(0, "/root/reference/pkg/tests")
    from test_sparse import random_clique_system
    from intact.sparse import clique_contributions, pcg_solve
    out = {}
    n, k = 40, 60
    cl = np.array([rng.choice(n, size=4, replace=False) for _ in range(k)])
    grids = np.empty((k, 4, 4, 3, 3))
    for c in range(k):
        a = rng.standard_normal((12, 12))
        grids[c] = (a @ a.T).reshape(4, 3, 4, 3).transpose(0, 2, 1, 3)
    r, c_, b = clique_contributions(cl, grids)
    out.update(cliques=cl, grids=grids, trip_rows=r, trip_cols=c_, trip_blocks=b)
    matrix, dense = random_clique_system(rng, 30, 25)
    out.update(rows=matrix.rows, cols=matrix.cols, blocks=matrix.blocks, dense=dense, n=np.array(30))
    xs = rng.standard_normal((4, 30, 3))
    out["mv_x"] = xs
    out["mv_y"] = np.stack([matrix.matvec(x) for x in xs])
    rhs = rng.standard_normal((30, 3))
    for tag, tol, cap in (("a", 1e-8, None), ("b", 1e-3, None), ("c", 1e-12, 5)):
        p, info = pcg_solve(matrix, rhs, tol, cap)
        out.update({f"pcg_{tag}_x": p, f"pcg_{tag}_info": np.array(
            [info.iterations, float(info.converged), info.rel_residual])})
    out["rhs"] = rhs
    save("sparse.npz", **out)


def gen_trajectory(rng):
    """A small SNH box dropped on a fixed LIN slab: per-step states and records."""
    from intact.contact import ActiveSet
    from intact.elasticity import Material, MaterialModel
    from intact.mesh import compute_rest_data
    from intact.primitives import box_mesh, transformed
    from intact.solver import ElasticRegion
    from intact.stepper import BoundaryCondition, Simulation, StepParams, System
    from intact.mesh import SimState
    slab = box_mesh(2, 2, 1, size=(0.3, 0.3, 0.05), origin=(-0.15, -0.15, -0.05))
    cube = transformed(box_mesh(3, 3, 3, size=0.1), translate=(-0.05, -0.05, 0.0025))
    bodies = [(slab, Material(MaterialModel.LIN, 1e7, 0.3)),
              (cube, Material(MaterialModel.SNH, 1e5, 0.3))]
    masses, regions, tris, edges, verts, xs = [], [], [], [], [], []
    off = 0
    for mesh, mat in bodies:
        rest = compute_rest_data(mesh, 1000.0)
        regions.append(ElasticRegion(mat, mesh.tets + off, rest.shape_rows, rest.volumes))
        masses.append(rest.masses)
        tris.append(mesh.surface_tris + off)
        edges.append(mesh.surface_edges + off)
        verts.append(mesh.surface_verts + off)
        xs.append(mesh.rest_positions)
        off += mesh.n_verts
    n_slab = slab.n_verts
    system = System(np.concatenate(masses), regions, np.vstack(tris), np.vstack(edges),
                    np.concatenate(verts), [BoundaryCondition(np.arange(n_slab))])
    x0 = np.vstack(xs)
    v0 = np.zeros_like(x0)
    v0[n_slab:, 2] = -0.5
    params = StepParams(h=0.01, offset=1e-3, min_iterations=2)
    sim = Simulation(system, params, SimState(x0.copy(), v0.copy()), ActiveSet())
    out = {"x0": x0, "v0": v0, "masses": system.masses, "tris": system.surface_triangles,
           "edges": system.surface_edges, "verts": system.surface_vertices,
           "n_slab": np.array(n_slab)}
    for i, reg in enumerate(regions):
        out[f"reg{i}_tets"] = reg.tets
        out[f"reg{i}_rows"] = reg.shape_rows
        out[f"reg{i}_vols"] = reg.volumes
    steps = 6
    xs_out, vs_out, recs, keys = [], [], [], []
    for _ in range(steps):
        d = sim.advance()
        xs_out.append(sim.state.x.copy())
        vs_out.append(sim.state.v.copy())
        recs.append(np.array([[r.alpha, r.beta, r.n_constraints, r.newton_iters, r.cg_iters]
                              for r in d.iterations]))
        keys.append(sorted(c.key for c in sim.active_set))
    out["xs"], out["vs"] = np.stack(xs_out), np.stack(vs_out)
    for i, r in enumerate(recs):
        out[f"rec{i}"] = r
        out[f"keys{i}"] = np.array([[k[0], *k[1]] for k in keys[i]], dtype=np.int64).reshape(-1, 5)
    save("trajectory.npz", **out)


def gen_activeset(rng):
    from intact.ccd import BlockingPairs
    from intact.contact import ActiveSet, admission_filter
    out = {}
    nv = 30
    aset = ActiveSet()
    for it in range(5):
        nb = 40
        kinds = rng.integers(0, 2, nb).astype(np.int64)
        quads = np.array([rng.choice(nv, 4, replace=False) for _ in range(nb)], dtype=np.int64)
        tois = np.round(rng.uniform(0.0, 1.0, nb), 1)   # many exact ties
        if it > 0:   # re-submit some resident pairs
            res = list(aset)[:5]
            for j, con in enumerate(res):
                kinds[j] = int(con.kind)
                quads[j] = con.indices
        adm, pruned = aset.update(BlockingPairs(kinds, quads, tois))
        for j, con in enumerate(aset):  # decay some weights to exercise pruning
            if j % 3 == 0:
                con.gamma *= 0.005 if it % 2 else 0.5
        out.update({f"k{it}": kinds, f"q{it}": quads, f"t{it}": tois,
                    f"adm{it}": np.array([adm, pruned]),
                    f"keys{it}": np.array([[int(c.kind), *c.indices] for c in aset],
                                          dtype=np.int64).reshape(-1, 5),
                    f"gamma{it}": np.array([c.gamma for c in aset])})
    quads = np.array([rng.choice(nv, 4, replace=False) for _ in range(200)])
    tois = np.round(rng.uniform(0, 1, 200), 2)
    out["af_q"], out["af_t"], out["af_keep"] = quads, tois, admission_filter(quads, tois)
    save("activeset.npz", **out)


def gen_intersect(rng):
    """static_intersection_test (intact/intersect.py:125-140) on two-body
    surfaces: interpenetrating, coplanar face contact, separated, jittered."""
    from intact.intersect import static_intersection_test
    from intact.primitives import box_mesh, sphere_mesh, transformed
    out = {}
    a = box_mesh(3, 3, 3, size=0.1)
    cases = [transformed(box_mesh(3, 3, 3, size=0.1), translate=(0.04, 0.03, 0.06)),   # interpenetrating
             transformed(box_mesh(2, 2, 2, size=0.1), translate=(0.0, 0.0, 0.1)),      # coplanar face contact
             transformed(box_mesh(3, 3, 3, size=0.1), translate=(0.0, 0.0, 0.1001)),   # separated by 1e-4
             transformed(sphere_mesh(3, radius=0.06), translate=(0.05, 0.05, 0.1))]    # sphere through a face
    for c, b in enumerate(cases):
        x = np.vstack([a.rest_positions, b.rest_positions])
        if c == 3:
            x = x + rng.uniform(-1e-4, 1e-4, x.shape)
        tris = np.vstack([a.surface_tris, b.surface_tris + a.n_verts])
        pairs = static_intersection_test(x, tris)
        pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))] if len(pairs) else pairs.reshape(0, 2)
        out.update({f"x{c}": x, f"tris{c}": tris, f"pairs{c}": pairs.astype(np.int64)})
    out["n"] = np.array(len(cases))
    save("intersect.npz", **out)


def gen_friction(rng):
    """intact/friction.py: mollifier and frames on grids; energy / gradient /
    Hessian of random frozen terms; and a box sliding on a slab with
    mu_f = 0.5 (per-step states, active sets and precomputed terms)."""
    from intact.friction import FrictionTerms, f0, f0_over_y, f0_second, friction_precompute, tangent_basis
    from intact.contact import ActiveSet
    from intact.elasticity import Material, MaterialModel
    from intact.mesh import SimState, compute_rest_data
    from intact.primitives import box_mesh, transformed
    from intact.solver import ElasticRegion
    from intact.stepper import BoundaryCondition, Simulation, StepParams, System
    out = {}
    eps = 1e-4
    y = np.concatenate([np.linspace(0.0, 3 * eps, 61), [1e-20, eps * (1 - 1e-12), eps * (1 + 1e-12)]])
    out.update(y=y, eps=np.array(eps), f0=f0(y, eps), f0y=f0_over_y(y, eps), f0s=f0_second(y, eps))
    nrm = rng.standard_normal((200, 3))
    nrm[:5] = np.eye(3)[[0, 1, 2, 0, 2]] * np.array([[1], [-1], [1], [-2], [3]])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    out.update(normals=nrm, frames=tangent_basis(nrm))
    k, n = 50, 40
    idx = np.array([rng.choice(n, 4, replace=False) for _ in range(k)])
    w = rng.uniform(-1, 1, (k, 4))
    nn = rng.standard_normal((k, 3))
    nn /= np.linalg.norm(nn, axis=1, keepdims=True)
    terms = FrictionTerms(indices=idx, weights=w, frames=tangent_basis(nn), coeff=rng.uniform(0.1, 2, k),
                          ref=rng.standard_normal((k, 3)) * 1e-3, eps=eps)
    xr = rng.standard_normal((n, 3)) * 1e-3
    xr[idx[:5]] = 0.0     # a few terms at exactly zero slip
    terms.ref[:5] = 0.0
    out.update(t_idx=idx, t_w=w, t_frames=terms.frames, t_coeff=terms.coeff, t_ref=terms.ref, t_x=xr,
               t_energy=np.array(terms.energy(xr)), t_grad=terms.gradient_terms(xr), t_hess=terms.hessian_grids(xr))
    # sliding box
    slab = box_mesh(2, 2, 1, size=(0.4, 0.4, 0.05), origin=(-0.2, -0.2, -0.05))
    cube = transformed(box_mesh(2, 2, 2, size=0.08), translate=(-0.04, -0.04, 0.0012))
    masses, regions, tris, edges, verts, xs = [], [], [], [], [], []
    off = 0
    for mesh, mat in ((slab, Material(MaterialModel.LIN, 1e7, 0.3)), (cube, Material(MaterialModel.SNH, 1e5, 0.3))):
        rest = compute_rest_data(mesh, 1000.0)
        regions.append(ElasticRegion(mat, mesh.tets + off, rest.shape_rows, rest.volumes))
        masses.append(rest.masses)
        tris.append(mesh.surface_tris + off)
        edges.append(mesh.surface_edges + off)
        verts.append(mesh.surface_verts + off)
        xs.append(mesh.rest_positions)
        off += mesh.n_verts
    n_slab = slab.n_verts
    system = System(np.concatenate(masses), regions, np.vstack(tris), np.vstack(edges), np.concatenate(verts),
                    [BoundaryCondition(np.arange(n_slab))])
    x0 = np.vstack(xs)
    v0 = np.zeros_like(x0)
    v0[n_slab:] = [0.8, 0.3, -0.4]
    params = StepParams(h=0.01, offset=1e-3, min_iterations=2, friction_coefficient=0.5, eps_v=1e-3)
    sim = Simulation(system, params, SimState(x0.copy(), v0.copy()), ActiveSet())
    out.update(s_xinit=x0, s_vinit=v0, s_masses=system.masses, s_tris=system.surface_triangles,
               s_edges=system.surface_edges, s_verts=system.surface_vertices, s_n_slab=np.array(n_slab))
    for i, reg in enumerate(regions):
        out[f"s_reg{i}_tets"], out[f"s_reg{i}_rows"], out[f"s_reg{i}_vols"] = reg.tets, reg.shape_rows, reg.volumes
    steps = 5
    for k_ in range(steps):
        diag = sim.advance()
        out[f"s_x{k_}"] = sim.state.x.copy()
        out[f"s_newton{k_}"] = np.array([r.newton_iters for r in diag.iterations])
        fr = diag.friction
        out[f"s_nfr{k_}"] = np.array(0 if fr is None else len(fr))
        if fr is not None:
            out.update({f"s_fidx{k_}": fr.indices, f"s_fw{k_}": fr.weights, f"s_ffr{k_}": fr.frames,
                        f"s_fc{k_}": fr.coeff, f"s_fref{k_}": fr.ref})
        cons = list(sim.active_set)
        out[f"s_akind{k_}"] = np.array([int(c.kind) for c in cons], dtype=np.int64)
        out[f"s_aquad{k_}"] = np.array([c.indices for c in cons], dtype=np.int64).reshape(-1, 4)
        out[f"s_alam{k_}"] = np.array([c.lam for c in cons])
        out[f"s_mu{k_}"] = np.array(diag.mu)
        # identical-input precompute from this step's state and multipliers
        fr2 = friction_precompute(sim.state.x, sim.active_set, diag.mu, diag.offset, params.h, 0.5, 1e-3)
        assert (fr2 is None and fr is None) or np.array_equal(fr2.coeff, fr.coeff)
    out["s_steps"] = np.array(steps)
    save("friction.npz", **out)


def _surface_meshes(rng):
    """Tet sets for surface extraction: a box, a sphere, two bodies in one
    index space, a random ragged subset (holes, non-manifold edges), one tet,
    and tets in shuffled order."""
    from intact.primitives import box_mesh, sphere_mesh
    box = box_mesh(4, 3, 5, size=0.1)
    sph = sphere_mesh(4, radius=0.3)
    two = np.vstack([box.tets, sph.tets + box.n_verts])
    sub = box.tets[rng.random(len(box.tets)) < 0.55]
    shuffled = box.tets[rng.permutation(len(box.tets))]
    return [box.tets, sph.tets, two, sub, box.tets[:1], shuffled]


def gen_sceneio(rng):
    """extract_surface_arrays (intact/mesh.py:106-124) on several tet sets, and
    the exact bytes export_frame (intact/io_utils.py:35-43) writes, with
    coordinates covering repr's layouts (tiny, huge, integral, negative zero)."""
    import tempfile
    from intact.io_utils import export_frame
    from intact.mesh import extract_surface_arrays
    from intact.primitives import box_mesh
    out = {}
    meshes = _surface_meshes(rng)
    for c, tets in enumerate(meshes):
        tris, edges, verts = extract_surface_arrays(tets)
        out.update({f"tets{c}": tets, f"tris{c}": tris, f"edges{c}": edges, f"verts{c}": verts})
    out["n_meshes"] = np.array(len(meshes))
    box = box_mesh(3, 2, 2, size=0.1)
    x = box.rest_positions + rng.standard_normal(box.rest_positions.shape) * 1e-3
    special = [0.0, -0.0, 1.0, -2.0, 1e-5, 1e-4, 0.0001234, 123456789012345.6, 1e16, 1e15, 2.5e-300, -1.7e308,
               0.1, 1 / 3, 5e-324, 1e22, 9007199254740993.0, 1.5]
    x[:len(special) // 3 * 3].flat[:len(special)] = special[:len(special) // 3 * 3]
    x = x.reshape(-1, 3)
    x[-6:] *= 10.0 ** rng.integers(-12, 18, (6, 1))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "frame.obj")
        export_frame(x, box.surface_tris, path)
        with open(path, "rb") as f:
            data = f.read()
        export_frame(x, np.zeros((0, 3), np.int64), path)
        with open(path, "rb") as f:
            empty = f.read()
    out.update({"obj_x": x, "obj_tris": box.surface_tris, "obj_bytes": np.frombuffer(data, np.uint8),
                "obj_empty_bytes": np.frombuffer(empty, np.uint8)})
    save("sceneio.npz", **out)


GENERATORS = ["distance", "accd", "broadphase", "elastic", "sparse", "activeset", "trajectory", "intersect",
              "friction", "sceneio"]


def main():
    only = sys.argv[1:] or GENERATORS
    _ref()
    if only != GENERATORS:
        for k, name in enumerate(GENERATORS):
            if name in only:
                globals()[f"gen_{name}"](np.random.default_rng(SEED + k))
        return
    gen_distance(np.random.default_rng(SEED))
    gen_accd(np.random.default_rng(SEED + 1))
    gen_broadphase(np.random.default_rng(SEED + 2))
    gen_elastic(np.random.default_rng(SEED + 3))
    gen_sparse(np.random.default_rng(SEED + 4))
    gen_activeset(np.random.default_rng(SEED + 5))
    gen_trajectory(np.random.default_rng(SEED + 6))
    gen_intersect(np.random.default_rng(SEED + 7))
    gen_friction(np.random.default_rng(SEED + 8))
    gen_sceneio(np.random.default_rng(SEED + 9))


if __name__ == "__main__":
    main()
