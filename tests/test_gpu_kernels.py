"""GPU parity of the individual kernels against the reference's golden vectors
and the CPU oracle (run on a B200; marked gpu).

Bit-exact: distances, ACCD TOIs, broad-phase candidate sets, blocking pairs,
active-set keys, BSR coalescing.  FP64 tolerance (stated per test):
element Hessian blocks, gradients, matvec, PCG iterates.
"""

import numpy as np
import pytest

from oracle import blocksparse, contact as ocontact, geometry, material
from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ibf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_12151_b200 as pkg
    from paper_2512_12151_b200 import _lib
    _lib.lib()
    return pkg


def test_distance_bit_exact(ibf):
    from paper_2512_12151_b200 import distance
    g = golden("distance.npz")
    for tag, fn in (("vf", distance.vf_eval), ("ee", distance.ee_eval)):
        d, grad, w, dg = fn(g[f"{tag}_pts"])
        assert np.array_equal(d, g[f"{tag}_d"])
        assert np.array_equal(grad, g[f"{tag}_grad"])
        assert np.array_equal(w, g[f"{tag}_w"])
        assert np.array_equal(dg, g[f"{tag}_degen"])


def test_accd_bit_exact(ibf):
    from paper_2512_12151_b200 import ccd
    g = golden("accd.npz")
    for tag, kind in (("vf", 0), ("ee", 1)):
        gap = g[f"{tag}_gap"]
        for val in np.unique(gap):
            sel = gap == val
            toi = ccd.accd_batch(kind, g[f"{tag}_x0"][sel], g[f"{tag}_x1"][sel], float(val))
            assert np.array_equal(toi, g[f"{tag}_toi"][sel])


def test_accd_known_answers(ibf):
    """tests/test_ccd.py:19-53 of the reference."""
    from paper_2512_12151_b200 import ccd
    tri = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    x0 = np.vstack([[0.2, 0.2, 1.0], tri])
    x1 = x0.copy()
    x1[0, 2] -= 2.0
    a = ccd.accd_toi(0, x0, x1, 0.0)
    assert 0.5 * 0.9 - 1e-12 <= a <= 0.5
    x1 = x0.copy()
    x1[0, 0] += 3.0
    assert ccd.accd_toi(0, x0, x1, 0.0) == 1.0
    assert ccd.accd_toi(0, x0, x0, 0.01) == 1.0
    x0 = np.vstack([[0.2, 0.2, 0.05], tri])
    x1 = x0.copy()
    x1[0, 2] -= 1.0
    assert ccd.accd_toi(0, x0, x1, 0.05) == 0.0


def _keyset(quads, kind):
    return {(kind, tuple(sorted(q))) for q in np.asarray(quads).tolist()}


def test_broadphase_sets_and_step_limit(ibf):
    from paper_2512_12151_b200 import ccd
    g = golden("broadphase.npz")
    x, tris, edges, verts = g["x"], g["tris"], g["edges"], g["verts"]
    gap = float(g["min_gap"])
    for c in range(len(g["x_hat"])):
        xh = g["x_hat"][c]
        vf, ee = ccd.candidate_pairs(x, xh, tris, edges, verts, gap)
        assert {tuple(q) for q in vf.tolist()} == {tuple(q) for q in g[f"vf{c}"].tolist()}
        assert {tuple(q) for q in ee.tolist()} == {tuple(q) for q in g[f"ee{c}"].tolist()}
        assert len(vf) == len(g[f"vf{c}"]) and len(ee) == len(g[f"ee{c}"])
        alpha, bl = ccd.max_step_size(x, xh, tris, edges, verts, gap)
        assert alpha == float(g[f"alpha{c}"])
        ref = {(int(k), tuple(q), t) for k, q, t in zip(g[f"bk{c}"], g[f"bq{c}"].tolist(), g[f"bt{c}"])}
        got = {(int(k), tuple(q), t) for k, q, t in zip(bl.kinds, bl.indices.tolist(), bl.tois)}
        assert got == ref


def test_broadphase_large_random(ibf):
    """LBVH candidate set == brute force on a scene with thousands of prims."""
    from paper_2512_12151_b200 import ccd, scenes
    mesh = scenes.box_mesh(8, 8, 3, size=(0.4, 0.4, 0.1))
    rng = np.random.default_rng(7)
    x0 = mesh.rest_positions + rng.uniform(-0.004, 0.004, mesh.rest_positions.shape)
    x1 = x0 + rng.uniform(-0.01, 0.01, x0.shape)
    gap = 2e-3
    vf, ee = ccd.candidate_pairs(x0, x1, mesh.surface_tris, mesh.surface_edges, mesh.surface_verts, gap)
    rvf, ree = geometry.candidates(x0, x1, mesh.surface_tris, mesh.surface_edges, mesh.surface_verts, gap)
    assert {tuple(q) for q in vf.tolist()} == {tuple(q) for q in rvf.tolist()}
    assert {tuple(q) for q in ee.tolist()} == {tuple(q) for q in ree.tolist()}
    alpha, bl = ccd.max_step_size(x0, x1, mesh.surface_tris, mesh.surface_edges, mesh.surface_verts, gap)
    ra, rk, rq, rt = geometry.step_limit(x0, x1, mesh.surface_tris, mesh.surface_edges, mesh.surface_verts, gap)
    assert alpha == ra
    assert {(int(k), tuple(q), t) for k, q, t in zip(bl.kinds, bl.indices.tolist(), bl.tois)} == \
        {(int(k), tuple(q), t) for k, q, t in zip(rk, rq.tolist(), rt)}


def test_broadphase_refit_across_calls(ibf):
    """One CCD handle over 40 calls on a drifting, deforming scene: the VF/EE
    trees are refit between rebuilds (every 16 calls, csrc/ccd.cu), and every
    call's candidate set and step limit must still equal brute force."""
    from paper_2512_12151_b200 import ccd, scenes
    from paper_2512_12151_b200.device import to_dev
    mesh = scenes.box_mesh(6, 6, 3, size=(0.3, 0.3, 0.1))
    rng = np.random.default_rng(11)
    t, e, v = mesh.surface_tris, mesh.surface_edges, mesh.surface_verts
    h = ccd.CCD(t, e, v)
    x = mesh.rest_positions + rng.uniform(-0.003, 0.003, mesh.rest_positions.shape)
    vel = rng.uniform(-0.01, 0.01, x.shape)
    gap = 2e-3
    for k in range(40):
        x1 = x + vel + rng.uniform(-0.002, 0.002, x.shape)
        vf, ee = h.candidates(to_dev(x), to_dev(x1), gap)
        rvf, ree = geometry.candidates(x, x1, t, e, v, gap)
        assert {tuple(q) for q in vf.tolist()} == {tuple(q) for q in rvf.tolist()}, k
        assert {tuple(q) for q in ee.tolist()} == {tuple(q) for q in ree.tolist()}, k
        alpha = h.max_step_size(to_dev(x), to_dev(x1), gap)
        ra, _, _, _ = geometry.step_limit(x, x1, t, e, v, gap)
        assert alpha == ra, k
        x = x + 0.5 * (x1 - x)     # drift: the scene moves between calls


def test_bsr_coalesce_matvec_pcg(ibf):
    from paper_2512_12151_b200.sparse import BlockSparseMatrix, clique_contributions, pcg_solve
    g = golden("sparse.npz")
    r, c, b = clique_contributions(g["cliques"], g["grids"])
    assert np.array_equal(r, g["trip_rows"]) and np.array_equal(c, g["trip_cols"])
    n = int(g["n"])
    # coalescing in key order with sequential sums is bit-identical
    A = BlockSparseMatrix(n, g["rows"], g["cols"], g["blocks"])
    assert np.array_equal(A.rows, g["rows"]) and np.array_equal(A.blocks, g["blocks"])
    for x, y in zip(g["mv_x"], g["mv_y"]):
        np.testing.assert_allclose(A.matvec(x), y, rtol=1e-12, atol=1e-12)   # tests/test_sparse.py:50-54
    for tag, tol, cap in (("a", 1e-8, None), ("b", 1e-3, None), ("c", 1e-12, 5)):
        x, info = pcg_solve(A, g["rhs"], tol, cap)
        ref = g[f"pcg_{tag}_info"]
        assert abs(info.iterations - int(ref[0])) <= 1 and info.converged == bool(ref[1])
        np.testing.assert_allclose(x, g[f"pcg_{tag}_x"], rtol=1e-6, atol=1e-9)
    # identity: one iteration, exact (tests/test_sparse.py:67-75)
    eye = BlockSparseMatrix(5, np.arange(5), np.arange(5), np.tile(np.eye(3), (5, 1, 1)))
    rhs = np.random.default_rng(1).standard_normal((5, 3))
    x, info = pcg_solve(eye, rhs, 1e-10)
    assert info.iterations == 1 and info.converged and np.allclose(x, rhs)
    x, info = pcg_solve(eye, np.zeros((5, 3)), 1e-10)
    assert info.iterations == 0 and info.converged and not np.any(x)


def test_pcg_restart_chain(ibf):
    """260-vertex chain needs > 250 iterations: exercises the restart
    (tests/test_sparse.py:148-161)."""
    from paper_2512_12151_b200.sparse import BlockSparseMatrix, pcg_solve
    n = 260
    rows, cols, blocks = [], [], []
    for i in range(n):
        rows.append(i), cols.append(i), blocks.append(2.0 * np.eye(3))
        if i + 1 < n:
            rows.append(i), cols.append(i + 1), blocks.append(-1.0 * np.eye(3))
    A = BlockSparseMatrix(n, np.array(rows), np.array(cols), np.array(blocks))
    rhs = np.zeros((n, 3))
    rhs[0] = 1.0
    rhs[-1] = -2.0
    x, info = pcg_solve(A, rhs, 1e-10)
    Ao = blocksparse.SymBlockMatrix(n, np.array(rows), np.array(cols), np.array(blocks))
    xo, its, conv, _ = blocksparse.pcg(Ao, rhs, 1e-10)
    assert info.converged == conv and abs(info.iterations - its) <= 1
    np.testing.assert_allclose(x, xo, rtol=1e-8, atol=1e-10)


def _disjoint_system(F, rows, vols, model):
    """M disjoint tets whose deformation gradients are the golden F."""
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel
    M = len(F)
    X = np.zeros((M, 4, 3))
    for m in range(M):
        Ar = rows[m, 1:]                      # rows A_1..A_3
        E = F[m] @ np.linalg.inv(Ar)          # columns x_k - x_0
        X[m, 1:] = E.T
    tets = np.arange(4 * M).reshape(M, 4)
    reg = ElasticRegion(Material(MaterialModel(model), 1e5, 0.3), tets, rows, vols)
    return X.reshape(-1, 3), reg


@pytest.mark.parametrize("model", ["snh", "nh", "cor", "lin"])
def test_element_hessian_blocks(ibf, model):
    """PSD 12x12 vertex blocks vs the reference's (tests/test_elasticity.py:271-280: 1e-10)."""
    from paper_2512_12151_b200.solver import DeviceSystem
    from paper_2512_12151_b200.device import to_dev, empty, to_host
    g = golden("elastic.npz")
    x, reg = _disjoint_system(g[f"{model}_F"], g["shape_rows"], g["volumes"], model)
    n = len(x)
    dev = DeviceSystem(np.ones(n), [reg])
    xd = to_dev(x)
    gr = empty((n, 3))
    dev.assemble(None, xd, xd, 1.0, 1.0, 1.0, False, gr)
    rows, cols, blocks = dev.export_bsr()
    ref = g[f"{model}_blocks"]                # (M,4,4,3,3), h = 1
    scale = np.abs(ref).max()
    for r, c, b in zip(rows, cols, blocks):
        t, i, j = r // 4, r % 4, c % 4
        want = ref[t, i, j] + (np.eye(3) if r == c else 0.0)
        assert np.abs(b - want).max() <= 1e-10 * scale, (model, r, c)
    np.testing.assert_allclose(to_host(gr).reshape(-1, 4, 3), g[f"{model}_grad"], rtol=1e-9,
                               atol=1e-9 * np.abs(g[f"{model}_grad"]).max())


def test_inversion_cap(ibf):
    from paper_2512_12151_b200 import ElasticRegion, Material, MaterialModel
    from paper_2512_12151_b200.solver import DeviceSystem
    from paper_2512_12151_b200.device import to_dev
    g = golden("elastic.npz")
    reg = ElasticRegion(Material(MaterialModel.NH, 1e5, 0.3), g["inv_tets"], g["inv_rows"], np.ones(1))
    dev = DeviceSystem(np.ones(4), [reg])
    for p, want in zip(g["inv_p"], g["inv_alpha"]):
        got = dev.inversion_safe_step(to_dev(g["inv_x"]), to_dev(p))
        assert got == pytest.approx(want, rel=1e-9)


def test_active_set_sequence(ibf):
    from paper_2512_12151_b200.ccd import BlockingPairs
    from paper_2512_12151_b200.contact import ActiveSet
    g = golden("activeset.npz")
    aset = ActiveSet()
    aset.ensure(30)
    for it in range(5):
        adm, pr = aset.update(BlockingPairs(g[f"k{it}"], g[f"q{it}"], g[f"t{it}"]))
        assert [adm, pr] == g[f"adm{it}"].tolist()
        st = list(aset.export_state())
        keys = np.concatenate([st[0][:, None], st[1]], axis=1)
        assert np.array_equal(keys, g[f"keys{it}"])       # same order, same insertion semantics
        gam = st[3]
        for j in range(len(gam)):
            if j % 3 == 0:
                gam[j] *= 0.005 if it % 2 else 0.5
        aset.import_state(*st)
        assert np.array_equal(aset.export_state()[3], g[f"gamma{it}"])


def test_refresh_and_dual_sweep_match_oracle(ibf, rng):
    from paper_2512_12151_b200.contact import ActiveSet
    n = 40
    x = rng.uniform(-1, 1, (n, 3))
    kinds = rng.integers(0, 2, 60)
    quads = np.array([rng.choice(n, 4, replace=False) for _ in range(60)])
    quads[0] = quads[1]                                    # duplicate key: first wins
    tois = rng.uniform(0, 1, 60)
    o = ocontact.ConstraintSet(admit_all=True)
    o.update(kinds, quads, tois)
    a = ActiveSet(admit_all=True)
    a.ensure(n)
    a.update(__import__("paper_2512_12151_b200.ccd", fromlist=["x"]).BlockingPairs(kinds, quads, tois))
    assert len(a) == len(o)
    assert o.refresh_anchors(x) == a.refresh_anchors(x)
    st = a.export_state()
    assert np.array_equal(st[5], o.anchor_d) and np.array_equal(st[6], o.anchor_grad)
    x_hat = x + 0.01 * rng.standard_normal(x.shape)
    o.lam[:] = rng.uniform(0, 1, len(o))
    st = list(st)
    st[2] = o.lam.copy()
    a.import_state(*st)
    w_o = o.dual_sweep(x_hat, 0.05, 10.0, 0.9)
    w_a = a.dual_update_sweep(x_hat, 0.05, 10.0, 0.9)
    assert w_a == w_o
    st = a.export_state()
    assert np.array_equal(st[2], o.lam) and np.array_equal(st[3], o.gamma) and np.array_equal(st[4], o.s)


def test_static_intersection_matches_reference(ibf):
    """GPU tri-tri test vs the reference's static_intersection_test
    (golden: interpenetrating, coplanar face contact, separated by 1e-4,
    jittered sphere through a face) and vs the oracle on a larger random
    two-body case."""
    from oracle import intersect as ointersect
    from paper_2512_12151_b200.intersect import static_intersection_test
    from paper_2512_12151_b200 import scenes
    g = golden("intersect.npz")
    for c in range(int(g["n"])):
        got = static_intersection_test(g[f"x{c}"], g[f"tris{c}"])
        assert np.array_equal(got, g[f"pairs{c}"]), c
    rng = np.random.default_rng(7)
    a = scenes.box_mesh(8, 8, 6, size=0.2)
    b = scenes.transformed(scenes.shell_sphere(10, 0.07, layers=2), translate=(0.1, 0.1, 0.17))
    x = np.vstack([a.rest_positions, b.rest_positions]) + rng.uniform(-1e-4, 1e-4, (a.n_verts + b.n_verts, 3))
    tris = np.vstack([a.surface_tris, b.surface_tris + a.n_verts])
    want = ointersect.intersecting_pairs(x, tris)
    assert len(want) > 0
    assert np.array_equal(static_intersection_test(x, tris), want)


def test_min_distance_monitor_matches_oracle(ibf):
    """Nearest VF/EE pair within a radius: distance bit-identical to the
    oracle (same pair_dist arithmetic), on separated boxes and on a random
    drop scene."""
    from oracle import intersect as ointersect
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.ccd import CCD
    from paper_2512_12151_b200.device import to_dev
    g = golden("intersect.npz")
    x, tris = g["x2"], g["tris2"]
    edges = np.unique(np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1), axis=0)
    verts = np.unique(tris)
    h = CCD(tris, edges, verts)
    for radius in (1e-3, 5e-5):
        d, kind, q = h.min_distance(to_dev(x), radius)
        do, ko, qo = ointersect.min_distance(x, tris, edges, verts, radius)
        assert d == do and kind == ko
    system, state, _ = scenes.c5_scene(3, nx=5, ny=5, nz=4)
    x = state.x + np.random.default_rng(2).uniform(-1e-3, 1e-3, state.x.shape)
    h = CCD(system.surface_triangles, system.surface_edges, system.surface_vertices)
    d, kind, q = h.min_distance(to_dev(x), 0.01)
    do, ko, qo = ointersect.min_distance(x, system.surface_triangles, system.surface_edges, system.surface_vertices,
                                         0.01)
    assert d == do and kind == ko
