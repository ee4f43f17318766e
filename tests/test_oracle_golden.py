"""Pin the CPU oracle against golden vectors produced by the reference itself.

Bit-exact for distance / ACCD / broad phase / active set (integer and exact
FP64 decisions); LAPACK-backed quantities to the reference's own tolerances.
"""

import numpy as np
import pytest

from oracle import blocksparse, contact, geometry, material, newton, timestep
from tests.conftest import golden


def test_distance_bit_exact():
    g = golden("distance.npz")
    for tag, kind in (("vf", geometry.VF), ("ee", geometry.EE)):
        d, grad, w, dg = geometry.pair_eval(kind, g[f"{tag}_pts"])
        assert np.array_equal(d, g[f"{tag}_d"])
        assert np.array_equal(grad, g[f"{tag}_grad"])
        assert np.array_equal(w, g[f"{tag}_w"])
        assert np.array_equal(dg, g[f"{tag}_degen"])
        assert np.array_equal(geometry.pair_dist(kind, g[f"{tag}_pts"]), g[f"{tag}_d"])


def test_accd_bit_exact():
    g = golden("accd.npz")
    for tag, kind in (("vf", geometry.VF), ("ee", geometry.EE)):
        gap = g[f"{tag}_gap"]
        for val in np.unique(gap):
            sel = gap == val
            toi = geometry.accd(kind, g[f"{tag}_x0"][sel], g[f"{tag}_x1"][sel], float(val))
            assert np.array_equal(toi, g[f"{tag}_toi"][sel])


def test_broadphase_and_step_limit_bit_exact():
    g = golden("broadphase.npz")
    x, tris, edges, verts = g["x"], g["tris"], g["edges"], g["verts"]
    gap = float(g["min_gap"])
    for c in range(len(g["x_hat"])):
        xh = g["x_hat"][c]
        vf, ee = geometry.candidates(x, xh, tris, edges, verts, gap)
        assert np.array_equal(vf, g[f"vf{c}"])          # same order, not just same set
        assert np.array_equal(ee, g[f"ee{c}"])
        alpha, kinds, quads, tois = geometry.step_limit(x, xh, tris, edges, verts, gap)
        assert alpha == float(g[f"alpha{c}"])
        assert np.array_equal(kinds, g[f"bk{c}"])
        assert np.array_equal(quads, g[f"bq{c}"])
        assert np.array_equal(tois, g[f"bt{c}"])


def test_bruteforce_equals_tree_query():
    g = golden("broadphase.npz")
    x, xh, tris = g["x"], g["x_hat"][0], g["tris"]
    lo, hi = geometry.swept_prim_boxes(x, xh, tris, 1e-4)
    vlo, vhi = geometry.swept_prim_boxes(x, xh, g["verts"], 0.0)
    a = set(zip(*geometry.BoxTree(lo, hi).query(vlo, vhi)))
    qi, ti = geometry._dense_overlaps(vlo, vhi, lo, hi)
    assert a == set(zip(qi.tolist(), ti.tolist()))


@pytest.mark.parametrize("model", ["snh", "nh", "cor", "lin"])
def test_elastic_terms(model):
    g = golden("elastic.npz")
    mu, lam = material.lame(1e5, 0.3)
    F = g[f"{model}_F"]
    rows, vols = g["shape_rows"], g["volumes"]
    np.testing.assert_allclose(material.psi(model, mu, lam, F), g[f"{model}_psi"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(material.stress(model, mu, lam, F), g[f"{model}_P"], rtol=1e-10, atol=1e-7)
    np.testing.assert_allclose(material.elem_grad(model, mu, lam, F, rows, vols), g[f"{model}_grad"],
                               rtol=1e-10, atol=1e-6)
    ref = g[f"{model}_blocks"]
    got = material.vertex_blocks(model, mu, lam, F, rows, vols)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-10 * scale


def test_inversion_cap_known_answer():
    g = golden("elastic.npz")
    got = [material.inversion_cap("nh", g["inv_x"], p, g["inv_tets"], g["inv_rows"]) for p in g["inv_p"]]
    np.testing.assert_allclose(got, g["inv_alpha"], rtol=1e-12)
    assert abs(got[0] - 0.36) < 1e-9       # tests/test_elasticity.py:358-366 of the reference


def test_sparse_matvec_and_pcg():
    g = golden("sparse.npz")
    r, c, b = blocksparse.upper_triplets(g["cliques"], g["grids"])
    assert np.array_equal(r, g["trip_rows"]) and np.array_equal(c, g["trip_cols"])
    assert np.array_equal(b, g["trip_blocks"])
    n = int(g["n"])
    A = blocksparse.SymBlockMatrix(n, g["rows"], g["cols"], g["blocks"])
    assert np.allclose(A.dense(), g["dense"], atol=1e-12)
    for x, y in zip(g["mv_x"], g["mv_y"]):
        assert np.array_equal(A.matvec(x), y)
    for tag, tol, cap in (("a", 1e-8, None), ("b", 1e-3, None), ("c", 1e-12, 5)):
        x, its, conv, rel = blocksparse.pcg(A, g["rhs"], tol, cap)
        info = g[f"pcg_{tag}_info"]
        assert its == int(info[0]) and conv == bool(info[1])
        np.testing.assert_allclose(x, g[f"pcg_{tag}_x"], rtol=1e-12, atol=1e-14)
        assert rel == pytest.approx(info[2], rel=1e-12)


def test_active_set_sequence():
    g = golden("activeset.npz")
    aset = contact.ConstraintSet()
    for it in range(5):
        adm, pr = aset.update(g[f"k{it}"], g[f"q{it}"], g[f"t{it}"])
        assert [adm, pr] == g[f"adm{it}"].tolist()
        keys = np.concatenate([aset.kind[:, None], aset.quad], axis=1)
        assert np.array_equal(keys, g[f"keys{it}"])
        for j in range(len(aset)):
            if j % 3 == 0:
                aset.gamma[j] *= 0.005 if it % 2 else 0.5
        assert np.array_equal(aset.gamma, g[f"gamma{it}"])
    keep = contact.earliest_admission(g["af_q"], g["af_t"])
    assert np.array_equal(keep, g["af_keep"])


def _trajectory_scene(g):
    mu_l, lam_l = material.lame(1e7, 0.3)
    mu_s, lam_s = material.lame(1e5, 0.3)
    regions = [("lin", mu_l, lam_l, g["reg0_tets"], g["reg0_rows"], g["reg0_vols"]),
               ("snh", mu_s, lam_s, g["reg1_tets"], g["reg1_rows"], g["reg1_vols"])]
    n_slab = int(g["n_slab"])
    return timestep.Scene(g["masses"], regions, g["tris"], g["edges"], g["verts"],
                          [(np.arange(n_slab), None)])


def test_trajectory_matches_reference():
    g = golden("trajectory.npz")
    scene = _trajectory_scene(g)
    x, v = g["x0"].copy(), g["v0"].copy()
    aset = contact.ConstraintSet()
    for k in range(len(g["xs"])):
        x, v, rec, _, _ = timestep.step(x, v, scene, aset, h=0.01, offset=1e-3, k_min=2, step_index=k)
        np.testing.assert_allclose(x, g["xs"][k], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(v, g["vs"][k], rtol=1e-9, atol=1e-12)
        ref = g[f"rec{k}"]
        got = np.array([r[:5] for r in rec])
        assert got.shape == ref.shape
        np.testing.assert_allclose(got, ref, rtol=1e-12)
        keys = sorted(contact.key_of(kd, q) for kd, q in zip(aset.kind, aset.quad))
        assert np.array_equal(np.array([[kk[0], *kk[1]] for kk in keys]).reshape(-1, 5), g[f"keys{k}"])


def test_newton_lin_single_iteration():
    """LIN has a constant Hessian: one Newton step reaches the exact minimiser
    (tests/test_solver.py:76-90 of the reference)."""
    g = golden("trajectory.npz")
    mu, lam = material.lame(1e5, 0.3)
    reg = ("lin", mu, lam, g["reg1_tets"] - int(g["n_slab"]), g["reg1_rows"], g["reg1_vols"])
    x = g["x0"][int(g["n_slab"]):]
    masses = g["masses"][int(g["n_slab"]):]
    x_tilde = x + 0.001 * np.random.default_rng(0).standard_normal(x.shape)
    aset = contact.ConstraintSet()
    xh, nit, _, _, _ = newton.subproblem(x_tilde, x, x, masses, [reg], aset, 1.0, 1e-3, 0.01, cg_tol=1e-12)
    assert nit == 1
    gr, _ = newton.assemble(xh, x_tilde, masses, [reg], None, 1.0, 1e-3, 0.01)
    assert np.abs(gr).max() < 1e-9


def test_intersection_pairs_match_reference():
    """oracle/intersect.py vs the reference's static_intersection_test on
    interpenetrating, coplanar-contact, separated and jittered two-body
    surfaces (tests/golden/intersect.npz)."""
    from oracle import intersect
    g = golden("intersect.npz")
    for c in range(int(g["n"])):
        got = intersect.intersecting_pairs(g[f"x{c}"], g[f"tris{c}"])
        assert np.array_equal(got, g[f"pairs{c}"]), c


def test_min_distance_monitor_oracle():
    """Separated boxes 1e-4 apart: the closest VF/EE pair is exactly the gap;
    with a radius below the gap the inter-body pairs are not tested and the
    result is an intra-body pair beyond the radius (any untested pair is
    farther than the radius, so min(d, radius) bounds the true minimum)."""
    from oracle import intersect
    g = golden("intersect.npz")
    x, tris = g["x2"], g["tris2"]
    edges = np.unique(np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1), axis=0)
    verts = np.unique(tris)
    d, kind, q = intersect.min_distance(x, tris, edges, verts, 1e-3)
    assert d == pytest.approx(1e-4, rel=1e-6)
    assert intersect.min_distance(x, tris, edges, verts, 5e-5)[0] > 5e-5
