"""Pin the friction oracle (oracle/friction.py) against the reference's
intact/friction.py outputs (tests/golden/friction.npz, make_golden.py)."""

import numpy as np
import pytest

from oracle import contact, friction, material, timestep
from tests.conftest import golden


def test_mollifier_and_frames():
    g = golden("friction.npz")
    eps = float(g["eps"])
    np.testing.assert_array_equal(friction.f0(g["y"], eps), g["f0"])
    np.testing.assert_array_equal(friction.f0_over_y(g["y"], eps), g["f0y"])
    np.testing.assert_array_equal(friction.f0_second(g["y"], eps), g["f0s"])
    np.testing.assert_allclose(friction.tangent_frames(g["normals"]), g["frames"], rtol=0, atol=1e-15)


def test_terms_energy_gradient_hessian():
    g = golden("friction.npz")
    fs = friction.FrictionSet(g["t_idx"], g["t_w"], g["t_frames"], g["t_coeff"], g["t_ref"], float(g["eps"]))
    x = g["t_x"]
    assert fs.energy(x) == pytest.approx(float(g["t_energy"]), rel=1e-14)
    np.testing.assert_allclose(fs.grad_terms(x), g["t_grad"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(fs.hess_grids(x), g["t_hess"], rtol=1e-12, atol=1e-12 * np.abs(g["t_hess"]).max())


def _aset(g, k):
    a = contact.ConstraintSet()
    kinds, quads = g[f"s_akind{k}"], g[f"s_aquad{k}"]
    a._append(kinds, quads, [contact.key_of(kk, q) for kk, q in zip(kinds, quads)], lam=g[f"s_alam{k}"])
    return a


def test_precompute_identical_inputs():
    """friction_precompute from the reference's own accepted states and
    multipliers: same terms, same order."""
    g = golden("friction.npz")
    for k in range(int(g["s_steps"])):
        fr = friction.precompute(g[f"s_x{k}"], _aset(g, k), float(g[f"s_mu{k}"]), 1e-3, 0.01, 0.5, 1e-3)
        n = int(g[f"s_nfr{k}"])
        assert (0 if fr is None else len(fr)) == n
        if n:
            np.testing.assert_array_equal(fr.indices, g[f"s_fidx{k}"])
            np.testing.assert_array_equal(fr.weights, g[f"s_fw{k}"])
            np.testing.assert_allclose(fr.frames, g[f"s_ffr{k}"], rtol=0, atol=1e-14)
            np.testing.assert_allclose(fr.coeff, g[f"s_fc{k}"], rtol=1e-12)
            np.testing.assert_allclose(fr.ref, g[f"s_fref{k}"], rtol=1e-14, atol=1e-16)


def friction_scene(g):
    mu_l, lam_l = material.lame(1e7, 0.3)
    mu_s, lam_s = material.lame(1e5, 0.3)
    regions = [("lin", mu_l, lam_l, g["s_reg0_tets"], g["s_reg0_rows"], g["s_reg0_vols"]),
               ("snh", mu_s, lam_s, g["s_reg1_tets"], g["s_reg1_rows"], g["s_reg1_vols"])]
    return timestep.Scene(g["s_masses"], regions, g["s_tris"], g["s_edges"], g["s_verts"],
                          [(np.arange(int(g["s_n_slab"])), None)])


def test_sliding_box_trajectory():
    """Five steps of the box sliding on the slab with mu_f = 0.5: positions
    within 1e-9 relative of the reference, same friction term counts."""
    g = golden("friction.npz")
    scene = friction_scene(g)
    x, v = g["s_xinit"].copy(), g["s_vinit"].copy()
    aset = contact.ConstraintSet()
    fr = None
    scale = np.abs(g["s_xinit"]).max()
    for k in range(int(g["s_steps"])):
        out = []
        x, v, rec, _, _ = timestep.step(x, v, scene, aset, h=0.01, offset=1e-3, k_min=2, step_index=k,
                                        mu_f=0.5, eps_v=1e-3, friction=fr, friction_out=out)
        fr = out[0]
        assert np.abs(x - g[f"s_x{k}"]).max() <= 1e-9 * scale, k
        assert (0 if fr is None else len(fr)) == int(g[f"s_nfr{k}"])
