"""CPU tests: the C-ABI library loads and exports every declared symbol, and
the host-side logic (parameters, boundaries, scene generation, sparse index
bookkeeping) behaves like the reference's."""

import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "ibf.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|unsigned long long|int|void)\s+(ibf_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_12151_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2512_12151_b200.build import build
        build()
    return _lib.lib()


def test_library_exports_every_header_symbol(lib):
    syms = _declared_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2512_12151_b200 import _lib
    assert set(_lib.exported_symbols()) <= set(syms)
    assert lib.ibf_version().startswith(b"ibf-b200")


def test_library_is_sm100a_only():
    from paper_2512_12151_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2512_12151_b200 import distance
    with pytest.raises(RuntimeError):
        distance.vf_eval(np.zeros((1, 4, 3)))


def test_step_params_validation():
    from paper_2512_12151_b200 import StepParams
    StepParams(h=0.01, offset=1e-3)
    for bad in (dict(h=0.0, offset=1e-3), dict(h=0.01, offset=0.0), dict(h=0.01, offset=1e-3, epsilon=1.0),
                dict(h=0.01, offset=1e-3, min_iterations=0), dict(h=0.01, offset=1e-3, decay=1.5),
                dict(h=0.01, offset=1e-3, stiffness_constant=0.0), dict(h=0.01, offset=1e-3, gravity=(0, 0))):
        with pytest.raises(ValueError):
            StepParams(**bad)


def test_simulation_state_assignment_replaces_device_copy():
    """Simulation keeps the evolving state on the device between advances;
    assigning `sim.state` must still take effect, as on the reference's plain
    dataclass (intact/stepper.py:374-384)."""
    from paper_2512_12151_b200 import Simulation
    from paper_2512_12151_b200.mesh import SimState
    old = SimState(x=np.zeros((2, 3)), v=np.zeros((2, 3)))
    new = SimState(x=np.ones((2, 3)), v=np.ones((2, 3)))
    sim = Simulation(None, None, old)
    sim.__dict__["_x"] = sim.__dict__["_v"] = object()    # stands in for a device copy after advance()
    sim.state = new
    assert sim.__dict__["_x"] is None and sim.__dict__["_v"] is None
    assert sim.state is new


def test_beta_recursion_code_semantics():
    """beta_update is called with k-1 (intact/stepper.py:320): K_min passes exempt."""
    from paper_2512_12151_b200.stepper import beta_update
    beta = 1.0
    trace = []
    for k in range(4):
        beta = beta_update(beta, 0.5, k - 1, 2)
        trace.append(beta)
    assert trace == [1.0, 1.0, 0.5, 0.25]


def test_boundary_and_system_validation():
    from paper_2512_12151_b200.stepper import BoundaryCondition, System
    with pytest.raises(ValueError):
        BoundaryCondition([0], kind="moving")
    with pytest.raises(ValueError):
        BoundaryCondition([0], kind="scripted")
    with pytest.raises(ValueError):
        System(np.ones(3), [], np.zeros((0, 3), int), np.zeros((0, 2), int), np.zeros(0, int),
               [BoundaryCondition([0, 1]), BoundaryCondition([1, 2])])
    s = System(np.ones(3), [], np.zeros((0, 3), int), np.zeros((0, 2), int), np.zeros(0, int),
               [BoundaryCondition([0, 2])])
    assert s.dbc_mask.tolist() == [True, False, True]


def test_clique_contributions_match_oracle(rng):
    from oracle import blocksparse
    from paper_2512_12151_b200.sparse import clique_contributions
    ids = np.array([rng.choice(20, 4, replace=False) for _ in range(10)])
    grids = rng.standard_normal((10, 4, 4, 3, 3))
    a = clique_contributions(ids, grids)
    b = blocksparse.upper_triplets(ids, grids)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_shell_sphere_counts():
    """Hollow shell: 36n^2 - 72n + 48 tets."""
    from paper_2512_12151_b200.scenes import shell_sphere
    for n in (4, 8):
        m = shell_sphere(n, 0.1)
        assert m.n_tets == 36 * n * n - 72 * n + 48
        assert m.n_verts == 6 * n * n + 2 + 6 * (n - 2) ** 2 + 2
        r = np.linalg.norm(m.rest_positions, axis=1)
        assert r.max() == pytest.approx(0.1, rel=1e-12)


def test_scene_generators_match_reference_primitives():
    """box_mesh and rest data follow intact/primitives.py + intact/mesh.py."""
    from oracle import material
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.mesh import compute_rest_data
    m = scenes.box_mesh(3, 2, 2, size=(0.3, 0.2, 0.2))
    assert m.n_tets == 6 * 12 and m.n_verts == 4 * 3 * 3
    rest = compute_rest_data(m, 1000.0)
    assert rest.masses.sum() == pytest.approx(1000.0 * 0.3 * 0.2 * 0.2)
    F = material.def_grad(m.rest_positions, m.tets, rest.shape_rows)
    assert np.allclose(F, np.eye(3), atol=1e-12)
    system, state, params = scenes.c1_scene()
    assert sum(len(r.tets) for r in system.regions) == 4800 + 24
    assert params.min_iterations == 2


def test_sell_numbering_is_a_padding_reducing_permutation():
    """mesh.sell_numbering (the optional squishy-ball numbering):
    a permutation of the vertices that keeps the mesh (same tets up to
    renumbering) and lowers the sliced-ELL padding of the upper slots."""
    import numpy as np
    from paper_2512_12151_b200 import scenes
    from paper_2512_12151_b200.mesh import reorder_for_sell, sell_numbering

    ball = scenes.squishy_ball(n=8, shell=2, stem=4, tip=3, cell=0.02)
    n = ball.n_verts
    new_of = sell_numbering(n, ball.tets, window=128)
    assert np.array_equal(np.sort(new_of), np.arange(n))

    def upper_padding(tets):
        pairs = np.concatenate([tets[:, [i, j]] for i in range(4) for j in range(i + 1, 4)])
        key = np.unique(pairs.min(axis=1) * n + pairs.max(axis=1))
        up = np.bincount(key // n, minlength=n) + 1
        w = np.maximum.reduceat(up, np.arange(0, n, 32))
        return 1.0 - up.sum() / (32.0 * w.sum())

    re = reorder_for_sell(ball, window=128)
    assert re.n_verts == n and re.n_tets == ball.n_tets
    # same geometry: the renumbered positions are a permutation of the originals
    perm = np.empty_like(new_of)
    perm[new_of] = np.arange(n)
    assert np.array_equal(re.rest_positions, ball.rest_positions[perm])
    assert upper_padding(re.tets) < upper_padding(ball.tets)
