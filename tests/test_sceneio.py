"""Scene build and export: boundary-surface extraction
on the device and the native OBJ writer, bit-exact against the reference's
extract_surface_arrays (intact/mesh.py:106-124) and export_frame
(intact/io_utils.py:35-43) through golden fixtures (tests/golden/sceneio.npz,
made by tests/golden/make_golden.py from the reference itself).

The OBJ writer is host code in libibf.so and needs no GPU, so its parity
tests run on CPU; surface extraction is a CUDA path (marked gpu).
"""

import os

import numpy as np
import pytest

from oracle import sceneio
from tests.conftest import golden


def _meshes():
    g = golden("sceneio.npz")
    for c in range(int(g["n_meshes"])):
        yield c, g[f"tets{c}"], g[f"tris{c}"], g[f"edges{c}"], g[f"verts{c}"]


# ------------------------------------------------------------------ oracle


def test_oracle_surface_matches_reference():
    for c, tets, tris, edges, verts in _meshes():
        t, e, v, _ = sceneio.extract_surface_arrays(tets)
        assert np.array_equal(t, tris), c
        assert np.array_equal(e, edges), c
        assert np.array_equal(v, verts), c


def test_oracle_obj_matches_reference():
    g = golden("sceneio.npz")
    assert sceneio.obj_text(g["obj_x"], g["obj_tris"]).encode() == g["obj_bytes"].tobytes()
    assert sceneio.obj_text(g["obj_x"], np.zeros((0, 3), np.int64)).encode() == g["obj_empty_bytes"].tobytes()


# -------------------------------------------------------- native OBJ writer


def _write(tmp_path, x, tris, threads=0, name="f.obj"):
    from paper_2512_12151_b200.io_utils import export_frame
    path = tmp_path / name
    export_frame(x, tris, str(path), threads=threads)
    return path.read_bytes()


def test_export_frame_matches_reference_bytes(tmp_path):
    g = golden("sceneio.npz")
    for threads in (1, 3, 0):
        assert _write(tmp_path, g["obj_x"], g["obj_tris"], threads) == g["obj_bytes"].tobytes()
    assert _write(tmp_path, g["obj_x"], np.zeros((0, 3), np.int64)) == g["obj_empty_bytes"].tobytes()


def test_export_frame_repr_over_magnitudes(tmp_path, rng):
    # shortest round-trip digits and Python's positional/scientific switch
    # over the whole exponent range, subnormals and non-finite values
    n = 60000
    mant = rng.uniform(-10.0, 10.0, n)
    x = (mant * 10.0 ** rng.integers(-320, 308, n).astype(np.float64)).reshape(-1, 3)
    x[:200] = np.round(rng.uniform(-1e4, 1e4, (200, 3))) / 1e3
    x[200:400] = rng.integers(-10**17, 10**17, (200, 3)).astype(np.float64)
    x[400, :] = (np.nan, np.inf, -np.inf)
    x[401, :] = (5e-324, -2.2250738585072014e-308, 1.7976931348623157e308)
    tris = np.arange(len(x) - len(x) % 3).reshape(-1, 3)
    tris = tris[rng.permutation(len(tris))]
    got = _write(tmp_path, x, tris, threads=5)
    assert got == sceneio.obj_text(x, tris).encode()


def test_export_frame_compacts_unused_vertices(tmp_path, rng):
    x = rng.standard_normal((50, 3))
    tris = np.array([[40, 3, 7], [7, 3, 12], [49, 40, 12]])
    assert _write(tmp_path, x, tris) == sceneio.obj_text(x, tris).encode()


def test_export_frame_errors(tmp_path):
    from paper_2512_12151_b200.io_utils import export_frame
    x = np.zeros((4, 3))
    with pytest.raises(ValueError):
        export_frame(x, np.array([[0, 1, 4]]), str(tmp_path / "a.obj"))
    with pytest.raises(OSError):
        export_frame(x, np.array([[0, 1, 2]]), str(tmp_path / "missing_dir" / "a.obj"))


# ---------------------------------------------------- device surface extraction


@pytest.mark.gpu
def test_surface_extraction_matches_reference():
    from paper_2512_12151_b200.mesh import extract_surface_arrays
    for c, tets, tris, edges, verts in _meshes():
        t, e, v = extract_surface_arrays(tets)
        assert np.array_equal(t, tris), c
        assert np.array_equal(e, edges), c
        assert np.array_equal(v, verts), c


@pytest.mark.gpu
def test_surface_extraction_large_and_edge_cases(rng):
    """A 240k-tet box with shuffled tets and a ragged random subset against
    the oracle; an empty mesh; negative ids rejected."""
    from paper_2512_12151_b200.mesh import extract_surface_arrays
    from paper_2512_12151_b200.scenes import box_mesh
    box = box_mesh(40, 40, 25, size=1.0)
    for tets in (box.tets[rng.permutation(len(box.tets))], box.tets[rng.random(len(box.tets)) < 0.3]):
        t, e, v = extract_surface_arrays(tets)
        ot, oe, ov, _ = sceneio.extract_surface_arrays(tets)
        assert np.array_equal(t, ot) and np.array_equal(e, oe) and np.array_equal(v, ov)
    t, e, v = extract_surface_arrays(np.zeros((0, 4), np.int64))
    assert t.shape == (0, 3) and e.shape == (0, 2) and v.shape == (0,)
    with pytest.raises(ValueError):
        extract_surface_arrays(np.array([[0, 1, 2, -3]]))
