"""Procedural meshes and the synthetic benchmark scenes of BASELINE.json.

Primitives follow intact/primitives.py (Kuhn 6-tet boxes, cube-to-sphere
map); scenes follow SURVEY.md §8(d):

  C1  NH cube (box_mesh(10,10,8), 0.2 m, 4800 tets) dropped at 1 m/s from
      3 mm onto a Dirichlet-fixed LIN slab, h = 0.01.
  C4  five cube-to-sphere balls of 444,528 tets each (solid n = 42 grid,
      2.22M tets, 0.40M vertices in all), COR, rho 1e2, E 1e4, nu 0.4
      (PAPER.md:810), four in a 2x2 square on a fixed slab and one in the
      pocket above, compressed by a scripted top plate at 0.1 m/s.  The
      survey's one-cell hollow-shell proxy (n = 112, 0.74M vertices) is kept
      behind `layers=1`; it is not used for the benchmark because the
      reference algorithm itself blows up on it after a few frames (ultra-light
      shells escape tangentially under the linearised constraints; GPU and
      oracle agree on identical inputs — DESIGN.md §Scenes).
  C2  27 SNH cubes (3x3x3 stack, 131k tets) falling into a pinned box.
  C3  8 NH rods (491k tets) whose end layers are twisted in opposite senses
      by rotational scripted Dirichlet conditions.
  C5  randomized C1-like drops (seeded jitter of translation, rotation and
      velocity), one scene per seed.

Host-side setup only (numpy); nothing here runs in the timed hot path.
"""

from __future__ import annotations

import numpy as np

from .elasticity import Material, MaterialModel
from .mesh import SimState, TetMesh, build_tet_mesh, compute_rest_data, reorder_for_locality, reorder_for_sell
from .solver import ElasticRegion
from .stepper import BoundaryCondition, StepParams, System

_CUBE_TETS = np.array([[0, 1, 3, 7], [0, 3, 2, 7], [0, 2, 6, 7], [0, 6, 4, 7], [0, 4, 5, 7], [0, 5, 1, 7]],
                      dtype=np.int64)


def grid_points(nx, ny, nz, size):
    sx, sy, sz = (float(s) for s in np.broadcast_to(size, 3))
    g = np.stack(np.meshgrid(np.linspace(0.0, sx, nx + 1), np.linspace(0.0, sy, ny + 1),
                             np.linspace(0.0, sz, nz + 1), indexing="ij"), axis=-1)
    return g.reshape(-1, 3)


def cell_tets(nx, ny, nz, cells=None):
    """Kuhn tets of the given cells ((k,3) integer cell coords; all if None)."""
    if cells is None:
        i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
        cells = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1)
    i, j, k = cells[:, 0], cells[:, 1], cells[:, 2]

    def vid(a, b, c):
        return (a * (ny + 1) + b) * (nz + 1) + c

    corner = np.stack([vid(i, j, k), vid(i, j, k + 1), vid(i, j + 1, k), vid(i, j + 1, k + 1),
                       vid(i + 1, j, k), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k), vid(i + 1, j + 1, k + 1)],
                      axis=1)
    return corner[:, _CUBE_TETS].reshape(-1, 4)


def box_mesh(nx, ny, nz, size=1.0, origin=(0.0, 0.0, 0.0)) -> TetMesh:
    return build_tet_mesh(grid_points(nx, ny, nz, size) + np.asarray(origin, dtype=np.float64),
                          cell_tets(nx, ny, nz))


def rotation_matrix(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    c, s = np.cos(angle), np.sin(angle)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return c * np.eye(3) + s * k + (1 - c) * np.outer(a, a)


def transformed(mesh: TetMesh, translate=(0.0, 0.0, 0.0), rotate=None) -> TetMesh:
    v = mesh.rest_positions
    if rotate is not None:
        v = v @ np.asarray(rotate, dtype=np.float64).T
    return TetMesh(v + np.asarray(translate, dtype=np.float64), mesh.tets.copy(), mesh.surface_tris.copy(),
                   mesh.surface_edges.copy(), mesh.surface_verts.copy())


def shell_sphere(n, radius=0.1, center=(0.0, 0.0, 0.0), layers=1) -> TetMesh:
    """Hollow ball: the outermost `layers` Kuhn-cell layers of an n^3 grid on
    [-1,1]^3 (layers >= n/2 gives the solid ball), mapped radially onto a
    sphere (the intact/primitives.py:80-87 map)."""
    i, j, k = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    depth = np.minimum(np.minimum(np.minimum(i, j), k), np.minimum(np.minimum(n - 1 - i, n - 1 - j), n - 1 - k))
    on = depth < layers
    cells = np.stack([i[on], j[on], k[on]], axis=1)
    tets = cell_tets(n, n, n, cells)
    used, tets = np.unique(tets, return_inverse=True)
    tets = tets.reshape(-1, 4)
    verts = grid_points(n, n, n, 2.0)[used] - 1.0
    sup = np.abs(verts).max(axis=1)
    nrm = np.linalg.norm(verts, axis=1)
    verts = verts * np.where(nrm > 0.0, sup / np.maximum(nrm, 1e-300), 0.0)[:, None] * radius
    return build_tet_mesh(verts + np.asarray(center, dtype=np.float64), tets)


def _sphere_map(c, radius, blend=0.8):
    """Cube [-1,1]^3 -> rounded ball: each cube shell |c|_inf = r goes to
    `blend` x the sphere of radius r * radius under the smooth "spherified
    cube" map s_x sqrt(1 - s_y^2/2 - s_z^2/2 + s_y^2 s_z^2/3) of
    s = c / |c|_inf, plus (1 - blend) x the cube itself.  The full radial
    projection (intact/primitives.py:80-87, blend 1) flattens the Kuhn cells
    at the cube corners to 1e-3..1e-2 of the median volume; blend 0.8 keeps
    every tet above 0.29 of it."""
    sup = np.abs(c).max(axis=1)
    s = c / np.where(sup > 0.0, sup, 1.0)[:, None]
    q = s * s
    out = np.empty_like(s)
    out[:, 0] = s[:, 0] * np.sqrt(np.maximum(1 - q[:, 1] / 2 - q[:, 2] / 2 + q[:, 1] * q[:, 2] / 3, 0.0))
    out[:, 1] = s[:, 1] * np.sqrt(np.maximum(1 - q[:, 2] / 2 - q[:, 0] / 2 + q[:, 2] * q[:, 0] / 3, 0.0))
    out[:, 2] = s[:, 2] * np.sqrt(np.maximum(1 - q[:, 0] / 2 - q[:, 1] / 2 + q[:, 0] * q[:, 1] / 3, 0.0))
    return (blend * out * sup[:, None] + (1.0 - blend) * c) * radius


def squishy_ball(n=32, shell=2, stem=23, tip=16, pitch=3, cell=0.01, center=(0.0, 0.0, 0.0),
                 reorder=False, numbering="lattice") -> TetMesh:
    """Squishy ball: a hollow core with thin strands all over it.

    The core is the outer `shell` Kuhn-cell layers of an n^3 grid mapped onto
    a rounded ball of radius ~n/2 * cell (`_sphere_map`).  On every face of the grid, 2x2-cell strands
    start at a `pitch`-cell spacing (one free cell between neighbours); each
    runs `stem` cells out along the radial direction through its base centre,
    then narrows to a 1x1-cell `tip` of `tip` cells, centred on the same axis.
    All cells belong to one integer lattice, so the Kuhn (Freudenthal) split
    is conforming everywhere, strand bases included.

    Almost every vertex lies on the surface, as in the paper's squishy balls
    (0.87M vertices, 1.59M surface triangles, 2.25M tets for
    five balls): the defaults give 454k tets, 179k vertices and 319k surface
    triangles per ball.
    """
    L = stem + tip
    off = L                                   # lattice shift: coordinates >= 0
    dim = n + 2 * L                           # cells per axis of the enclosing lattice
    cells = []
    # hollow core
    i, j, k = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    depth = np.minimum(np.minimum(np.minimum(i, j), k), np.minimum(np.minimum(n - 1 - i, n - 1 - j), n - 1 - k))
    on = depth < shell
    cells.append(np.stack([i[on], j[on], k[on]], axis=1))
    # strand origins on a face: (a, b) lower corners of 2x2 patches
    starts = np.arange(1, n - 1, pitch)
    starts = starts[starts + 3 <= n]     # a free cell to the face edge on both sides
    starts = starts + (n - (starts[-1] + 2) - starts[0]) // 2   # centre the pattern
    A, B = np.meshgrid(starts, starts, indexing="ij")
    A, B = A.ravel(), B.ravel()
    for ax in range(3):
        u_ax, v_ax = [a for a in range(3) if a != ax]
        for sgn in (-1, 1):
            for l in range(L):
                w = 2 if l < stem else 1
                layer = n + l if sgn > 0 else -1 - l
                for du in range(w):
                    for dv in range(w):
                        c = np.empty((len(A), 3), dtype=np.int64)
                        c[:, ax] = layer
                        c[:, u_ax] = A + du
                        c[:, v_ax] = B + dv
                        cells.append(c)
    cells = np.concatenate(cells) + off
    tets = cell_tets(dim, dim, dim, cells)
    used, tets = np.unique(tets, return_inverse=True)
    tets = tets.reshape(-1, 4)
    g = np.stack(np.unravel_index(used, (dim + 1, dim + 1, dim + 1)), axis=1) - off   # lattice coords
    half = n / 2.0
    radius = half * cell
    pos = np.empty((len(g), 3))
    inside = ((g >= 0) & (g <= n)).all(axis=1)
    pos[inside] = _sphere_map((g[inside] - half) / half, radius)
    out = np.flatnonzero(~inside)
    go = g[out]
    # face of each strand vertex: the axis that leaves [0, n]
    ax = np.argmax((go < 0) | (go > n), axis=1)
    rows = np.arange(len(out))
    gax = go[rows, ax]
    sgn = np.where(gax > n, 1, -1)
    l = np.where(sgn > 0, gax - n, -gax)                     # layers out from the face
    base = go.copy()
    base[rows, ax] = np.where(sgn > 0, n, 0)
    uv = np.stack([base[rows, (ax + 1) % 3], base[rows, (ax + 2) % 3]], axis=1)
    # strand origin (lower corner) of each vertex: the start <= coordinate
    org = starts[np.clip(np.searchsorted(starts, uv, side="right") - 1, 0, len(starts) - 1)]
    centre = base.astype(np.float64)
    centre[rows, (ax + 1) % 3] = org[:, 0] + 1.0
    centre[rows, (ax + 2) % 3] = org[:, 1] + 1.0
    bc = _sphere_map((centre - half) / half, radius)
    axis = bc / np.linalg.norm(bc, axis=1)[:, None]
    # tip vertices (l > stem) sit on a half-size cross-section: map the 1x1
    # corner (a + du, b + dv), du, dv in {0, 1}, to the 2x2 corner (a + 2du, b + 2dv)
    # and take half its offset from the axis
    tipv = l > stem
    wide = base.astype(np.float64)
    wide[rows, (ax + 1) % 3] = np.where(tipv, org[:, 0] + 2 * (uv[:, 0] - org[:, 0]), uv[:, 0])
    wide[rows, (ax + 2) % 3] = np.where(tipv, org[:, 1] + 2 * (uv[:, 1] - org[:, 1]), uv[:, 1])
    bw = _sphere_map((wide - half) / half, radius)
    shift = np.where(tipv[:, None], 0.5 * (bw - bc), bw - bc)
    pos[out] = bc + shift + (l * cell)[:, None] * axis
    mesh = build_tet_mesh(pos + np.asarray(center, dtype=np.float64), tets)
    if reorder or numbering == "morton":
        return reorder_for_locality(mesh)
    if numbering == "sell":
        return reorder_for_sell(mesh)
    return mesh


def squishy_extent(n=32, stem=23, tip=16, cell=0.01):
    """Radius of the sphere holding a squishy_ball (strand tips included)."""
    return (n / 2.0 + stem + tip) * cell


def merge(bodies, boundary_bodies=(), scripted=None, h=0.01, scripted_stop=None):
    """Stack bodies [(mesh, material, density, velocity)] into a System.

    boundary_bodies: indices of bodies pinned entirely (fixed DBC);
    scripted: {body index: velocity} for bodies driven at constant velocity.
    """
    scripted = scripted or {}
    masses, regions, tris, edges, verts, xs, vs = [], [], [], [], [], [], []
    offs = [0]
    rest_cache = {}
    for mesh, mat, rho, vel in bodies:
        key = (id(mesh.tets), rho)
        rest = rest_cache.get(key)
        if rest is None or rest[0] is not mesh:
            rest = (mesh, compute_rest_data(mesh, rho))
        rest_cache[key] = rest
        rd = rest[1]
        off = offs[-1]
        regions.append(ElasticRegion(mat, mesh.tets + off, rd.shape_rows, rd.volumes))
        masses.append(rd.masses)
        tris.append(mesh.surface_tris + off)
        edges.append(mesh.surface_edges + off)
        verts.append(mesh.surface_verts + off)
        xs.append(mesh.rest_positions)
        vs.append(np.tile(np.asarray(vel, dtype=np.float64), (mesh.n_verts, 1)))
        offs.append(off + mesh.n_verts)
    x = np.vstack(xs)
    boundary = []
    for b in boundary_bodies:
        boundary.append(BoundaryCondition(np.arange(offs[b], offs[b + 1])))
    for b, vel in scripted.items():
        ids = np.arange(offs[b], offs[b + 1])
        traj = _ScriptedLine(x[ids].copy(), np.asarray(vel, dtype=np.float64), h,
                             None if scripted_stop is None else scripted_stop.get(b))
        boundary.append(BoundaryCondition(ids, kind="scripted", trajectory=traj))
    system = System(np.concatenate(masses), regions, np.vstack(tris), np.vstack(edges), np.concatenate(verts),
                    boundary)
    return system, SimState(x, np.vstack(vs)), np.asarray(offs)


class _ScriptedLine:
    """Constant-velocity target at the end of step k (intact/scene.py:459-466);
    h is bound by the scene builder.  t_stop (seconds) optionally halts the
    motion, e.g. a press that holds its minimum height."""

    def __init__(self, start, velocity, h=0.01, t_stop=None):
        self.start, self.velocity, self.h, self.t_stop = start, velocity, h, t_stop

    def __call__(self, step_index):
        t = (step_index + 1) * self.h
        if self.t_stop is not None:
            t = min(t, self.t_stop)
        return self.start + t * self.velocity


def _slab(size, corner, cells=(2, 2, 1), young=1e7):
    return (box_mesh(*cells, size=size, origin=corner), Material(MaterialModel.LIN, young, 0.3), 1000.0,
            (0.0, 0.0, 0.0))


def _pinned_slab(size, corner, cells, young, rho, edge):
    """A Dirichlet-pinned slab whose per-vertex mass and stiffness match a
    body of (young, rho) meshed at element size `edge`.

    Pinned vertices never move, but the reference's penalty stiffness
    mu = C_mu * max diag(M + h^2 K) is taken over ALL vertices, Dirichlet
    ones included (intact/stepper.py:191-200, :265-268).  A coarse dense
    stiff slab (decimetre cells, 1e3 kg/m^3, 1e7 Pa) would set mu ~1e4x above
    the balls' own diagonal and drive the AL iteration into divergence;
    scaling E by edge/cell and rho by (edge/cell)^3 gives the slab's
    vertices the balls' diagonal scale, as for a press modelled as a moving
    boundary.
    """
    cell = max(float(np.max(np.asarray(size, dtype=float) / np.asarray(cells, dtype=float))), edge)
    ratio = edge / cell
    return (box_mesh(*cells, size=size, origin=corner), Material(MaterialModel.LIN, young * ratio, 0.3),
            rho * ratio ** 3, (0.0, 0.0, 0.0))


def c1_scene(nx=10, ny=10, nz=8, size=0.2, height=0.003, speed=1.0):
    """NH cube dropped onto a fixed LIN slab."""
    cube = box_mesh(nx, ny, nz, size=size, origin=(-size / 2, -size / 2, height))
    bodies = [_slab((0.6, 0.6, 0.05), (-0.3, -0.3, -0.05)),
              (cube, Material(MaterialModel.NH, 1e5, 0.3), 1000.0, (0.0, 0.0, -speed))]
    system, state, offs = merge(bodies, boundary_bodies=[0])
    params = StepParams(h=0.01, offset=1e-3, min_iterations=2)
    return system, state, params


def c4_scene(n=42, radius=0.1, gap=0.001, plate_speed=0.1, h=0.01, layers=None, plate_stop=None):
    """Five squishy-ball proxies compressed by a moving plate.
    layers=None builds solid balls; layers=k keeps the outer k cell layers.

    Four shells sit in a 2x2 square on a fixed slab, the fifth in the pocket
    above them; a scripted top plate starts one gap above the top shell and
    moves down at plate_speed; with plate_stop (metres) it halts once its
    underside reaches that height and holds the compression (the press of
    PAPER.md:596 shrinking the container to a minimum height).
    """
    ball = shell_sphere(n, radius, layers=(n + 1) // 2 if layers is None else layers)
    mat = Material(MaterialModel.COR, 1e4, 0.4)
    rho = 1e2
    c = radius + gap / 2
    z0 = radius + gap
    centers = [(-c, -c, z0), (c, -c, z0), (-c, c, z0), (c, c, z0)]
    dz = np.sqrt((2 * radius + gap) ** 2 - 2 * c * c)
    centers.append((0.0, 0.0, z0 + dz + gap))
    edge = 2.0 * radius / n
    # plates meshed at ~4 cm: long plate edges would each overlap thousands of
    # ball edges in the EE broad phase
    bodies = [_pinned_slab((1.0, 1.0, 0.05), (-0.5, -0.5, -0.05), (24, 24, 1), mat.young, rho, edge)]
    for ctr in centers:
        bodies.append((transformed(ball, translate=ctr), mat, rho, (0.0, 0.0, 0.0)))
    top = centers[-1][2] + radius + gap
    bodies.append(_pinned_slab((0.6, 0.6, 0.03), (-0.3, -0.3, top), (16, 16, 1), mat.young, rho, edge))
    stop = None
    if plate_stop is not None:
        stop = {len(bodies) - 1: max(0.0, (top - plate_stop) / plate_speed)}
    system, state, offs = merge(bodies, boundary_bodies=[0], scripted={len(bodies) - 1: (0.0, 0.0, -plate_speed)},
                                h=h, scripted_stop=stop)
    params = StepParams(h=h, offset=1e-3, min_iterations=2)
    return system, state, params


def squishy_scene(cell=0.02, n=32, stem=23, tip=16, shell=2, gap=None, plate_speed=1.0, plate_stop=None, h=0.01,
                  walls=True, seed=7, balls=5, reorder=False, numbering="lattice"):
    """C4, paper-scale: five squishy balls in a box, pressed by a plate.

    Each ball is a `squishy_ball` (hollow core + 600 strands; the defaults
    give 2.27M tets, 0.89M vertices and 1.60M surface triangles for five
    balls, within 3 % of the paper's 2.25M / 0.87M / 1.59M),
    COR with the paper's rho 1e2, E 1e4, nu 0.4, h = 0.01, offset 1e-3,
    K_min 2.  Each ball gets a seeded random rotation so no strands of two
    balls are aligned.  Four balls rest one gap above a pinned floor in a
    2x2 square and the fifth in the pocket above; four pinned walls (with
    slits between them, as in c2_scene) hold the stack, and a scripted plate
    starts one gap above it and moves down at plate_speed, holding once its
    underside reaches plate_stop (the container shrinking to a minimum
    height).  Physical scale: `cell` is the strand cell edge;
    2 cm puts block-Jacobi PCG at ~90-110 CG iterations per solve (the
    paper's average is 28, its peak 146), see DESIGN.md.
    `numbering` = the ball's vertex numbering: "lattice" (default), "sell"
    (lattice order with 1024-vertex windows sorted for even sliced-ELL
    slices, mesh.sell_numbering; measured slower) or "morton".
    """
    rng = np.random.default_rng(seed)
    base = squishy_ball(n=n, shell=shell, stem=stem, tip=tip, cell=cell, reorder=reorder, numbering=numbering)
    R = float(np.linalg.norm(base.rest_positions, axis=1).max())
    gap = 2.0 * cell if gap is None else gap
    mat = Material(MaterialModel.COR, 1e4, 0.4)
    rho = 1e2
    rots = [rotation_matrix(rng.standard_normal(3), rng.uniform(-np.pi, np.pi)) for _ in range(balls)]
    c = R + gap / 2
    # the bottom four rest one gap above the floor (lowest vertex), the fifth
    # sits in their pocket, its bounding sphere one gap above theirs
    lows = [float((base.rest_positions @ Rm.T)[:, 2].min()) for Rm in rots]
    centers = [(-c, -c, gap - lows[0]), (c, -c, gap - lows[1]), (-c, c, gap - lows[2]), (c, c, gap - lows[3])]
    z0 = max(ct[2] for ct in centers[:4])
    dz = np.sqrt((2 * R + gap) ** 2 - 2 * c * c)
    centers.append((0.0, 0.0, z0 + dz + gap))
    centers = centers[:balls]
    meshes = [transformed(base, translate=ct, rotate=Rm) for ct, Rm in zip(centers, rots)]
    top = max(float(m.rest_positions[:, 2].max()) for m in meshes) + gap
    half = 2 * R + 2 * gap                      # inner half-width of the box
    wall, slit = 4 * cell, 2 * cell
    pc = 8                                      # wall / plate cells per ~8 ball cells
    nc = max(2, int(round(2 * (half + wall) / (pc * cell))))
    hc = max(2, int(round(top / (pc * cell))))
    bodies = [_pinned_slab((2 * (half + wall), 2 * (half + wall), wall), (-half - wall, -half - wall, -wall),
                           (nc, nc, 1), mat.young, rho, cell)]
    n_fixed = 1
    if walls:
        height = top + 2 * cell
        for sx, sy, cx, cy in ((wall, 2 * half - 2 * slit, -half - wall, -half + slit),
                               (wall, 2 * half - 2 * slit, half, -half + slit),
                               (2 * half, wall, -half, -half - wall),
                               (2 * half, wall, -half, half)):
            bodies.append(_pinned_slab((sx, sy, height), (cx, cy, slit),
                                       (1 if sx == wall else nc, 1 if sy == wall else nc, hc), mat.young, rho, cell))
        n_fixed = 5
    for m in meshes:
        bodies.append((m, mat, rho, (0.0, 0.0, 0.0)))
    pl = half - slit
    bodies.append(_pinned_slab((2 * pl, 2 * pl, wall), (-pl, -pl, top), (nc, nc, 1), mat.young, rho, cell))
    stop = None
    if plate_stop is not None:
        stop = {len(bodies) - 1: max(0.0, (top - plate_stop) / plate_speed)}
    system, state, offs = merge(bodies, boundary_bodies=list(range(n_fixed)),
                                scripted={len(bodies) - 1: (0.0, 0.0, -plate_speed)}, h=h, scripted_stop=stop)
    params = StepParams(h=h, offset=1e-3, min_iterations=2)
    system.scene_info = {"ball_tets": int(base.n_tets), "ball_verts": int(base.n_verts),
                         "ball_tris": int(len(base.surface_tris)), "balls": len(centers), "ball_radius": R,
                         "plate_top": float(top), "cell": cell}
    return system, state, params


class _ScriptedTwist:
    """Rotation of fixed start positions about a vertical axis through
    `center` by omega * t at the end of step k (a rotational scripted DBC,
    SURVEY.md §8(d) C3; the reference's Python BoundaryCondition API,
    intact/stepper.py:78-100)."""

    def __init__(self, start, center, omega, h=0.01):
        self.start = np.asarray(start, dtype=np.float64)
        self.center = np.zeros(3)
        self.center[:2] = np.asarray(center, dtype=np.float64)[:2]
        self.omega, self.h = float(omega), float(h)

    def __call__(self, step_index):
        a = self.omega * (step_index + 1) * self.h
        c, s_ = np.cos(a), np.sin(a)
        d = self.start - self.center
        out = self.start.copy()
        out[:, 0] = self.center[0] + c * d[:, 0] - s_ * d[:, 1]
        out[:, 1] = self.center[1] + s_ * d[:, 0] + c * d[:, 1]
        return out


def c2_scene(grid=3, cells=(9, 9, 10), size=(0.09, 0.09, 0.1), gap=0.002, h=0.01):
    """Stack of grid^3 SNH cubes falling into a pinned box of five slabs
    (27 x 4,860 tets = 131k tets, dense multi-body
    contact and active-set churn)."""
    size = np.asarray(size, dtype=np.float64)
    mat = Material(MaterialModel.SNH, 1e5, 0.3)
    rho = 1000.0
    edge = float(np.min(size / np.asarray(cells)))
    pitch = size + gap
    span = grid * pitch - gap
    lo = -0.5 * span[:2]
    cube = box_mesh(*cells, size=size)
    bodies = []
    wall = 0.02
    inner = span[:2] + 2 * 0.01
    height = grid * pitch[2] + 0.05
    # floor and four walls, pinned (per-vertex diagonal matched to the cubes).
    # The five slabs keep a slit between one another: the reference's CCD
    # also tests pairs of pinned primitives, and touching slabs would pin
    # alpha at 0 for good (TOI 0, intact/ccd.py:64-66).
    slit = 0.002
    bodies.append(_pinned_slab((inner[0] + 2 * wall, inner[1] + 2 * wall, wall),
                               (-inner[0] / 2 - wall, -inner[1] / 2 - wall, -wall), (12, 12, 1), mat.young, rho, edge))
    for sx, sy, cx, cy in ((wall, inner[1] - 2 * slit, -inner[0] / 2 - wall, -inner[1] / 2 + slit),
                           (wall, inner[1] - 2 * slit, inner[0] / 2, -inner[1] / 2 + slit),
                           (inner[0], wall, -inner[0] / 2, -inner[1] / 2 - wall),
                           (inner[0], wall, -inner[0] / 2, inner[1] / 2)):
        bodies.append(_pinned_slab((sx, sy, height), (cx, cy, slit),
                                   (1 if sx == wall else 12, 1 if sy == wall else 12, 10), mat.young, rho, edge))
    for k in range(grid):
        for j in range(grid):
            for i in range(grid):
                org = (lo[0] + i * pitch[0], lo[1] + j * pitch[1], gap + k * pitch[2])
                bodies.append((transformed(cube, translate=org), mat, rho, (0.0, 0.0, 0.0)))
    system, state, _ = merge(bodies, boundary_bodies=list(range(5)), h=h)
    return system, state, StepParams(h=h, offset=1e-3, min_iterations=2)


def c3_scene(rows=2, cols=4, cells=(8, 8, 160), size=(0.02, 0.02, 0.4), gap=0.002, omega=np.pi, h=0.01):
    """Bundle of NH rods (rho 1e3, E 1e6, nu 0.3, offset 2e-4)
    whose end layers are twisted in opposite senses about the bundle axis by
    rotational scripted Dirichlet conditions (~500k tets,
    self-contact with edge-edge dominated CCD)."""
    size = np.asarray(size, dtype=np.float64)
    mat = Material(MaterialModel.NH, 1e6, 0.3)
    rho = 1e3
    rod = box_mesh(*cells, size=size)
    pitch = size[:2] + gap
    bodies = []
    for j in range(rows):
        for i in range(cols):
            org = (-0.5 * (cols * pitch[0] - gap) + i * pitch[0], -0.5 * (rows * pitch[1] - gap) + j * pitch[1], 0.0)
            bodies.append((transformed(rod, translate=org), mat, rho, (0.0, 0.0, 0.0)))
    system, state, offs = merge(bodies, h=h)
    x = state.x
    bottom = np.flatnonzero(np.isclose(x[:, 2], 0.0))
    top = np.flatnonzero(np.isclose(x[:, 2], size[2]))
    boundary = [BoundaryCondition(bottom, kind="scripted", trajectory=_ScriptedTwist(x[bottom], (0, 0), -omega, h)),
                BoundaryCondition(top, kind="scripted", trajectory=_ScriptedTwist(x[top], (0, 0), omega, h))]
    system = System(system.masses, system.regions, system.surface_triangles, system.surface_edges,
                    system.surface_vertices, boundary)
    return system, state, StepParams(h=h, offset=2e-4, min_iterations=2)


def c5_scene(seed, nx=10, ny=10, nz=8):
    """One randomized C1-like drop."""
    rng = np.random.default_rng(seed)
    size = 0.2
    cube = box_mesh(nx, ny, nz, size=size, origin=(-size / 2, -size / 2, -size / 2))
    axis = rng.standard_normal(3)
    R = rotation_matrix(axis, rng.uniform(-np.pi, np.pi))
    cube = transformed(cube, rotate=R)
    lift = -cube.rest_positions[:, 2].min() + 0.003
    shift = rng.uniform(-0.005, 0.005, 3)
    cube = transformed(cube, translate=(shift[0], shift[1], lift + abs(shift[2])))
    speed = rng.uniform(0.5, 2.0)
    bodies = [_slab((0.6, 0.6, 0.05), (-0.3, -0.3, -0.05)),
              (cube, Material(MaterialModel.NH, 1e5, 0.3), 1000.0, (0.0, 0.0, -speed))]
    system, state, _ = merge(bodies, boundary_bodies=[0])
    return system, state, StepParams(h=0.01, offset=1e-3, min_iterations=2)
