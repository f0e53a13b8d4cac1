"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only describes the five
synthetic scenes of BASELINE.json ``configs`` (SURVEY.md section 8(d), table
d.1) as plain dicts, rounds them to the float32 values the device path sees,
and draws seeded random debug records.  Both ``oracle/`` and
``paper_2402_03106_b200/`` consume it; neither imports the other.

Every scene stands in for the paper's mesh scenes (GLOSSY DRAGON, STAIRCASE,
CORNELL BOX), which are not available; see DESIGN.md
section 4 for the recipe.
"""
from __future__ import annotations

import copy

import numpy as np

# R22 caps, R21 spp semantics, R29 direction modes, R8 table axes.
CONFIGS = {
    1: dict(
        name="cfg1_infinite_detector",
        sigma_s=0.9, sigma_a=0.1, g=0.0,
        medium="infinite",
        emitters=[((0.0, 0.0, 0.0), 0.0, 1.0)],
        camera="detector", cam_pos=(2.0, 0.0, 0.0), det_radius=0.05,
        width=1, height=1,
        t0=2.0, t1=12.0, n_bins=128, warped=1,
        spp=2048, spp_mode="cell", max_bounces=64, seed=0,
        direction_mode="reuse",
    ),
    2: dict(
        name="cfg2_sphere_unwarped",
        sigma_s=4.75, sigma_a=0.25, g=0.5,
        medium="sphere", center=(0.0, 0.0, 0.0), radius=1.0,
        emitters=[((0.0, 0.0, -3.0), 0.0, 1.0)],
        camera="pinhole", cam_pos=(0.0, 0.0, 4.0), fov_y_deg=40.0,
        width=64, height=64,
        t0=0.0, t1=20.0, n_bins=256, warped=0,
        spp=16, spp_mode="cell", max_bounces=512, seed=1,
        direction_mode="reuse",
    ),
    3: dict(
        name="cfg3_slab_warped",
        sigma_s=9.9, sigma_a=0.1, g=0.8,
        medium="box", bmin=(-2.0, -2.0, 0.0), bmax=(2.0, 2.0, 1.0),
        emitters=[((0.0, 0.0, -2.0), 0.0, 1.0)],
        camera="pinhole", cam_pos=(0.0, 0.0, -2.0), fov_y_deg=60.0,
        width=256, height=256,
        t0=4.0, t1=40.0, n_bins=512, warped=1,
        spp=64, spp_mode="cell", max_bounces=1024, seed=2,
        direction_mode="split",
    ),
    4: dict(
        name="cfg4_cube_walls_gate",
        sigma_s=1.8, sigma_a=0.2, g=0.3,
        medium="box", bmin=(-1.0, -1.0, -1.0), bmax=(1.0, 1.0, 1.0),
        # faces: 0 -x, 1 +x, 2 -y, 3 +y, 4 -z (open front), 5 +z
        wall_mask=0b101111, wall_albedo=(0.7, 0.7, 0.7, 0.7, 0.0, 0.7),
        emitters=[((-0.5, 0.8, 0.0), 0.0, 1.0), ((0.5, 0.8, 0.0), 1.5, 1.0)],
        camera="pinhole", cam_pos=(0.0, 0.0, -4.0), fov_y_deg=45.0,
        width=512, height=512,
        t0=6.0, t1=6.1, n_bins=1, warped=1,
        spp=256, spp_mode="cell", max_bounces=128, seed=3,
        direction_mode="reuse",
    ),
    5: dict(
        name="cfg5_fogbox_warped",
        sigma_s=19.98, sigma_a=0.02, g=0.9,
        medium="box", bmin=(-5.0, -5.0, -5.0), bmax=(5.0, 5.0, 5.0),
        emitters=[((0.0, 0.0, -6.0), 0.0, 1.0)],
        camera="pinhole", cam_pos=(0.0, 0.0, -8.0), fov_y_deg=50.0,
        width=1024, height=1024,
        t0=0.0, t1=100.0, n_bins=1000, warped=1,
        spp=1024, spp_mode="pixel", max_bounces=4096, seed=4,
        direction_mode="split",
    ),
}

_DEFAULTS = dict(
    center=(0.0, 0.0, 0.0), radius=1.0, bmin=(0.0, 0.0, 0.0), bmax=(0.0, 0.0, 0.0),
    wall_mask=0, wall_albedo=(0.0,) * 6, look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0),
    fov_y_deg=45.0, det_radius=0.0, strategy="darts", n_ris=8, alpha=0.5,
    parity_r_excl=0.0, parity_s_excess=0.0, table_nr=16, table_ns=16,
    crop=None, table_smin=None, table_smax=None, response=None, mesh=None,
    conn_sampling="exp",   # "exp": truncated exponential P of S; "uniform": ablation
)


def config(idx: int, **overrides) -> dict:
    """Full scene dict for config ``idx`` (1..5; 6 = mesh_config) with defaults and overrides."""
    if idx == 6:
        return mesh_config(**overrides)
    c = copy.deepcopy(_DEFAULTS)
    c.update(copy.deepcopy(CONFIGS[idx]))
    c.update(overrides)
    sigma_t = c["sigma_s"] + c["sigma_a"]
    if c["table_smin"] is None:
        c["table_smin"] = 1e-2 / sigma_t                     # R8
    if c["table_smax"] is None:
        c["table_smax"] = c["t1"] - min(e[1] for e in c["emitters"])
    if c["crop"] is None:
        c["crop"] = (0, 0, c["width"], c["height"])
    return c


def _f32(x):
    return float(np.float32(x))


def as_f32(c: dict) -> dict:
    """Round every real scene parameter to float32 (what the device sees), so
    the fp64 oracle integrates the identical scene."""
    out = copy.deepcopy(c)
    for k, v in c.items():
        if isinstance(v, float):
            out[k] = _f32(v)
        elif isinstance(v, tuple) and v and all(isinstance(t, float) for t in v):
            out[k] = tuple(_f32(t) for t in v)
    out["emitters"] = [(tuple(_f32(t) for t in p), _f32(te), _f32(en)) for p, te, en in c["emitters"]]
    return out


def crop_center(c: dict, w: int, h: int) -> dict:
    """Centre crop of w x h pixels (oracle sub-workloads)."""
    out = dict(c)
    x0 = (c["width"] - w) // 2
    y0 = (c["height"] - h) // 2
    out["crop"] = (x0, y0, x0 + w, y0 + h)
    return out


def two_peak_response(n_bins: int, t0: float, t1: float, peaks=((5.0, 0.15, 1.0), (7.0, 0.15, 0.6)),
                      floor: float = 1e-3) -> np.ndarray:
    """A two-peak sensor response W(t) (the setting of PAPER.md:302-310, Fig. 6:
    "the temporal response weight comprises two peaks"), tabulated at the bin
    centres as a sum of Gaussians (centre, sigma, height), zeroed where it is
    below floor x its maximum so that it has exact zeros between the peaks.
    Rounded to float32 (what the device sees)."""
    tc = t0 + (np.arange(n_bins) + 0.5) * (t1 - t0) / n_bins
    w = np.zeros(n_bins)
    for mu, sg, h in peaks:
        w += h * np.exp(-0.5 * ((tc - mu) / sg) ** 2)
    w[w < floor * w.max()] = 0.0
    return w.astype(np.float32).astype(np.float64)


def response_config(**overrides) -> dict:
    """The rejection experiment: config 4's cube with walls and
    two emitters, a 3..9 time window of 120 bins and the two-peak W; spp paths
    per pixel, each drawing its bin with probability ~ W (R31)."""
    c = config(4, t0=3.0, t1=9.0, n_bins=120, spp=64, spp_mode="response", name="cfg4_two_peak_response")
    c.update(overrides)
    c["response"] = two_peak_response(c["n_bins"], c["t0"], c["t1"])
    return c


# ----------------------------------------------------------------------------
# triangle meshes (R32, R33): synthetic stand-ins for the
# paper's GLOSSY DRAGON and STAIRCASE scenes (Table 1),
# whose geometry is not available: a glossy icosphere and a plastic staircase.
def icosphere(center, radius, subdiv: int) -> np.ndarray:
    """Triangles (n, 3, 3) of a subdivided icosahedron, vertices projected on the sphere."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
         (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    tris = [[np.asarray(v[i], float) / np.linalg.norm(v[i]) for i in tri] for tri in f]
    for _ in range(subdiv):
        nxt = []
        for a, b, c in tris:
            ab, bc, ca = [(p + q) / np.linalg.norm(p + q) for p, q in ((a, b), (b, c), (c, a))]
            nxt += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        tris = nxt
    return np.asarray(center, float) + radius * np.asarray(tris)


def staircase(x0, x1, y0, z0, n_steps: int, rise: float, run: float) -> np.ndarray:
    """Triangles of n steps rising along +y and receding along +z (two per tread, two per riser)."""
    out = []
    for k in range(n_steps):
        ylo, yhi = y0 + k * rise, y0 + (k + 1) * rise
        za, zb = z0 + k * run, z0 + (k + 1) * run
        riser = [(x0, ylo, za), (x1, ylo, za), (x1, yhi, za), (x0, yhi, za)]
        tread = [(x0, yhi, za), (x1, yhi, za), (x1, yhi, zb), (x0, yhi, zb)]
        for q in (riser, tread):
            out += [[q[0], q[1], q[2]], [q[0], q[2], q[3]]]
    return np.asarray(out, float)


def mesh_config(ico_subdiv: int = 2, **overrides) -> dict:
    """Config 6: config 4's fog cube with walls and two
    emitters, plus a glossy icosphere (rho 0.8, ks 0.9, Phong n 40; 320
    triangles) and a plastic staircase (rho 0.6, ks 0.25, n 15; 16 triangles),
    time-gated in two bins of width 0.1.  ico_subdiv 4 / 6: 5120 / 81920
    sphere triangles (BVH depth checks)."""
    ico = icosphere((0.35, -0.45, 0.2), 0.35, ico_subdiv)
    st = staircase(-0.9, -0.1, -0.98, -0.2, 4, 0.2, 0.25)
    tris = np.concatenate([ico, st]).astype(np.float32).astype(np.float64)
    mat = np.concatenate([np.zeros(len(ico), np.int32), np.ones(len(st), np.int32)])
    c = config(4, t0=5.0, t1=5.2, n_bins=2, spp=64, width=256, height=256, name="cfg6_mesh_glossy_stairs", seed=6)
    c["mesh"] = dict(tris=tris.reshape(-1, 9), tri_mat=mat, mats=[(0.8, 0.9, 40.0), (0.6, 0.25, 15.0)])
    c.update(overrides)
    return c


def sphere_mesh_config(**overrides) -> dict:
    """Config 2's sphere (unwarped camera) with a glossy icosphere (r 0.3, 80
    triangles) and a Lambertian square plate (two triangles) inside: meshes in a
    SPHERE medium and the R17 shell intervals cut at a surface."""
    ico = icosphere((0.2, 0.1, 0.25), 0.3, 1)
    q = [(-0.6, -0.6, -0.3), (0.6, -0.6, -0.3), (0.6, 0.6, -0.3), (-0.6, 0.6, -0.3)]
    plate = np.array([[q[0], q[1], q[2]], [q[0], q[2], q[3]]], float)
    tris = np.concatenate([ico, plate]).astype(np.float32).astype(np.float64)
    mat = np.concatenate([np.zeros(len(ico), np.int32), np.ones(2, np.int32)])
    c = config(2, name="cfg2_sphere_mesh")
    c["mesh"] = dict(tris=tris.reshape(-1, 9), tri_mat=mat, mats=[(0.8, 0.7, 30.0), (0.7, 0.0, 1.0)])
    c.update(overrides)
    return c


def plate_config(mats, **overrides) -> dict:
    """A 4 x 4 square plate (two triangles) at z = 0 in an infinite, almost
    non-scattering medium (sigma_s = 1e-4), a pulse emitter and a fluence
    detector above it: the single-bounce surface case of the mesh pins."""
    c = config(1, sigma_s=1e-4, sigma_a=0.05, emitters=[((0.5, 0.0, 1.0), 0.0, 1.0)], cam_pos=(-0.5, 0.0, 1.0),
               det_radius=0.02, t0=2.0, t1=6.0, n_bins=40, name="plate_single_bounce")
    q = [(-2.0, -2.0, 0.0), (2.0, -2.0, 0.0), (2.0, 2.0, 0.0), (-2.0, 2.0, 0.0)]
    tris = np.array([q[0] + q[1] + q[2], q[0] + q[2] + q[3]], float)
    c["mesh"] = dict(tris=tris, tri_mat=np.zeros(2, np.int32), mats=mats)
    c.update(overrides)
    return c


def small(c: dict, width: int, height: int, n_bins: int | None = None, t1: float | None = None) -> dict:
    """A reduced-size variant of a config (same medium and geometry) for parity
    runs the oracle finishes in seconds."""
    out = dict(c)
    out["width"], out["height"] = width, height
    out["crop"] = (0, 0, width, height)
    if n_bins is not None:
        out["n_bins"] = n_bins
    if t1 is not None:
        out["t1"] = t1
    return out


# ----------------------------------------------------------------------------
# seeded debug records: positions in the medium, E in [0, R_M),
# random directions and raw 32-bit uniforms.
def _unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def debug_records(c: dict, n: int, seed: int, kinds=("camera", "medium", "wall", "surface")) -> dict:
    """Random vertex states for ``dts_sample_debug`` parity.  Returns a dict of
    numpy arrays (kind, face, bin, emitter, x[n,3], w[n,3], E, beta, r[n,12]).
    Surface records (mesh scenes): a uniform point of a random triangle, moved
    1e-4 off it on the side the incoming direction arrives from (R33)."""
    rng = np.random.default_rng(seed)
    kind = np.zeros(n, np.int32)
    face = np.full(n, -1, np.int32)
    x = np.zeros((n, 3))
    w = _unit(rng, n)
    names = {"camera": 0, "medium": 1, "wall": 2, "surface": 3}
    allowed = [names[k] for k in kinds]
    if c.get("mesh") is None and 3 in allowed:
        allowed.remove(3)
    if c["medium"] == "box" and c["wall_mask"] == 0 and 2 in allowed:
        allowed.remove(2)
    if c["medium"] != "box" and 2 in allowed:
        allowed.remove(2)
    kind[:] = rng.choice(allowed, size=n)
    ne = len(c["emitters"])
    emitter = rng.integers(0, ne, size=n).astype(np.int32)
    b = rng.integers(0, c["n_bins"], size=n).astype(np.int32)
    for i in range(n):
        if kind[i] == 0:
            if c["camera"] == "pinhole":
                x[i] = c["cam_pos"]
                tgt = rng.uniform(-0.5, 0.5, 3) * np.asarray(_extent(c))
                d = tgt - np.asarray(c["cam_pos"])
                w[i] = d / np.linalg.norm(d)
            else:
                x[i] = np.asarray(c["cam_pos"]) + _unit(rng, 1)[0] * c["det_radius"] * rng.uniform() ** (1 / 3)
        elif kind[i] == 1:
            x[i] = _inside(c, rng)
        elif kind[i] == 3:
            tris = np.asarray(c["mesh"]["tris"], float).reshape(-1, 3, 3)
            t = int(rng.integers(0, len(tris)))
            face[i] = t
            u, v = rng.uniform(size=2)
            if u + v > 1.0:
                u, v = 1.0 - u, 1.0 - v
            pt = tris[t, 0] + u * (tris[t, 1] - tris[t, 0]) + v * (tris[t, 2] - tris[t, 0])
            nrm = np.cross(tris[t, 1] - tris[t, 0], tris[t, 2] - tris[t, 0])
            nrm /= np.linalg.norm(nrm)
            if w[i] @ nrm > 0.0:
                nrm = -nrm
            x[i] = pt + 1e-4 * nrm
        else:
            faces = [f for f in range(6) if (c["wall_mask"] >> f) & 1]
            f = int(rng.choice(faces))
            face[i] = f
            p = _inside(c, rng)
            a = f // 2
            p[a] = c["bmax"][a] if (f & 1) else c["bmin"][a]
            x[i] = p
    dt = (c["t1"] - c["t0"]) / c["n_bins"]
    E = np.zeros(n)
    for i in range(n):
        te = c["emitters"][emitter[i]][1]
        RM = c["t0"] + (b[i] + 1) * dt - te
        C = np.linalg.norm(x[i] - np.asarray(c["emitters"][emitter[i]][0]))
        if kind[i] != 0 and RM - C > 0:
            E[i] = rng.uniform(0.0, RM - C)
    r = rng.integers(0, 2**32, size=(n, 12), dtype=np.uint64).astype(np.uint32)
    beta = np.ones(n)
    # the device stores positions/directions in float32: hand both sides the
    # identical (float32-representable) values
    x = x.astype(np.float32).astype(np.float64)
    w = w.astype(np.float32).astype(np.float64)
    return dict(kind=kind, face=face, bin=b, emitter=emitter, x=x, w=w, E=E, beta=beta, r=r)


def _extent(c):
    if c["medium"] == "sphere":
        return (2 * c["radius"],) * 3
    if c["medium"] == "box":
        return tuple(c["bmax"][i] - c["bmin"][i] for i in range(3))
    return (4.0, 4.0, 4.0)


def _inside(c, rng):
    if c["medium"] == "sphere":
        u = _unit(rng, 1)[0] * c["radius"] * rng.uniform() ** (1 / 3)
        return np.asarray(c["center"]) + u
    if c["medium"] == "box":
        return rng.uniform(np.asarray(c["bmin"]), np.asarray(c["bmax"]))
    # infinite: around the emitter / detector region
    return rng.uniform(-3.0, 3.0, 3)


def n_cells(c: dict) -> int:
    x0, y0, x1, y1 = c["crop"]
    return (x1 - x0) * (y1 - y0) * c["n_bins"]
