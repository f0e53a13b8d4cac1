"""ctypes wrapper of the fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It never imports the CUDA
package ``paper_2402_03106_b200`` and the CUDA package never imports it.  Scene
dicts come from the neutral input module ``dts_inputs``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdts_oracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "dts_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-shared", "-fPIC", "-pthread",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.or_uniform.restype = ctypes.c_double
        _lib.or_sobol.restype = ctypes.c_double
        _lib.or_da_flux.restype = ctypes.c_double
        _lib.or_hg_eval.restype = ctypes.c_double
        _lib.or_hg_eval.argtypes = [ctypes.c_double, ctypes.c_double]
        _lib.or_polar_distance.restype = ctypes.c_double
        _lib.or_polar_distance.argtypes = [ctypes.c_double] * 3
        _lib.or_table_integrand.restype = ctypes.c_double
        _lib.or_hg_sample_cos.restype = ctypes.c_double
        _lib.or_hg_sample_cos.argtypes = [ctypes.c_double, ctypes.c_double]
    return _lib


D3 = ctypes.c_double * 3


class OrScene(ctypes.Structure):
    _fields_ = [
        ("sigma_s", ctypes.c_double), ("sigma_a", ctypes.c_double), ("g", ctypes.c_double),
        ("medium_shape", ctypes.c_int32),
        ("center", D3), ("radius", ctypes.c_double), ("bmin", D3), ("bmax", D3),
        ("wall_mask", ctypes.c_uint32), ("wall_albedo", ctypes.c_double * 6),
        ("n_emitters", ctypes.c_int32),
        ("em_pos", D3 * 8), ("em_t", ctypes.c_double * 8), ("em_energy", ctypes.c_double * 8),
        ("camera_kind", ctypes.c_int32),
        ("cam_pos", D3), ("look_at", D3), ("up", D3), ("fov_y_deg", ctypes.c_double),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("det_radius", ctypes.c_double),
        ("crop", ctypes.c_int32 * 4),
        ("t0", ctypes.c_double), ("t1", ctypes.c_double),
        ("n_bins", ctypes.c_int32), ("warped", ctypes.c_int32),
        ("strategy", ctypes.c_int32), ("n_ris", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("max_bounces", ctypes.c_int32), ("direction_mode", ctypes.c_int32), ("spp_mode", ctypes.c_int32),
        ("parity_r_excl", ctypes.c_double), ("parity_s_excess", ctypes.c_double),
        ("table_nr", ctypes.c_int32), ("table_ns", ctypes.c_int32),
        ("table_smin", ctypes.c_double), ("table_smax", ctypes.c_double),
        ("conn_sampling", ctypes.c_int32),
        ("response", ctypes.c_void_p),
        ("n_tris", ctypes.c_int32), ("tris", ctypes.c_void_p), ("tri_mat", ctypes.c_void_p),
        ("n_mats", ctypes.c_int32), ("mats", D3 * 8),
        ("bin_window", ctypes.c_int32 * 2),
    ]


class OrStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "paths", "camera_miss", "vertices", "conn_nonempty", "ris_all_invalid",
        "early_exit", "escapes", "cap_hits", "nonfinite", "wall_nee", "samples", "rejected")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


DEBUG_IN = np.dtype([
    ("kind", np.int32), ("face", np.int32), ("bin", np.int32), ("emitter", np.int32),
    ("x", np.float64, 3), ("w", np.float64, 3), ("E", np.float64), ("beta", np.float64),
    ("r", np.uint32, 12),
], align=True)

DEBUG_OUT = np.dtype([
    ("tech", np.int32), ("gamma", np.float64), ("p_eda", np.float64), ("p_hg", np.float64),
    ("p_mix", np.float64), ("wc", np.float64, 3), ("ww", np.float64, 3), ("beta_dir", np.float64),
    ("wconn", np.float64),
    ("t_lo", np.float64), ("t_hi", np.float64), ("tc_lo", np.float64), ("tc_hi", np.float64),
    ("hit", np.int32), ("face_hit", np.int32),
    ("S_lo", np.float64), ("S_hi", np.float64), ("S", np.float64), ("t", np.float64),
    ("x_ell", np.float64, 3), ("p_t", np.float64), ("contrib", np.float64), ("nee", np.float64),
    ("conn_valid", np.int32),
    ("p_m", np.float64), ("event", np.int32),
    ("cand_d", np.float64, 8), ("cand_wn", np.float64, 8), ("istar", np.int32),
    ("d", np.float64), ("x_next", np.float64, 3), ("beta_ris", np.float64), ("E_next", np.float64),
    ("beta_out", np.float64), ("terminate", np.int32),
    ("m_event", np.float64), ("m_select", np.float64), ("m_tech", np.float64), ("m_cell", np.float64),
    ("m_hgbin", np.float64), ("m_valid", np.float64), ("m_conn", np.float64), ("m_term", np.float64),
    ("m_cond", np.float64),
], align=True)

_MED = {"infinite": 0, "sphere": 1, "box": 2}
_CAM = {"pinhole": 0, "detector": 1}
_STRAT = {"darts": 0, "vanilla": 1, "da_only": 2, "eda_only": 3}
_CONN = {"exp": 0, "uniform": 1}
_DIR = {"reuse": 0, "split": 1}
_SPP = {"cell": 0, "pixel": 1, "response": 2}


def scene(c: dict) -> OrScene:
    s = OrScene()
    s.sigma_s, s.sigma_a, s.g = c["sigma_s"], c["sigma_a"], c["g"]
    s.medium_shape = _MED[c["medium"]]
    s.center[:] = c["center"]
    s.radius = c["radius"]
    s.bmin[:] = c["bmin"]
    s.bmax[:] = c["bmax"]
    s.wall_mask = c["wall_mask"]
    s.wall_albedo[:] = c["wall_albedo"]
    s.n_emitters = len(c["emitters"])
    for i, (p, te, en) in enumerate(c["emitters"]):
        s.em_pos[i][:] = p
        s.em_t[i] = te
        s.em_energy[i] = en
    s.camera_kind = _CAM[c["camera"]]
    s.cam_pos[:] = c["cam_pos"]
    s.look_at[:] = c["look_at"]
    s.up[:] = c["up"]
    s.fov_y_deg = c["fov_y_deg"]
    s.width, s.height = c["width"], c["height"]
    s.det_radius = c["det_radius"]
    s.crop[:] = c["crop"]
    s.t0, s.t1 = c["t0"], c["t1"]
    s.n_bins, s.warped = c["n_bins"], c["warped"]
    s.strategy = _STRAT[c["strategy"]]
    s.n_ris = c["n_ris"]
    s.alpha = c["alpha"]
    s.max_bounces = c["max_bounces"]
    s.direction_mode = _DIR[c["direction_mode"]]
    s.spp_mode = _SPP[c["spp_mode"]]
    s.parity_r_excl, s.parity_s_excess = c["parity_r_excl"], c["parity_s_excess"]
    s.table_nr, s.table_ns = c["table_nr"], c["table_ns"]
    s.table_smin, s.table_smax = c["table_smin"], c["table_smax"]
    s.conn_sampling = _CONN[c.get("conn_sampling", "exp")]
    if c.get("response") is not None:
        w = np.ascontiguousarray(np.asarray(c["response"], dtype=np.float64))
        assert w.shape == (c["n_bins"],)
        s._response_keepalive = w
        s.response = w.ctypes.data
    if c.get("bin_window") is not None:
        s.bin_window[:] = c["bin_window"]
    m = c.get("mesh")
    if m is not None and len(m["tris"]):
        tris = np.ascontiguousarray(np.asarray(m["tris"], dtype=np.float64).reshape(-1, 9))
        mat = np.ascontiguousarray(np.asarray(m["tri_mat"], dtype=np.int32))
        assert mat.shape == (tris.shape[0],) and 1 <= len(m["mats"]) <= 8
        s._mesh_keepalive = (tris, mat)
        s.n_tris = tris.shape[0]
        s.tris = tris.ctypes.data
        s.tri_mat = mat.ctypes.data
        s.n_mats = len(m["mats"])
        for i, mm in enumerate(m["mats"]):
            s.mats[i][:] = mm
    return s


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def uniform(r: int) -> float:
    return lib().or_uniform(ctypes.c_uint32(r))


def sobol(row: int, col: int) -> float:
    return lib().or_sobol(ctypes.c_int(row), ctypes.c_int(col))


def da_flux(c: dict, r2: float, dt: float) -> float:
    s = scene(c)
    return lib().or_da_flux(ctypes.byref(s), ctypes.c_double(r2), ctypes.c_double(dt))


def hg_eval(g: float, mu: float) -> float:
    return lib().or_hg_eval(g, mu)


def hg_sample_cos(g: float, u: float) -> float:
    return lib().or_hg_sample_cos(g, u)


def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    lib().or_gauss_legendre(ctypes.c_int(n), _p(x), _p(w))
    return x, w


def polar_distance(C: float, S: float, mu: float) -> float:
    return lib().or_polar_distance(C, S, mu)


def intersect(c: dict, o, d):
    s = scene(c)
    lo, hi = ctypes.c_double(), ctypes.c_double()
    face = ctypes.c_int()
    hit = lib().or_intersect(ctypes.byref(s), D3(*o), D3(*d), ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(face))
    return hit, lo.value, hi.value, face.value


def mesh_hit(c: dict, o, d, t_max: float = float("inf")):
    """(triangle, t) of the nearest triangle hit with 0 < t < t_max, or (-1, None)."""
    sc = scene(c)
    t = ctypes.c_double()
    lib().or_mesh_hit.restype = ctypes.c_int
    tri = lib().or_mesh_hit(ctypes.byref(sc), D3(*o), D3(*d), ctypes.c_double(t_max), ctypes.byref(t))
    return (tri, t.value) if tri >= 0 else (-1, None)


def bsdf_eval(c: dict, tri: int, w, wo) -> float:
    sc = scene(c)
    lib().or_bsdf_eval.restype = ctypes.c_double
    return lib().or_bsdf_eval(ctypes.byref(sc), ctypes.c_int(tri), D3(*w), D3(*wo))


def bsdf_sample(c: dict, tri: int, w, u4: float, u5: float, u6: float):
    """(wo, f cos / p) of the R32 sampling."""
    sc = scene(c)
    wo = D3()
    lib().or_bsdf_sample.restype = ctypes.c_double
    wgt = lib().or_bsdf_sample(ctypes.byref(sc), ctypes.c_int(tri), D3(*w), ctypes.c_double(u4),
                               ctypes.c_double(u5), ctypes.c_double(u6), wo)
    return np.array(wo[:]), wgt


def table_integrand(c: dict, C: float, S: float, mu: float) -> float:
    s = scene(c)
    return lib().or_table_integrand(ctypes.byref(s), ctypes.c_double(C), ctypes.c_double(S), ctypes.c_double(mu))


def build_table(c: dict, nthreads: int | None = None):
    """Returns (q uint16 [nr*ns*256], mass float64 [nr*ns*256])."""
    s = scene(c)
    n = c["table_nr"] * c["table_ns"] * 256
    q = np.zeros(n, np.uint16)
    mass = np.zeros(n, np.float64)
    rc = lib().or_table_build(ctypes.byref(s), _p(mass), _p(q), ctypes.c_int(nthreads or os.cpu_count()))
    if rc != 0:
        raise RuntimeError(f"or_table_build failed: {rc}")
    return q, mass


def debug(c: dict, q: np.ndarray | None, recs: dict) -> np.ndarray:
    s = scene(c)
    n = len(recs["kind"])
    a = np.zeros(n, DEBUG_IN)
    for k in ("kind", "face", "bin", "emitter", "x", "w", "E", "beta", "r"):
        a[k] = recs[k]
    out = np.zeros(n, DEBUG_OUT)
    qq = q if q is not None else np.zeros(256, np.uint16)
    lib().or_debug(ctypes.byref(s), _p(qq), ctypes.c_int(n), _p(a), _p(out))
    return out


def render(c: dict, q: np.ndarray | None, spp: int, seed: int, s_begin: int = 0, s_end: int | None = None,
           n_orders: int = 0, sq: bool = True, nthreads: int | None = None) -> dict:
    """Oracle render of the crop in ``c``; returns hist [h, w, bins] (float64),
    hist_sq, order_hist [n_orders, h, w, bins] and stats."""
    s = scene(c)
    x0, y0, x1, y1 = c["crop"]
    shape = (y1 - y0, x1 - x0, c["n_bins"])
    cells = int(np.prod(shape))
    hist = np.zeros(cells)
    hsq = np.zeros(cells) if sq else None
    oh = np.zeros(cells * n_orders) if n_orders else None
    st = OrStats()
    if s_end is None:
        s_end = spp
    qq = q if q is not None else np.zeros(256, np.uint16)
    rc = lib().or_render(ctypes.byref(s), _p(qq), ctypes.c_uint64(spp), ctypes.c_uint64(seed),
                         ctypes.c_uint64(s_begin), ctypes.c_uint64(s_end), _p(hist),
                         _p(hsq) if hsq is not None else None, _p(oh) if oh is not None else None,
                         ctypes.c_int(n_orders), ctypes.byref(st), ctypes.c_int(nthreads or os.cpu_count()))
    if rc != 0:
        raise RuntimeError(f"or_render failed: {rc}")
    return dict(hist=hist.reshape(shape), hist_sq=None if hsq is None else hsq.reshape(shape),
                order_hist=None if oh is None else oh.reshape((n_orders,) + shape), stats=st.as_dict())


def uniform_index(n: int, r: int) -> int:
    lib().or_uniform_index.restype = ctypes.c_int
    return lib().or_uniform_index(ctypes.c_int(n), ctypes.c_uint32(r))


def pixel_offset(c: dict, seed: int, p: int) -> int:
    """R21: the bin offset o_p of image pixel p (row-major)."""
    s = scene(c)
    lib().or_pixel_offset.restype = ctypes.c_int
    return lib().or_pixel_offset(ctypes.byref(s), ctypes.c_uint64(seed), ctypes.c_uint64(p))


def cell_count(c: dict, spp: int, o_p: int, b: int) -> int:
    """R21: n_pb, the samples of a pixel with offset o_p that land in bin b."""
    s = scene(c)
    lib().or_cell_count.restype = ctypes.c_uint64
    return int(lib().or_cell_count(ctypes.byref(s), ctypes.c_uint64(spp), ctypes.c_int(o_p), ctypes.c_int(b)))


def render_ids(c: dict, q: np.ndarray, spp: int, seed: int, ids: np.ndarray):
    s = scene(c)
    ids = np.ascontiguousarray(ids, np.uint64)
    acc = np.zeros(len(ids))
    nv = np.zeros(len(ids), np.uint32)
    lib().or_render_ids(ctypes.byref(s), _p(q), ctypes.c_uint64(spp), ctypes.c_uint64(seed), _p(ids),
                        ctypes.c_int(len(ids)), _p(acc), _p(nv))
    return acc, nv
