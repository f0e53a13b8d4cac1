"""Thin ctypes binding of libdts.so (include/dts.h).  Argument marshalling
only: every step of the path runs in the library's kernels.  Names follow the
C ABI (dts_scene_create -> scene_create, ...).  Device buffers are passed as
raw pointers (torch tensors are accepted and their ``data_ptr()`` is used);
torch is plumbing (memory, streams), never part of the compute path."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DTS_LIB selects an alternative in-tree build of the same library (launch
# geometry sweeps); the default is the one __graft_entry__.build() produces.
LIB_PATH = os.path.join(_HERE, os.environ.get("DTS_LIB", "libdts.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                      "There is no CPU fallback.")
_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------- ABI structs
F3 = ctypes.c_float * 3
MAX_EMITTERS = 8
NUM_COUNTERS = 15
COUNTER_NAMES = ("paths", "camera_miss", "vertices", "conn_nonempty", "ris_invalid", "early_exit", "escapes",
                 "cap_hits", "nonfinite", "wall_nee", "samples", "rejected", "walk_vertices",
                 "camera_vertices", "wall_vertices")


class SceneDesc(ctypes.Structure):
    _fields_ = [
        ("sigma_s", ctypes.c_float), ("sigma_a", ctypes.c_float), ("g", ctypes.c_float),
        ("medium_shape", ctypes.c_int32),
        ("center", F3), ("radius", ctypes.c_float), ("bmin", F3), ("bmax", F3),
        ("wall_mask", ctypes.c_uint32), ("wall_albedo", ctypes.c_float * 6),
        ("n_emitters", ctypes.c_int32),
        ("em_pos", F3 * MAX_EMITTERS), ("em_t", ctypes.c_float * MAX_EMITTERS),
        ("em_energy", ctypes.c_float * MAX_EMITTERS),
        ("camera_kind", ctypes.c_int32),
        ("cam_pos", F3), ("look_at", F3), ("up", F3), ("fov_y_deg", ctypes.c_float),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("det_radius", ctypes.c_float),
        ("crop", ctypes.c_int32 * 4),
        ("t0", ctypes.c_float), ("t1", ctypes.c_float),
        ("n_bins", ctypes.c_int32), ("warped", ctypes.c_int32),
        ("strategy", ctypes.c_int32), ("n_ris", ctypes.c_int32), ("alpha", ctypes.c_float),
        ("max_bounces", ctypes.c_int32), ("direction_mode", ctypes.c_int32), ("spp_mode", ctypes.c_int32),
        ("parity_r_excl", ctypes.c_float), ("parity_s_excess", ctypes.c_float),
        ("conn_sampling", ctypes.c_int32),
        ("n_tris", ctypes.c_int32), ("tris", ctypes.c_void_p), ("tri_mat", ctypes.c_void_p),
        ("n_mats", ctypes.c_int32), ("mats", (ctypes.c_float * 3) * 8),
    ]


class TableDesc(ctypes.Structure):
    _fields_ = [("n_ratio", ctypes.c_int32), ("n_s", ctypes.c_int32),
                ("s_min", ctypes.c_float), ("s_max", ctypes.c_float)]


DEBUG_IN = np.dtype([
    ("kind", np.int32), ("face", np.int32), ("bin", np.int32), ("emitter", np.int32),
    ("x", np.float32, 3), ("w", np.float32, 3), ("E", np.float64), ("beta", np.float32), ("pad_", np.float32),
    ("r", np.uint32, 12),
], align=True)

DEBUG_OUT = np.dtype([
    ("tech", np.int32), ("gamma", np.float32), ("p_eda", np.float32), ("p_hg", np.float32), ("p_mix", np.float32),
    ("wc", np.float32, 3), ("ww", np.float32, 3), ("beta_dir", np.float32), ("wconn", np.float32),
    ("t_lo", np.float32), ("t_hi", np.float32), ("tc_lo", np.float32), ("tc_hi", np.float32),
    ("hit", np.int32), ("face_hit", np.int32),
    ("S_lo", np.float32), ("S_hi", np.float32), ("S", np.float32), ("t", np.float32), ("x_ell", np.float32, 3),
    ("p_t", np.float32), ("contrib", np.float32), ("nee", np.float32), ("conn_valid", np.int32),
    ("p_m", np.float32), ("event", np.int32), ("cand_d", np.float32, 8), ("cand_wn", np.float32, 8),
    ("istar", np.int32), ("d", np.float32), ("x_next", np.float32, 3), ("beta_ris", np.float32),
    ("E_next", np.float64), ("beta_out", np.float32), ("terminate", np.int32),
], align=True)

_VP = ctypes.c_void_p
_U64 = ctypes.c_uint64
_lib.dts_scene_create.argtypes = [ctypes.POINTER(SceneDesc), ctypes.POINTER(_VP)]
_lib.dts_scene_destroy.argtypes = [_VP]
_lib.dts_table_build.argtypes = [_VP, ctypes.POINTER(TableDesc), _VP]
_lib.dts_table_export.argtypes = [_VP, _VP, ctypes.c_size_t]
_lib.dts_table_size.argtypes = [_VP]
_lib.dts_table_size.restype = ctypes.c_size_t
_lib.dts_hist_cells.argtypes = [_VP]
_lib.dts_hist_cells.restype = ctypes.c_size_t
_lib.dts_render.argtypes = [_VP, _U64, _U64, _U64, _U64, _VP, _VP, _VP, _VP]
_lib.dts_render_host.argtypes = [_VP, _U64, _U64, _U64, _U64, _VP, _VP, _VP]
_lib.dts_render_rows.argtypes = [_VP, _U64, _U64, _U64, _U64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP,
                                 _VP, _VP]
_lib.dts_sample_debug.argtypes = [_VP, ctypes.c_int32, _VP, _VP, _VP]
_lib.dts_last_launch.argtypes = [ctypes.POINTER(ctypes.c_int32)] * 4
_lib.dts_set_response.argtypes = [_VP, _VP, ctypes.c_int32]
_lib.dts_check_failures.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
_lib.dts_enable_peer.argtypes = [ctypes.c_int32]
_lib.dts_pool_release.argtypes = []
_lib.dts_status_string.restype = ctypes.c_char_p
_lib.dts_status_string.argtypes = [ctypes.c_int]
_lib.dts_last_error.restype = ctypes.c_char_p
_lib.dts_abi_version.restype = ctypes.c_int32

EXPORTED = ("dts_scene_create", "dts_scene_destroy", "dts_set_response", "dts_table_build", "dts_table_export",
            "dts_table_size", "dts_check_failures", "dts_enable_peer", "dts_pool_release",
            "dts_hist_cells", "dts_render", "dts_render_rows", "dts_render_host", "dts_sample_debug", "dts_last_launch",
            "dts_status_string", "dts_last_error", "dts_abi_version")


class DtsError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != 0:
        raise DtsError(f"{what}: {_lib.dts_status_string(st).decode()}: {_lib.dts_last_error().decode()}")


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(stream) -> int | None:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


_MED = {"infinite": 0, "sphere": 1, "box": 2}
_CAM = {"pinhole": 0, "detector": 1}
_STRAT = {"darts": 0, "vanilla": 1, "da_only": 2, "eda_only": 3}
_CONN = {"exp": 0, "uniform": 1}
_DIR = {"reuse": 0, "split": 1}
_SPP = {"cell": 0, "pixel": 1, "response": 2}


def scene_desc(c: dict) -> SceneDesc:
    """Scene dict (``dts_inputs.config``) -> dts_scene_desc."""
    d = SceneDesc()
    d.sigma_s, d.sigma_a, d.g = c["sigma_s"], c["sigma_a"], c["g"]
    d.medium_shape = _MED[c["medium"]]
    d.center[:] = c["center"]
    d.radius = c["radius"]
    d.bmin[:] = c["bmin"]
    d.bmax[:] = c["bmax"]
    d.wall_mask = c["wall_mask"]
    d.wall_albedo[:] = c["wall_albedo"]
    d.n_emitters = len(c["emitters"])
    for i, (p, te, en) in enumerate(c["emitters"]):
        d.em_pos[i][:] = p
        d.em_t[i] = te
        d.em_energy[i] = en
    d.camera_kind = _CAM[c["camera"]]
    d.cam_pos[:] = c["cam_pos"]
    d.look_at[:] = c["look_at"]
    d.up[:] = c["up"]
    d.fov_y_deg = c["fov_y_deg"]
    d.width, d.height = c["width"], c["height"]
    d.det_radius = c["det_radius"]
    d.crop[:] = c["crop"]
    d.t0, d.t1 = c["t0"], c["t1"]
    d.n_bins, d.warped = c["n_bins"], c["warped"]
    d.strategy = _STRAT[c["strategy"]]
    d.n_ris = c["n_ris"]
    d.alpha = c["alpha"]
    d.max_bounces = c["max_bounces"]
    d.direction_mode = _DIR[c["direction_mode"]]
    d.spp_mode = _SPP[c["spp_mode"]]
    d.parity_r_excl, d.parity_s_excess = c["parity_r_excl"], c["parity_s_excess"]
    d.conn_sampling = _CONN[c.get("conn_sampling", "exp")]
    m = c.get("mesh")
    if m is not None and len(m["tris"]):
        tris = np.ascontiguousarray(np.asarray(m["tris"], dtype=np.float32).reshape(-1, 9))
        mat = np.ascontiguousarray(np.asarray(m["tri_mat"], dtype=np.int32))
        d._mesh_keepalive = (tris, mat)   # read by dts_scene_create (copied there)
        d.n_tris = tris.shape[0]
        d.tris = tris.ctypes.data
        d.tri_mat = mat.ctypes.data
        d.n_mats = len(m["mats"])
        for i, mm in enumerate(m["mats"]):
            d.mats[i][:] = mm
    return d


class Scene:
    """Owns one dts_scene_t."""

    def __init__(self, c: dict):
        self.config = dict(c)
        self._desc = scene_desc(c)
        h = _VP()
        _check(_lib.dts_scene_create(ctypes.byref(self._desc), ctypes.byref(h)), "dts_scene_create")
        self.handle = h.value
        if c.get("response") is not None:
            self.set_response(c["response"])

    def close(self):
        if getattr(self, "handle", None):
            _lib.dts_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls with the C names -------------------------------------------------
    def table_build(self, n_ratio: int | None = None, n_s: int | None = None, s_min: float | None = None,
                    s_max: float | None = None, stream=None):
        c = self.config
        td = TableDesc(n_ratio or c.get("table_nr", 16), n_s or c.get("table_ns", 16),
                       s_min if s_min is not None else c.get("table_smin") or 0.0,
                       s_max if s_max is not None else c.get("table_smax") or 0.0)
        _check(_lib.dts_table_build(self.handle, ctypes.byref(td), _stream(stream)), "dts_table_build")

    def set_response(self, w) -> None:
        a = np.ascontiguousarray(np.asarray(w, dtype=np.float32))
        _check(_lib.dts_set_response(self.handle, a.ctypes.data, a.size), "dts_set_response")

    def table_size(self) -> int:
        return int(_lib.dts_table_size(self.handle))

    def table_export(self) -> np.ndarray:
        n = self.table_size()
        q = np.zeros(n, np.uint16)
        _check(_lib.dts_table_export(self.handle, q.ctypes.data, n), "dts_table_export")
        return q

    def hist_cells(self) -> int:
        return int(_lib.dts_hist_cells(self.handle))

    def hist_shape(self) -> tuple:
        x0, y0, x1, y1 = self.config["crop"]
        return (y1 - y0, x1 - x0, self.config["n_bins"])

    def render(self, spp: int, seed: int, sample_begin: int, sample_end: int, hist, hist_sq=None, counters=None,
               stream=None):
        _check(_lib.dts_render(self.handle, spp, seed, sample_begin, sample_end, _ptr(hist), _ptr(hist_sq),
                               _ptr(counters), _stream(stream)), "dts_render")

    def render_rows(self, spp: int, seed: int, sample_begin: int, sample_end: int, row0: int, row1: int, band: int,
                    hist_band, counters=None, stream=None):
        """dts_render over crop rows [row0, row1) into hist_band (that band's cells)."""
        _check(_lib.dts_render_rows(self.handle, spp, seed, sample_begin, sample_end, row0, row1, band,
                                    _ptr(hist_band), _ptr(counters), _stream(stream)), "dts_render_rows")

    def render_host(self, spp: int, seed: int, sample_begin: int, sample_end: int, h_hist: np.ndarray,
                    h_counters: np.ndarray | None = None, stream=None):
        assert h_hist.dtype == np.float32 and h_hist.size == self.hist_cells()
        _check(_lib.dts_render_host(self.handle, spp, seed, sample_begin, sample_end, h_hist.ctypes.data,
                                    None if h_counters is None else h_counters.ctypes.data, _stream(stream)),
               "dts_render_host")

    def sample_debug(self, d_in, d_out, n: int, stream=None):
        _check(_lib.dts_sample_debug(self.handle, n, _ptr(d_in), _ptr(d_out), _stream(stream)), "dts_sample_debug")


def last_launch() -> dict:
    v = [ctypes.c_int32() for _ in range(4)]
    _lib.dts_last_launch(*[ctypes.byref(x) for x in v])
    return dict(n_launches=v[0].value, grid=v[1].value, block=v[2].value, smem=v[3].value)


def check_failures() -> int:
    """Failed device-side bounds checks since the last call (check builds only)."""
    v = ctypes.c_uint64()
    _check(_lib.dts_check_failures(ctypes.byref(v)), "dts_check_failures")
    return int(v.value)


def pool_release() -> None:
    """dts_pool_release: frees the library's pooled device buffers."""
    _check(_lib.dts_pool_release(), "dts_pool_release")


def enable_peer(peer: int) -> None:
    """dts_enable_peer: peer access from the current device to device ``peer``."""
    _check(_lib.dts_enable_peer(int(peer)), "dts_enable_peer")


def abi_version() -> int:
    return int(_lib.dts_abi_version())


def status_string(code: int) -> str:
    return _lib.dts_status_string(code).decode()


def lib_handle():
    return _lib


# ----------------------------------------------------------------- torch convenience (plumbing only)
def debug_records_to_device(recs: dict):
    """Pack a ``dts_inputs.debug_records`` dict as dts_debug_in on the device."""
    import torch
    n = len(recs["kind"])
    a = np.zeros(n, DEBUG_IN)
    for k in ("kind", "face", "bin", "emitter", "x", "w", "E", "beta", "r"):
        a[k] = recs[k]
    d_in = torch.from_numpy(a.view(np.uint8)).cuda()
    d_out = torch.zeros(n * DEBUG_OUT.itemsize, dtype=torch.uint8, device="cuda")
    return d_in, d_out


def debug(scene: Scene, recs: dict) -> np.ndarray:
    """Run dts_sample_debug on host records; returns a DEBUG_OUT array."""
    import torch
    n = len(recs["kind"])
    d_in, d_out = debug_records_to_device(recs)
    scene.sample_debug(d_in, d_out, n)
    torch.cuda.synchronize()
    return d_out.cpu().numpy().view(DEBUG_OUT)


def render_to_tensor(scene: Scene, spp: int, seed: int, sample_begin: int = 0, sample_end: int | None = None,
                     with_sq: bool = False, stream=None):
    """Allocate a zeroed device histogram with torch, render into it; returns
    (hist [h, w, bins], hist_sq or None, counters dict)."""
    import torch
    shape = scene.hist_shape()
    h = torch.zeros(shape, dtype=torch.float32, device="cuda")
    hs = torch.zeros(shape, dtype=torch.float32, device="cuda") if with_sq else None
    ctr = torch.zeros(NUM_COUNTERS, dtype=torch.int64, device="cuda")
    scene.render(spp, seed, sample_begin, spp if sample_end is None else sample_end, h, hs, ctr, stream)
    return h, hs, ctr


def counters_dict(ctr) -> dict:
    v = ctr.cpu().numpy() if hasattr(ctr, "cpu") else np.asarray(ctr)
    return {n: int(x) for n, x in zip(COUNTER_NAMES, v)}
