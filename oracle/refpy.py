"""ctypes bindings for oracle/_ref/libtacchi_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (/root/reference/proj, compiled by
oracle/Makefile against the Eigen-subset shim). Only tests/, smoke() and the
bench's reference / cpu_baseline legs import this module; the product never
does. Arrays use the "row layout" documented in oracle/ref_driver.cpp.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtacchi_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_lp = C.POINTER(C.c_long)
_vpp = C.POINTER(C.c_void_p)

_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.c_double, C.c_int, _vpp]
        L.ref_build_parts.argtypes = [_ip, C.c_double, _dp, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_int, _dp, C.c_double, _dp, _ip, _dp, _dp,
                                      C.c_long, _dp, C.c_int, _vpp]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_num_particles.argtypes = [C.c_void_p]
        L.ref_num_particles.restype = C.c_long
        L.ref_elastomer_count.argtypes = [C.c_void_p]
        L.ref_elastomer_count.restype = C.c_long
        L.ref_set_threads.argtypes = [C.c_void_p, C.c_int]
        L.ref_get_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _u8p]
        L.ref_set_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.ref_step.argtypes = [C.c_void_p, _dp, C.c_int]
        L.ref_phase.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_get_diag.argtypes = [C.c_void_p, _dp, _dp, _lp, _dp]
        L.ref_grid_info.argtypes = [C.c_void_p, _ip, _dp, _dp, _ip, _ip]
        L.ref_get_grid.argtypes = [C.c_void_p, _ip, _ip, _dp, _dp, _dp]
        L.ref_surface.argtypes = [C.c_void_p, _ip, _ip, _dp, _u32p]
        L.ref_capture.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, _dp, _u8p, _ip, _ip]
        L.ref_extract_depth.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, _dp, _ip, _ip]
        L.ref_crop_align.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_surface_normals.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
        L.ref_phong.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_char_p, _u8p]
        L.ref_config_lights.argtypes = [C.c_char_p, _dp, _ip]
        L.ref_generate_cloud.argtypes = [C.c_char_p, C.c_long, C.c_uint64, _dp]
        L.ref_placed_indenter.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.c_double, _dp, _lp]
        L.ref_polar_rotation.argtypes = [_dp, _dp]
        L.ref_polar_rotation_svd.argtypes = [_dp, _dp]
        L.ref_corotated_stress.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp]
        L.ref_oracle_step.argtypes = [C.c_long, _dp, _dp, _dp, _dp, _dp, _dp, _u8p, C.c_int,
                                      C.c_int, C.c_int, C.c_double, _dp, C.c_double, C.c_double,
                                      C.c_double, _dp, _dp, _dp, _dp]
        _lib = L
    return _lib


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def cfg_json(cfg) -> bytes:
    return (cfg if isinstance(cfg, str) else json.dumps(cfg or {})).encode()


class RefSim:
    """The reference SimState, built by build_sim / init_scene."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @classmethod
    def from_config(cls, cfg=None, obj="", off_x=0.0, off_y=0.0, threads=0):
        h = C.c_void_p()
        _check(lib().ref_build(cfg_json(cfg), obj.encode(), off_x, off_y, threads, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_parts(cls, res, grid_edge, lat_dims, lat_counts, lat_origin, ind_pos, *, dt,
                   E=1.45e5, nu=0.45, rho=1000.0, fixed_bottom_layers=2, gravity=(0, 0, 0),
                   indenter_mass_scale=80.0, grid_origin=(0, 0, 0), ind_v0=(0, 0, 0), threads=0):
        h = C.c_void_p()
        ind = _d(ind_pos).reshape(-1, 3)
        _check(lib().ref_build_parts(
            _p(np.asarray(res, np.int32), _ip), grid_edge, _p(_d(grid_origin)), E, nu, rho, dt,
            fixed_bottom_layers, _p(_d(gravity)), indenter_mass_scale, _p(_d(lat_dims)),
            _p(np.asarray(lat_counts, np.int32), _ip), _p(_d(lat_origin)), _p(ind),
            ind.shape[0], _p(_d(ind_v0)), threads, C.byref(h)))
        return cls(h.value)

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().ref_destroy(self.h)
            self.h = None

    @property
    def n(self):
        return lib().ref_num_particles(self.h)

    @property
    def n_elastomer(self):
        return lib().ref_elastomer_count(self.h)

    def set_threads(self, n):
        lib().ref_set_threads(self.h, n)

    def state(self):
        n = self.n
        s = dict(x=np.empty((n, 3)), v=np.empty((n, 3)), C=np.empty((n, 3, 3)),
                 F=np.empty((n, 3, 3)), mass=np.empty(n), vol0=np.empty(n),
                 tag=np.empty(n, np.uint8))
        _check(lib().ref_get_state(self.h, _p(s["x"]), _p(s["v"]), _p(s["C"]), _p(s["F"]),
                                   _p(s["mass"]), _p(s["vol0"]), _p(s["tag"], _u8p)))
        return s

    def set_state(self, x=None, v=None, Cm=None, F=None):
        arrs = [None if a is None else _d(a) for a in (x, v, Cm, F)]
        _check(lib().ref_set_state(self.h, *[_p(a) for a in arrs]))

    def step(self, vind, n=1):
        _check(lib().ref_step(self.h, _p(_d(vind)), n))

    def phase(self, pid, vind=(0, 0, 0)):
        _check(lib().ref_phase(self.h, pid, _p(_d(vind))))

    def diag(self):
        a, b, c, v = C.c_double(), C.c_double(), C.c_long(), np.empty(3)
        lib().ref_get_diag(self.h, C.byref(a), C.byref(b), C.byref(c), _p(v))
        return dict(min_det_f=a.value, max_speed=b.value, step_count=c.value,
                    indenter_velocity=v)

    def grid_info(self):
        res, o, lo, hi = (np.empty(3, np.int32), np.empty(3), np.empty(3, np.int32),
                          np.empty(3, np.int32))
        dx = C.c_double()
        lib().ref_grid_info(self.h, _p(res, _ip), C.byref(dx), _p(o), _p(lo, _ip), _p(hi, _ip))
        return dict(res=res, dx=dx.value, origin=o, lo=lo, hi=hi)

    def grid(self, lo, hi):
        lo = np.asarray(lo, np.int32)
        hi = np.asarray(hi, np.int32)
        shp = tuple(int(v) for v in (hi - lo))
        m, mom, vel = np.empty(shp), np.empty(shp + (3,)), np.empty(shp + (3,))
        _check(lib().ref_get_grid(self.h, _p(lo, _ip), _p(hi, _ip), _p(m), _p(mom), _p(vel)))
        return m, mom, vel

    def surface(self):
        nx, ny, geom = C.c_int(), C.c_int(), np.empty(5)
        lib().ref_surface(self.h, C.byref(nx), C.byref(ny), _p(geom), None)
        idx = np.empty(nx.value * ny.value, np.uint32)
        lib().ref_surface(self.h, C.byref(nx), C.byref(ny), _p(geom), _p(idx, _u32p))
        return dict(nx=nx.value, ny=ny.value, x0=geom[0], y0=geom[1], sx=geom[2], sy=geom[3],
                    z0=geom[4], particle=idx)

    def capture(self, cfg=None, obj=""):
        w, h = C.c_int(), C.c_int()
        rp = (cfg or {}).get("render", {}) if isinstance(cfg, dict) else {}
        W, H = rp.get("image_width", 640), rp.get("image_height", 480)
        depth = np.empty((H, W))
        rgb = np.empty((H, W, 3), np.uint8)
        _check(lib().ref_capture(self.h, cfg_json(cfg), obj.encode(), _p(depth), _p(rgb, _u8p),
                                 C.byref(w), C.byref(h)))
        return depth, rgb

    def extract_depth(self, r, w=0, h=0):
        ow, oh = C.c_int(), C.c_int()
        _check(lib().ref_extract_depth(self.h, w, h, r, None, C.byref(ow), C.byref(oh)))
        out = np.empty((oh.value, ow.value))
        _check(lib().ref_extract_depth(self.h, w, h, r, _p(out), C.byref(ow), C.byref(oh)))
        return out


def crop_align(src, r, offset=(0.0, 0.0), scale=1.0, out_w=640, out_h=480):
    src = _d(src)
    out = np.empty((out_h, out_w))
    r_out = C.c_double()
    _check(lib().ref_crop_align(_p(src), src.shape[1], src.shape[0], r, offset[0], offset[1],
                                scale, out_w, out_h, _p(out), C.byref(r_out)))
    return out, r_out.value


def surface_normals(depth, r):
    d = _d(depth)
    out = np.empty(d.shape + (3,))
    _check(lib().ref_surface_normals(_p(d), d.shape[1], d.shape[0], r, _p(out)))
    return out


def phong(depth, r, cfg=None):
    d = _d(depth)
    out = np.empty(d.shape + (3,), np.uint8)
    _check(lib().ref_phong(_p(d), d.shape[1], d.shape[0], r, cfg_json(cfg), _p(out, _u8p)))
    return out


def config_lights(cfg=None):
    n = C.c_int()
    _check(lib().ref_config_lights(cfg_json(cfg), None, C.byref(n)))
    out = np.empty((n.value, 9))
    _check(lib().ref_config_lights(cfg_json(cfg), _p(out), C.byref(n)))
    return out


def generate_cloud(shape, n, seed):
    out = np.empty((n, 3))
    _check(lib().ref_generate_cloud(shape.encode(), n, seed, _p(out)))
    return out


def bridge_run(messages, base_cfg=None, session_root="."):
    """The reference's bridge::run_protocol over in-memory lines; parsed replies.
    Images are written as binary PPM under the .png name (ref_driver.cpp)."""
    L = lib()
    L.ref_bridge_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
    L.ref_free.argtypes = [C.c_void_p]
    lines = [m if isinstance(m, str) else json.dumps(m) for m in messages]
    out = C.c_void_p()
    _check(L.ref_bridge_run(cfg_json(base_cfg), session_root.encode(),
                            ("\n".join(lines) + "\n").encode(), C.byref(out)))
    try:
        text = C.string_at(out.value).decode()
    finally:
        L.ref_free(out)
    return [json.loads(x) for x in text.splitlines() if x]


def run_press_dataset(cfg, out_dir):
    """The reference's dataset::run_press_dataset; returns (rows, skipped)."""
    L = lib()
    L.ref_run_press_dataset.argtypes = [C.c_char_p, C.c_char_p, _lp, _lp]
    rows, skipped = C.c_long(), C.c_long()
    _check(L.ref_run_press_dataset(cfg_json(cfg), str(out_dir).encode(), C.byref(rows),
                                   C.byref(skipped)))
    return rows.value, skipped.value


def image_metrics(a, b):
    """metrics::compare -> (ssim, psnr_db, mae_pct)."""
    L = lib()
    L.ref_image_metrics.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _dp]
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    out = np.zeros(3)
    _check(L.ref_image_metrics(_p(a, _u8p), _p(b, _u8p), a.shape[1], a.shape[0], _p(out)))
    return tuple(out)


def load_ppm(path):
    with open(path, "rb") as f:
        data = f.read()
    parts = data.split(b"\n", 3)
    w, h = map(int, parts[1].split())
    return np.frombuffer(parts[3], dtype=np.uint8)[: w * h * 3].reshape(h, w, 3)


def placed_indenter(cfg=None, obj="", off_x=0.0, off_y=0.0):
    n = C.c_long()
    _check(lib().ref_placed_indenter(cfg_json(cfg), obj.encode(), off_x, off_y, None, C.byref(n)))
    out = np.empty((n.value, 3))
    _check(lib().ref_placed_indenter(cfg_json(cfg), obj.encode(), off_x, off_y, _p(out),
                                     C.byref(n)))
    return out


def polar_rotation(F):
    R = np.empty((3, 3))
    _check(lib().ref_polar_rotation(_p(_d(F)), _p(R)))
    return R


def polar_rotation_svd(F):
    R = np.empty((3, 3))
    _check(lib().ref_polar_rotation_svd(_p(_d(F)), _p(R)))
    return R


def corotated_stress(F, E=1.45e5, nu=0.45, rho=1000.0):
    S = np.empty((3, 3))
    _check(lib().ref_corotated_stress(_p(_d(F)), E, nu, rho, _p(S)))
    return S


def oracle_step(state, res, dx, origin, mu, lam, dt, vind):
    """tests/oracle/reference_mpm.cpp:reference_step; returns (state', grid)."""
    s = {k: np.array(state[k], dtype=np.float64 if k != "tag" else np.uint8, copy=True)
         for k in ("x", "v", "C", "F", "mass", "vol0", "tag")}
    nx, ny, nz = (int(r) for r in res)
    gm, gmom, gvel = np.empty((nx, ny, nz)), np.empty((nx, ny, nz, 3)), np.empty((nx, ny, nz, 3))
    _check(lib().ref_oracle_step(len(s["mass"]), _p(s["x"]), _p(s["v"]), _p(s["C"]), _p(s["F"]),
                                 _p(s["mass"]), _p(s["vol0"]), _p(s["tag"], _u8p), nx, ny, nz, dx,
                                 _p(_d(origin)), mu, lam, dt, _p(_d(vind)), _p(gm), _p(gmom),
                                 _p(gvel)))
    return s, (gm, gmom, gvel)
