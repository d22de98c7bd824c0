"""ctypes bindings for the C restatement oracle/_build/libtacchi_oracle.so.

TEST INFRASTRUCTURE ONLY: the parity checker for the CUDA product. Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this. Layout and error codes as oracle/tacchi_oracle.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libtacchi_oracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)


class Params(C.Structure):
    _fields_ = [("res", C.c_int * 3), ("dx", C.c_double), ("origin", C.c_double * 3),
                ("mu", C.c_double), ("lam", C.c_double), ("dt", C.c_double),
                ("gravity", C.c_double * 3)]


class Diag(C.Structure):
    _fields_ = [("min_det_f", C.c_double), ("max_speed", C.c_double), ("step_count", C.c_int64)]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.to_polar_rotation.argtypes = [_dp, _dp]
        L.to_polar_rotation_svd.argtypes = [_dp, _dp]
        L.to_corotated_stress.argtypes = [_dp, C.c_double, C.c_double, _dp]
        L.to_stencil.argtypes = [_dp, _dp, C.c_double, _ip, _dp, _dp]
        L.to_window.argtypes = [C.POINTER(Params), C.c_long, _dp, _ip, _ip]
        L.to_p2g.argtypes = [C.POINTER(Params), C.c_long, _dp, _dp, _dp, _dp, _dp, _dp, _u8p, _ip,
                             _ip, _dp, _dp, _dp]
        L.to_grid_update.argtypes = [C.POINTER(Params), _ip, _ip, _dp, _dp, _dp]
        L.to_g2p.argtypes = [C.POINTER(Params), C.c_long, _dp, _dp, _dp, _dp, _u8p, _ip, _ip, _dp]
        L.to_apply_boundary.argtypes = [C.c_long, _dp, _u8p, _dp]
        L.to_advect.argtypes = [C.POINTER(Params), C.c_long, _dp, _dp, _dp]
        L.to_step.argtypes = [C.POINTER(Params), C.c_long, _dp, _dp, _dp, _dp, _dp, _dp, _u8p, _dp,
                              C.c_int, C.POINTER(Diag)]
        L.to_extract_depth.argtypes = [C.c_int, C.c_int, _dp, _u32p, _dp, C.c_int, C.c_int,
                                       C.c_double, _dp]
        L.to_full_depth_size.argtypes = [C.c_int, C.c_int, _dp, C.c_double, _ip, _ip]
        L.to_crop_align.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.c_int, _dp]
        L.to_surface_normals.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
        L.to_phong.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp, C.c_int, _dp, _u8p, _u8p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error {code}")
        self.code = code


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def params(res, dx, origin=(0, 0, 0), E=1.45e5, nu=0.45, dt=1e-5, gravity=(0, 0, 0)):
    P = Params()
    P.res[:] = [int(r) for r in res]
    P.dx = dx
    P.origin[:] = list(origin)
    P.mu = E / (2.0 * (1.0 + nu))
    P.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    P.dt = dt
    P.gravity[:] = list(gravity)
    return P


class OracleSim:
    """Host state + the serial restatement of mpm::step."""

    def __init__(self, P: Params, x, v, mass, vol0, tag, C_=None, F=None):
        n = len(mass)
        self.P = P
        self.x = _d(x).reshape(n, 3).copy()
        self.v = _d(v).reshape(n, 3).copy()
        self.C = np.zeros((n, 3, 3)) if C_ is None else _d(C_).reshape(n, 3, 3).copy()
        self.F = (np.tile(np.eye(3), (n, 1, 1)) if F is None else _d(F).reshape(n, 3, 3).copy())
        self.mass = _d(mass).copy()
        self.vol0 = _d(vol0).copy()
        self.tag = np.ascontiguousarray(tag, np.uint8).copy()
        self.diag = Diag(1.0, 0.0, 0)

    @property
    def n(self):
        return len(self.mass)

    def step(self, vind, n_substeps=1):
        rc = lib().to_step(C.byref(self.P), self.n, _p(self.x), _p(self.v), _p(self.C),
                           _p(self.F), _p(self.mass), _p(self.vol0), _p(self.tag, _u8p),
                           _p(_d(vind)), n_substeps, C.byref(self.diag))
        if rc:
            raise OracleError(rc)

    def window(self):
        lo, hi = np.empty(3, np.int32), np.empty(3, np.int32)
        rc = lib().to_window(C.byref(self.P), self.n, _p(self.x), _p(lo, _ip), _p(hi, _ip))
        if rc:
            raise OracleError(rc)
        return lo, hi

    def p2g(self, lo, hi):
        shp = tuple(int(v) for v in np.asarray(hi) - np.asarray(lo))
        gm, gp = np.zeros(shp), np.zeros(shp + (3,))
        mdf = C.c_double()
        lo_ = np.ascontiguousarray(lo, np.int32)
        hi_ = np.ascontiguousarray(hi, np.int32)
        rc = lib().to_p2g(C.byref(self.P), self.n, _p(self.x), _p(self.v), _p(self.C), _p(self.F),
                          _p(self.mass), _p(self.vol0), _p(self.tag, _u8p), _p(lo_, _ip),
                          _p(hi_, _ip), _p(gm), _p(gp), C.byref(mdf))
        if rc:
            raise OracleError(rc)
        return gm, gp, mdf.value

    def grid_update(self, lo, hi, gm, gp):
        gv = np.zeros(gp.shape)
        lo_ = np.ascontiguousarray(lo, np.int32)
        hi_ = np.ascontiguousarray(hi, np.int32)
        lib().to_grid_update(C.byref(self.P), _p(lo_, _ip), _p(hi_, _ip), _p(_d(gm)), _p(_d(gp)),
                             _p(gv))
        return gv

    def g2p(self, lo, hi, gv):
        lo_ = np.ascontiguousarray(lo, np.int32)
        hi_ = np.ascontiguousarray(hi, np.int32)
        lib().to_g2p(C.byref(self.P), self.n, _p(self.x), _p(self.v), _p(self.C), _p(self.F),
                     _p(self.tag, _u8p), _p(lo_, _ip), _p(hi_, _ip), _p(_d(gv)))

    def apply_boundary(self, vind):
        lib().to_apply_boundary(self.n, _p(self.v), _p(self.tag, _u8p), _p(_d(vind)))

    def advect(self):
        ms = C.c_double()
        rc = lib().to_advect(C.byref(self.P), self.n, _p(self.x), _p(self.v), C.byref(ms))
        self.diag.max_speed = ms.value
        self.diag.step_count += 1
        if rc:
            raise OracleError(rc)


def polar_rotation(F):
    R = np.empty((3, 3))
    rc = lib().to_polar_rotation(_p(_d(F)), _p(R))
    if rc:
        raise OracleError(rc)
    return R


def corotated_stress(F, E=1.45e5, nu=0.45):
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    S = np.empty((3, 3))
    rc = lib().to_corotated_stress(_p(_d(F)), mu, lam, _p(S))
    if rc:
        raise OracleError(rc)
    return S


def stencil(x, origin, dx):
    base = np.empty(3, np.int32)
    w = np.empty((3, 3))
    fx = np.empty(3)
    lib().to_stencil(_p(_d(x)), _p(_d(origin)), 1.0 / dx, _p(base, _ip), _p(w), _p(fx))
    return base, w, fx


def full_depth_size(nx, ny, geom, r):
    w, h = C.c_int(), C.c_int()
    lib().to_full_depth_size(nx, ny, _p(_d(geom)), r, C.byref(w), C.byref(h))
    return w.value, h.value


def extract_depth(surface, x, r, w=0, h=0):
    geom = _d([surface["x0"], surface["y0"], surface["sx"], surface["sy"], surface["z0"]])
    if w <= 0 or h <= 0:
        w, h = full_depth_size(surface["nx"], surface["ny"], geom, r)
    out = np.empty((h, w))
    idx = np.ascontiguousarray(surface["particle"], np.uint32)
    rc = lib().to_extract_depth(surface["nx"], surface["ny"], _p(geom), _p(idx, _u32p),
                                _p(_d(x)), w, h, r, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def crop_align(src, offset=(0.0, 0.0), scale=1.0, out_w=640, out_h=480):
    src = _d(src)
    out = np.empty((out_h, out_w))
    rc = lib().to_crop_align(_p(src), src.shape[1], src.shape[0], offset[0], offset[1], scale,
                             out_w, out_h, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def surface_normals(depth, r):
    d = _d(depth)
    out = np.empty(d.shape + (3,))
    rc = lib().to_surface_normals(_p(d), d.shape[1], d.shape[0], r, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def phong(depth, r, lights, render, background=None):
    """render = [ka, kd, ks, shininess, ambient(3), view(3)]; lights n x 9."""
    d = _d(depth)
    L = _d(lights).reshape(-1, 9)
    out = np.empty(d.shape + (3,), np.uint8)
    bg = None if background is None else np.ascontiguousarray(background, np.uint8)
    rc = lib().to_phong(_p(d), d.shape[1], d.shape[0], r, _p(L), L.shape[0], _p(_d(render)),
                        _p(bg, _u8p), _p(out, _u8p))
    if rc:
        raise OracleError(rc)
    return out


def default_lights():
    """scene_config.cpp:42-57 (restated)."""
    e = np.sqrt(0.5)
    tints = [(0.80, 0.12, 0.10), (0.10, 0.80, 0.12), (0.12, 0.10, 0.80)]
    out = []
    for m in range(3):
        az = 2.0 * np.pi * m / 3.0
        out.append([e * np.cos(az), e * np.sin(az), -e, *tints[m], *(0.5 * np.array(tints[m]))])
    return np.array(out)


DEFAULT_RENDER = [1.0, 0.55, 0.25, 24.0, 0.34, 0.37, 0.44, 0.0, 0.0, -1.0]


def capture(surface, x, r=2.8125e-5, offset=(0.0, 0.0), scale=1.0, out_w=640, out_h=480,
            lights=None, render=None):
    """sim::capture restated: extract (full) -> crop -> Phong."""
    full = extract_depth(surface, x, r)
    crop = crop_align(full, offset, scale, out_w, out_h)
    img = phong(crop, r * scale, default_lights() if lights is None else lights,
                DEFAULT_RENDER if render is None else render)
    return crop, img
