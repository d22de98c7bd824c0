"""tacchi_b200 — B200-native (sm_100a) Tacchi hot path, Python mirror of the
reference C++ API over the C-ABI in include/tacchi_cuda.h.

Names follow the reference (/root/reference/proj): ``mpm.step``,
``mpm.particle_to_grid`` …, ``render.extract_surface_depth``,
``sim.build_sim`` / ``sim.capture``; errors are the reference's exception
classes (errors.hpp:9-39). Every compute call runs on the GPU through
``_lib/libtacchi_cuda.so``; there is no CPU fallback — importing on a machine
without the built library raises, and creating a simulation without an
sm_100 device raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TACCHI_LIB") or os.path.join(_HERE, "_lib", "libtacchi_cuda.so")

# ---------------------------------------------------------------------------
# Errors (errors.hpp:9-39)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """tacchi::Error"""


class GridTooSmall(Error): ...
class EmptyScene(Error): ...
class OutOfGrid(Error): ...
class DegenerateF(Error): ...
class ParseError(Error): ...
class EmptyCloud(Error): ...
class NoSurface(Error): ...
class CropOutOfBounds(Error): ...
class ShapeMismatch(Error): ...
class ConfigError(Error): ...
class IoError(Error): ...
class CudaError(Error): ...
class InvalidArgument(Error): ...
class SessionNotInitialized(Error): ...
class NonMonotonicTime(Error): ...
class ProtocolError(Error): ...
class ManifestMismatch(Error): ...


ERRORS = {1: GridTooSmall, 2: EmptyScene, 3: OutOfGrid, 4: DegenerateF, 5: ConfigError,
          6: NoSurface, 7: CropOutOfBounds, 8: ShapeMismatch, 9: EmptyCloud, 10: ParseError,
          11: IoError, 12: SessionNotInitialized, 13: NonMonotonicTime, 14: ProtocolError,
          15: ManifestMismatch, 20: CudaError, 21: InvalidArgument}

PHASES = dict(zero_grid=0, particle_to_grid=1, grid_update=2, grid_to_particle=3,
              apply_boundary=4, advect=5)

# ---------------------------------------------------------------------------
# ctypes plumbing
# ---------------------------------------------------------------------------

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)


class TgParams(C.Structure):
    _fields_ = [("res", C.c_int * 3), ("dx", C.c_double), ("origin", C.c_double * 3),
                ("youngs_modulus", C.c_double), ("poisson_ratio", C.c_double),
                ("density", C.c_double), ("dt", C.c_double), ("gravity", C.c_double * 3)]


class TgParticles(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_elastomer", C.c_int64), ("x", _dp), ("v", _dp),
                ("C", _dp), ("F", _dp), ("mass", _dp), ("volume0", _dp), ("tag", _u8p),
                ("indenter_velocity", C.c_double * 3)]


class TgSurface(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("x0", C.c_double), ("y0", C.c_double),
                ("sx", C.c_double), ("sy", C.c_double), ("z0", C.c_double),
                ("particle", C.POINTER(C.c_uint32))]


class TgSceneParams(C.Structure):
    """mpm::SceneParams (sim_state.hpp:81-98)."""
    _fields_ = [("grid_resolution", C.c_int * 3), ("grid_edge", C.c_double),
                ("grid_origin", C.c_double * 3), ("youngs_modulus", C.c_double),
                ("poisson_ratio", C.c_double), ("density", C.c_double), ("dt", C.c_double),
                ("fixed_bottom_layers", C.c_int), ("gravity", C.c_double * 3),
                ("indenter_mass_scale", C.c_double)]


class TgLattice(C.Structure):
    """An elastomer ParticleSet with its LatticeMeta (particle_set.hpp:18-30)."""
    _fields_ = [("counts", C.c_int * 3), ("dims", C.c_double * 3), ("origin", C.c_double * 3),
                ("positions", _dp)]


class TgRender(C.Structure):
    _fields_ = [("pixel_to_meter", C.c_double), ("crop_offset", C.c_double * 2),
                ("crop_scale", C.c_double), ("width", C.c_int), ("height", C.c_int),
                ("ambient_k", C.c_double), ("diffuse_k", C.c_double),
                ("specular_k", C.c_double), ("shininess", C.c_double),
                ("ambient_rgb", C.c_double * 3), ("view_dir", C.c_double * 3),
                ("n_lights", C.c_int), ("lights", (C.c_double * 9) * 8),
                ("background", _u8p)]


EXPORTED = [
    "tg_create", "tg_build_sim", "tg_destroy", "tg_step", "tg_phase", "tg_num_particles",
    "tg_num_elastomer", "tg_download", "tg_upload", "tg_diag", "tg_grid_window",
    "tg_download_grid", "tg_render_from_config", "tg_capture", "tg_extract_depth",
    "tg_crop_align", "tg_surface_normals", "tg_phong_render", "tg_step_many", "tg_step_capture_many", "tg_sync",
    "tg_stream", "tg_kernel_launches", "tg_set_graphs", "tg_last_error", "tg_version",
    "tg_generate_cloud", "tg_placed_indenter", "tg_time_phases", "tg_polar", "tg_init_scene",
    "tg_build_sim_points", "tg_download_constants", "tg_set_keep_grid", "tg_stats",
    "tg_build_episodes", "tg_set_deterministic", "tg_generate_cloud_device",
    "tg_step_capture_submit", "tg_step_capture_wait",
]

PHASE_TIMING_NAMES = ["p2g_elastomer_first", "p2g_indenter_first", "grid_update",
                      "g2p2g_elastomer", "indenter_move_p2g", "finalize"]

_lib = None


def lib():
    """Loads the sm_100a library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.tg_last_error.restype = C.c_char_p
        L.tg_version.restype = C.c_char_p
        L.tg_create.argtypes = [C.c_int, C.POINTER(TgParams), C.POINTER(TgParticles),
                                C.POINTER(TgSurface), C.POINTER(C.c_void_p)]
        L.tg_build_sim.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_double, C.c_double,
                                   C.POINTER(C.c_void_p)]
        L.tg_destroy.argtypes = [C.c_void_p]
        L.tg_step.argtypes = [C.c_void_p, _dp, C.c_int]
        L.tg_phase.argtypes = [C.c_void_p, C.c_int, _dp]
        L.tg_num_particles.argtypes = [C.c_void_p]
        L.tg_num_particles.restype = C.c_int64
        L.tg_num_elastomer.argtypes = [C.c_void_p]
        L.tg_num_elastomer.restype = C.c_int64
        L.tg_download.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.tg_upload.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.tg_diag.argtypes = [C.c_void_p, _dp, _dp, _i64p, _dp]
        L.tg_grid_window.argtypes = [C.c_void_p, _ip, _ip]
        L.tg_download_grid.argtypes = [C.c_void_p, _ip, _ip, _dp, _dp, _dp]
        L.tg_render_from_config.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(TgRender)]
        L.tg_capture.argtypes = [C.c_void_p, C.POINTER(TgRender), _dp, _u8p]
        L.tg_capture_buffers.argtypes = [C.c_void_p, C.POINTER(TgRender),
                                         C.POINTER(C.POINTER(C.c_double)),
                                         C.POINTER(C.POINTER(C.c_uint8))]
        L.tg_step_capture.argtypes = [C.c_void_p, _dp, C.c_int, C.POINTER(TgRender), _dp, _u8p]
        L.tg_extract_depth.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, _dp, _ip, _ip]
        L.tg_crop_align.argtypes = [C.c_int, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_int, C.c_int, _dp]
        L.tg_surface_normals.argtypes = [C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp]
        L.tg_phong_render.argtypes = [C.c_int, _dp, C.c_int, C.c_int, C.c_double,
                                      C.POINTER(TgRender), _u8p]
        L.tg_step_many.argtypes = [C.POINTER(C.c_void_p), C.c_int, _dp, C.c_int]
        L.tg_step_capture_many.argtypes = [C.POINTER(C.c_void_p), C.c_int, _dp, C.c_int,
                                           C.POINTER(TgRender), C.c_int,
                                           C.POINTER(_dp), C.POINTER(_u8p),
                                           C.POINTER(C.c_int)]
        L.tg_sync.argtypes = [C.c_void_p]
        L.tg_stream.argtypes = [C.c_void_p]
        L.tg_stream.restype = C.c_void_p
        L.tg_kernel_launches.argtypes = [C.c_void_p]
        L.tg_kernel_launches.restype = C.c_int64
        L.tg_set_graphs.argtypes = [C.c_void_p, C.c_int]
        L.tg_time_phases.argtypes = [C.c_void_p, _dp, C.c_int, _dp]
        L.tg_init_scene.argtypes = [C.c_int, C.POINTER(TgSceneParams), C.POINTER(TgLattice), _dp,
                                    C.c_int64, _dp, C.POINTER(C.c_void_p)]
        L.tg_build_sim_points.argtypes = [C.c_int, C.c_char_p, _dp, C.c_int64,
                                          C.POINTER(C.c_void_p)]
        L.tg_download_constants.argtypes = [C.c_void_p, _dp, _dp, _u8p]
        L.tg_set_keep_grid.argtypes = [C.c_void_p, C.c_int]
        L.tg_stats.argtypes = [C.c_void_p, _i64p]
        L.tg_set_deterministic.argtypes = [C.c_void_p, C.c_int]
        L.tg_generate_cloud_device.argtypes = [C.c_int, C.c_char_p, C.c_int64, C.c_uint64, _dp]
        L.tg_step_capture_submit.argtypes = [C.c_void_p, _dp, C.c_int, C.POINTER(TgRender),
                                             C.c_int, _i64p]
        L.tg_step_capture_wait.argtypes = [C.c_void_p, C.c_int64, C.POINTER(_dp),
                                           C.POINTER(_u8p)]
        L.tg_build_episodes.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_int, _dp,
                                        C.POINTER(C.c_void_p)]
        L.tg_polar.argtypes = [C.c_int, _dp, C.c_int64, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.tg_generate_cloud.argtypes = [C.c_char_p, C.c_int64, C.c_uint64, _dp]
        L.tg_placed_indenter.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.c_double, _dp,
                                         _i64p]
        L.tg_bridge_run.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p,
                                    C.POINTER(C.c_void_p)]
        L.tg_bridge_serve.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_int, C.c_int]
        L.tg_free.argtypes = [C.c_void_p]
        L.tg_run_press_dataset.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_int, _i64p,
                                           _i64p]
        L.tg_compare_datasets.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, _dp]
        L.tg_image_metrics.argtypes = [C.c_int, _u8p, _u8p, C.c_int, C.c_int, C.c_int, _dp]
        L.tg_load_png.argtypes = [C.c_char_p, _u8p, _ip, _ip]
        L.tg_save_png.argtypes = [C.c_char_p, _u8p, C.c_int, C.c_int]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().tg_last_error().decode(errors="replace")
        raise ERRORS.get(rc, Error)(msg)


def _d(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a if shape is None else a.reshape(shape)


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _cfg(cfg) -> bytes:
    if cfg is None:
        return b""
    return (cfg if isinstance(cfg, str) else json.dumps(cfg)).encode()


# ---------------------------------------------------------------------------
# mpm::SimState (sim_state.hpp:59-79), device resident
# ---------------------------------------------------------------------------


class SimState:
    """Device-resident simulation state. Host views are produced on demand
    (``state()``); they are snapshots, not live mirrors."""

    def __init__(self, handle: int, device: int = 0):
        self._h = C.c_void_p(handle)
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.tg_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return int(lib().tg_num_particles(self._h))

    @property
    def elastomer_count(self) -> int:
        return int(lib().tg_num_elastomer(self._h))

    def state(self) -> dict:
        n = self.n
        s = dict(x=np.empty((n, 3)), v=np.empty((n, 3)), C=np.empty((n, 3, 3)),
                 F=np.empty((n, 3, 3)))
        _check(lib().tg_download(self._h, _p(s["x"]), _p(s["v"]), _p(s["C"]), _p(s["F"])))
        return s

    def positions(self) -> np.ndarray:
        x = np.empty((self.n, 3))
        _check(lib().tg_download(self._h, _p(x), None, None, None))
        return x

    def set_state(self, x=None, v=None, Cm=None, F=None):
        n = self.n
        arrs = [None if a is None else _d(a, (n, k)) for a, k in ((x, 3), (v, 3), (Cm, 9), (F, 9))]
        _check(lib().tg_upload(self._h, *[_p(a) for a in arrs]))

    def constants(self) -> dict:
        """ParticleStore::mass / volume0 / tag (reference order)."""
        n = self.n
        out = dict(mass=np.empty(n), volume0=np.empty(n), tag=np.empty(n, np.uint8))
        _check(lib().tg_download_constants(self._h, _p(out["mass"]), _p(out["volume0"]),
                                           _p(out["tag"], _u8p)))
        return out

    def stats(self) -> dict:
        """Instrumentation counters (tg_stats)."""
        out = np.zeros(7, np.int64)
        _check(lib().tg_stats(self._h, _p(out, _i64p)))
        keys = ["kernel_launches", "regrows", "grid_bytes", "walk_fixups", "grid_nodes",
                "graphs", "indenter_walked"]
        return dict(zip(keys, (int(v) for v in out)))

    def set_deterministic(self, enabled: bool = True):
        """Fixed-point node accumulation, bit-identical reruns
        (tg_set_deterministic; build_sim follows SceneConfig.deterministic)."""
        _check(lib().tg_set_deterministic(self._h, int(bool(enabled))))

    def set_keep_grid(self, enabled: bool = True):
        """Keep the reference's post-step grid (tg_set_keep_grid): the last
        substep of each step runs the phase path."""
        _check(lib().tg_set_keep_grid(self._h, int(bool(enabled))))

    @property
    def diag(self) -> SimpleNamespace:
        a, b, c, v = C.c_double(), C.c_double(), C.c_int64(), np.empty(3)
        _check(lib().tg_diag(self._h, C.byref(a), C.byref(b), C.byref(c), _p(v)))
        return SimpleNamespace(min_det_f=a.value, max_speed=b.value, step_count=c.value,
                               indenter_velocity=v)

    @property
    def step_count(self) -> int:
        return self.diag.step_count

    def grid_window(self):
        lo, hi = np.empty(3, np.int32), np.empty(3, np.int32)
        _check(lib().tg_grid_window(self._h, _p(lo, _ip), _p(hi, _ip)))
        return lo, hi

    def grid(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.int32)
        hi = np.ascontiguousarray(hi, np.int32)
        shp = tuple(int(v) for v in hi - lo)
        m, mom, vel = np.empty(shp), np.empty(shp + (3,)), np.empty(shp + (3,))
        _check(lib().tg_download_grid(self._h, _p(lo, _ip), _p(hi, _ip), _p(m), _p(mom), _p(vel)))
        return m, mom, vel

    @property
    def stream(self) -> int:
        return int(lib().tg_stream(self._h) or 0)

    @property
    def kernel_launches(self) -> int:
        return int(lib().tg_kernel_launches(self._h))

    def set_graphs(self, enabled: bool):
        _check(lib().tg_set_graphs(self._h, int(bool(enabled))))

    def sync(self):
        _check(lib().tg_sync(self._h))

    def time_phases(self, indenter_velocity, reps: int = 10) -> dict:
        out = np.zeros(len(PHASE_TIMING_NAMES))
        _check(lib().tg_time_phases(self._h, _p(_vec(indenter_velocity)), int(reps), _p(out)))
        return dict(zip(PHASE_TIMING_NAMES, out.tolist()))


def init_scene(params: dict, particles: dict, surface: dict | None = None, device: int = 0):
    """mpm::init_scene from explicit arrays (row layout, reference order).

    params: res, dx, origin, E, nu, rho, dt, gravity.
    particles: x, v, (C, F), mass, volume0, tag, n_elastomer, indenter_velocity.
    surface: nx, ny, x0, y0, sx, sy, z0, particle.
    """
    P = TgParams()
    P.res[:] = [int(r) for r in params["res"]]
    P.dx = float(params["dx"])
    P.origin[:] = list(params.get("origin", (0, 0, 0)))
    P.youngs_modulus = float(params.get("E", 1.45e5))
    P.poisson_ratio = float(params.get("nu", 0.45))
    P.density = float(params.get("rho", 1000.0))
    P.dt = float(params["dt"])
    P.gravity[:] = list(params.get("gravity", (0, 0, 0)))
    n = len(particles["mass"])
    keep = dict(x=_d(particles["x"], (n, 3)), v=_d(particles.get("v", np.zeros((n, 3))), (n, 3)),
                mass=_d(particles["mass"]), vol=_d(particles["volume0"]),
                tag=np.ascontiguousarray(particles["tag"], np.uint8))
    keep["C"] = None if particles.get("C") is None else _d(particles["C"], (n, 9))
    keep["F"] = None if particles.get("F") is None else _d(particles["F"], (n, 9))
    T = TgParticles()
    T.n = n
    T.n_elastomer = int(particles["n_elastomer"])
    T.x, T.v = _p(keep["x"]), _p(keep["v"])
    T.C, T.F = _p(keep["C"]), _p(keep["F"])
    T.mass, T.volume0, T.tag = _p(keep["mass"]), _p(keep["vol"]), _p(keep["tag"], _u8p)
    T.indenter_velocity[:] = list(particles.get("indenter_velocity", (0, 0, 0)))
    S = None
    if surface is not None:
        idx = np.ascontiguousarray(surface["particle"], np.uint32)
        keep["surf"] = idx
        S = TgSurface(int(surface["nx"]), int(surface["ny"]), surface["x0"], surface["y0"],
                      surface["sx"], surface["sy"], surface["z0"],
                      idx.ctypes.data_as(C.POINTER(C.c_uint32)))
    h = C.c_void_p()
    _check(lib().tg_create(device, C.byref(P), C.byref(T), C.byref(S) if S else None,
                           C.byref(h)))
    return SimState(h.value, device)


# ---------------------------------------------------------------------------
# namespaces mirroring the reference
# ---------------------------------------------------------------------------


def _vec(v):
    return _d(v, (3,))


class mpm:  # noqa: N801 — mirrors tacchi::mpm
    """engine.hpp:10-35, sim_state.hpp:102-104"""

    @staticmethod
    def init_scene(params: dict, elastomer: dict, indenter, indenter_velocity=(0.0, 0.0, 0.0),
                   device: int = 0) -> SimState:
        """mpm::init_scene(SceneParams, elastomer lattice, indenter points, v0)
        (scene.cpp:28-87): masses, rest volumes, tags and the surface lattice
        are derived here as the reference does.

        params: grid_resolution, grid_edge, [grid_origin], [E, nu, rho], dt,
        [fixed_bottom_layers = 2], [gravity], [indenter_mass_scale = 80].
        elastomer: counts, dims, origin, [positions] (lattice order; default
        make_elastomer_lattice). indenter: n x 3 placed points (m)."""
        P = TgSceneParams()
        P.grid_resolution[:] = [int(r) for r in params["grid_resolution"]]
        P.grid_edge = float(params["grid_edge"])
        P.grid_origin[:] = list(params.get("grid_origin", (0.0, 0.0, 0.0)))
        P.youngs_modulus = float(params.get("E", 1.45e5))
        P.poisson_ratio = float(params.get("nu", 0.45))
        P.density = float(params.get("rho", 1000.0))
        P.dt = float(params["dt"])
        P.fixed_bottom_layers = int(params.get("fixed_bottom_layers", 2))
        P.gravity[:] = list(params.get("gravity", (0.0, 0.0, 0.0)))
        P.indenter_mass_scale = float(params.get("indenter_mass_scale", 80.0))
        L = TgLattice()
        L.counts[:] = [int(c) for c in elastomer["counts"]]
        L.dims[:] = list(elastomer["dims"])
        L.origin[:] = list(elastomer["origin"])
        pos = elastomer.get("positions")
        pos = None if pos is None else _d(pos, (-1, 3))
        L.positions = _p(pos)
        ind = _d(indenter, (-1, 3))
        h = C.c_void_p()
        _check(lib().tg_init_scene(device, C.byref(P), C.byref(L), _p(ind), len(ind),
                                   _p(_vec(indenter_velocity)), C.byref(h)))
        return SimState(h.value, device)

    @staticmethod
    def zero_grid(state: SimState):
        _check(lib().tg_phase(state.handle, 0, None))

    @staticmethod
    def particle_to_grid(state: SimState):
        _check(lib().tg_phase(state.handle, 1, None))

    @staticmethod
    def grid_update(state: SimState):
        _check(lib().tg_phase(state.handle, 2, None))

    @staticmethod
    def grid_to_particle(state: SimState):
        _check(lib().tg_phase(state.handle, 3, None))

    @staticmethod
    def apply_boundary(state: SimState, indenter_velocity):
        _check(lib().tg_phase(state.handle, 4, _p(_vec(indenter_velocity))))

    @staticmethod
    def advect(state: SimState):
        _check(lib().tg_phase(state.handle, 5, None))

    @staticmethod
    def step(state: SimState, indenter_velocity, n_substeps: int = 1):
        _check(lib().tg_step(state.handle, _p(_vec(indenter_velocity)), int(n_substeps)))

    @staticmethod
    def step_many(states, velocities, n_substeps: int = 1):
        hs = (C.c_void_p * len(states))(*[s.handle.value for s in states])
        v = _d(velocities, (len(states), 3))
        _check(lib().tg_step_many(hs, len(states), _p(v), int(n_substeps)))


def render_params(cfg=None, obj: str = "") -> TgRender:
    """Resolves capture's render inputs from a SceneConfig (scene_config.cpp:70-81)."""
    r = TgRender()
    _check(lib().tg_render_from_config(_cfg(cfg), obj.encode(), C.byref(r)))
    return r


class render:  # noqa: N801 — mirrors tacchi::render
    @staticmethod
    def extract_surface_depth(state: SimState, pixel_to_meter: float, width: int = 0,
                              height: int = 0) -> np.ndarray:
        w, h = C.c_int(), C.c_int()
        _check(lib().tg_extract_depth(state.handle, width, height, pixel_to_meter, None,
                                      C.byref(w), C.byref(h)))
        out = np.empty((h.value, w.value))
        _check(lib().tg_extract_depth(state.handle, w.value, h.value, pixel_to_meter, _p(out),
                                      None, None))
        return out

    @staticmethod
    def crop_align(src, alignment=(0.0, 0.0, 1.0), out_width=640, out_height=480, device=0):
        src = _d(src)
        out = np.empty((out_height, out_width))
        ox, oy, sc = alignment
        _check(lib().tg_crop_align(device, _p(src), src.shape[1], src.shape[0], ox, oy, sc,
                                   out_width, out_height, _p(out)))
        return out

    @staticmethod
    def surface_normals(depth, pixel_to_meter, device=0):
        d = _d(depth)
        out = np.empty(d.shape + (3,))
        _check(lib().tg_surface_normals(device, _p(d), d.shape[1], d.shape[0], pixel_to_meter,
                                        _p(out)))
        return out

    @staticmethod
    def phong_render(depth, pixel_to_meter, params: TgRender | None = None, background=None,
                     device=0):
        d = _d(depth)
        rp = params if params is not None else render_params()
        bg = None
        if background is not None:
            bg = np.ascontiguousarray(background, np.uint8)
            if bg.shape != d.shape + (3,):
                raise ShapeMismatch("phong_render: background image size differs from the depth map")
            rp.background = bg.ctypes.data_as(_u8p)
        out = np.empty(d.shape + (3,), np.uint8)
        _check(lib().tg_phong_render(device, _p(d), d.shape[1], d.shape[0], pixel_to_meter,
                                     C.byref(rp), _p(out, _u8p)))
        return out


_VIEWS: dict = {}


def _pinned_view(addr: int, shape, dtype) -> np.ndarray:
    """numpy view of a pinned host buffer owned by the library (cached per
    address: the slots are reused frame after frame)."""
    key = (addr, shape, np.dtype(dtype).str)
    v = _VIEWS.get(key)
    if v is None:
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        buf = (C.c_char * n).from_address(addr)
        v = np.frombuffer(buf, dtype=dtype).reshape(shape)
        if len(_VIEWS) > 4096:
            _VIEWS.clear()
        _VIEWS[key] = v
    return v


class sim:  # noqa: N801 — mirrors tacchi::sim
    @staticmethod
    def build_sim(cfg=None, obj: str = "", offset_x: float = 0.0, offset_y: float = 0.0,
                  device: int = 0) -> SimState:
        """build_sim(cfg, place_for_press(cfg, indenter_cloud_for(cfg, obj), ox, oy))."""
        h = C.c_void_p()
        _check(lib().tg_build_sim(device, _cfg(cfg), obj.encode(), offset_x, offset_y,
                                  C.byref(h)))
        return SimState(h.value, device)

    @staticmethod
    def build_episodes(cfg, obj: str, poses, device: int = 0) -> list:
        """Episodes of one object sharing one indenter cloud (tg_build_episodes):
        poses is n x 3 (offset_x, offset_y, z_rotation_rad)."""
        P = _d(poses, (-1, 3))
        hs = (C.c_void_p * len(P))()
        _check(lib().tg_build_episodes(device, _cfg(cfg), obj.encode(), len(P), _p(P), hs))
        return [SimState(h, device) for h in hs]

    @staticmethod
    def build_sim_points(cfg, indenter, device: int = 0) -> SimState:
        """sim::build_sim(cfg, indenter) with caller-placed indenter points
        (scene_builder.cpp:63-78)."""
        ind = _d(indenter, (-1, 3))
        h = C.c_void_p()
        _check(lib().tg_build_sim_points(device, _cfg(cfg), _p(ind), len(ind), C.byref(h)))
        return SimState(h.value, device)

    @staticmethod
    def capture(state: SimState, cfg=None, obj: str = "", params: TgRender | None = None,
                want_depth=True, want_image=True):
        """sim::capture -> (depth HxW fp64, image HxWx3 uint8)."""
        rp = params if params is not None else render_params(cfg, obj)
        depth = np.empty((rp.height, rp.width)) if want_depth else None
        img = np.empty((rp.height, rp.width, 3), np.uint8) if want_image else None
        _check(lib().tg_capture(state.handle, C.byref(rp), _p(depth), _p(img, _u8p)))
        return depth, img

    @staticmethod
    def _pinned_views(state: SimState, rp: TgRender):
        """numpy views of the handle's pinned capture buffers (tg_capture_buffers);
        valid until the next capture on this state."""
        dptr, rptr = C.c_void_p(), C.c_void_p()
        _check(lib().tg_capture_buffers(state.handle, C.byref(rp), C.cast(C.pointer(dptr), C.POINTER(_dp)),
                                        C.cast(C.pointer(rptr), C.POINTER(_u8p))))
        return (_pinned_view(dptr.value, (rp.height, rp.width), np.float64),
                _pinned_view(rptr.value, (rp.height, rp.width, 3), np.uint8))

    @staticmethod
    def step_capture(state: SimState, indenter_velocity, n_substeps: int, cfg=None, obj: str = "",
                     params: TgRender | None = None, zero_copy: bool = False,
                     want_depth: bool = True, want_image: bool = True):
        """One Session control step (session.cpp:86, 42): mpm::step then
        sim::capture with a single host sync -> (depth, image). zero_copy
        returns views of pinned buffers that the next capture overwrites;
        want_* False keeps that output on the device."""
        rp = params if params is not None else render_params(cfg, obj)
        if zero_copy:
            depth, img = sim._pinned_views(state, rp)
        else:
            depth = np.empty((rp.height, rp.width))
            img = np.empty((rp.height, rp.width, 3), np.uint8)
        depth = depth if want_depth else None
        img = img if want_image else None
        _check(lib().tg_step_capture(state.handle, _p(_vec(indenter_velocity)), int(n_substeps),
                                     C.byref(rp), _p(depth), _p(img, _u8p)))
        return depth, img


    @staticmethod
    def step_capture_submit(state: SimState, indenter_velocity, n_substeps: int,
                            params: TgRender, read_back: bool = True) -> int:
        """Pipelined control step (tg_step_capture_submit): enqueue step +
        capture (+ read-back), return the frame's ticket at once."""
        t = C.c_int64()
        _check(lib().tg_step_capture_submit(state.handle, _p(_vec(indenter_velocity)),
                                            int(n_substeps), C.byref(params), int(bool(read_back)),
                                            C.byref(t)))
        return t.value

    @staticmethod
    def step_capture_wait(state: SimState, ticket: int, params: TgRender):
        """Outputs of a submitted frame (tickets in order): (depth, image) views
        of its pinned slot, valid until the submit after next."""
        dptr, rptr = C.c_void_p(), C.c_void_p()
        _check(lib().tg_step_capture_wait(state.handle, int(ticket), C.cast(C.pointer(dptr), C.POINTER(_dp)),
                                          C.cast(C.pointer(rptr), C.POINTER(_u8p))))
        if not dptr.value:  # submitted with read_back=False
            return None, None
        return (_pinned_view(dptr.value, (params.height, params.width), np.float64),
                _pinned_view(rptr.value, (params.height, params.width, 3), np.uint8))

    @staticmethod
    def step_capture_many(states, velocities, n_substeps: int, params, want_depth: bool = True,
                          want_image: bool = True, zero_copy: bool = False):
        """Batched control step (tg_step_capture_many): every state steps with
        its velocity row and is captured with `params` (one TgRender for all,
        or one per state); all submitted before any wait; zero_copy returns
        views of each handle's pinned buffers (overwritten by its next capture). Returns
        (outputs, status): outputs[i] = (depth, image) (None where not
        wanted), status[i] = the handle's error code (0 = OK). Raises the
        first failing handle's error after every handle was processed."""
        n = len(states)
        ps = list(params) if isinstance(params, (list, tuple)) else [params]
        if len(ps) not in (1, n):
            raise ValueError("params: one TgRender or one per state")
        renders = (TgRender * len(ps))(*ps)
        v = _d(velocities, (n, 3))
        outs, dptr, iptr = [], (_dp * n)(), (_u8p * n)()
        for i in range(n):
            rp = ps[0] if len(ps) == 1 else ps[i]
            if zero_copy:  # views of the handle's pinned buffers (next capture overwrites)
                d, im = sim._pinned_views(states[i], rp)
                d = d if want_depth else None
                im = im if want_image else None
            else:
                d = np.empty((rp.height, rp.width)) if want_depth else None
                im = np.empty((rp.height, rp.width, 3), np.uint8) if want_image else None
            dptr[i] = _p(d)
            iptr[i] = _p(im, _u8p)
            outs.append((d, im))
        hs = (C.c_void_p * n)(*[s.handle.value for s in states])
        status = (C.c_int * n)()
        rc = lib().tg_step_capture_many(hs, n, _p(v), int(n_substeps), renders, len(ps), dptr,
                                        iptr, status)
        st = list(status)
        if rc:
            _check(rc)
        return outs, st


class material:  # noqa: N801 — mirrors tacchi::mpm material functions (material.hpp)
    @staticmethod
    def polar_rotation(F, svd: bool = False, E: float = 1.45e5, nu: float = 0.45,
                       device: int = 0):
        """polar_rotation (or polar_rotation_svd when svd) and corotated_stress
        of a batch of 3x3 F on the device -> (R, S), each n x 3 x 3."""
        F = _d(F).reshape(-1, 9)
        R = np.empty_like(F)
        S = np.empty_like(F)
        _check(lib().tg_polar(device, _p(F), len(F), 1 if svd else 0, E, nu, _p(R), _p(S)))
        return R.reshape(-1, 3, 3), S.reshape(-1, 3, 3)


class geo:  # noqa: N801 — mirrors tacchi::geo (host setup)
    @staticmethod
    def generate_shape_cloud(name: str, n: int, seed: int) -> np.ndarray:
        out = np.empty((n, 3))
        _check(lib().tg_generate_cloud(name.encode(), n, seed, _p(out)))
        return out

    @staticmethod
    def generate_shape_cloud_device(name: str, n: int, seed: int, device: int = 0) -> np.ndarray:
        """generate_shape_cloud on the GPU (bit-identical to the host's)."""
        out = np.empty((n, 3))
        _check(lib().tg_generate_cloud_device(device, name.encode(), n, seed, _p(out)))
        return out

    @staticmethod
    def placed_indenter(cfg=None, obj: str = "", offset_x=0.0, offset_y=0.0) -> np.ndarray:
        n = C.c_int64()
        _check(lib().tg_placed_indenter(_cfg(cfg), obj.encode(), offset_x, offset_y, None,
                                        C.byref(n)))
        out = np.empty((n.value, 3))
        _check(lib().tg_placed_indenter(_cfg(cfg), obj.encode(), offset_x, offset_y, _p(out),
                                        C.byref(n)))
        return out


class bridge:  # noqa: N801 — mirrors tacchi::bridge (server.hpp, session.hpp)
    """Co-simulation protocol "tacchi/1" over the B200 path (§8 row f1)."""

    @staticmethod
    def run_protocol(messages, base_cfg=None, session_root: str = ".", device: int = 0) -> list:
        """bridge::run_protocol (server.cpp:49-113) over in-memory lines.

        `messages` are dicts (serialised with json.dumps) or raw strings; the
        reply lines come back parsed."""
        lines = [m if isinstance(m, str) else json.dumps(m) for m in messages]
        out = C.c_void_p()
        _check(lib().tg_bridge_run(device, _cfg(base_cfg), session_root.encode(),
                                   ("\n".join(lines) + "\n").encode(), C.byref(out)))
        try:
            text = C.string_at(out.value).decode()
        finally:
            lib().tg_free(out)
        return [json.loads(l) for l in text.splitlines() if l]

    @staticmethod
    def serve(base_cfg=None, session_root: str = ".", port: int = -1, max_connections: int = 0,
              device: int = 0):
        """serve_stdio (port < 0) or serve_tcp on 127.0.0.1:port (server.cpp:115-182)."""
        _check(lib().tg_bridge_serve(device, _cfg(base_cfg), session_root.encode(), port,
                                     max_connections))


def load_depth_map(path: str):
    """render::load_depth_map (depth_map.cpp:40-60): (values HxW float64, pixel_to_meter)."""
    with open(path, "rb") as f:
        header = json.loads(f.readline())
        w, h = header["width"], header["height"]
        buf = np.frombuffer(f.read(), dtype=np.float32)
    if w <= 0 or h <= 0 or buf.size < w * h:
        raise ParseError(f"{path}: bad depth map")
    return buf[: w * h].astype(np.float64).reshape(h, w), header["pixel_to_meter"]


def load_png(path: str) -> np.ndarray:
    """render::load_png (image.cpp:51-90) -> H x W x 3 uint8."""
    w, h = C.c_int(), C.c_int()
    _check(lib().tg_load_png(path.encode(), None, C.byref(w), C.byref(h)))
    out = np.empty((h.value, w.value, 3), dtype=np.uint8)
    _check(lib().tg_load_png(path.encode(), _p(out, _u8p), C.byref(w), C.byref(h)))
    return out


def save_png(image: np.ndarray, path: str):
    """render::save_png (image.cpp:23-49) of an H x W x 3 uint8 image."""
    img = np.ascontiguousarray(image, dtype=np.uint8)
    _check(lib().tg_save_png(path.encode(), _p(img, _u8p), img.shape[1], img.shape[0]))


class metrics:  # noqa: N801 — mirrors tacchi::metrics (image_metrics.hpp)
    @staticmethod
    def compare_batch(a, b, device: int = 0) -> np.ndarray:
        """ssim, psnr_db, mae_pct for each of a batch of image pairs (B x H x W x 3
        uint8 each), one device launch (image_metrics.cpp:57-112)."""
        a = np.ascontiguousarray(a, dtype=np.uint8)
        b = np.ascontiguousarray(b, dtype=np.uint8)
        if a.ndim == 3:
            a, b = a[None], b[None]
        if a.shape != b.shape:
            raise ShapeMismatch(f"image shapes differ: {a.shape[1:]} vs {b.shape[1:]}")
        out = np.zeros((a.shape[0], 3))
        _check(lib().tg_image_metrics(device, _p(a, _u8p), _p(b, _u8p), a.shape[2], a.shape[1],
                                      a.shape[0], _p(out)))
        return out

    @staticmethod
    def compare(a, b, device: int = 0):
        """metrics::compare -> (ssim, psnr_db, mae_pct)."""
        return tuple(metrics.compare_batch(a, b, device)[0])


class dataset:  # noqa: N801 — mirrors tacchi::dataset (harness.hpp)
    @staticmethod
    def run_press_dataset(cfg, out_dir: str, batch: int = 0, device: int = 0):
        """dataset::run_press_dataset (harness.cpp:159-245) on the device;
        returns (rows, skipped_positions)."""
        rows, skipped = C.c_int64(), C.c_int64()
        _check(lib().tg_run_press_dataset(device, _cfg(cfg), str(out_dir).encode(), batch,
                                          C.byref(rows), C.byref(skipped)))
        return rows.value, skipped.value

    @staticmethod
    def compare_datasets(dir_a: str, dir_b: str, csv_out: str = "", device: int = 0) -> dict:
        """dataset::compare_datasets (harness.cpp:247-321)."""
        out = np.zeros(7)
        _check(lib().tg_compare_datasets(device, str(dir_a).encode(), str(dir_b).encode(),
                                         str(csv_out).encode(), _p(out)))
        keys = ["pairs", "ssim_mean", "ssim_std", "psnr_mean", "psnr_std", "mae_mean", "mae_std"]
        d = dict(zip(keys, out.tolist()))
        d["pairs"] = int(d["pairs"])
        return d


def version() -> str:
    return lib().tg_version().decode()
