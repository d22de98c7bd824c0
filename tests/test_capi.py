"""The C-ABI library (libtacchi_cuda.so): loads, exports every symbol
include/tacchi_cuda.h declares, and its host-side setup reproduces the
reference's inputs bit for bit. CPU only (no kernel launches)."""
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT, has_gpu
from tests.scenes import PLACED_ROT, SHAPES, sha


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "tacchi_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2301_08343_b200 as tb

    L = tb.lib()
    names = _declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(tb.EXPORTED) <= set(names) | {"tg_generate_cloud", "tg_placed_indenter"}
    assert "sm_100a" in tb.version()


def test_library_is_built_for_sm100a():
    import subprocess

    import paper_2301_08343_b200 as tb

    out = subprocess.run(["cuobjdump", "--list-elf", tb.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_generated_clouds_match_reference_bit_exact(golden):
    import paper_2301_08343_b200 as tb

    k = golden("kat.npz")
    for i, s in enumerate(SHAPES):
        pts = tb.geo.generate_shape_cloud(s, 2000, 7)
        np.testing.assert_array_equal(pts[:4], k["cloud_head"][i])
        assert sha(pts) == str(k["cloud_hash"][i]), s


def test_placed_indenter_matches_reference_bit_exact(golden):
    import paper_2301_08343_b200 as tb

    k = golden("kat.npz")
    pts = tb.geo.placed_indenter({}, "")
    assert len(pts) == int(k["placed_n"]) and sha(pts) == str(k["placed_hash"])
    pts = tb.geo.placed_indenter(*PLACED_ROT)
    assert len(pts) == int(k["placed_rot_n"]) and sha(pts) == str(k["placed_rot_hash"])


def test_unknown_shape_is_an_error():
    import paper_2301_08343_b200 as tb

    with pytest.raises(tb.ConfigError):
        tb.geo.generate_shape_cloud("dodecahedron", 10, 1)


def test_render_params_from_config_defaults():
    import paper_2301_08343_b200 as tb

    r = tb.render_params({}, "")
    assert (r.width, r.height, r.n_lights) == (640, 480, 3)
    assert (r.ambient_k, r.diffuse_k, r.specular_k, r.shininess) == (1.0, 0.55, 0.25, 24.0)
    assert list(r.ambient_rgb) == [0.34, 0.37, 0.44]
    assert r.pixel_to_meter == 2.8125e-5 and r.crop_scale == 1.0
    e = np.sqrt(0.5)
    np.testing.assert_allclose(list(r.lights[0])[:3], [e, 0, -e], atol=1e-15)
    r2 = tb.render_params({"alignment": {"dots": {"offset_px": [3, -2], "scale": 1.1}}}, "dots")
    assert (r2.crop_offset[0], r2.crop_offset[1], r2.crop_scale) == (3.0, -2.0, 1.1)
    with pytest.raises(tb.ConfigError):
        tb.render_params("{not json", "")


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    import paper_2301_08343_b200 as tb

    with pytest.raises(tb.CudaError):
        tb.sim.build_sim({"time": {"dt_s": 2e-6}, "indenter": {"source_points": 2000,
                                                                 "target_points": 1000}})


def test_render_background_image_from_config(tmp_path):
    """render_params_struct's background_image (scene_config.cpp:77-78): loaded
    once, passed to the capture; a size other than the image's is the
    reference's ShapeMismatch (phong.cpp:46-48)."""
    import ctypes

    import numpy as np

    import paper_2301_08343_b200 as tb
    from tests.scenes import SMALL

    bg = np.random.default_rng(4).integers(0, 256, (120, 160, 3), dtype=np.uint8)
    path = str(tmp_path / "bg.png")
    tb.save_png(bg, path)
    cfg = {**SMALL, "render": {**SMALL["render"], "background_image": path}}
    rp = tb.render_params(cfg, "")
    assert rp.background
    got = np.ctypeslib.as_array(ctypes.cast(rp.background, ctypes.POINTER(ctypes.c_uint8)),
                                shape=(120, 160, 3))
    np.testing.assert_array_equal(got, bg)
    tb.save_png(bg[:60], path)  # rewritten with another size: reloaded, rejected
    with pytest.raises(tb.ShapeMismatch):
        tb.render_params(cfg, "")
    with pytest.raises(tb.IoError):
        tb.render_params({**cfg, "render": {"background_image": str(tmp_path / "none.png")}}, "")


def test_point_cloud_files_match_reference(golden, tmp_path):
    """Indenters from point-cloud files (geo::load_point_cloud, ASCII PLY and
    plain XYZ in millimetres; scene_builder.cpp:33-50: cloud_path, or the
    object name as a path), placed bit-identically to the reference; its
    errors for malformed files."""
    import paper_2301_08343_b200 as tb

    g = golden("clouds.npz")
    paths = {}
    for k in ("ply", "xyz", "binary", "empty", "short"):
        paths[k] = str(tmp_path / f"cloud_{k}.{'ply' if k in ('ply', 'binary') else 'xyz'}")
        with open(paths[k], "w") as f:
            f.write(str(g[f"text_{k}"]))
    for k in ("ply", "xyz"):
        placed = tb.geo.placed_indenter({"indenter": {"cloud_path": paths[k],
                                                      "target_points": 2000}})
        assert len(placed) == int(g[f"{k}_n"]) and sha(placed) == str(g[f"{k}_hash"])
        obj = tb.geo.placed_indenter({"indenter": {"target_points": 2000}}, paths[k])
        assert sha(obj) == str(g[f"{k}_obj_hash"])
        sub = tb.geo.placed_indenter({"indenter": {"cloud_path": paths[k], "target_points": 1000,
                                                   "z_rotation_rad": 0.3}})
        assert sha(sub) == str(g[f"{k}_sub_hash"])
    errors = {10: tb.ParseError, 9: tb.EmptyCloud}
    for k in ("binary", "empty", "short"):
        code, msg = str(g[f"{k}_err"]).split(":", 1)
        with pytest.raises(errors[int(code)]) as e:
            tb.geo.placed_indenter({"indenter": {"cloud_path": paths[k]}})
        assert str(e.value).replace(paths[k], "<path>") == msg
