"""The header-only C++ mirror (include/tacchi_b200.hpp) driven by real C++
callers: tools/mirror_demo.cpp (init_scene from the reference's inputs,
build_sim with caller points, keep_grid + grid, RenderSetup capture) and
tools/press_demo.cpp (the Session-shaped step + capture loop)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2301_08343_b200", "_lib")


def _run(exe, *args):
    out = subprocess.run([os.path.join(LIB, exe), *args], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_mirror_demo_setup_grid_and_capture():
    r = _run("mirror_demo")
    assert r["same_setup"] and r["same_init"]  # caller points / own inputs == config path
    assert r["particles"] == 31 * 31 * 7 + 3000 and r["step_count"] == 20
    # the kept post-step grid carries every particle's mass (P2G conserves it)
    assert abs(r["grid_mass"] - r["total_mass"]) <= 1e-10 * r["total_mass"]
    lo, hi = r["window"][:3], r["window"][3:]
    assert all(h > l for l, h in zip(lo, hi))
    assert r["image"] == [160, 120] and r["max_depth_m"] > 0.0


def test_press_demo_session_loop():
    r = _run("press_demo", json.dumps({"time": {"dt_s": 2e-6}}), "5")
    assert r["particles"] == 314221 and r["control_steps"] == 5 and r["step_count"] == 50
    assert 0.0 < r["min_det_f"] <= 1.0
