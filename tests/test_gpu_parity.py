"""Parity of the CUDA path (through the C-ABI) against the oracle and the
reference's golden fixtures. Needs a B200: run with `pytest -m gpu`.

Tolerances (BASELINE.json north_star): particle positions relative <= 1e-4
(we hold a far tighter displacement-relative bound, stated per test), height
map <= 1e-7 m, tactile image max abs diff <= 2/255. The capture path itself is
bit-exact for identical particle positions.
"""
import numpy as np
import pytest

from tests.scenes import (CONFIG1, CONFIG1_STEPS, CONFIG1_V, LIGHT_CFG, SMALL, SMALL_STEPS,
                          SMALL_V, render_inputs, sha)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tb():
    import paper_2301_08343_b200 as tb

    return tb


def _small_oracle(oracle, g):
    P = oracle.params((64, 64, 64), 12e-3 / 64, dt=2e-6)
    n = len(g["mass"])
    return oracle.OracleSim(P, g["x0"], np.zeros((n, 3)), g["mass"], g["vol0"], g["tag"])


def _surface_of(g, nx=31, ny=31):
    geom = g["surf_geom"]
    return dict(nx=nx, ny=ny, x0=geom[0], y0=geom[1], sx=geom[2], sy=geom[3], z0=geom[4],
                particle=g["surf_particle"])


def test_build_sim_reproduces_reference_setup(tb, golden):
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    st = s.state()
    np.testing.assert_array_equal(st["x"], g["x0"])
    assert s.elastomer_count == 31 * 31 * 7
    np.testing.assert_array_equal(st["F"], np.tile(np.eye(3), (s.n, 1, 1)))
    assert not st["v"].any() and not st["C"].any()


def test_small_scene_matches_reference(tb, golden):
    """200 substeps of the SMALL press vs the reference (golden)."""
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, SMALL_STEPS)
    st = s.state()
    disp = np.abs(g["x"] - g["x0"]).max()
    err = np.abs(st["x"] - g["x"]).max()
    assert err <= 1e-9 * disp, (err, disp)  # displacement-relative 1e-9
    assert np.abs(st["x"] - g["x"]).max() / np.abs(g["x"]).max() <= 1e-4  # north_star bar
    np.testing.assert_allclose(st["v"], g["v"], rtol=0, atol=1e-8 * np.abs(g["v"]).max())
    np.testing.assert_allclose(st["C"], g["C"], rtol=0, atol=1e-8 * np.abs(g["C"]).max())
    np.testing.assert_allclose(st["F"], g["F"], rtol=0, atol=1e-11)
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-12)
    assert d.max_speed == pytest.approx(float(g["max_speed"]), rel=1e-12)
    lo, hi = s.grid_window()
    np.testing.assert_array_equal(lo, g["win_lo"])
    np.testing.assert_array_equal(hi, g["win_hi"])
    depth, img = tb.sim.capture(s, SMALL)
    assert np.abs(depth - g["depth"]).max() <= 1e-7
    assert np.abs(depth - g["depth"]).max() <= 1e-9 * np.abs(g["depth"]).max()
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


@pytest.mark.parametrize("env", [{"TACCHI_FULL_INDENTER": "1"}, {"TACCHI_SCATTER": "1"},
                                 {"TACCHI_FULL_INDENTER": "1", "TACCHI_SCATTER": "1"}])
def test_alternative_scatter_paths_match_reference(tb, golden, monkeypatch, env):
    """The alternative device paths (read at tg_create): every indenter
    particle scattered by k_ind_move_p2g instead of the column walks, and the
    per-particle RED.F64 elastomer scatter instead of the shared tile."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, SMALL_STEPS // 2)
    tb.mpm.step(s, SMALL_V, SMALL_STEPS // 2)
    st = s.state()
    disp = np.abs(g["x"] - g["x0"]).max()
    assert np.abs(st["x"] - g["x"]).max() <= 1e-9 * disp
    np.testing.assert_allclose(st["F"], g["F"], rtol=0, atol=1e-11)
    assert s.diag.step_count == int(g["step_count"])
    depth, img = tb.sim.capture(s, SMALL)
    assert np.abs(depth - g["depth"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


def test_capture_bit_exact_for_identical_positions(tb, golden, oracle):
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, 60)
    x = s.positions()
    depth, img = tb.sim.capture(s, SMALL)
    od, oi = oracle.capture(_surface_of(g), x, out_w=160, out_h=120)
    np.testing.assert_array_equal(depth, od)
    np.testing.assert_array_equal(img, oi)
    full = tb.render.extract_surface_depth(s, 2.8125e-5)
    np.testing.assert_array_equal(full, oracle.extract_depth(_surface_of(g), x, 2.8125e-5))
    part = tb.render.extract_surface_depth(s, 3e-5, 50, 40)
    np.testing.assert_array_equal(part, oracle.extract_depth(_surface_of(g), x, 3e-5, 50, 40))


def test_phases_match_oracle(tb, golden, oracle):
    """Each engine.hpp phase through tg_phase vs the restated phase."""
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, 30)
    st = s.state()
    o = _small_oracle(oracle, g)
    o.x, o.v, o.C, o.F = st["x"].copy(), st["v"].copy(), st["C"].copy(), st["F"].copy()
    tb.mpm.zero_grid(s)
    lo, hi = o.window()
    glo, ghi = s.grid_window()
    np.testing.assert_array_equal(glo, lo)
    np.testing.assert_array_equal(ghi, hi)
    tb.mpm.particle_to_grid(s)
    om, op, mdf = o.p2g(lo, hi)
    m, mom, _ = s.grid(lo, hi)
    np.testing.assert_allclose(m, om, rtol=1e-12, atol=1e-14 * om.max())
    np.testing.assert_allclose(mom, op, rtol=0, atol=1e-10 * np.abs(op).max())
    assert s.diag.min_det_f == pytest.approx(mdf, abs=1e-14)
    tb.mpm.grid_update(s)
    _, _, vel = s.grid(lo, hi)
    ov = o.grid_update(lo, hi, m, mom)
    np.testing.assert_array_equal(vel, ov)  # same inputs -> IEEE division, bit-exact
    tb.mpm.grid_to_particle(s)
    o.g2p(lo, hi, vel)
    st = s.state()
    np.testing.assert_allclose(st["v"], o.v, rtol=0, atol=1e-12 * np.abs(o.v).max())
    np.testing.assert_allclose(st["C"], o.C, rtol=0, atol=1e-11 * np.abs(o.C).max())
    np.testing.assert_allclose(st["F"], o.F, rtol=0, atol=1e-14)
    tb.mpm.apply_boundary(s, SMALL_V)
    o.apply_boundary(SMALL_V)
    tb.mpm.advect(s)
    o.v = s.state()["v"]  # advect from identical velocities
    x_before = st["x"].copy()
    o.x = x_before.copy()
    o.advect()
    np.testing.assert_array_equal(s.positions(), o.x)
    assert s.diag.max_speed == pytest.approx(o.diag.max_speed, rel=1e-15)


def test_step_chains_with_uploads_match_oracle(tb, golden, oracle):
    """Step calls interleaved with state uploads, velocity changes and odd
    substep counts vs the serial oracle on the same inputs. The step path
    carries the next substep's scatter, each tile's staging box and (before
    each elastomer kernel's grid-dependency wait) the particle state from one
    launch to the next; an upload must discard all of it."""
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    o = _small_oracle(oracle, g)
    rng = np.random.default_rng(7)
    plan = [(SMALL_V, 10, None), (SMALL_V, 7, "x"), ((0.0, 0.0, -0.02), 13, None),
            ((0.001, 0.0, -0.01), 1, "F"), (SMALL_V, 20, "v"), (SMALL_V, 9, None)]
    for vind, n, upload in plan:
        el = o.tag != 2  # elastomer (the indenter stays rigid)
        if upload == "x":
            x = s.state()["x"].copy()
            x[el] += rng.uniform(-2e-7, 2e-7, (int(el.sum()), 3))
            s.set_state(x=x)
            o.x = x.copy()
        elif upload == "F":
            st = s.state()
            F = st["F"].reshape(-1, 3, 3).copy()
            F[el] += rng.uniform(-1e-6, 1e-6, (int(el.sum()), 3, 3))
            s.set_state(F=F.reshape(-1, 9))
            o.F = F.copy()
        elif upload == "v":
            st = s.state()
            v = st["v"].copy()
            v[el] += rng.uniform(-1e-4, 1e-4, (int(el.sum()), 3))
            s.set_state(v=v)
            o.v = v.copy()
        tb.mpm.step(s, vind, n)
        o.step(vind, n)
        x = s.positions()
        disp = np.abs(o.x - g["x0"]).max()
        err = np.abs(x - o.x).max()
        assert err <= 1e-8 * disp, (upload, n, err, disp)
        st = s.state()
        np.testing.assert_allclose(st["F"].reshape(-1, 3, 3), o.F, rtol=0, atol=1e-11)
        assert s.step_count == o.diag.step_count


def test_step_graph_and_plain_launches_agree(tb):
    a = tb.sim.build_sim(SMALL)
    b = tb.sim.build_sim(SMALL)
    b.set_graphs(False)
    for _ in range(3):
        tb.mpm.step(a, SMALL_V, 10)
        tb.mpm.step(b, SMALL_V, 10)
    xa, xb = a.positions(), b.positions()
    assert np.abs(xa - xb).max() <= 1e-15
    assert a.step_count == b.step_count == 30
    assert a.kernel_launches > 0


def test_step_capture_matches_step_then_capture(tb):
    """tg_step_capture (one sync per control step) == mpm::step + sim::capture
    (to the atomic-order rounding of two independent runs); zero-copy outputs
    are views of the handle's pinned buffers."""
    a, b = tb.sim.build_sim(SMALL), tb.sim.build_sim(SMALL)
    rp = tb.render_params(SMALL, "")

    def same(da, ia, db, ib):
        np.testing.assert_allclose(da, db, rtol=0, atol=1e-12)
        assert np.abs(ia.astype(int) - ib).max() <= 1

    for _ in range(3):
        tb.mpm.step(a, SMALL_V, 10)
        da, ia = tb.sim.capture(a, params=rp)
        db, ib = tb.sim.step_capture(b, SMALL_V, 10, params=rp)
        same(da, ia, db, ib)
    dz, iz = tb.sim.step_capture(b, SMALL_V, 10, params=rp, zero_copy=True)
    tb.mpm.step(a, SMALL_V, 10)
    da, ia = tb.sim.capture(a, params=rp)
    same(da, ia, dz, iz)
    np.testing.assert_allclose(a.state()["x"], b.state()["x"], rtol=0, atol=1e-15)
    _, none = tb.sim.step_capture(b, SMALL_V, 250, params=rp, want_image=False)  # > 200: chunked
    assert none is None and b.step_count == a.step_count + 250


def test_handles_stepped_from_concurrent_threads(tb, golden):
    """One control thread per handle: four host threads each
    drive their own simulation at the same time; each matches the reference."""
    import threading

    g = golden("small_scene.npz")
    results, errors = {}, []

    def run(i):
        try:
            s = tb.sim.build_sim(SMALL)
            for _ in range(SMALL_STEPS // 10):
                tb.mpm.step(s, SMALL_V, 10)
            results[i] = s.state()["x"]
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    disp = np.abs(g["x"] - g["x0"]).max()
    for x in results.values():
        assert np.abs(x - g["x"]).max() <= 1e-9 * disp


def test_step_many_matches_individual_steps(tb):
    sims = [tb.sim.build_sim(SMALL, "", 1e-4 * i, 0.0) for i in range(3)]
    ref = [tb.sim.build_sim(SMALL, "", 1e-4 * i, 0.0) for i in range(3)]
    vel = np.array([[0, 0, -0.05], [0, 0, -0.03], [0.01, 0, -0.05]])
    tb.mpm.step_many(sims, vel, 20)
    for r, v in zip(ref, vel):
        tb.mpm.step(r, v, 20)
    for s, r in zip(sims, ref):
        assert np.abs(s.positions() - r.positions()).max() <= 1e-15


def test_degenerate_f_leaves_state_at_failing_substep(tb):
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, 5)
    st = s.state()
    F = st["F"].copy()
    F[7] = np.diag([1.0, 1.0, -1.0])  # det < 0
    s.set_state(F=F.reshape(-1, 9))
    x_before = s.positions()
    with pytest.raises(tb.DegenerateF):
        tb.mpm.step(s, SMALL_V, 3)
    np.testing.assert_array_equal(s.positions(), x_before)
    assert s.step_count == 5
    with pytest.raises(tb.DegenerateF):  # still degenerate on retry
        tb.mpm.step(s, SMALL_V, 1)


def test_step_capture_many_matches_single_handles(tb):
    """tg_step_capture_many (every handle submitted before any wait) == one
    tg_step_capture per handle; per-handle status, and a failing handle
    (OutOfGrid, the out-of-grid setup below) does not stop the others."""
    rp = tb.render_params(SMALL, "")
    vs = np.array([SMALL_V, (0.002, 0.0, -0.04), (0.0, -0.003, -0.02)])
    batch = [tb.sim.build_sim(SMALL) for _ in vs]
    single = [tb.sim.build_sim(SMALL) for _ in vs]
    for _ in range(3):
        outs, status = tb.sim.step_capture_many(batch, vs, 10, rp)
        assert status == [0, 0, 0]
        for s, v, (d, im) in zip(single, vs, outs):
            ds, ims = tb.sim.step_capture(s, v, 10, params=rp)
            np.testing.assert_allclose(d, ds, rtol=0, atol=1e-12)
            assert np.abs(im.astype(int) - ims).max() <= 1
    outs, status = tb.sim.step_capture_many(batch, vs, 5, [rp] * 3, want_depth=False)
    assert all(d is None and im is not None for d, im in outs)
    # handle 1 runs out of the grid; 0 and 2 still step and capture
    x = batch[1].positions()
    x[-1, 2] = (64 - 3) * (12e-3 / 64) + 0.49 * (12e-3 / 64)
    batch[1].set_state(x=x)
    before = [s.step_count for s in batch]
    up = vs.copy()
    up[1] = (0.0, 0.0, 1.0)
    with pytest.raises(tb.OutOfGrid):
        tb.sim.step_capture_many(batch, up, 200, rp)
    assert batch[0].step_count == before[0] + 200 and batch[2].step_count == before[2] + 200
    assert before[1] < batch[1].step_count < before[1] + 200


def test_out_of_grid_after_advect(tb):
    s = tb.sim.build_sim(SMALL)
    x = s.positions()
    # push one indenter particle right to the top of the stencil-safe margin
    dx = 12e-3 / 64
    x[-1, 2] = (64 - 3) * dx + 0.49 * dx  # base = 61 -> base + 2 = 63 < 64 still in range
    s.set_state(x=x)
    with pytest.raises(tb.OutOfGrid):
        tb.mpm.step(s, (0, 0, 1.0), 200)  # moves up by 2e-6 * 1.0 per substep
    assert 1 <= s.step_count < 200


def test_elastomer_moving_cells_per_substep_matches_oracle(tb, golden, oracle):
    """The indenter's look-ahead walks use the previous elastomer box widened
    by one node; when the elastomer moves further in one substep (here the
    whole scene translates at 300 m/s, 3.2 cells per substep), finalize
    scatters the indenter particles the walks missed, so the step continues
    as the reference's does (engine.cpp:268-286 raises nothing there)."""
    g = golden("small_scene.npz")
    s = tb.sim.build_sim(SMALL)
    tb.mpm.step(s, SMALL_V, 4)
    st = s.state()
    vfast = (300.0, -120.0, 0.0)
    v = st["v"].copy()
    v[:] += np.array(vfast)
    v[s.elastomer_count:] = vfast  # uniform indenter velocity (the command)
    s.set_state(v=v)
    o = _small_oracle(oracle, g)
    o.x, o.v, o.C, o.F = st["x"].copy(), v.copy(), st["C"].copy(), st["F"].copy()
    tb.mpm.step(s, vfast, 3)
    o.step(vfast, 3)
    x = s.positions()
    moved = np.abs(x - st["x"]).max()
    assert moved > 3 * 3 * 12e-3 / 64  # > 3 cells per substep
    assert np.abs(x - o.x).max() <= 1e-9 * moved
    np.testing.assert_allclose(s.state()["F"], o.F, rtol=0, atol=1e-11)
    assert s.step_count == 7
    st = s.stats()
    assert st["walk_fixups"] >= 1  # finalize completed the walks
    assert st["regrows"] >= 1      # the node arrays followed the elastomer


def test_windowed_node_arrays_match_dense(tb, monkeypatch):
    """The node arrays cover the elastomer's box plus the walks' reach and
    grow on demand; a dense res^3 allocation (TACCHI_DENSE_GRID=1) gives the
    same trajectory (to summation order), and a default config-1 scene needs
    a tenth of the dense 1.07 GB."""
    from tests.scenes import CONFIG1

    s = tb.sim.build_sim(CONFIG1)
    st = s.stats()
    assert st["grid_bytes"] < 160e6, st
    monkeypatch.setenv("TACCHI_DENSE_GRID", "1")
    d = tb.sim.build_sim(SMALL)
    monkeypatch.delenv("TACCHI_DENSE_GRID")
    w = tb.sim.build_sim(SMALL)
    assert d.stats()["grid_nodes"] == 64 ** 3 > w.stats()["grid_nodes"]
    for sim in (d, w):
        tb.mpm.step(sim, SMALL_V, 100)
        tb.mpm.step(sim, (0.02, -0.01, -0.05), 100)
    x0 = tb.sim.build_sim(SMALL).positions()
    disp = np.abs(d.positions() - x0).max()
    assert np.abs(d.positions() - w.positions()).max() <= 1e-11 * disp


def test_capture_with_background_image_matches_reference(tb, golden, tmp_path):
    """sim::capture with render.background_image (the image starts from
    k_a * background, phong.cpp:61-64), bit-exact on identical positions."""
    g = golden("background.npz")
    path = str(tmp_path / "bg.png")
    tb.save_png(g["background"], path)
    cfg = {**SMALL, "render": {**SMALL["render"], "background_image": path}}
    s = tb.sim.build_sim(cfg)
    depth, img = tb.sim.capture(s, cfg)
    assert sha(depth) == str(g["depth_sha"])
    np.testing.assert_array_equal(img, g["image"])


def test_render_functions_match_reference(tb, golden):
    k = golden("kat.npz")
    r, hemi, ramp, src = render_inputs()
    assert sha(tb.render.surface_normals(hemi, r)) == str(k["normals_hemi_sha"])
    rp = tb.render_params({}, "")
    np.testing.assert_array_equal(tb.render.phong_render(hemi, r, rp), k["img_hemi"])
    np.testing.assert_array_equal(tb.render.phong_render(ramp, r, rp), k["img_ramp"])
    img_l = tb.render.phong_render(hemi, r, tb.render_params(LIGHT_CFG, ""))
    assert np.abs(img_l.astype(int) - k["img_hemi_l"]).max() <= 1
    assert sha(tb.render.crop_align(src, (0.0, 0.0, 1.0))) == str(k["crop_c_sha"])
    assert sha(tb.render.crop_align(src, (12.25, -7.5, 1.07))) == str(k["crop_o_sha"])
    with pytest.raises(tb.CropOutOfBounds):
        tb.render.crop_align(np.zeros((100, 100)), (0, 0, 1.0))


def test_config1_hundred_frames_match_reference(tb, golden):
    """Config 1 at full size (314,221 particles, 256^3): 100 frames (1000
    substeps, SURVEY §8(d) CI parity) vs the reference; positions, F, height
    map and image."""
    g = golden("config1.npz")
    s = tb.sim.build_sim(CONFIG1)
    assert s.n == int(g["n"]) and s.elastomer_count == int(g["n_elastomer"])
    x0 = s.positions()
    assert sha(x0) == str(g["x0_hash"])
    for _ in range(CONFIG1_STEPS // 10):
        tb.mpm.step(s, CONFIG1_V, 10)
    st = s.state()
    sub = g["subset"]
    disp = np.abs(g["x_subset"] - x0[sub]).max()
    err = np.abs(st["x"][sub] - g["x_subset"]).max()
    assert err <= 1e-6 * disp, (err, disp)  # displacement-relative
    assert err / np.abs(g["x_subset"]).max() <= 1e-4  # north_star bar
    surf_err = np.abs(st["x"][_default_surface()] - g["x_surface"]).max()
    assert surf_err <= 1e-6 * disp
    np.testing.assert_allclose(st["F"][sub], g["F_subset"], rtol=0, atol=1e-9)
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-12)
    depth, img = tb.sim.capture(s, CONFIG1)
    assert np.abs(depth[::16, ::16] - g["depth_sample"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


def test_reruns_agree_to_rounding(tb):
    """Fast mode (deterministic off): two runs of the config-1 press (1000
    frames, gap crossed, 0.1 mm into the gel) from the same inputs. The node
    sums are fp64 adds in hardware order (tile bulk reductions from
    neighbouring CTAs, RED.F64), so reruns are not bit-identical;
    this pins how far apart they are: positions within 1e-11 of the
    displacement (measured ~3e-13), height maps within 1e-15 m (measured
    ~3e-17 m), images within 1 LSB (measured equal)."""
    from tests.scenes import CONFIG1_DEEP_STEPS

    out = []
    for _ in range(2):
        s = tb.sim.build_sim({**CONFIG1, "deterministic": False})
        x0 = s.positions()
        for _ in range(CONFIG1_DEEP_STEPS // 10):
            tb.mpm.step(s, CONFIG1_V, 10)
        depth, img = tb.sim.capture(s, CONFIG1)
        out.append((s.positions(), depth, img.astype(int)))
        del s
    (xa, da, ia), (xb, db, ib) = out
    disp = np.abs(xa - x0).max()
    assert disp > 1e-4
    assert np.abs(xa - xb).max() <= 1e-11 * disp
    assert np.abs(da - db).max() <= 1e-15
    assert np.abs(ia - ib).max() <= 1


def test_config1_thousand_frames_pressing_matches_reference(tb, golden):
    """Config 1 for 1000 frames (10,000 substeps): the indenter crosses the
    0.1 mm gap and presses 0.1 mm into the gel; positions, F, height map and
    image vs the reference."""
    from tests.scenes import CONFIG1_DEEP_STEPS

    g = golden("config1_deep.npz")
    s = tb.sim.build_sim(CONFIG1)
    x0 = s.positions()
    assert sha(x0) == str(g["x0_hash"])
    for _ in range(CONFIG1_DEEP_STEPS // 10):
        tb.mpm.step(s, CONFIG1_V, 10)
    st = s.state()
    sub = g["subset"]
    disp = np.abs(g["x_subset"] - g["x0_subset"]).max()
    err = np.abs(st["x"][sub] - g["x_subset"]).max()
    print(f"config1 deep: err {err:.3e} m, displacement {disp:.3e} m")
    assert err <= 1e-9 * disp, (err, disp)  # measured ~5e-12 of the displacement
    assert np.abs(st["x"][_default_surface()] - g["x_surface"]).max() <= 1e-9 * disp
    np.testing.assert_allclose(st["F"].reshape(-1, 9)[sub], g["F_subset"], rtol=0, atol=1e-9)
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-9)
    depth, img = tb.sim.capture(s, CONFIG1)
    assert np.abs(depth[::8, ::8] - g["depth_sample"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


def _default_surface(nx=101, ny=101, nz=21):
    return np.array([(i * ny + j) * nz + nz - 1 for i in range(nx) for j in range(ny)])


@pytest.mark.parametrize("shape", ["cylinder", "cylinder_shell", "wave1", "dots"])
def test_config3_press_and_slide_match_reference(tb, golden, shape):
    """Config 3 indenters (cylinder, ring, wave, dot grid) pressed then slid
    laterally (sticky grid contact drags the gel), scaled to SMALL3; the slide
    exercises the indenter column walk under lateral motion."""
    from tests.scenes import SMALL3, SMALL3_PRESS, SMALL3_SLIDE

    g = golden("config3.npz")
    s = tb.sim.build_sim(SMALL3, shape)
    x0 = s.positions()
    assert sha(x0) == str(g[f"{shape}_x0_sha"])
    tb.mpm.step(s, SMALL3_PRESS[1], SMALL3_PRESS[0])
    tb.mpm.step(s, SMALL3_SLIDE[1], SMALL3_SLIDE[0])
    st = s.state()
    sub = g[f"{shape}_subset"]
    disp = np.abs(g[f"{shape}_x_subset"] - x0[sub]).max()
    assert np.abs(st["x"][sub] - g[f"{shape}_x_subset"]).max() <= 1e-8 * disp
    nx = ny = 51
    surf = np.array([(i * ny + j) * 7 + 6 for i in range(nx) for j in range(ny)])
    assert np.abs(st["x"][surf] - g[f"{shape}_x_surface"]).max() <= 1e-8 * disp
    np.testing.assert_allclose(st["F"][sub], g[f"{shape}_F_subset"], rtol=0, atol=1e-11)
    assert s.step_count == int(g[f"{shape}_step_count"])
    assert s.diag.min_det_f == pytest.approx(float(g[f"{shape}_min_det_f"]), abs=1e-12)
    depth, img = tb.sim.capture(s, SMALL3, shape)
    assert np.abs(depth[::8, ::8] - g[f"{shape}_depth_sample"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g[f"{shape}_image"]).max() <= 2


def test_config5_large_gel_matches_reference(tb, golden):
    """Config 5 (large-area gel, 948,421 particles, 512^3 grid): press then
    move laterally vs the reference (tests/scenes.py CONFIG5)."""
    from tests.scenes import CONFIG5, CONFIG5_MOVE, CONFIG5_PRESS

    g = golden("config5.npz")
    s = tb.sim.build_sim(CONFIG5)
    assert s.n == int(g["n"]) and s.elastomer_count == int(g["n_elastomer"])
    x0 = s.positions()
    assert sha(x0) == str(g["x0_hash"])
    tb.mpm.step(s, CONFIG5_PRESS[1], CONFIG5_PRESS[0])
    tb.mpm.step(s, CONFIG5_MOVE[1], CONFIG5_MOVE[0])
    st = s.state()
    sub = g["subset"]
    disp = np.abs(g["x_subset"] - x0[sub]).max()
    assert disp > 1e-5
    assert np.abs(st["x"][sub] - g["x_subset"]).max() <= 1e-8 * disp
    surf = _default_surface(201, 201, 21)[::7]
    assert np.abs(st["x"][surf] - g["x_surface"]).max() <= 1e-8 * disp
    np.testing.assert_allclose(st["F"][sub], g["F_subset"], rtol=0, atol=1e-11)
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-12)
    assert d.max_speed == pytest.approx(float(g["max_speed"]), rel=1e-9)
    depth, img = tb.sim.capture(s, CONFIG5)
    assert np.abs(depth[::16, ::16] - g["depth_sample"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


def test_config2b_dense_gel_matches_reference(tb, golden):
    """Config 2b (171 x 171 x 35 gel at 0.91 grid cells spacing + sphere 1e5,
    1,123,435 particles): a quarter of the gel particles share a base cell, so
    the scatter's duplicate path carries real load. Press then slide vs the
    reference (tests/scenes.py CONFIG2B)."""
    from tests.scenes import CONFIG2B, CONFIG2B_PRESS, CONFIG2B_SLIDE

    g = golden("config2b.npz")
    s = tb.sim.build_sim(CONFIG2B)
    assert s.n == int(g["n"]) and s.elastomer_count == int(g["n_elastomer"])
    x0 = s.positions()
    assert sha(x0) == str(g["x0_hash"])
    tb.mpm.step(s, CONFIG2B_PRESS[1], CONFIG2B_PRESS[0])
    tb.mpm.step(s, CONFIG2B_SLIDE[1], CONFIG2B_SLIDE[0])
    st = s.state()
    sub = g["subset"]
    disp = np.abs(g["x_subset"] - x0[sub]).max()
    assert disp > 1e-5
    assert np.abs(st["x"][sub] - g["x_subset"]).max() <= 1e-8 * disp
    surf = _default_surface(171, 171, 35)[::7]
    assert np.abs(st["x"][surf] - g["x_surface"]).max() <= 1e-8 * disp
    np.testing.assert_allclose(st["F"][sub], g["F_subset"], rtol=0, atol=1e-11)
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-12)
    assert d.max_speed == pytest.approx(float(g["max_speed"]), rel=1e-9)
    depth, img = tb.sim.capture(s, CONFIG2B)
    assert np.abs(depth[::16, ::16] - g["depth_sample"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


@pytest.mark.parametrize("with_surface", [True, False])
def test_init_scene_parts_gravity_nonuniform_indenter(tb, golden, with_surface):
    """mpm::init_scene from explicit arrays (tests/scenes.py PARTS) with gravity,
    an indenter moving at creation and a non-uniform indenter velocity (the
    direct indenter scatter), 21 x 19 x 6 lattice; with the surface lattice
    (lattice-block CTA tiling) and without (flat tiling)."""
    from tests.scenes import PARTS, PARTS_STEPS, PARTS_V

    g = golden("parts.npz")
    P = PARTS
    params = dict(res=P["res"], dx=P["grid_edge"] / P["res"][0], origin=(0, 0, 0), dt=P["dt"],
                  gravity=P["gravity"])
    particles = dict(x=g["x0"], v=g["v0"], mass=g["mass"], volume0=g["vol0"], tag=g["tag"],
                     n_elastomer=int(g["n_elastomer"]))
    surface = None
    if with_surface:
        geom = g["surf_geom"]
        surface = dict(nx=int(g["surf_n"][0]), ny=int(g["surf_n"][1]), x0=geom[0], y0=geom[1],
                       sx=geom[2], sy=geom[3], z0=geom[4], particle=g["surf_particle"])
    s = tb.init_scene(params, particles, surface)
    tb.mpm.step(s, PARTS_V, PARTS_STEPS)
    st = s.state()
    disp = np.abs(g["x"] - g["x0"]).max()
    assert np.abs(st["x"] - g["x"]).max() <= 1e-8 * disp
    ne = int(g["n_elastomer"])
    np.testing.assert_allclose(st["F"].reshape(-1, 9)[:ne], g["F"][:ne], rtol=0, atol=1e-11)
    np.testing.assert_allclose(st["v"], g["v"], rtol=0, atol=1e-7 * np.abs(g["v"]).max())
    d = s.diag
    assert d.step_count == int(g["step_count"])
    assert d.min_det_f == pytest.approx(float(g["min_det_f"]), abs=1e-12)
    assert d.max_speed == pytest.approx(float(g["max_speed"]), rel=1e-9)


def test_config2a_conserves_mass_and_momentum(tb):
    """Config 2a (1,214,221 particles): size-independent P2G invariants
    (SPEC.md:147-148): sum of node mass = sum of particle mass; with zero
    stress (F = I) and C = 0, sum of node momentum = sum of m v."""
    from tests.scenes import CONFIG2A

    s = tb.sim.build_sim(CONFIG2A)
    assert s.n == 1214221
    n, ne = s.n, s.elastomer_count
    rng = np.random.default_rng(0)
    v = rng.standard_normal((n, 3)) * 1e-3
    s.set_state(v=v, Cm=np.zeros((n, 9)), F=np.tile(np.eye(3).ravel(), (n, 1)))
    tb.mpm.zero_grid(s)
    tb.mpm.particle_to_grid(s)
    lo, hi = s.grid_window()
    m, mom, _ = s.grid(lo, hi)
    # particle masses (init_scene, scene.cpp:48-66)
    gel_m = 1000.0 * (0.02 * 0.02 * 0.004) / ne
    x = s.positions()
    ind = x[ne:]
    ext = ind.max(0) - ind.min(0)
    ind_m = 1000.0 * (ext[0] * ext[1] * ext[2] / (n - ne)) * 80.0
    total_m = gel_m * ne + ind_m * (n - ne)
    assert m.sum() == pytest.approx(total_m, rel=1e-10)
    pm = np.concatenate([gel_m * v[:ne], ind_m * v[ne:]]).sum(0)
    np.testing.assert_allclose(mom.reshape(-1, 3).sum(0), pm, rtol=1e-9, atol=1e-12 * np.abs(pm).max())


def test_rest_state_is_a_fixed_point(tb):
    """zero indenter velocity, untouched gel -> no drift."""
    cfg = dict(SMALL)
    cfg = {**SMALL, "indenter": {**SMALL["indenter"], "gap_mm": 0.5}}
    s = tb.sim.build_sim(cfg)
    x0 = s.positions()
    tb.mpm.step(s, (0, 0, 0), 100)
    assert np.abs(s.positions() - x0).max() <= 1e-9
    assert s.diag.max_speed < 1e-9


def test_polar_rotation_and_svd_fallback_match_reference(tb, golden):
    """material.cpp:18-89 on the device (the functions the P2G kernels call)
    vs the reference (kat.npz, 63 deformation gradients from identity to
    strongly sheared): the scaled Newton polar rotation, the corotated stress,
    and the SVD fallback polar_rotation_svd forced directly (the Newton loop
    reaches it only for |det F| <= 1e-300 or no convergence in 40 iterations,
    which no well-posed press produces)."""
    g = golden("kat.npz")
    F = g["F"]
    R, S = tb.material.polar_rotation(F)
    np.testing.assert_allclose(R, g["R"], rtol=0, atol=1e-13)
    smax = np.abs(g["S"]).max()
    np.testing.assert_allclose(S, g["S"], rtol=0, atol=1e-12 * smax)
    Rs, Ss = tb.material.polar_rotation(F, svd=True)
    np.testing.assert_allclose(Rs, g["R_svd"], rtol=0, atol=1e-12)
    # the two paths agree, and the fallback's rotation is proper
    np.testing.assert_allclose(Rs, R, rtol=0, atol=1e-10)
    np.testing.assert_allclose(np.einsum("nji,njk->nik", Rs, Rs), np.tile(np.eye(3), (len(F), 1, 1)),
                               rtol=0, atol=1e-13)
    assert np.all(np.linalg.det(Rs) > 0)
    np.testing.assert_allclose(Ss, S, rtol=0, atol=1e-8 * smax)


def test_init_scene_from_reference_inputs(tb, golden):
    """mpm::init_scene from its own inputs (SceneParams, the elastomer
    lattice, the placed indenter points and v0; scene.cpp:28-87) computes the
    reference's masses, rest volumes, tags and initial velocities bit for bit
    (parts.npz was made by the reference's init_scene from the same inputs),
    and the scene then steps as the reference's."""
    from tests.scenes import PARTS, PARTS_STEPS, PARTS_V

    g = golden("parts.npz")
    P = PARTS
    params = dict(grid_resolution=P["res"], grid_edge=P["grid_edge"], dt=P["dt"],
                  gravity=P["gravity"])
    lattice = dict(counts=P["lat_counts"], dims=P["lat_dims"], origin=P["lat_origin"])
    s = tb.mpm.init_scene(params, lattice, g["ind"], P["ind_v0"])
    st = s.state()
    k = s.constants()
    np.testing.assert_array_equal(st["x"], g["x0"])
    np.testing.assert_array_equal(k["mass"], g["mass"])
    np.testing.assert_array_equal(k["volume0"], g["vol0"])
    np.testing.assert_array_equal(k["tag"], g["tag"])
    ne = int(g["n_elastomer"])
    assert s.elastomer_count == ne
    assert not st["v"][:ne].any()
    np.testing.assert_array_equal(st["v"][ne:], np.tile(P["ind_v0"], (s.n - ne, 1)))
    s.set_state(v=g["v0"])  # the golden's non-uniform indenter velocity
    tb.mpm.step(s, PARTS_V, PARTS_STEPS)
    disp = np.abs(g["x"] - g["x0"]).max()
    assert np.abs(s.positions() - g["x"]).max() <= 1e-8 * disp
    # explicit lattice positions give the same scene
    pos = g["x0"][:ne]
    s2 = tb.mpm.init_scene(params, dict(lattice, positions=pos), g["ind"], P["ind_v0"])
    np.testing.assert_array_equal(s2.state()["x"], g["x0"])
    with pytest.raises(tb.EmptyScene):
        tb.mpm.init_scene(params, lattice, np.zeros((0, 3)))
    with pytest.raises(tb.GridTooSmall):
        tb.mpm.init_scene(params, lattice, g["ind"] + np.array([0.0, 0.0, 0.1]))


def test_build_sim_from_caller_points(tb, golden):
    """sim::build_sim(cfg, indenter) with the caller's placed points equals
    the config path that places the indenter itself."""
    g = golden("small_scene.npz")
    placed = tb.geo.placed_indenter(SMALL, "")
    s = tb.sim.build_sim_points(SMALL, placed)
    np.testing.assert_array_equal(s.state()["x"], g["x0"])
    tb.mpm.step(s, SMALL_V, SMALL_STEPS)
    disp = np.abs(g["x"] - g["x0"]).max()
    assert np.abs(s.positions() - g["x"]).max() <= 1e-9 * disp


def test_post_step_grid_matches_reference(tb, golden):
    """After mpm::step the grid holds the last substep's P2G and grid_update
    (engine.cpp:180-205) and zeros outside the active window: with keep_grid
    the last substep runs the phase path, and tg_download_grid returns that
    grid; after a fused step (the default) the grid is not retained and the
    call says so."""
    g = golden("grid_post_step.npz")
    s = tb.sim.build_sim(SMALL)
    s.set_keep_grid(True)
    for tag, n in (("a", 20), ("b", 7)):
        tb.mpm.step(s, SMALL_V, n)
        lo, hi = s.grid_window()
        np.testing.assert_array_equal(lo, g[f"{tag}_win_lo"])
        np.testing.assert_array_equal(hi, g[f"{tag}_win_hi"])
        m, mom, vel = s.grid(g[f"{tag}_lo"], g[f"{tag}_hi"])
        gm = g[f"{tag}_mass"]
        assert (m == 0).sum() == (gm == 0).sum()  # the same massless nodes
        np.testing.assert_allclose(m, gm, rtol=0, atol=1e-12 * gm.max())
        pmax = np.abs(g[f"{tag}_mom"]).max()
        np.testing.assert_allclose(mom, g[f"{tag}_mom"], rtol=0, atol=1e-9 * pmax)
        vmax = np.abs(g[f"{tag}_vel"]).max()
        np.testing.assert_allclose(vel, g[f"{tag}_vel"], rtol=0, atol=1e-9 * vmax)
        disp = np.abs(g[f"{tag}_x"] - s.state()["x"]).max()
        assert disp <= 1e-15
    s.set_keep_grid(False)
    tb.mpm.step(s, SMALL_V, 3)
    with pytest.raises(tb.InvalidArgument):
        s.grid(g["a_lo"], g["a_hi"])


def _check_checkpoint(tb, s, g, prefix, cfg, obj="", tol=1e-8, label=""):
    """Positions (subset and top surface) within tol x the displacement, F,
    diagnostics, height map <= 1e-7 m and image <= 2/255 vs a reference
    checkpoint of make_golden._checkpoint."""
    st = s.state()
    sub = g[f"{prefix}subset"]
    disp = np.abs(g[f"{prefix}x_subset"] - g[f"{prefix}x0_subset"]).max()
    err = np.abs(st["x"][sub] - g[f"{prefix}x_subset"]).max()
    surf = _default_surface()
    serr = np.abs(st["x"][surf] - g[f"{prefix}x_surface"]).max()
    print(f"{label} {prefix}: x err {err:.3e} m, surface {serr:.3e} m, displacement {disp:.3e} m")
    assert disp > 0
    assert err <= tol * disp, (err, disp)
    assert serr <= tol * disp, (serr, disp)
    assert err / np.abs(g[f"{prefix}x_subset"]).max() <= 1e-4  # north_star bar
    np.testing.assert_allclose(st["F"].reshape(-1, 9)[sub], g[f"{prefix}F_subset"], rtol=0, atol=1e-9)
    d = s.diag
    assert d.step_count == int(g[f"{prefix}step_count"])
    assert d.min_det_f == pytest.approx(float(g[f"{prefix}min_det_f"]), abs=1e-9)
    depth, img = tb.sim.capture(s, cfg, obj)
    assert np.abs(depth[::8, ::8] - g[f"{prefix}depth_sample"]).max() <= 1e-7
    assert depth.max() == pytest.approx(float(g[f"{prefix}depth_max"]), abs=1e-9)
    assert np.abs(img.astype(int) - g[f"{prefix}image"]).max() <= 2


def test_config2a_bench_workload_matches_reference(tb, golden):
    """Config 2a, the bench workload (1,214,221 particles: the sphere at 1e6
    points), stepped exactly as bench.py steps it (tg_step_capture, 10
    substeps + capture per frame) for 100 frames and on to 600 (past the
    0.1 mm gap) vs the reference at both checkpoints."""
    from tests.scenes import CONFIG2A, CONFIG2A_FRAMES, CONFIG2A_V

    g = golden("config2a.npz")
    s = tb.sim.build_sim(CONFIG2A)
    assert s.n == int(g["n"]) and s.elastomer_count == int(g["n_elastomer"])
    assert sha(s.positions()) == str(g["x0_hash"])
    rp = tb.render_params(CONFIG2A, "")
    done = 0
    for f in CONFIG2A_FRAMES:
        for _ in range(f - done):
            tb.sim.step_capture(s, CONFIG2A_V, 10, params=rp, want_depth=False, want_image=False)
        done = f
        _check_checkpoint(tb, s, g, f"f{f}_", CONFIG2A, label="config2a")


def test_config4_episodes_match_reference(tb, golden):
    """Config 4: the first episodes of the 1024-episode batch (mt19937_64
    draws: lateral offset over +-1 mm and z-rotation of the indenter),
    stepped together with tg_step_capture_many for 200 frames, each vs the
    reference's episode."""
    from paper_2301_08343_b200 import episodes as E
    from tests.scenes import CONFIG1, CONFIG1_V, CONFIG4_EPISODES, CONFIG4_FRAMES

    g = golden("config4.npz")
    eps = [E.make_episode(e) for e in range(CONFIG4_EPISODES)]
    sims, cfgs = [], []
    for e, ep in enumerate(eps):
        np.testing.assert_array_equal(
            g[f"e{e}_pose"], [ep.offset_x_m, ep.offset_y_m, ep.z_rotation_rad, ep.depth_m])
        cfg = E.episode_config(CONFIG1, ep)
        s = tb.sim.build_sim(cfg, "", ep.offset_x_m, ep.offset_y_m)
        assert sha(s.positions()) == str(g[f"e{e}_x0_hash"])
        sims.append(s)
        cfgs.append(cfg)
    # the batched builder (one shared cloud) gives the same episodes
    poses = [[ep.offset_x_m, ep.offset_y_m, ep.z_rotation_rad] for ep in eps[:2]]
    for e, b in enumerate(tb.sim.build_episodes(CONFIG1, "", poses)):
        assert sha(b.positions()) == str(g[f"e{e}_x0_hash"])
    rps = [tb.render_params(c, "") for c in cfgs]
    vel = np.tile(CONFIG1_V, (len(sims), 1))
    for _ in range(CONFIG4_FRAMES):
        outs, status = tb.sim.step_capture_many(sims, vel, 10, rps, want_depth=False)
        assert status == [0] * len(sims)
    for e, (s, cfg) in enumerate(zip(sims, cfgs)):
        _check_checkpoint(tb, s, g, f"e{e}_", cfg, label=f"config4 episode {e}")
        assert np.abs(outs[e][1].astype(int) - g[f"e{e}_image"]).max() <= 2


def test_config3_full_size_dots_press_and_slide(tb, golden):
    """Config 3 at full size: the dot-grid indenter (3 x 3 studs, 1e5 points)
    on the default gel and 256^3 grid, pressed until the commanded travel is
    gap + 0.3 mm (20,000 substeps), then slid +x at 5 mm/s for 200 frames,
    vs the reference after the press and after the slide."""
    from tests.scenes import CONFIG1, CONFIG3_FULL_PRESS, CONFIG3_FULL_SHAPE, CONFIG3_FULL_SLIDE

    g = golden("config3_full.npz")
    shape = CONFIG3_FULL_SHAPE
    s = tb.sim.build_sim(CONFIG1, shape)
    assert sha(s.positions()) == str(g["x0_hash"])
    tb.mpm.step(s, CONFIG3_FULL_PRESS[1], CONFIG3_FULL_PRESS[0])
    _check_checkpoint(tb, s, g, "press_", CONFIG1, shape, label="config3 dots")
    rp = tb.render_params(CONFIG1, shape)
    for _ in range(CONFIG3_FULL_SLIDE[0] // 10):
        tb.sim.step_capture(s, CONFIG3_FULL_SLIDE[1], 10, params=rp, want_depth=False,
                            want_image=False)
    _check_checkpoint(tb, s, g, "slide_", CONFIG1, shape, label="config3 dots")


def test_deterministic_reruns_bit_identical(tb):
    """SPEC acceptance 10 / "Concurrency Model": in deterministic mode
    (SceneConfig.deterministic, the default) two runs of the config-1 press
    (1000 frames: gap crossed, 0.1 mm into the gel) give byte-identical
    particle states, height maps and images."""
    from tests.scenes import CONFIG1_DEEP_STEPS

    out = []
    for _ in range(2):
        s = tb.sim.build_sim(CONFIG1)  # deterministic: true by default
        for _ in range(CONFIG1_DEEP_STEPS // 10):
            tb.mpm.step(s, CONFIG1_V, 10)
        depth, img = tb.sim.capture(s, CONFIG1)
        st = s.state()
        out.append((st["x"].tobytes(), st["v"].tobytes(), st["C"].tobytes(), st["F"].tobytes(),
                    depth.tobytes(), img.tobytes()))
        del s
    assert out[0] == out[1]


def test_deterministic_reruns_bit_identical_with_duplicates(tb):
    """Deterministic mode where gel particles share base cells (config 2b:
    0.91-cell spacing, about a quarter of the particles are duplicates): the
    duplicates' contributions reach the grid as their own fixed-point REDs,
    the owner's inside the tile sum, so the owner must not be chosen by
    timing (the highest thread of the CTA takes the cell). Two runs of the
    press + slide slice give byte-identical states, height maps and images."""
    from tests.scenes import CONFIG2B, CONFIG2B_PRESS, CONFIG2B_SLIDE

    out = []
    for _ in range(2):
        s = tb.sim.build_sim({**CONFIG2B, "deterministic": True})
        for n, v in (CONFIG2B_PRESS, CONFIG2B_SLIDE):
            for _ in range(n):
                tb.mpm.step(s, v, 10)
        depth, img = tb.sim.capture(s, CONFIG2B)
        st = s.state()
        out.append((st["x"].tobytes(), st["v"].tobytes(), st["C"].tobytes(), st["F"].tobytes(),
                    depth.tobytes(), img.tobytes()))
        del s
    assert out[0] == out[1]


_WALK_CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
import paper_2301_08343_b200 as tb
from tests.scenes import CONFIG2A, CONFIG2A_V
s = tb.sim.build_sim({**CONFIG2A, "deterministic": True})
for _ in range(30):
    tb.mpm.step(s, CONFIG2A_V, 10)
st = s.state()
print(json.dumps({k: hashlib.sha1(st[k].tobytes()).hexdigest() for k in ("x", "v", "C", "F")}))
"""


def test_storage_orders_byte_identical():
    """The elastomer's storage order within each CTA's slots (dealt for the
    shared-memory banks, TACCHI_GEL_LANES=2 the default; 1 within warps; 0
    lattice order) only changes which thread handles which particle: in
    deterministic mode (fixed-point node sums) 300 substeps of config 2a
    give byte-identical particle states in every order (downloaded through
    the permutation). Config 2a's gel has no duplicate base cells; where
    there are duplicates the cell's owner is the CTA's highest thread, a
    function of the storage order, and the rounding of the fixed-point sums
    follows it."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("0", "1", "2"):
        p = subprocess.run([sys.executable, "-c", _WALK_CHILD % root], capture_output=True,
                           text=True, env={**os.environ, "TACCHI_GEL_LANES": mode}, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        out[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["0"] == out["1"] == out["2"]


def test_walk_plans_byte_identical():
    """The indenter's look-ahead walks as extra blocks of the elastomer kernel
    (TACCHI_WALKS=fused) or as their own kernel on a forked stream
    (TACCHI_WALKS=fork, the default; double-buffered M_I) scatter the same
    contributions: in deterministic mode 300 substeps of config 2a give
    byte-identical particle states (one process per plan: the switch is read
    at tg_create)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for plan in ("fused", "fork"):
        p = subprocess.run([sys.executable, "-c", _WALK_CHILD % root], capture_output=True,
                           text=True, env={**os.environ, "TACCHI_WALKS": plan}, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        out[plan] = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["fused"] == out["fork"]


@pytest.mark.parametrize("det", [False, True])
def test_small_scene_both_accumulation_modes_match_reference(tb, golden, det):
    """The fp64 fast mode and the fixed-point deterministic mode both match
    the reference (200 substeps of the SMALL press)."""
    g = golden("small_scene.npz")
    s = tb.sim.build_sim({**SMALL, "deterministic": det})
    tb.mpm.step(s, SMALL_V, SMALL_STEPS // 2)
    tb.mpm.step(s, SMALL_V, SMALL_STEPS // 2)
    st = s.state()
    disp = np.abs(g["x"] - g["x0"]).max()
    assert np.abs(st["x"] - g["x"]).max() <= 1e-9 * disp
    np.testing.assert_allclose(st["F"], g["F"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(st["v"], g["v"], rtol=0, atol=1e-8 * np.abs(g["v"]).max())
    depth, img = tb.sim.capture(s, SMALL)
    assert np.abs(depth - g["depth"]).max() <= 1e-7
    assert np.abs(img.astype(int) - g["image"]).max() <= 2


def test_device_shape_clouds_bit_identical(tb, golden):
    """f3, episode setup on the GPU: the rejection sampler on the device
    (mt19937_64 stream twisted in shared memory, candidates tested and
    compacted in stream order) reproduces the host restatement -- and so the
    reference (kat.npz cloud hashes) -- bit for bit for all 21 shapes, and at
    the 1e6-point source size of the sphere, the dot grid, the wave and the
    bump field (the shapes whose tests call libm)."""
    from tests.scenes import SHAPES

    k = golden("kat.npz")
    for i, shape in enumerate(SHAPES):
        d = tb.geo.generate_shape_cloud_device(shape, 2000, 7)
        np.testing.assert_array_equal(d, tb.geo.generate_shape_cloud(shape, 2000, 7))
        assert sha(d) == str(k["cloud_hash"][i]), shape
    for shape in ("sphere", "dots", "wave1", "random", "pacman"):
        d = tb.geo.generate_shape_cloud_device(shape, 1000000, 20230115)
        h = tb.geo.generate_shape_cloud(shape, 1000000, 20230115)
        assert np.array_equal(d, h), shape


def test_device_and_host_setup_build_the_same_scene(tb, golden, monkeypatch):
    """build_sim / build_episodes with the device setup (default) and the host
    restatement (TACCHI_HOST_SETUP=1): identical particles for a rotated,
    offset, subsampled indenter (config-4 pose)."""
    from paper_2301_08343_b200 import episodes as E
    from tests.scenes import CONFIG1

    ep = E.make_episode(5)
    cfg = E.episode_config(CONFIG1, ep)
    dev = tb.sim.build_sim(cfg, "dots", ep.offset_x_m, ep.offset_y_m).positions()
    dev_eps = tb.sim.build_episodes(CONFIG1, "dots", [[ep.offset_x_m, ep.offset_y_m,
                                                       ep.z_rotation_rad]])[0].positions()
    monkeypatch.setenv("TACCHI_HOST_SETUP", "1")
    host = tb.sim.build_sim(cfg, "dots", ep.offset_x_m, ep.offset_y_m).positions()
    np.testing.assert_array_equal(dev, host)
    np.testing.assert_array_equal(dev_eps, host)
    np.testing.assert_array_equal(host[-100000:], tb.geo.placed_indenter(cfg, "dots", ep.offset_x_m,
                                                                          ep.offset_y_m))


def test_pipelined_step_capture_matches_synchronous(tb):
    """tg_step_capture_submit / _wait (two frames in flight, the read-back of
    frame k overlapping frame k+1) gives the frames of tg_step_capture;
    order and capacity rules; an error surfaces at its frame's wait and at
    the wait of the frame submitted after it."""
    rp = tb.render_params(SMALL, "")
    a, b = tb.sim.build_sim(SMALL), tb.sim.build_sim(SMALL)
    ref = [tb.sim.step_capture(b, SMALL_V, 10, params=rp) for _ in range(6)]
    t = [tb.sim.step_capture_submit(a, SMALL_V, 10, rp)]
    got = []
    for k in range(1, 6):
        t.append(tb.sim.step_capture_submit(a, SMALL_V, 10, rp))
        if k == 1:
            with pytest.raises(tb.InvalidArgument):  # a third frame in flight
                tb.sim.step_capture_submit(a, SMALL_V, 10, rp)
        d, im = tb.sim.step_capture_wait(a, t[k - 1], rp)
        got.append((d.copy(), im.copy()))
    d, im = tb.sim.step_capture_wait(a, t[-1], rp)
    got.append((d.copy(), im.copy()))
    for (d, im), (dr, imr) in zip(got, ref):
        np.testing.assert_allclose(d, dr, rtol=0, atol=1e-12)
        assert np.abs(im.astype(int) - imr).max() <= 1
    t_open = tb.sim.step_capture_submit(a, SMALL_V, 10, rp, read_back=False)
    with pytest.raises(tb.InvalidArgument):  # the handle is busy while frames are in flight
        tb.mpm.step(a, SMALL_V, 1)
    assert tb.sim.step_capture_wait(a, t_open, rp) == (None, None)
    tb.mpm.step(b, SMALL_V, 10)
    assert a.step_count == b.step_count == 70
    # an error in frame k: reported at its wait and at the next frame's
    x = a.positions()
    x[-1, 2] = (64 - 3) * (12e-3 / 64) + 0.49 * (12e-3 / 64)
    a.set_state(x=x)
    t1 = tb.sim.step_capture_submit(a, (0.0, 0.0, 1.0), 200, rp)
    t2 = tb.sim.step_capture_submit(a, (0.0, 0.0, 1.0), 10, rp)
    with pytest.raises(tb.OutOfGrid):
        tb.sim.step_capture_wait(a, t1, rp)
    with pytest.raises(tb.OutOfGrid):
        tb.sim.step_capture_wait(a, t2, rp)


def test_pipelined_frames_across_a_regrow(tb):
    """A pipelined frame whose scatter outgrows the node arrays (the scene
    translating 3.2 cells per substep) is finished after the regrow and the
    frame submitted behind it is replayed: the frames equal the synchronous
    ones."""
    rp = tb.render_params(SMALL, "")
    sims = [tb.sim.build_sim(SMALL), tb.sim.build_sim(SMALL)]
    vfast = (300.0, -120.0, 0.0)
    for s in sims:
        tb.mpm.step(s, SMALL_V, 4)
        v = s.state()["v"]
        v[:] += np.array(vfast)
        v[s.elastomer_count:] = vfast
        s.set_state(v=v)
    a, b = sims
    before = a.stats()["regrows"]
    t1 = tb.sim.step_capture_submit(a, vfast, 2, rp)
    t2 = tb.sim.step_capture_submit(a, vfast, 1, rp)
    d1, i1 = (x.copy() for x in tb.sim.step_capture_wait(a, t1, rp))
    d2, i2 = (x.copy() for x in tb.sim.step_capture_wait(a, t2, rp))
    r1 = tb.sim.step_capture(b, vfast, 2, params=rp)
    r2 = tb.sim.step_capture(b, vfast, 1, params=rp)
    assert a.stats()["regrows"] > before
    np.testing.assert_allclose(d1, r1[0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(d2, r2[0], rtol=0, atol=1e-12)
    assert np.abs(i2.astype(int) - r2[1]).max() <= 1
    assert a.step_count == b.step_count == 7
    assert np.abs(a.positions() - b.positions()).max() <= 1e-12
