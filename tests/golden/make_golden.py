"""Generates the committed golden fixtures from the UNMODIFIED reference.

The reference ships no golden vectors (its unit tests are empty stubs,
SURVEY.md §4), so the fixtures here are produced by running the reference's
own C++ code, compiled from /root/reference/proj by oracle/Makefile into
oracle/_ref/libtacchi_ref.so. Run in the build container (where
/root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures (all numpy .npz):
  kat.npz          polar_rotation / corotated_stress on a spread of F,
                   render KATs (crop_align, surface_normals, phong_render)
                   on synthetic depth maps, and hashes of the 21 generated
                   indenter clouds + the default placed indenter.
  small_scene.npz  SMALL config, 200 substeps at v = (0, 0, -0.05) m/s:
                   full particle state, diagnostics, capture depth + image.
  config3.npz      SMALL3 scene per config-3 shape (cylinder, ring, wave,
                   dots): press then slide; full positions, F, image.
  config1_deep.npz default config, 10,000 substeps (1000 frames) at the default
                   press velocity: 0.1 mm into the gel; elastomer subset, surface
                   positions, image and depth.
  config5.npz      large-area gel (848,421 + 1e5 particles, 512^3 grid):
                   50 substeps pressing + 30 moving laterally; seeded
                   4096-particle subset, every 7th surface particle, image.
  bridge.npz       the reference's bridge (server.cpp / session.cpp) driven
                   by tests/scenes.bridge_script on the SMALL scene, plus the
                   init errors of BAD_CONFIGS: replies, steps.jsonl, the
                   .depth files (bytes) and the images (pixels).
  clouds.npz       indenters from point-cloud files (ASCII PLY, XYZ) and the
                   reference's errors for malformed files.
  background.npz   sim::capture with a render background image (SMALL scene).
  parts.npz        mpm::init_scene from explicit parts (PARTS: gravity, moving
                   indenter at creation, then a non-uniform indenter velocity):
                   initial arrays and the state after PARTS_STEPS substeps.
  harness.npz      the reference's dataset::run_press_dataset on HARNESS
                   (2 objects x 2 positions x 3 depths): manifest.csv,
                   config.json, every image and .depth file; metrics::compare
                   on image pairs and on a seeded noise pair.
  config2a.npz     the bench workload (sphere 1e6, 1,214,221 particles) at
                   100 and 600 frames: subset x / F / v, surface, image, depth.
  config4.npz      config-4 episodes 0-3 (mt19937_64 pose draws, offset and
                   z-rotation), 200 frames each.
  config3_full.npz the dot-grid indenter at full size, pressed 20,000
                   substeps then slid 2,000.
  config1.npz      default config (dt 2e-6), 1000 substeps (100 frames) at the
                   default press velocity: surface-particle positions, a
                   seeded 4096-particle subset of x and F, diagnostics, the
                   640x480 capture image and depth.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refpy as R  # noqa: E402
from tests.scenes import (BAD_CONFIGS, CONFIG1_DEEP_STEPS, HARNESS, PARTS, PARTS_STEPS, PARTS_V, CONFIG1, CONFIG2B, CONFIG2B_PRESS, CONFIG2B_SLIDE, CONFIG5, CONFIG5_MOVE, CONFIG5_PRESS, bridge_script, CONFIG1_STEPS, CONFIG1_V, LIGHT_CFG, PLACED_ROT, SHAPES,  # noqa: E402
                          SMALL, SMALL3, SMALL3_PRESS, SMALL3_SHAPES, SMALL3_SLIDE, SMALL_STEPS,
                          SMALL_V, render_inputs, sha)

OUT = os.path.dirname(os.path.abspath(__file__))


def kat():
    rng = np.random.default_rng(20230115)
    Fs = [np.eye(3), np.diag([0.9, 1.0, 1.0]), np.diag([1.2, 0.8, 1.05])]
    th = 0.7
    rot = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
    Fs.append(rot)
    Fs.append(rot @ np.diag([1.1, 0.95, 0.9]))
    for _ in range(40):
        Fs.append(np.eye(3) + 0.05 * rng.standard_normal((3, 3)))
    for _ in range(20):
        Fs.append(np.eye(3) + 0.4 * rng.standard_normal((3, 3)))
    Fs = [F for F in Fs if np.linalg.det(F) > 0]
    Fs = np.array(Fs)
    Rs = np.array([R.polar_rotation(F) for F in Fs])
    Ss = np.array([R.corotated_stress(F) for F in Fs])
    Rsvd = np.array([R.polar_rotation_svd(F) for F in Fs])

    r, hemi, ramp, src = render_inputs()
    normals_hemi = R.surface_normals(hemi, r)
    img_hemi = R.phong(hemi, r, None)
    img_ramp = R.phong(ramp, r, None)
    img_hemi_l = R.phong(hemi, r, LIGHT_CFG)
    crop_c, r_c = R.crop_align(src, r, (0.0, 0.0), 1.0, 640, 480)
    crop_o, r_o = R.crop_align(src, r, (12.25, -7.5), 1.07, 640, 480)
    cloud_hash, cloud_head = [], []
    for s in SHAPES:
        pts = R.generate_cloud(s, 2000, 7)
        cloud_hash.append(sha(pts))
        cloud_head.append(pts[:4])
    placed = R.placed_indenter({}, "")
    placed_rot = R.placed_indenter(*PLACED_ROT)
    np.savez_compressed(
        os.path.join(OUT, "kat.npz"), F=Fs, R=Rs, R_svd=Rsvd, S=Ss,
        normals_hemi_sha=sha(normals_hemi), normals_hemi_sample=normals_hemi[::37, ::41],
        img_hemi=img_hemi, img_ramp=img_ramp, img_hemi_l=img_hemi_l,
        crop_c_sha=sha(crop_c), crop_o_sha=sha(crop_o), crop_o_sample=crop_o[::29, ::31],
        r_c=r_c, r_o=r_o, cloud_hash=np.array(cloud_hash), cloud_head=np.array(cloud_head),
        placed_hash=sha(placed), placed_n=len(placed), placed_rot_hash=sha(placed_rot),
        placed_rot_n=len(placed_rot))


def small_scene():
    sim = R.RefSim.from_config(SMALL, "", threads=0)
    s0 = sim.state()
    sim.step(SMALL_V, SMALL_STEPS)
    s1 = sim.state()
    d = sim.diag()
    gi = sim.grid_info()
    depth, img = sim.capture(SMALL)
    surf = sim.surface()
    np.savez_compressed(
        os.path.join(OUT, "small_scene.npz"), x0=s0["x"], tag=s0["tag"], mass=s0["mass"],
        vol0=s0["vol0"], x=s1["x"], v=s1["v"], C=s1["C"], F=s1["F"], min_det_f=d["min_det_f"],
        max_speed=d["max_speed"], step_count=d["step_count"], win_lo=gi["lo"], win_hi=gi["hi"],
        depth=depth, image=img, surf_particle=surf["particle"],
        surf_geom=np.array([surf["x0"], surf["y0"], surf["sx"], surf["sy"], surf["z0"]]))


def config3():
    """Config 3 shapes (press then slide), scaled (tests/scenes.py SMALL3)."""
    out = {}
    for shape in SMALL3_SHAPES:
        sim = R.RefSim.from_config(SMALL3, shape, threads=0)
        x0 = sim.state()["x"]
        sim.step(SMALL3_PRESS[1], SMALL3_PRESS[0])
        sim.step(SMALL3_SLIDE[1], SMALL3_SLIDE[0])
        st = sim.state()
        d = sim.diag()
        depth, img = sim.capture(SMALL3, shape)
        rng = np.random.default_rng(3)
        sub = np.sort(rng.choice(sim.n, 2000, replace=False))
        surf = sim.surface()["particle"]
        out[f"{shape}_x0_sha"] = sha(x0)
        out[f"{shape}_subset"] = sub
        out[f"{shape}_x_subset"] = st["x"][sub]
        out[f"{shape}_F_subset"] = st["F"][sub]
        out[f"{shape}_x_surface"] = st["x"][surf]
        out[f"{shape}_min_det_f"] = d["min_det_f"]
        out[f"{shape}_step_count"] = d["step_count"]
        out[f"{shape}_image"] = img
        out[f"{shape}_depth_sample"] = depth[::8, ::8]
    np.savez_compressed(os.path.join(OUT, "config3.npz"), **out)


def config1():
    sim = R.RefSim.from_config(CONFIG1, "", threads=0)
    s0 = sim.state()
    sim.step(CONFIG1_V, CONFIG1_STEPS)
    s1 = sim.state()
    d = sim.diag()
    depth, img = sim.capture(CONFIG1)
    surf = sim.surface()
    rng = np.random.default_rng(1)
    subset = np.sort(rng.choice(sim.n, 4096, replace=False))
    np.savez_compressed(
        os.path.join(OUT, "config1.npz"), n=sim.n, n_elastomer=sim.n_elastomer,
        x0_hash=sha(s0["x"]), subset=subset,
        x_subset=s1["x"][subset], F_subset=s1["F"][subset], v_subset=s1["v"][subset],
        x_surface=s1["x"][surf["particle"]], min_det_f=d["min_det_f"], max_speed=d["max_speed"],
        step_count=d["step_count"], image=img, depth_sha=sha(depth),
        depth_sample=depth[::16, ::16])


def config1_deep():
    sim = R.RefSim.from_config(CONFIG1, "", threads=0)
    s0 = sim.state()
    sim.step(CONFIG1_V, CONFIG1_DEEP_STEPS)
    s1 = sim.state()
    d = sim.diag()
    depth, img = sim.capture(CONFIG1)
    surf = sim.surface()
    rng = np.random.default_rng(2)
    subset = np.sort(rng.choice(sim.n_elastomer, 4096, replace=False))
    np.savez_compressed(
        os.path.join(OUT, "config1_deep.npz"), x0_hash=sha(s0["x"]), subset=subset,
        x0_subset=s0["x"][subset], x_subset=s1["x"][subset],
        F_subset=s1["F"].reshape(-1, 9)[subset], x_surface=s1["x"][surf["particle"]],
        min_det_f=d["min_det_f"], max_speed=d["max_speed"], step_count=d["step_count"],
        image=img, depth_sample=depth[::8, ::8], depth_max=depth.max())


def config5():
    sim = R.RefSim.from_config(CONFIG5, "", threads=0)
    s0 = sim.state()
    sim.step(CONFIG5_PRESS[1], CONFIG5_PRESS[0])
    sim.step(CONFIG5_MOVE[1], CONFIG5_MOVE[0])
    s1 = sim.state()
    d = sim.diag()
    depth, img = sim.capture(CONFIG5)
    surf = sim.surface()
    rng = np.random.default_rng(5)
    subset = np.sort(rng.choice(sim.n, 4096, replace=False))
    np.savez_compressed(
        os.path.join(OUT, "config5.npz"), n=sim.n, n_elastomer=sim.n_elastomer,
        x0_hash=sha(s0["x"]), subset=subset, x0_subset=s0["x"][subset],
        x_subset=s1["x"][subset], F_subset=s1["F"][subset],
        x_surface=s1["x"][surf["particle"]][::7], min_det_f=d["min_det_f"],
        max_speed=d["max_speed"], step_count=d["step_count"], image=img,
        depth_sample=depth[::16, ::16])


def config2b():
    sim = R.RefSim.from_config(CONFIG2B, "", threads=0)
    s0 = sim.state()
    sim.step(CONFIG2B_PRESS[1], CONFIG2B_PRESS[0])
    sim.step(CONFIG2B_SLIDE[1], CONFIG2B_SLIDE[0])
    s1 = sim.state()
    d = sim.diag()
    depth, img = sim.capture(CONFIG2B)
    surf = sim.surface()
    rng = np.random.default_rng(6)
    subset = np.sort(rng.choice(sim.n, 4096, replace=False))
    np.savez_compressed(
        os.path.join(OUT, "config2b.npz"), n=sim.n, n_elastomer=sim.n_elastomer,
        x0_hash=sha(s0["x"]), subset=subset, x_subset=s1["x"][subset],
        F_subset=s1["F"][subset], x_surface=s1["x"][surf["particle"]][::7],
        min_det_f=d["min_det_f"], max_speed=d["max_speed"], step_count=d["step_count"],
        image=img, depth_sample=depth[::16, ::16])


def _checkpoint(sim, cfg, obj, x0, rng_seed, prefix, out):
    """Subset positions / F, the surface, diagnostics, the capture image and
    a depth sample of the reference state (keys prefixed)."""
    st = sim.state()
    d = sim.diag()
    depth, img = sim.capture(cfg, obj)
    surf = sim.surface()["particle"]
    rng = np.random.default_rng(rng_seed)
    sub = np.sort(rng.choice(sim.n_elastomer, 4096, replace=False))
    out[f"{prefix}subset"] = sub
    out[f"{prefix}x0_subset"] = x0[sub]
    out[f"{prefix}x_subset"] = st["x"][sub]
    out[f"{prefix}F_subset"] = st["F"].reshape(-1, 9)[sub]
    out[f"{prefix}v_subset"] = st["v"][sub]
    out[f"{prefix}x_surface"] = st["x"][surf]
    out[f"{prefix}min_det_f"] = d["min_det_f"]
    out[f"{prefix}max_speed"] = d["max_speed"]
    out[f"{prefix}step_count"] = d["step_count"]
    out[f"{prefix}image"] = img
    out[f"{prefix}depth_sample"] = depth[::8, ::8]
    out[f"{prefix}depth_max"] = depth.max()


def config2a():
    """The bench workload (1,214,221 particles) at 100 frames and 600 frames
    (past the gap), 10 substeps per frame as the bench steps it."""
    from tests.scenes import CONFIG2A, CONFIG2A_FRAMES, CONFIG2A_V

    sim = R.RefSim.from_config(CONFIG2A, "", threads=0)
    s0 = sim.state()
    out = {"n": sim.n, "n_elastomer": sim.n_elastomer, "x0_hash": sha(s0["x"]),
           "frames": np.array(CONFIG2A_FRAMES)}
    done = 0
    for f in CONFIG2A_FRAMES:
        sim.step(CONFIG2A_V, 10 * (f - done))
        done = f
        _checkpoint(sim, CONFIG2A, "", s0["x"], 7, f"f{f}_", out)
        print("config2a frame", f, flush=True)
    np.savez_compressed(os.path.join(OUT, "config2a.npz"), **out)


def config4():
    """The first CONFIG4_EPISODES episodes of the config-4 batch (mt19937_64
    pose draws: lateral offset and z-rotation), CONFIG4_FRAMES frames each."""
    from paper_2301_08343_b200 import episodes as E
    from tests.scenes import CONFIG1, CONFIG1_V, CONFIG4_EPISODES, CONFIG4_FRAMES

    out = {"episodes": CONFIG4_EPISODES, "frames": CONFIG4_FRAMES}
    for e in range(CONFIG4_EPISODES):
        ep = E.make_episode(e)
        cfg = E.episode_config(CONFIG1, ep)
        sim = R.RefSim.from_config(cfg, "", ep.offset_x_m, ep.offset_y_m, threads=0)
        s0 = sim.state()
        out[f"e{e}_pose"] = np.array([ep.offset_x_m, ep.offset_y_m, ep.z_rotation_rad, ep.depth_m])
        out[f"e{e}_x0_hash"] = sha(s0["x"])
        sim.step(CONFIG1_V, 10 * CONFIG4_FRAMES)
        _checkpoint(sim, cfg, "", s0["x"], 40 + e, f"e{e}_", out)
        print("config4 episode", e, flush=True)
    np.savez_compressed(os.path.join(OUT, "config4.npz"), **out)


def config3_full():
    """Config 3 at full size: the dot-grid indenter (1e5 points) on the
    default gel and 256^3 grid, pressed to gap + 0.3 mm, then slid +x."""
    from tests.scenes import CONFIG1, CONFIG3_FULL_PRESS, CONFIG3_FULL_SHAPE, CONFIG3_FULL_SLIDE

    shape = CONFIG3_FULL_SHAPE
    sim = R.RefSim.from_config(CONFIG1, shape, threads=0)
    s0 = sim.state()
    out = {"shape": shape, "n": sim.n, "x0_hash": sha(s0["x"])}
    sim.step(CONFIG3_FULL_PRESS[1], CONFIG3_FULL_PRESS[0])
    _checkpoint(sim, CONFIG1, shape, s0["x"], 31, "press_", out)
    print("config3 full: pressed", flush=True)
    sim.step(CONFIG3_FULL_SLIDE[1], CONFIG3_FULL_SLIDE[0])
    _checkpoint(sim, CONFIG1, shape, s0["x"], 32, "slide_", out)
    np.savez_compressed(os.path.join(OUT, "config3_full.npz"), **out)


def grid_post_step():
    """The reference's Grid after mpm::step (SMALL scene, 20 substeps, then
    7 more): active window, mass / momentum / velocity over the window plus
    a 2-node margin (zero outside the window)."""
    sim = R.RefSim.from_config(SMALL, "", threads=0)
    out = {}
    for tag, n in (("a", 20), ("b", 7)):
        sim.step(SMALL_V, n)
        gi = sim.grid_info()
        lo, hi = gi["lo"] - 2, gi["hi"] + 2
        m, mom, vel = sim.grid(lo, hi)
        out.update({f"{tag}_win_lo": gi["lo"], f"{tag}_win_hi": gi["hi"], f"{tag}_lo": lo,
                    f"{tag}_hi": hi, f"{tag}_mass": m, f"{tag}_mom": mom, f"{tag}_vel": vel,
                    f"{tag}_x": sim.state()["x"]})
    np.savez_compressed(os.path.join(OUT, "grid_post_step.npz"), **out)


def acceptance3():
    """SPEC acceptance 3 scene: 60 particles on an 8^3 grid, one step of the
    reference's serial SVD oracle (tests/oracle/reference_mpm.cpp)."""
    rng = np.random.default_rng(3)
    n = 60
    dx = 1e-3
    x = 2.5e-3 + rng.random((n, 3)) * 3e-3
    v = rng.standard_normal((n, 3)) * 0.01
    Cm = rng.standard_normal((n, 3, 3)) * 0.5
    F = np.eye(3) + rng.standard_normal((n, 3, 3)) * 0.02
    tag = np.where(np.arange(n) < 40, 0, 2).astype(np.uint8)
    tag[:5] = 1
    Cm[tag == 2] = 0
    F[tag == 2] = np.eye(3)
    mass = np.where(tag == 2, 2e-6, 1e-6)
    vol0 = np.full(n, 1e-9)
    E, nu, dt = 1.45e5, 0.45, 1e-5
    mu = E / (2 * (1 + nu))
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    st = dict(x=x, v=v, C=Cm, F=F, mass=mass, vol0=vol0, tag=tag)
    ref, _ = R.oracle_step(st, (8, 8, 8), dx, (0, 0, 0), mu, lam, dt, (0, 0, -0.01))
    np.savez_compressed(os.path.join(OUT, "acceptance3.npz"), dx=dx, dt=dt, E=E, nu=nu,
                        vind=np.array([0, 0, -0.01]), x0=x, v0=v, C0=Cm, F0=F, tag=tag,
                        mass=mass, vol0=vol0, x=ref["x"], v=ref["v"], C=ref["C"], F=ref["F"])


def harness():
    import shutil
    import tempfile

    root = tempfile.mkdtemp(prefix="tacchi_dataset_")
    try:
        rows, skipped = R.run_press_dataset(HARNESS, root)
        with open(os.path.join(root, "manifest.csv")) as f:
            manifest = f.read()
        with open(os.path.join(root, "config.json")) as f:
            config_json = f.read()
        arrays = {}
        for line in manifest.splitlines()[1:]:
            f = line.split(",")
            key = f"{f[0]}_p{int(f[1])}_d{int(f[4])}"
            arrays[f"image_{key}"] = R.load_ppm(os.path.join(root, f[8]))
            with open(os.path.join(root, f[9]), "rb") as fh:
                arrays[f"depth_{key}"] = np.frombuffer(fh.read(), dtype=np.uint8)
        # metrics::compare on image pairs of this dataset + a synthetic pair
        keys = sorted(k for k in arrays if k.startswith("image_"))
        pairs = [(keys[0], keys[2]), (keys[3], keys[5]), (keys[1], keys[7]), (keys[4], keys[4])]
        metric_a = np.array([arrays[a] for a, _ in pairs])
        metric_b = np.array([arrays[b] for _, b in pairs])
        rng = np.random.default_rng(11)
        na = rng.integers(0, 256, (37, 53, 3), dtype=np.uint8)
        nb = np.clip(na.astype(int) + rng.integers(-9, 10, na.shape), 0, 255).astype(np.uint8)
        metrics = np.array([R.image_metrics(a, b) for a, b in zip(metric_a, metric_b)])
        noise_metrics = np.array(R.image_metrics(na, nb))
        np.savez_compressed(
            os.path.join(OUT, "harness.npz"), rows=rows, skipped=skipped, manifest=manifest,
            config_json=config_json, metric_pairs=np.array(pairs), metrics=metrics,
            noise_a=na, noise_b=nb, noise_metrics=noise_metrics, **arrays)
    finally:
        shutil.rmtree(root)


def parts_indenter():
    P = PARTS
    pts = R.generate_cloud(P["ind_shape"], P["ind_points"], 11) * P["ind_scale"]
    top = P["lat_origin"][2] + P["lat_dims"][2]
    centre = np.array(P["lat_origin"][:2]) + 0.5 * np.array(P["lat_dims"][:2])
    pts[:, :2] += centre - 0.5 * (pts[:, :2].min(0) + pts[:, :2].max(0))
    pts[:, 2] += top + P["gap"] - pts[:, 2].min()
    return pts


def parts():
    P = PARTS
    ind = parts_indenter()
    sim = R.RefSim.from_parts(P["res"], P["grid_edge"], P["lat_dims"], P["lat_counts"],
                              P["lat_origin"], ind, dt=P["dt"], gravity=P["gravity"],
                              ind_v0=P["ind_v0"], threads=0)
    s0 = sim.state()
    ne = sim.n_elastomer
    rng = np.random.default_rng(21)
    v = s0["v"].copy()
    v[ne:] += rng.uniform(-0.01, 0.01, v[ne:].shape)  # non-uniform indenter velocity
    sim.set_state(v=v)
    sim.step(PARTS_V, PARTS_STEPS)
    s1 = sim.state()
    d = sim.diag()
    surf = sim.surface()
    np.savez_compressed(
        os.path.join(OUT, "parts.npz"), ind=ind, n_elastomer=ne, x0=s0["x"], v0=v,
        mass=s0["mass"], vol0=s0["vol0"], tag=s0["tag"], x=s1["x"], v=s1["v"],
        F=s1["F"].reshape(-1, 9), C=s1["C"].reshape(-1, 9), min_det_f=d["min_det_f"],
        max_speed=d["max_speed"], step_count=d["step_count"], surf_particle=surf["particle"],
        surf_geom=np.array([surf["x0"], surf["y0"], surf["sx"], surf["sy"], surf["z0"]]),
        surf_n=np.array([surf["nx"], surf["ny"]]))


def background_pixels(h=120, w=160):
    yy, xx = np.mgrid[0:h, 0:w]
    return np.stack([(xx * 7 + yy * 3) % 256, (xx * 2 + yy * 11) % 256, (xx * yy) % 256],
                    axis=2).astype(np.uint8)


def background():
    """sim::capture with a render background image (render_params_struct loads
    it, phong_render starts from k_a * background): SMALL scene at creation."""
    import tempfile

    bg = background_pixels()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "bg.png")
        with open(path, "wb") as f:  # binary PPM under the .png name (ref_driver load_png)
            f.write(b"P6\n160 120\n255\n" + bg.tobytes())
        cfg = {**SMALL, "render": {**SMALL["render"], "background_image": path}}
        sim = R.RefSim.from_config(cfg, "", threads=0)
        depth, img = sim.capture(cfg)
    np.savez_compressed(os.path.join(OUT, "background.npz"), background=bg, image=img,
                        depth_sha=sha(depth))


def cloud_files():
    """Point-cloud files as indenters (geo::load_point_cloud, scene_builder.cpp:
    33-50): an ASCII PLY with extra properties and comments, a plain XYZ file
    with blank lines; the placed indenters the reference builds from them and
    its errors for malformed files."""
    import tempfile

    rng = np.random.default_rng(9)
    pts = rng.uniform(-2.0, 2.0, (3000, 3))
    pts = (pts[np.linalg.norm(pts, axis=1) < 2.0] * np.array([1.0, 1.0, 0.5])).tolist()
    ply = ["ply", "format ascii 1.0", "comment test cloud", f"element vertex {len(pts)}",
           "property float nx", "property double x", "property double y", "property double z",
           "element face 0", "property list uchar int vertex_indices", "end_header"]
    ply += [f"0.5 {x!r} {y!r} {z!r}" for x, y, z in pts]
    xyz = ["", "  "] + [f"{x:.9f}\t{y:.9f} {z:.9f}" + ("" if k % 7 else "\n") for k, (x, y, z) in
                         enumerate(pts)]
    texts = {"ply": "\n".join(ply) + "\n", "xyz": "\n".join(xyz) + "\n",
             "binary": "ply\nformat binary_little_endian 1.0\nelement vertex 1\nend_header\n",
             "empty": "\n\n", "short": "1.0 2.0\n"}
    out = {}
    with tempfile.TemporaryDirectory() as d:
        paths = {}
        for k, t in texts.items():
            paths[k] = os.path.join(d, f"cloud_{k}.{'ply' if k in ('ply', 'binary') else 'xyz'}")
            with open(paths[k], "w") as f:
                f.write(t)
        for k in ("ply", "xyz"):
            cfg = {"indenter": {"cloud_path": paths[k], "target_points": 2000}}
            placed = R.placed_indenter(cfg, "")
            out[f"{k}_hash"] = sha(placed)
            out[f"{k}_n"] = len(placed)
            # the object name as a file path (no cloud_path)
            placed2 = R.placed_indenter({"indenter": {"target_points": 2000}}, paths[k])
            out[f"{k}_obj_hash"] = sha(placed2)
            sub = R.placed_indenter({"indenter": {"cloud_path": paths[k], "target_points": 1000,
                                                  "z_rotation_rad": 0.3}}, "")
            out[f"{k}_sub_hash"] = sha(sub)
        for k in ("binary", "empty", "short"):
            try:
                R.placed_indenter({"indenter": {"cloud_path": paths[k]}}, "")
                out[f"{k}_err"] = "none"
            except R.RefError as e:
                out[f"{k}_err"] = f"{e.code}:" + e.msg.replace(paths[k], "<path>")
    np.savez_compressed(os.path.join(OUT, "clouds.npz"), **{f"text_{k}": v for k, v in texts.items()},
                        **out)


def bridge():
    import json
    import shutil
    import tempfile

    root = tempfile.mkdtemp(prefix="tacchi_bridge_")
    try:
        sdir = os.path.join(root, "s0")
        replies = R.bridge_run(bridge_script(sdir), session_root=root)
        bad = R.bridge_run([{"type": "init", "config": c} for c in BAD_CONFIGS] + [{"type": "end"}],
                           session_root=root)
        with open(os.path.join(sdir, "steps.jsonl")) as f:
            steps_jsonl = f.read().replace(sdir, "<dir>")
        arrays = {}
        for r in replies:
            if r.get("type") == "reply" and r["image"]:
                k = r["step"]
                with open(r["depth_map"], "rb") as f:
                    arrays[f"depth_{k}"] = np.frombuffer(f.read(), dtype=np.uint8)
                arrays[f"image_{k}"] = R.load_ppm(r["image"])
        np.savez_compressed(
            os.path.join(OUT, "bridge.npz"),
            replies=json.dumps(replies).replace(sdir, "<dir>"), bad_configs=json.dumps(bad),
            steps_jsonl=steps_jsonl, **arrays)
    finally:
        shutil.rmtree(root)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kat", "small", "config1", "config3", "config5", "config2b", "acceptance3", "bridge", "harness", "parts", "background", "clouds"]
    if "config2b" in which:
        config2b()
    if "grid_post_step" in which:
        grid_post_step()
    if "config2a" in which:
        config2a()
    if "config4" in which:
        config4()
    if "config3_full" in which:
        config3_full()
    if "acceptance3" in which:
        acceptance3()
    if "config5" in which:
        config5()
    if "config1_deep" in which:
        config1_deep()
    if "bridge" in which:
        bridge()
    if "harness" in which:
        harness()
    if "parts" in which:
        parts()
    if "background" in which:
        background()
    if "clouds" in which:
        cloud_files()
    if "kat" in which:
        kat()
    if "small" in which:
        small_scene()
    if "config1" in which:
        config1()
    if "config3" in which:
        config3()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
