"""Scene definitions shared by the tests, the golden generator and bench.py.

All are SceneConfig JSON overrides of the reference's default_config()
(scene_config.cpp:118-122). Every config pins a stable dt (SURVEY.md §0
finding 4: the shipped dt = 1e-4 diverges).
"""

# Small CPU-oracle-sized scene: 31x31x7 gel (6 x 6 x 1.2 mm, 0.2 mm spacing)
# + 3000-point sphere2 indenter on a 64^3 grid of 12 mm edge.
SMALL = {
    "elastomer": {"size_mm": [6, 6, 1.2], "particle_counts": [31, 31, 7]},
    "grid": {"nodes_per_axis": [64, 64, 64], "edge_mm": 12.0},
    "time": {"dt_s": 2e-6},
    "render": {"image_width": 160, "image_height": 120},
    "indenter": {"generated_shape": "sphere2", "source_points": 20000, "target_points": 3000,
                 "gap_mm": 0.02},
}
SMALL_STEPS = 200
SMALL_V = (0.0, 0.0, -0.05)

# Config 1 (BASELINE.json configs[0]): default gel 101x101x21, sphere 1e6 ->
# 1e5 points, 256^3 / 33 mm, dt 2e-6, press velocity (0, 0, -0.01) m/s.
CONFIG1 = {"time": {"dt_s": 2e-6}}
CONFIG1_STEPS = 1000  # 100 frames (SURVEY §8(d) CI parity)
CONFIG1_V = (0.0, 0.0, -0.01)
# 1000 frames: the indenter crosses the 0.1 mm gap after 500 and presses
# 0.1 mm into the gel by the end (contact, the part 100 frames never reach).
CONFIG1_DEEP_STEPS = 10000

# Config 2a (BASELINE.json configs[1]): same gel, sphere at the reference's
# finest indenter density (1e6 points, no subsampling) -> 1,214,221 particles.
CONFIG2A = {"time": {"dt_s": 2e-6}, "indenter": {"target_points": 1000000}}
CONFIG2A_V = (0.0, 0.0, -0.01)

# Config 2b (BASELINE.json configs[2]): isotropic 0.1176 mm gel spacing,
# 171 x 171 x 35 = 1,023,435 gel particles + sphere 1e5 = 1,123,435. The gel
# spacing is 0.91 grid cells, so about a quarter of the gel particles share a
# base cell with a neighbour (the scatter's duplicate path). Parity slice:
# gap 2 um, press at 0.3 m/s, then slide while pressed.
CONFIG2B = {"elastomer": {"particle_counts": [171, 171, 35]}, "time": {"dt_s": 2e-6},
            "indenter": {"gap_mm": 0.002}}
CONFIG2B_PRESS = (40, (0.0, 0.0, -0.3))
CONFIG2B_SLIDE = (20, (0.2, -0.1, 0.0))

SUBSTEPS_PER_FRAME = 10  # scene_config.hpp:36, session.cpp:86

# Config 2a parity (the bench workload): 100 frames (SURVEY §8(d) CI length)
# and a checkpoint at 600 frames, past the gap (the indenter crosses the
# 0.1 mm gap after 500 frames).
CONFIG2A_FRAMES = (100, 600)

# Config 4 parity: the first episodes of the 1024-episode batch (config-1
# geometry, mt19937_64 pose draws, paper_2301_08343_b200/episodes.py), each
# stepped for the throughput cap of 200 frames at the press velocity.
CONFIG4_EPISODES = 4
CONFIG4_FRAMES = 200

# Config 3 at full size (default gel 101x101x21, 1e5-point dot-grid
# indenter, 256^3): pressed until the commanded travel is gap + 0.3 mm
# (20,000 substeps at 0.01 m/s), then slid +x at 5 mm/s for 200 frames
# (SURVEY §8(d)).
CONFIG3_FULL_SHAPE = "dots"
CONFIG3_FULL_PRESS = (20000, (0.0, 0.0, -0.01))
CONFIG3_FULL_SLIDE = (2000, (0.005, 0.0, 0.0))

# Config 5 (BASELINE.json configs[4]): large-area gel 40 x 40 x 4 mm at the
# same 0.2 mm spacing (201 x 201 x 21 = 848,421 gel particles) + sphere 1e5,
# 512^3 grid of 66 mm edge (same dx as config 1). The parity slice is short
# enough for the CPU reference (80 substeps, ~30 s): gap 2 um, press at
# 0.3 m/s, then move the indenter laterally while pressed.
CONFIG5 = {"elastomer": {"size_mm": [40, 40, 4], "particle_counts": [201, 201, 21]},
           "grid": {"nodes_per_axis": [512, 512, 512], "edge_mm": 66.0},
           "time": {"dt_s": 2e-6}, "indenter": {"gap_mm": 0.002}}
CONFIG5_PRESS = (50, (0.0, 0.0, -0.3))
CONFIG5_MOVE = (30, (0.3, 0.1, 0.0))

# Config 3 (textured / defect indenters, press then slide), scaled so the
# reference finishes in seconds: 10 x 10 x 1.2 mm gel on a 96^3 / 16 mm grid,
# 4000-point indenters; press 150 substeps at 0.05 m/s, then slide +x.
SMALL3 = {
    "elastomer": {"size_mm": [10, 10, 1.2], "particle_counts": [51, 51, 7]},
    "grid": {"nodes_per_axis": [96, 96, 96], "edge_mm": 16.0},
    "time": {"dt_s": 2e-6},
    "render": {"image_width": 320, "image_height": 240},
    "indenter": {"source_points": 40000, "target_points": 4000, "gap_mm": 0.005},
}
SMALL3_SHAPES = ["cylinder", "cylinder_shell", "wave1", "dots"]
SMALL3_PRESS = (150, (0.0, 0.0, -0.05))
SMALL3_SLIDE = (150, (0.05, 0.0, 0.0))


def render_inputs():
    """Synthetic depth maps for the render KATs: a
    hemispherical dimple, a ramp, and a 713x713 source for crop_align."""
    import numpy as np

    H, W = 480, 640
    r = 2.8125e-5
    yy, xx = np.mgrid[0:H, 0:W]
    rr = np.hypot(xx - 301.3, yy - 233.7) * r
    rad = 2.0e-3
    hemi = np.where(rr < rad, np.sqrt(np.maximum(rad**2 - rr**2, 0.0)) * 0.25, 0.0)
    ramp = 1e-5 * (xx * 0.37 - yy * 0.21) * r * 40
    sy, sx = np.mgrid[0:713, 0:713]
    src = np.sin(sx * 0.031) * np.cos(sy * 0.017) * 1e-4 + (sx - sy) * 1e-8
    return r, hemi, ramp, src


LIGHT_CFG = {"lights": [{"direction": [0.3, -0.2, -1.0], "diffuse_rgb": [0.9, 0.7, 0.5],
                         "specular_rgb": [0.4, 0.4, 0.4]}],
             "render": {"ambient_k": 0.8, "diffuse_k": 0.6, "specular_k": 0.5, "shininess": 12.0,
                        "ambient_rgb": [0.2, 0.25, 0.3], "view_dir": [0.05, 0.0, -1.0]}}

SHAPES = ["cone", "cross_lines", "curved_surface", "cylinder", "cylinder_shell", "cylinder_side",
          "dot_in", "dots", "flat_slab", "hexagon", "line", "moon", "pacman", "parallel_lines",
          "prism", "random", "sphere", "sphere2", "torus", "triangle", "wave1"]

PLACED_ROT = ({"indenter": {"z_rotation_rad": 0.6, "target_points": 20000}}, "dots", 0.0007,
              -0.0004)


def sha(a) -> str:
    import hashlib

    import numpy as np

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# Bridge session script (§8 row f1, protocol "tacchi/1", server.cpp:49-113):
# velocity and position commands, a non-monotonic sim_time, an image request
# before and at the terminal depth, a frozen step after it, protocol errors.
# SMALL scene, 10 substeps per control step (2e-5 s), gap 0.02 mm.
BRIDGE_MAX_DEPTH = 2.0e-5


def bridge_script(session_dir: str):
    return [
        {"type": "step", "vector": [0, 0, 0]},
        "not json",
        {"type": "init", "config": SMALL, "max_depth_m": BRIDGE_MAX_DEPTH,
         "session_dir": session_dir},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0, -0.5], "sim_time": 0.0,
         "request_image": True},
        {"type": "step", "mode": "position", "vector": [0.0, 0.0, -2.5e-5], "sim_time": 2e-5},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0, -0.5], "sim_time": 1e-5},
        {"type": "step", "mode": "sideways", "vector": [0.0, 0.0, -0.5]},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0]},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0, -0.5], "sim_time": 4e-5,
         "request_image": True},
        {"type": "step", "mode": "position", "vector": [0.0, 0.0, -9e-5], "request_image": True},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0, -0.5], "sim_time": 6e-5},
        {"type": "step", "mode": "velocity", "vector": [0.0, 0.0, float("nan")]},
        {"type": "end"},
    ]


# SceneConfig::validate failures (scene_config.cpp:83-116) reported by init.
BAD_CONFIGS = [
    {"elastomer": {"poisson_ratio": 0.5}},
    {"elastomer": {"youngs_modulus_pa": 0.0}},
    {"elastomer": {"density_kg_m3": -1.0}},
    {"elastomer": {"particle_counts": [1, 5, 5]}},
    {"grid": {"nodes_per_axis": [7, 64, 64]}},
    {"time": {"substeps_per_control_step": 0}},
    {"indenter": {"generated_shape": "no_such_shape"}},
    {"press_grid": {"depths_mm": []}},
    {"press_grid": {"positions_x": 0}},
    {"time": {"dt_s": 0.0}},
    {"lights": []},
    {"render": {"image_width": 1}},
    {"elastomer": {"fixed_bottom_layers": 21}},
]


# Dataset harness (§8 row f2, harness.cpp:159-245) on the SMALL scene: two
# objects x 2 press positions x 3 depth levels, press at 50 mm/s (1e-7 m per
# substep -> captures at substeps 200, 250, 300), a crop alignment for one
# object.
HARNESS = {**SMALL,
           "time": {"dt_s": 2e-6, "press_speed_mm_s": 50.0},
           "objects": ["sphere2", "dots"],
           "press_grid": {"positions_x": 2, "positions_y": 1, "step_mm": 0.5,
                          "depths_mm": [0.0, 0.005, 0.01]},
           "alignment": {"dots": {"offset_px": [3.0, -2.0], "scale": 1.05}}}


# init_scene from explicit parts (mpm::init_scene, scene.cpp:28-87) with the
# options the config path does not exercise: gravity, a moving indenter at
# creation and a non-uniform indenter velocity (set after creation), on a
# non-cubic-count lattice. Torus indenter 1 um above a 4 x 4 x 1 mm gel.
PARTS = dict(res=(48, 48, 48), grid_edge=0.0096, lat_dims=(0.004, 0.004, 0.001),
             lat_counts=(21, 19, 6), lat_origin=(0.0028, 0.0028, 0.0038), dt=2e-6,
             gravity=(0.0, 0.0, -9.81), ind_v0=(0.0, 0.0, -0.02), ind_shape="torus",
             ind_points=2500, ind_scale=0.5, gap=1e-6)
PARTS_STEPS = 120
PARTS_V = (0.02, -0.01, -0.1)
