"""Long-horizon parity against the reference on the full-length protocols of
SURVEY.md §8(d) (the tests run the same scenes over shorter slices):

  config1-deep : config 1, press at (0, 0, -0.01) m/s for 3000 frames
                 (30,000 substeps: 0.6 mm travel, 0.5 mm into the gel)
  config3-<s>  : config 1 gel, shape s (cylinder, cylinder_shell, wave1, dots),
                 press until the travel is gap + 0.3 mm (2000 frames), then
                 slide at (+0.005, 0, 0) m/s for 200 frames
  config5      : 40 x 40 mm gel on 512^3, press 2000 frames, then move at
                 (0.01, 0, 0) m/s for 500 frames
  config2a     : config 1 with the 1e6-point sphere, press 2000 frames
  config2b     : 171 x 171 x 35 gel (0.91 grid cells spacing: duplicate base
                 cells), press 2000 frames, then slide 200 frames
  config4-<e>  : config 1 with episode e's config-4 draw (lateral offset,
                 z-rotation; a non-symmetric "dots" indenter so the rotation
                 matters), pressed 700 frames (0.14 mm of travel, 0.04 mm into the gel)

The reference (oracle/_ref, all host threads) and the CUDA path run the same
step calls (10 substeps per frame); at every checkpoint both are captured and
compared. One JSON line per checkpoint:

    python tools/long_parity.py [case ...] > gpurun_out/long_parity.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from oracle import refpy  # noqa: E402  (checker only)
from tests.scenes import CONFIG1, CONFIG2A  # noqa: E402

CONFIG5_FULL = {"elastomer": {"size_mm": [40, 40, 4], "particle_counts": [201, 201, 21]},
                "grid": {"nodes_per_axis": [512, 512, 512], "edge_mm": 66.0},
                "time": {"dt_s": 2e-6}}
CONFIG2B_FULL = {"elastomer": {"particle_counts": [171, 171, 35]}, "time": {"dt_s": 2e-6}}
PRESS = (0.0, 0.0, -0.01)


def cases():
    yield "config1-deep", CONFIG1, "", [(3000, PRESS)], 500
    for shape in ("cylinder", "cylinder_shell", "wave1", "dots"):
        yield f"config3-{shape}", CONFIG1, shape, [(2000, PRESS), (200, (0.005, 0.0, 0.0))], 550
    yield "config5", CONFIG5_FULL, "", [(2000, PRESS), (500, (0.01, 0.0, 0.0))], 500
    yield "config2a", CONFIG2A, "", [(2000, PRESS)], 500
    from paper_2301_08343_b200 import episodes
    for e in range(8):
        ep = episodes.make_episode(e)
        cfg = episodes.episode_config(CONFIG1, ep)
        yield f"config4-{e}", cfg, ("dots", ep.offset_x_m, ep.offset_y_m), [(700, PRESS)], 700
    yield "config2b", CONFIG2B_FULL, "", [(2000, PRESS), (200, (0.005, 0.0, 0.0))], 550


def main(selected):
    threads = os.cpu_count() or 1
    div = int(os.environ.get("LP_DIV", "1"))  # shrink every phase (smoke runs)
    for name, cfg, obj, plan, every in cases():
        if selected and name not in selected and name.split("-")[0] not in selected:
            continue
        plan = [(max(f // div, 1), v) for f, v in plan]
        every = max(every // div, 1)
        t0 = time.perf_counter()
        ox = oy = 0.0
        if isinstance(obj, tuple):
            obj, ox, oy = obj
        ref = refpy.RefSim.from_config(cfg, obj, ox, oy, threads=threads)
        gpu = tb.sim.build_sim(cfg, obj, ox, oy)
        x0 = ref.state()["x"]
        assert np.array_equal(gpu.positions(), x0), "setup differs"
        frame = 0
        for frames, v in plan:
            for _ in range(frames):
                ref.step(v, 10)
                tb.mpm.step(gpu, v, 10)
                frame += 1
                if frame % every and not (frame == sum(f for f, _ in plan)):
                    continue
                rs = ref.state()
                x = gpu.positions()
                disp = float(np.abs(rs["x"] - x0).max())
                err = float(np.abs(x - rs["x"]).max())
                rd, ri = ref.capture(cfg, obj)
                gd, gi = tb.sim.capture(gpu, cfg, obj)
                F = gpu.state()["F"]
                print(json.dumps({
                    "case": name, "frame": frame, "particles": int(ref.n),
                    "disp_m": disp, "x_err_m": err, "x_err_rel_disp": err / disp,
                    "x_err_rel_pos": err / float(np.abs(rs["x"]).max()),
                    "F_err": float(np.abs(F - rs["F"]).max()),
                    "depth_err_m": float(np.abs(gd - rd).max()),
                    "max_depth_m": float(rd.max()),
                    "image_err_lsb": int(np.abs(gi.astype(int) - ri).max()),
                    "step_count": [int(gpu.step_count), int(ref.diag()["step_count"])],
                    "elapsed_s": round(time.perf_counter() - t0, 1)}), flush=True)
        del ref, gpu


if __name__ == "__main__":
    main(sys.argv[1:])
