"""Episode setup: indenter cloud generation + placement on
the host restatement vs on the GPU, for the 1e6-point source clouds of the
configs (sphere: config 1/2a; dots: config 3), and a config-4 batch build.

    python tools/bench_setup.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from paper_2301_08343_b200 import episodes as E  # noqa: E402
from tests.scenes import CONFIG1  # noqa: E402


def timed(f, reps=3):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        best = min(best, time.perf_counter() - t0)
    return best, out


def main():
    tb.geo.generate_shape_cloud_device("sphere", 1000, 1)  # context + module load
    for shape in ("sphere", "dots", "wave1"):
        th, h = timed(lambda: tb.geo.generate_shape_cloud(shape, 1000000, 20230115))
        td, d = timed(lambda: tb.geo.generate_shape_cloud_device(shape, 1000000, 20230115))
        print(json.dumps({"shape": shape, "points": 1000000, "host_s": th, "device_s": td,
                          "identical": bool(np.array_equal(h, d))}), flush=True)
    poses = [[E.make_episode(e).offset_x_m, E.make_episode(e).offset_y_m,
              E.make_episode(e).z_rotation_rad] for e in range(64)]
    for mode in ("device", "host"):
        if mode == "host":
            os.environ["TACCHI_HOST_SETUP"] = "1"
        t0 = time.perf_counter()
        sims = tb.sim.build_episodes(CONFIG1, "", poses)
        dt = time.perf_counter() - t0
        print(json.dumps({"build_episodes": len(sims), "setup": mode, "s": dt,
                          "s_per_episode": dt / len(sims)}), flush=True)
        del sims
        t0 = time.perf_counter()
        s = tb.sim.build_sim(CONFIG1)
        print(json.dumps({"build_sim": "config1", "setup": mode,
                          "s": time.perf_counter() - t0}), flush=True)
        del s
    os.environ.pop("TACCHI_HOST_SETUP", None)


if __name__ == "__main__":
    main()
