"""SPEC acceptance 8 (the paper's Fig. 6 particle-density effect) on the B200
path: the config-1 sphere at 1e4 / 1e5 / 1e6 indenter points (Tacchi_1 / 10 /
100) pressed to the same depth; prints the image metrics of each against the
1e6 run. The ordering MAE(1e4 vs 1e6) > MAE(1e5 vs 1e6) > 0 is asserted by
tests/test_spec_kat.py.

    python tools/density_ordering.py [--depth-mm D] [--speed MM_S]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_08343_b200 as tb  # noqa: E402


def press_images(depth_mm=1.0, speed_mm_s=50.0, points=(10000, 100000, 1000000)):
    dt = 2e-6
    out = {}
    for n in points:
        cfg = {"time": {"dt_s": dt}, "indenter": {"target_points": n}}
        s = tb.sim.build_sim(cfg)
        steps = round((0.1 + depth_mm) * 1e-3 / (speed_mm_s * 1e-3 * dt))
        rp = tb.render_params(cfg, "")
        done = 0
        while steps - done > 200:
            tb.mpm.step(s, (0, 0, -speed_mm_s * 1e-3), 200)
            done += 200
        _, img = tb.sim.step_capture(s, (0, 0, -speed_mm_s * 1e-3), steps - done, params=rp)
        out[n] = img
        del s
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth-mm", type=float, default=1.0)
    ap.add_argument("--speed", type=float, default=50.0)
    args = ap.parse_args()
    imgs = press_images(args.depth_mm, args.speed)
    ref = imgs[1000000]
    for n in (10000, 100000):
        ssim, psnr, mae = tb.metrics.compare(imgs[n], ref)
        print(json.dumps({"points": n, "vs": 1000000, "ssim": ssim, "psnr_db": psnr,
                          "mae_pct": mae}))


if __name__ == "__main__":
    main()
