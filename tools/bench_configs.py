"""Throughput of the step + capture frame on each BASELINE.json config shape
(one episode per GPU): config 1 (default gel, sphere 1e5), config 2a (sphere
1e6), config 2b (171 x 171 x 35 gel), config 3 (default gel, cylinder / ring / wave / dot-grid indenters,
1e5 points), config 5 (large-area gel on 512^3). Prints one JSON line each.

    python tools/bench_configs.py [--frames F]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG1, CONFIG2A, CONFIG2B, CONFIG5, SUBSTEPS_PER_FRAME  # noqa: E402

CASES = [
    ("config1", CONFIG1, "", (0.0, 0.0, -0.01)),
    ("config2a", CONFIG2A, "", (0.0, 0.0, -0.01)),
    ("config2b", CONFIG2B, "", (0.0, 0.0, -0.01)),
    ("config3-cylinder", CONFIG1, "cylinder", (0.0, 0.0, -0.01)),
    ("config3-ring", CONFIG1, "cylinder_shell", (0.0, 0.0, -0.01)),
    ("config3-wave", CONFIG1, "wave1", (0.0, 0.0, -0.01)),
    ("config3-dots", CONFIG1, "dots", (0.0, 0.0, -0.01)),
    ("config5", CONFIG5, "", (0.01, 0.0, -0.01)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=50)
    args = ap.parse_args()
    for name, cfg, obj, v in CASES:
        s = tb.sim.build_sim(cfg, obj)
        rp = tb.render_params(cfg, obj)
        for _ in range(3):
            tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, want_depth=False,
                                want_image=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.frames):
            tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, want_depth=False,
                                want_image=False)
        dt = time.perf_counter() - t0
        print(json.dumps({"config": name, "particles": s.n, "elastomer": s.elastomer_count,
                          "frames_per_s": args.frames / dt,
                          "particle_substeps_per_s": s.n * SUBSTEPS_PER_FRAME * args.frames / dt,
                          "elastomer_particle_substeps_per_s":
                              s.elastomer_count * SUBSTEPS_PER_FRAME * args.frames / dt}),
              flush=True)
        del s


if __name__ == "__main__":
    main()
