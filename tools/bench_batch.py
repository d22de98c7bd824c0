"""Batched independent episodes on one GPU:
K config-1 episodes with the config-4 pose draws (episodes.make_episode),
stepped and captured together with tg_step_capture_many (every handle's
substep graph and capture submitted before any wait), every frame. Prints one JSON line per K.

    python tools/bench_batch.py [K ...] [--frames F] [--warmup W]

Not the bench.py contract line (that is config 2a, BASELINE.json metric);
this measures how the per-GPU throughput of config 4 scales with the batch.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from paper_2301_08343_b200 import episodes  # noqa: E402
from tests.scenes import CONFIG1, CONFIG1_V, SUBSTEPS_PER_FRAME  # noqa: E402


def run(k, frames, warmup):
    sims, eps = [], []
    for e in range(k):
        ep = episodes.make_episode(e)
        sims.append(tb.sim.build_sim(episodes.episode_config(CONFIG1, ep), "", ep.offset_x_m,
                                     ep.offset_y_m))
        eps.append(ep)
    rp = tb.render_params(CONFIG1, "")
    v = np.tile(np.asarray(CONFIG1_V, dtype=np.float64), (k, 1))

    def frame():
        tb.sim.step_capture_many(sims, v, SUBSTEPS_PER_FRAME, rp, want_depth=False,
                                 want_image=False)

    for _ in range(warmup):
        frame()
    torch.cuda.synchronize()
    t0 = time.perf_counter()  # the handles run on their own streams: wall clock
    for _ in range(frames):
        frame()
    for s in sims:
        s.sync()
    ms = (time.perf_counter() - t0) * 1e3
    n = sims[0].n
    units = float(n) * k * SUBSTEPS_PER_FRAME * frames
    return {"workload": f"config4-style: {k} x config1 ({n} particles each), 10 substeps + capture "
                        "per frame, tg_step_capture_many",
            "episodes": k, "frames": frames, "ms": ms,
            "particle_substeps_per_s": units / (ms * 1e-3),
            "episode_frames_per_s": k * frames / (ms * 1e-3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("k", nargs="*", type=int, default=[1, 2, 4, 8, 16])
    ap.add_argument("--frames", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    for k in args.k:
        print(json.dumps(run(k, args.frames, args.warmup)), flush=True)


if __name__ == "__main__":
    main()
