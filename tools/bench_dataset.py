"""Dataset-harness throughput: the paper's press protocol
(one object, 3 x 3 press grid, 11 depth levels 0..1 mm) on the config-1 scene,
run through tg_run_press_dataset on the GPU, next to the reference harness's
cost on the host, extrapolated from a timed sample of its own per-substep
stepping (the full reference run takes hours).

    python tools/bench_dataset.py [--speed MM_S] [--out DIR] [--ref-substeps N]

Prints one JSON line.
"""
import argparse
import json
import math
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG1  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--speed", type=float, default=50.0, help="press speed, mm/s")
    ap.add_argument("--out", default="")
    ap.add_argument("--ref-substeps", type=int, default=20)
    args = ap.parse_args()
    cfg = {**CONFIG1, "time": {"dt_s": 2e-6, "press_speed_mm_s": args.speed},
           "objects": ["sphere"]}
    out = args.out or tempfile.mkdtemp(prefix="tacchi_ds_")
    t0 = time.perf_counter()
    rows, skipped = tb.dataset.run_press_dataset(cfg, out)
    gpu_s = time.perf_counter() - t0
    per_step = args.speed * 1e-3 * 2e-6
    substeps = round((0.1e-3 + 1.0e-3) / per_step)  # gap + deepest level
    positions = 9
    line = {"workload": f"press dataset: sphere, 3x3 positions, 11 depths, config-1 scene, "
                        f"press {args.speed} mm/s ({substeps} substeps per position)",
            "rows": rows, "positions": positions, "substeps_per_position": substeps,
            "gpu_wall_s": gpu_s, "gpu_substeps_per_s": positions * substeps / gpu_s}
    try:
        from oracle import refpy as R
        if R.available():
            import os as _os
            sim = R.RefSim.from_config(cfg, "sphere", threads=_os.cpu_count() or 1)
            sim.step((0, 0, -args.speed * 1e-3), 2)
            t1 = time.perf_counter()
            sim.step((0, 0, -args.speed * 1e-3), args.ref_substeps)
            ref_per = (time.perf_counter() - t1) / args.ref_substeps
            line["reference"] = {
                "kind": "reference (oracle/_ref), harness cost extrapolated from a timed sample",
                "threads": _os.cpu_count(), "sample_substeps": args.ref_substeps,
                "s_per_substep": ref_per,
                "extrapolated_wall_s": ref_per * substeps * positions}
            line["speedup_extrapolated"] = line["reference"]["extrapolated_wall_s"] / gpu_s
    except Exception as e:  # reference library absent on this machine
        line["reference"] = {"unavailable": str(e)[:200]}
    print(json.dumps(line))
    if not args.out:
        shutil.rmtree(out, ignore_errors=True)


if __name__ == "__main__":
    main()
