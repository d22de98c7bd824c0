"""Dataset-harness throughput: the paper's press protocol
(one object, 3 x 3 press grid, 11 depth levels 0..1 mm) on the config-1 scene,
run through tg_run_press_dataset on the GPU, next to the reference harness's
cost on the host extrapolated from its per-substep time (pass it with
--ref-s-per-substep; DESIGN.md §9.2 used 12.8 ms measured on the GPU box's
16 host threads).

    python tools/bench_dataset.py [--speed MM_S] [--out DIR] [--ref-s-per-substep S]

Prints one JSON line.
"""
import argparse
import json
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
    ap.add_argument("--ref-s-per-substep", type=float, default=0.0,
                    help="reference seconds per config-1 substep, for the extrapolation")
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
    if args.ref_s_per_substep > 0:
        # the reference's per-substep time on config 1 measured separately
        # (only tests/, smoke() and bench.py may run the reference library)
        line["reference_extrapolated_wall_s"] = args.ref_s_per_substep * substeps * positions
        line["speedup_extrapolated"] = line["reference_extrapolated_wall_s"] / gpu_s
    print(json.dumps(line))
    if not args.out:
        shutil.rmtree(out, ignore_errors=True)


if __name__ == "__main__":
    main()
