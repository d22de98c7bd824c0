"""Hash of a deterministic-mode config-2a episode (positions, v, C, F after
`--frames` frames of 10 substeps): the same hash from two libraries
(TACCHI_LIB) shows a change left deterministic mode's results bit-identical.

    python tools/det_hash.py [--frames 30] [--cfg config2a|config2b]
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG2A, CONFIG2A_V, CONFIG2B, CONFIG2B_PRESS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--cfg", default="config2a")
    a = ap.parse_args()
    cfg, v = {"config2a": (CONFIG2A, CONFIG2A_V), "config2b": (CONFIG2B, CONFIG2B_PRESS[1])}[a.cfg]
    s = tb.sim.build_sim({**cfg, "deterministic": True})
    for _ in range(a.frames):
        tb.mpm.step(s, v, 10)
    st = s.state()
    h = hashlib.sha256()
    for k in sorted(st):
        h.update(st[k].tobytes())
    print(json.dumps({"cfg": a.cfg, "frames": a.frames, "sha256": h.hexdigest(),
                      "lib": os.environ.get("TACCHI_LIB", "in-tree")}))


if __name__ == "__main__":
    main()
