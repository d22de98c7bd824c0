"""Hash of a deterministic-mode config-2a episode (positions, v, C, F after
`--frames` frames of 10 substeps): the same hash from two libraries
(TACCHI_LIB) shows a change left deterministic mode's results bit-identical.

    python tools/det_hash.py [--frames 30] [--cfg config2a|config2b|config3|config5]
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_08343_b200 as tb  # noqa: E402
from tests import scenes as S  # noqa: E402

# (config, object, [(substeps, indenter velocity), ...]); --frames scales the
# first phase of 2a / 2b (frames of 10 substeps)
SCENES = {
    "config2a": (S.CONFIG2A, "", None, S.CONFIG2A_V),
    "config2b": (S.CONFIG2B, "", None, S.CONFIG2B_PRESS[1]),
    "config3": (S.CONFIG1, S.CONFIG3_FULL_SHAPE, [S.CONFIG3_FULL_PRESS, S.CONFIG3_FULL_SLIDE], None),
    "config5": (S.CONFIG5, "", [S.CONFIG5_PRESS, S.CONFIG5_MOVE], None),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--cfg", default="config2a", choices=sorted(SCENES))
    a = ap.parse_args()
    cfg, obj, phases, v = SCENES[a.cfg]
    phases = phases or [(10 * a.frames, v)]
    s = tb.sim.build_sim({**cfg, "deterministic": True}, obj)
    for n, vel in phases:
        tb.mpm.step(s, vel, n)
    st = s.state()
    h = hashlib.sha256()
    for k in sorted(st):
        h.update(st[k].tobytes())
    print(json.dumps({"cfg": a.cfg, "substeps": sum(n for n, _ in phases), "sha256": h.hexdigest(),
                      "lib": os.environ.get("TACCHI_LIB", "in-tree")}))


if __name__ == "__main__":
    main()
