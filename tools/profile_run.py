"""Short driver for ncu: build a scene, warm up, run a few frames.

    python tools/profile_run.py [config2a|config1] [frames]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG1, CONFIG2A, CONFIG2A_V, SUBSTEPS_PER_FRAME  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2a"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
# the bench's accumulation mode (fp64); "-det" selects the deterministic mode
cfg = dict(CONFIG2A if name.startswith("config2a") else CONFIG1)
cfg["deterministic"] = name.endswith("-det")
s = tb.sim.build_sim(cfg)
rp = tb.render_params(cfg, "")
v = np.array(CONFIG2A_V)
for _ in range(frames):
    tb.mpm.step(s, v, SUBSTEPS_PER_FRAME)
    tb.sim.capture(s, params=rp, want_depth=False, want_image=False)
s.sync()
print("ok", s.n, s.step_count, s.kernel_launches)
