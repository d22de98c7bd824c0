import sys, numpy as np
sys.path.insert(0, ".")
import paper_2301_08343_b200 as tb
from tests.scenes import SMALL, SMALL_V
g = np.load("tests/golden/grid_post_step.npz")
for det in (False, True):
    s = tb.sim.build_sim({**SMALL, "deterministic": det})
    s.set_keep_grid(True)
    for tag, n in (("a", 20), ("b", 7)):
        tb.mpm.step(s, SMALL_V, n)
        m, mom, vel = s.grid(g[f"{tag}_lo"], g[f"{tag}_hi"])
        gm = g[f"{tag}_mass"]
        d = m - gm
        bad = np.abs(d) > 1e-12 * gm.max()
        print(det, tag, "bad", bad.sum(), "sum d", d.sum(), "sum gm", gm.sum(), "max|d|", np.abs(d).max(),
              "d>0", (d[bad] > 0).sum(), "d<0", (d[bad] < 0).sum(), "stats", s.stats())
