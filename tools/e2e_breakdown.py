"""Where an end-to-end frame goes: tg_step_capture on config 2a with no
read-back, RGB only, depth only, both, and mpm::step alone (ms per frame,
two repetitions). DESIGN.md §8.

    python tools/e2e_breakdown.py
"""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2301_08343_b200 as tb
from tests.scenes import CONFIG2A, CONFIG2A_V, SUBSTEPS_PER_FRAME
s = tb.sim.build_sim(CONFIG2A)
rp = tb.render_params(CONFIG2A, "")
v = np.array(CONFIG2A_V)
def run(k, **kw):
    for _ in range(5): tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, zero_copy=True, **kw)
    t0 = time.perf_counter()
    for _ in range(k): tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, zero_copy=True, **kw)
    return (time.perf_counter() - t0) / k * 1e3
out = {}
for rep in range(2):
    out[f"none{rep}"] = run(200, want_depth=False, want_image=False)
    out[f"rgb{rep}"] = run(200, want_depth=False, want_image=True)
    out[f"depth{rep}"] = run(200, want_depth=True, want_image=False)
    out[f"both{rep}"] = run(200)
    t0 = time.perf_counter()
    for _ in range(200): tb.mpm.step(s, v, SUBSTEPS_PER_FRAME)
    out[f"step_only{rep}"] = (time.perf_counter() - t0) / 200 * 1e3
print(json.dumps({k: round(x, 4) for k, x in out.items()}))
