"""Fork vs fused walks: positions after a step and the post-step grid, in
deterministic mode (both must be byte-identical) — one process per mode."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, hashlib, json
sys.path.insert(0, %r)
import numpy as np
import paper_2301_08343_b200 as tb
from tests.scenes import SMALL, SMALL_V, CONFIG2A, CONFIG2A_V
out = {}
for name, cfg, v, n in (("small", SMALL, SMALL_V, 20), ("config2a", CONFIG2A, CONFIG2A_V, 100)):
    for keep in (False, True):
        s = tb.sim.build_sim({**cfg, "deterministic": True})
        s.set_keep_grid(keep)
        tb.mpm.step(s, v, n)
        tb.mpm.step(s, v, 7)
        x = s.positions()
        r = {"x": hashlib.sha1(x.tobytes()).hexdigest()[:12], "stats": s.stats()}
        if keep:
            lo, hi = s.grid_window()
            m, mom, vel = s.grid(lo, hi)
            r["m"] = hashlib.sha1(m.tobytes()).hexdigest()[:12]
            r["msum"] = float(m.sum())
        out[f"{name}_keep{int(keep)}"] = r
print(json.dumps(out))
"""
res = {}
for mode in ("fused", "fork"):
    env = {**os.environ, "TACCHI_WALKS": mode}
    p = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
    res[mode] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-2000:]
print(json.dumps(res, indent=1))
