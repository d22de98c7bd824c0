"""Per-kernel device times of the config-2a substep (tg_time_phases) under the
TACCHI_SCATTER A/B switches; prints one JSON line.

    TACCHI_SCATTER=<mode> python tools/ab_phases.py [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG2A, CONFIG2A_V  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
s = tb.sim.build_sim(CONFIG2A)
tb.mpm.step(s, CONFIG2A_V, 30)
ph = s.time_phases(CONFIG2A_V, reps)
print(json.dumps({"mode": os.environ.get("TACCHI_SCATTER", "0"),
                  **{k: round(v * 1e3, 2) for k, v in ph.items()}}))
