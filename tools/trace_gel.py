"""Per-CTA stage timeline of the elastomer kernel (k_g2p2g_gel) from a
diagnostic build (-DTACCHI_TRACE, `make -C paper_2301_08343_b200/csrc
OUT=$PWD/paper_2301_08343_b200/_lib_trace EXTRA_NVFLAGS=-DTACCHI_TRACE`).

    TACCHI_LIB=paper_2301_08343_b200/_lib_trace/libtacchi_cuda.so python tools/trace_gel.py

Marks (thread 0 of each CTA, clock64), in time order: 0 entry, 1 after
griddepcontrol.wait, 2 velocity tile staged, 8 G2P gather done, 9 F update
+ stores done, 3 motion reduction done, 4 stress payload done, 5 P2G tile
box + zeroing done, 6 27 scatter phases done, 7 bulk reductions issued +
tile read.
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG2A, CONFIG2A_V, SUBSTEPS_PER_FRAME  # noqa: E402

# the bench mode (fast) unless TRACE_DET=1 (SceneConfig's default deterministic mode)
s = tb.sim.build_sim({**CONFIG2A, "deterministic": os.environ.get("TRACE_DET") == "1"})
for _ in range(5):
    tb.mpm.step(s, CONFIG2A_V, SUBSTEPS_PER_FRAME)
s.sync()
L = tb.lib()
fn = L.tg_debug_trace
fn.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((16384, 16), dtype=np.uint64)
n = fn(buf.ctypes.data, 16384)
assert n > 0
t = buf[buf[:, 15] > 0].astype(np.int64)
gel = t[t[:, 15] == 1]
ind = t[t[:, 15] == 2]
ghz = float(sys.argv[1]) if len(sys.argv) > 1 else 1.965
t0 = t[:, 0].min()
span = (t[:, 14].max() - t0) / 1e3
out = {"ctas_gel": int(len(gel)), "ctas_ind": int(len(ind)), "kernel_span_us": round(span, 2)}
order = [0, 1, 2, 8, 9, 3, 4, 5, 6, 7]
marks = gel[:, [2 + i for i in order]]
d = np.diff(marks, axis=1) / (ghz * 1e3)  # us
names = ["pdl_wait", "staging_wait", "gather", "update_store", "motion_reduce", "payload",
         "tilebox_zero", "phases27", "flush"]
out["stage_us_mean"] = {k: round(float(v), 3) for k, v in zip(names, d.mean(0))}
out["stage_us_p90"] = {k: round(float(v), 3) for k, v in zip(names, np.percentile(d, 90, 0))}
out["cta_us_mean"] = round(float(((marks[:, -1] - marks[:, 0]) / (ghz * 1e3)).mean()), 3)
out["cta_wall_us_mean"] = round(float(((gel[:, 14] - gel[:, 0]) / 1e3).mean()), 3)
st = (gel[:, 0] - t0) / 1e3
en = (gel[:, 14] - t0) / 1e3
out["gel_start_us_pct"] = [round(float(x), 2) for x in np.percentile(st, [0, 25, 50, 75, 90, 100])]
out["gel_end_us_pct"] = [round(float(x), 2) for x in np.percentile(en, [0, 25, 50, 75, 90, 100])]
if len(ind):
    out["ind_block_us_mean"] = round(float(((ind[:, 14] - ind[:, 0]) / 1e3).mean()), 2)
    out["ind_start_end_us"] = [round(float((ind[:, 0].min() - t0) / 1e3), 2),
                               round(float((ind[:, 14].max() - t0) / 1e3), 2)]
# concurrency: gel CTAs resident over time (1 us bins)
bins = np.arange(0, span + 1, 1.0)
conc = [int(((st <= b) & (en > b)).sum()) for b in bins]
out["gel_ctas_resident_per_us"] = conc
sm = gel[:, 1]
out["ctas_per_sm_max"] = int(np.bincount(sm).max())
print(json.dumps(out))
