"""A/B of environment switches on the config-2a frame: each variant runs in
its own process (the switches are read at tg_create), interleaved `--rounds`
times; prints frames/s and the per-kernel device times (tg_time_phases).

    python tools/ab_env.py --variant base: --variant dense:TACCHI_DENSE_GRID=1

AB_CFG: SceneConfig overrides as JSON, or @file holding them (for JSON with
commas, which the variant syntax splits on). AB_PREALLOC_KB: device memory
allocated before the handle (moves its allocations' addresses).
Without AB_CFG the scene runs in SceneConfig's default deterministic mode;
the bench's headline is fast mode: AB_CFG='{"deterministic": false}'.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, time
sys.path.insert(0, %r)
import torch
import paper_2301_08343_b200 as tb
from tests.scenes import CONFIG2A, CONFIG2A_V
_ab = os.environ.get("AB_CFG", "{}")
cfg = {**CONFIG2A, **json.loads(open(_ab[1:]).read() if _ab.startswith("@") else _ab)}
_pre = int(os.environ.get("AB_PREALLOC_KB", "0"))  # shifts the handle's allocations
_buf = torch.cuda.caching_allocator_alloc(_pre << 10) if _pre else None
s = tb.sim.build_sim(cfg)
rp = tb.render_params(cfg, "")
for _ in range(5):
    tb.sim.step_capture(s, CONFIG2A_V, 10, params=rp, want_depth=False, want_image=False)
frames = %d
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(s.stream)
e0.record(st)
for _ in range(frames):
    tb.sim.step_capture(s, CONFIG2A_V, 10, params=rp, want_depth=False, want_image=False)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ph = s.time_phases(CONFIG2A_V, reps=20)
print(json.dumps({"fps": frames / ms * 1e3, "phases_us": {k: round(v * 1e3, 2) for k, v in ph.items()},
                  "stats": s.stats()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", action="append", required=True, help="name:K=V,K=V")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--frames", type=int, default=100)
    args = ap.parse_args()
    variants = []
    for v in args.variant:
        name, _, kv = v.partition(":")
        env = dict(p.split("=", 1) for p in kv.split(",") if p)
        variants.append((name, env))
    for r in range(args.rounds):
        for name, env in variants:
            e = dict(os.environ)
            e.update(env)
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, args.frames)], env=e,
                                 capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
            print(json.dumps({"round": r, "variant": name, "result": line}), flush=True)


if __name__ == "__main__":
    main()
