"""End-to-end frame rate of config 2a (fp64 mode) through the public API in
its forms: device-resident, synchronous step_capture with the read-back
(zero-copy pinned views), and the pipelined submit / wait; wall clock and
stream events. One JSON line per mode.

    python tools/e2e_modes.py [frames]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_08343_b200 as tb  # noqa: E402
from tests.scenes import CONFIG2A, CONFIG2A_V  # noqa: E402


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    cfg = {**CONFIG2A, "deterministic": False}
    s = tb.sim.build_sim(cfg)
    rp = tb.render_params(cfg, "")
    v = np.array(CONFIG2A_V)
    st = torch.cuda.ExternalStream(s.stream)

    def run(name, body):
        for _ in range(3):
            body(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        body(frames)
        e1.record(st)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(json.dumps({"mode": name, "frames_per_s_events": frames / (e0.elapsed_time(e1) * 1e-3),
                          "frames_per_s_wall": frames / wall}), flush=True)

    def device(k):
        for _ in range(k):
            tb.sim.step_capture(s, v, 10, params=rp, want_depth=False, want_image=False)

    def sync_zero_copy(k):
        c = 0
        for _ in range(k):
            d, im = tb.sim.step_capture(s, v, 10, params=rp, zero_copy=True)
            c += int(im[240, 320, 0])

    def sync_rgb_only(k):
        for _ in range(k):
            tb.sim.step_capture(s, v, 10, params=rp, zero_copy=True, want_depth=False)

    def pipelined(k):
        c = 0
        prev = tb.sim.step_capture_submit(s, v, 10, rp)
        for _ in range(k - 1):
            cur = tb.sim.step_capture_submit(s, v, 10, rp)
            d, im = tb.sim.step_capture_wait(s, prev, rp)
            c += int(im[240, 320, 0])
            prev = cur
        tb.sim.step_capture_wait(s, prev, rp)

    for name, body in (("device", device), ("sync_zero_copy", sync_zero_copy),
                       ("sync_rgb_only", sync_rgb_only), ("pipelined", pipelined),
                       ("device_again", device)):
        run(name, body)


if __name__ == "__main__":
    main()
