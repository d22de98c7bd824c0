"""bench.py — Tacchi hot-path throughput on B200 (BASELINE.json metric).

Default workload (config 2a, BASELINE.json configs[1]): the default 20x20x4 mm
gel (101x101x21) + the sphere indenter at the reference's finest density (1e6
points, no subsampling) = 1,214,221 particles on the 256^3 / 33 mm grid,
dt = 2e-6 s, press velocity (0, 0, -0.01) m/s. One bench "step" = one tactile
frame = mpm::step(state, v, 10) + sim::capture (session.cpp:86, 42).

  value  particle-substeps/s with the state resident in HBM; device time on
         the handle's stream (CUDA events), max over ranks.
  e2e    the same metric through the C-ABI as a caller uses it: the command
         velocity goes in from host memory and the 640x480 depth (fp64) + RGB
         image come back to host buffers every frame, inside the timed region.

--workload config1 / config2b run the same protocol on those scenes;
--workload config4 runs the batch of --episodes (1024) independent config-1
episodes with mt19937_64 pose draws (episodes.py), episode e on rank
e mod N, all of a rank's episodes resident and stepped together
(tg_step_capture_many: one step = one frame of every episode).

Multi-GPU: one process per GPU (torchrun; `--gpus N` without a torchrun
environment spawns the N ranks itself). Episodes are independent: no
data-path collective; the per-rank device times are max-reduced.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, unmodified sources, OpenMP) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tests.scenes import (CONFIG1, CONFIG1_V, CONFIG2A, CONFIG2A_V, CONFIG2B,  # noqa: E402
                          SUBSTEPS_PER_FRAME)

# The bench runs the fp64 fast mode (SPEC "Concurrency Model": the default
# fast mode may relax to tolerance-level reproducibility); the fixed-point
# deterministic mode, which SceneConfig.deterministic selects, is reported as
# a secondary line of the same run.
FAST = {"deterministic": False}

METRIC = "particle-substeps/sec"
UNIT = "particle-substeps/s"
PRESS_V = (0.0, 0.0, -0.01)
WORKLOADS = {
    "config2a": ({**CONFIG2A, **FAST}, CONFIG2A_V,
                 "config2a: default gel 101x101x21 + sphere 1e6 pts (1,214,221 particles), 256^3 "
                 "grid, dt 2e-6, 10 substeps + capture per frame"),
    "config1": ({**CONFIG1, **FAST}, CONFIG1_V,
                "config1: default gel 101x101x21 + sphere 1e5 pts (314,221 particles), 256^3 grid, "
                "dt 2e-6, 10 substeps + capture per frame"),
    "config2b": ({**CONFIG2B, **FAST}, PRESS_V,
                 "config2b: gel 171x171x35 (0.1176 mm spacing) + sphere 1e5 (1,123,435 particles), "
                 "256^3 grid, dt 2e-6, 10 substeps + capture per frame"),
}
CONFIG4_WORKLOAD = ("config4: {n} independent episodes of config1 (314,221 particles each, "
                    "mt19937_64 pose draws: offset +-1 mm, z-rotation), episode e on rank e mod N, "
                    "one step = 10 substeps + capture of every episode")


def _dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clocks and clock-event (throttle) reasons sampled every ~5 ms by a
    thread from before the warm-up until after the timed regions
    (B200_PROFILING.md's clocks line). NVML (nvidia_ml_py, the library
    nvidia-smi reads) when it loads, else one-shot `nvidia-smi --query-gpu`
    calls; every sample is also written to gpurun_out/clocks_rank<i>.csv.
    (A streaming `nvidia-smi -lms` child block-buffers its output into a
    file and lost its samples when terminated.)"""

    # nvmlClocksEventReason* bits
    _BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        import threading

        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [t.strip() for t in vis.split(",") if t.strip()]
        self.phys = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.source = None
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.phys)
            self.nvml = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.source = "nvml"
        except Exception:
            self.source = "nvidia-smi"
        self.stop_ev = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _sample(self):
        if self.nvml is not None:
            p = self.nvml
            sm = float(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
            try:
                bits = int(p.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except AttributeError:
                bits = int(p.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
            return sm, self.max_mhz, bits
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.phys}", f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=10).stdout.strip().splitlines()[0]
        parts = [t.strip() for t in out.split(",")]
        bits = 0
        for bit, val in zip((0x8, 0x40, 0x20, 0x4), parts[2:6]):
            if val.lower() == "active":
                bits |= bit
        return float(parts[0]), float(parts[1]), bits

    def _run(self):
        with open(self.path, "w") as f:
            f.write("t_s,sm_mhz,sm_max_mhz,reasons_bits\n")
            t0 = time.perf_counter()
            while not self.stop_ev.is_set():
                try:
                    smp = self._sample()
                    self.samples.append(smp)
                    f.write(f"{time.perf_counter() - t0:.3f},{smp[0]:.0f},{smp[1]:.0f},{smp[2]:#x}\n")
                except Exception:
                    pass
                self.stop_ev.wait(0.005)

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=15)
        if not self.samples:
            return None
        # under load: samples without the GpuIdle reason (bit 0x1)
        sm = [x[0] for x in self.samples if not x[2] & 0x1] or [x[0] for x in self.samples]
        reasons = sorted({nm for _, _, b in self.samples for bit, nm in self._BITS.items() if b & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": reasons, "samples": len(sm), "samples_total": len(self.samples),
                "source": self.source}


# SURVEY §8(d) official yardstick: per substep every particle's persistent
# state is read once and written once: gel x(3) + F(9) doubles = 192 B,
# indenter x(3) = 48 B (v and C are transient; the grid is L2 scratch).
GEL_BYTES = 24 * 8
IND_BYTES = 6 * 8


def _roofline(s, phase_ms, walked_per_substep, n_el, n_ind, window_nodes):
    """roofline of the dominant kernel by §8(d) bytes: the elastomer kernel
    moves every gel particle's x and F in and out (192 B) and advects the
    indenter particles its column walks visit (48 B each); grid_update's
    algorithmic bytes are the node box's A + M_I read and V written."""
    peak, peak_src = _peaks()
    per_kernel = {
        "g2p2g_elastomer": n_el * GEL_BYTES + walked_per_substep * IND_BYTES,
        "grid_update": window_nodes * 64,
        "indenter_move_p2g": walked_per_substep * IND_BYTES,
    }
    dom = max(per_kernel, key=lambda k: phase_ms.get(k, 0.0))
    dom_ms = phase_ms[dom]
    achieved = per_kernel[dom] / (dom_ms * 1e-3) / 1e9
    per_substep = n_el * GEL_BYTES + n_ind * IND_BYTES
    substep_ms = (phase_ms["grid_update"] + phase_ms["g2p2g_elastomer"] + phase_ms["finalize"])
    traffic = shared = atomics = fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        kname = {"g2p2g_elastomer": "k_g2p2g_gel", "grid_update": "k_grid_update_boxes"}.get(dom)
        if kname in tr:
            traffic = tr[kname]["dram_bytes_per_launch"]
            if "shared_wavefronts_per_launch" in tr[kname]:
                shared = {"wavefronts_per_launch": tr[kname]["shared_wavefronts_per_launch"],
                          "pct_of_peak_sustained": tr[kname]["shared_wavefronts_pct_of_peak"]}
            f = tr[kname].get("fp64")
            if f and "peak_tflops" in f:
                # the kernel's fp64 work (ncu op counts per launch, a property
                # of the code and the config) over its live time
                ach = f["flop_per_launch"] / (dom_ms * 1e-3) / 1e12
                fp64 = {"achieved": ach, "peak": f["peak_tflops"], "unit": "TFLOP/s",
                        "frac": ach / f["peak_tflops"], "flop_per_launch": f["flop_per_launch"],
                        "source": f["source"], "peak_source": f["peak_source"]}
            red = tr[kname].get("l2_reduction")
            if red:
                atomics = {
                    "l2_reduction_requests_per_launch": red["lts__t_requests_op_red.sum"],
                    "l2_reduction_bytes_per_launch": 32 * red["lts__t_sectors_op_red.sum"],
                    "l2_atomic_unit_active_pct_of_peak":
                        red["lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"],
                    "bulk_reductions_per_launch": red["sm__sass_inst_executed_op_tma_red.sum"],
                    "redg_instructions_per_launch": red["smsp__sass_inst_executed_op_global_red.sum"],
                    "source": "profiles/traffic.json l2_reduction (ncu lts__t_*_op_red, "
                              "lts__d_atomic_input_cycles_active; profiles/r2_atomics.md)"}
    except Exception:
        pass
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": "profiles/traffic.json (ncu --set full, dram__bytes read+write per "
                              "launch of the same kernel)",
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": per_kernel[dom],
            "algorithmic_bytes_formula": "SURVEY §8(d): 192 B per elastomer particle (x, F read + "
                                         "written) + 48 B per indenter particle the launch "
                                         "advects (x read + written)",
            "indenter_particles_advected_per_launch": walked_per_substep,
            "traffic_over_algorithmic": (traffic / per_kernel[dom]) if traffic else None,
            "shared_memory": shared, "atomics": atomics, "fp64_compute": fp64, "kernel_ms": dom_ms,
            "substep": {"ms": substep_ms, "algorithmic_bytes": per_substep,
                        "achieved_gbs": per_substep / (substep_ms * 1e-3) / 1e9,
                        "frac": per_substep / (substep_ms * 1e-3) / 1e9 / peak,
                        "formula": "every particle once per substep: 192 B per elastomer, 48 B "
                                   "per indenter particle, over grid_update + elastomer kernel + "
                                   "finalize device time"},
            "phase_ms": phase_ms}


def _time_pipelined(tb, s, v, rp, steps, read_back):
    """Device time of `steps` pipelined frames (tg_step_capture_submit /
    _wait, two in flight): from before the first submit to after the last
    frame's shading (and read-back) on the handle's streams; the host reads
    every frame it gets back. Returns (ms, checksum, last outputs)."""
    import torch

    stream = torch.cuda.ExternalStream(s.stream, device=s.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    checksum = 0
    e0.record(stream)
    prev = tb.sim.step_capture_submit(s, v, SUBSTEPS_PER_FRAME, rp, read_back)
    out = (None, None)
    for _ in range(steps - 1):
        cur = tb.sim.step_capture_submit(s, v, SUBSTEPS_PER_FRAME, rp, read_back)
        out = tb.sim.step_capture_wait(s, prev, rp)
        if read_back:
            checksum += int(out[1][rp.height // 2, rp.width // 2, 0]) + int(out[0][0, 0] > 0)
        prev = cur
    out = tb.sim.step_capture_wait(s, prev, rp)  # waits for the frame's last stream
    e1.record(stream)
    torch.cuda.synchronize(s.device)
    return e0.elapsed_time(e1), checksum, out


def _time_frames(tb, s, v, rp, steps, want):
    """Device time (CUDA events on the handle's stream) of `steps` frames."""
    import torch

    stream = torch.cuda.ExternalStream(s.stream, device=s.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = None
    for _ in range(steps):
        out = tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, zero_copy=want,
                                  want_depth=want, want_image=want)
    e1.record(stream)
    torch.cuda.synchronize(s.device)
    return e0.elapsed_time(e1), out


def _secondary(tb, device, steps):
    """Short device-resident lines for config 1 and config 2b (the config-2a
    headline is dominated by its 1e6 rigid indenter particles; these show the
    elastomer-bound scenes) and for config 2a in the deterministic mode."""
    out = []
    cfg2a, v2a, desc2a = WORKLOADS["config2a"]
    cases = [(name, *WORKLOADS[name]) for name in ("config1", "config2b")]
    cases.append(("config2a-deterministic", {**cfg2a, "deterministic": True}, v2a,
                  desc2a + "; deterministic mode (fixed-point node sums, bit-identical reruns)"))
    for name, cfg, v, desc in cases:
        s = tb.sim.build_sim(cfg, device=device)
        rp = tb.render_params(cfg, "")
        for _ in range(3):
            tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, want_depth=False,
                                want_image=False)
        ms, _ = _time_frames(tb, s, v, rp, steps, False)
        out.append({"workload": desc, "value": s.n * SUBSTEPS_PER_FRAME * steps / (ms * 1e-3),
                    "unit": UNIT, "frames_per_sec": steps / (ms * 1e-3),
                    "ms_per_step": ms / steps, "particles": s.n, "elastomer": s.elastomer_count})
        del s
    return out


def _init_dist(world, local, backend="nccl"):
    import torch
    import torch.distributed as dist

    if world > 1:
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)


def run_single(args):
    """One scene per rank (config 2a / 1 / 2b): rank r runs its own episode
    (config-4 pose draw r; rank 0 the centred press)."""
    import torch

    import paper_2301_08343_b200 as tb
    from paper_2301_08343_b200 import episodes

    rank, world, local = _dist_env()
    _init_dist(world, local)
    device = local
    torch.cuda.set_device(device)
    cfg, v, desc = WORKLOADS[args.workload]
    ep = episodes.make_episode(rank) if world > 1 else episodes.Episode(0, 0.0, 0.0, 0.0, 0.0)
    s = tb.sim.build_sim(episodes.episode_config(cfg, ep), "", ep.offset_x_m, ep.offset_y_m,
                         device=device)
    n, n_el = s.n, s.elastomer_count
    rp = tb.render_params(cfg, "")
    v = np.array(v)

    clocks = Clocks(device)  # sampled from before warm-up until after the timed regions
    # warm-up through both call forms (graphs, pinned slots, the copy stream)
    for _ in range(args.warmup):
        tb.sim.step_capture(s, v, SUBSTEPS_PER_FRAME, params=rp, want_depth=False, want_image=False)
    _time_pipelined(tb, s, v, rp, args.warmup, True)
    torch.cuda.synchronize(device)

    # --- timed region 1: device-resident (value): pipelined frames, step +
    # capture with the outputs left on the device ---
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    k0 = s.kernel_launches
    dev_ms, _, _ = _time_pipelined(tb, s, v, rp, args.steps, False)
    launches = s.kernel_launches - k0
    dev_sync_ms, _ = _time_frames(tb, s, v, rp, args.steps, False)  # one sync per call

    # --- timed region 2: end to end through the C-ABI with host buffers ---
    # Pipelined control steps (tg_step_capture_submit / _wait): frame k's
    # depth + RGB come back to pinned host memory while frame k+1 runs; the
    # host reads every frame. Timed on the handle's stream from before the
    # first submit to after the last frame's read-back, and on the wall clock.
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    e2e_ms, _, (depth, img) = _time_pipelined(tb, s, v, rp, args.steps, True)
    e2e_wall = (time.perf_counter() - t0) * 1e3
    # the synchronous call (one control step, one host sync: the Session's
    # shape), for reference
    sync_ms, _ = _time_frames(tb, s, v, rp, args.steps, True)
    clk = clocks.stop()

    # --- per-kernel timing for the roofline (after the timed regions) ---
    w0 = s.stats()["indenter_walked"]
    reps = 20
    phase_ms = s.time_phases(v, reps=reps)
    walked = (s.stats()["indenter_walked"] - w0) / reps
    lo, hi = s.grid_window()
    window_nodes = int(np.prod(hi - lo))
    stats = s.stats()

    if world > 1:
        dev_ms = episodes.max_over_ranks(dev_ms, device=f"cuda:{device}")
        e2e_ms = episodes.max_over_ranks(e2e_ms, device=f"cuda:{device}")
        sync_ms = episodes.max_over_ranks(sync_ms, device=f"cuda:{device}")
        dev_sync_ms = episodes.max_over_ranks(dev_sync_ms, device=f"cuda:{device}")
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    units = float(n) * SUBSTEPS_PER_FRAME * args.steps * world
    line = {
        "metric": METRIC, "value": units / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "particles_per_gpu": n, "elastomer": n_el,
                   "grid": [256, 256, 256], "grid_node_arrays_bytes": stats["grid_bytes"],
                   "substeps_per_step": SUBSTEPS_PER_FRAME, "dt_s": 2e-6,
                   "accumulation": "fp64 fast mode (deterministic: false); the deterministic "
                                   "mode is the `secondary` config2a-deterministic line",
                   "parallelism": f"independent episodes x{world} (one per GPU), no collective",
                   "l2": "no flush; per substep the particle state streams ~62 MB and the node "
                         "box ~60 MB through the 126 MB L2 (warm-cache DRAM traffic ~200 MB per "
                         "substep: elastomer kernel 136 MB, grid_update 58 MB, ncu "
                         "--cache-control none, DESIGN.md 4): inputs are not L2-resident between "
                         "steps"},
        "frames_per_sec": args.steps * world / (dev_ms * 1e-3),
        "value_api": "pipelined tg_step_capture_submit / _wait with read_back = 0 (step + capture "
                     "per frame, outputs stay in HBM)",
        "value_synchronous": {"value": units / (dev_sync_ms * 1e-3),
                              "frames_per_sec": args.steps * world / (dev_sync_ms * 1e-3),
                              "api": "tg_step_capture with no outputs, one host sync per frame"},
        "e2e": {"value": units / (e2e_ms * 1e-3), "unit": UNIT,
                "frames_per_sec": args.steps * world / (e2e_ms * 1e-3),
                "h2d_bytes_per_step": 3 * 8, "d2h_bytes_per_step": depth.nbytes + img.nbytes,
                "wall_ms_per_step": e2e_wall / args.steps,
                "api": "tb.sim.step_capture_submit / _wait -> tg_step_capture_submit / "
                       "tg_step_capture_wait (step + capture + depth f64 + RGB8 D2H into pinned "
                       "host slots each step, two frames in flight, the host reads every frame)",
                "synchronous": {"value": units / (sync_ms * 1e-3),
                                "frames_per_sec": args.steps * world / (sync_ms * 1e-3),
                                "api": "tb.sim.step_capture -> tg_step_capture (one control step, "
                                       "one host sync per call)"}},
        "gpu_launches": int(launches),
        "roofline": _roofline(s, phase_ms, walked, n_el, n - n_el, window_nodes),
    }
    if clk:
        line["clocks"] = clk
    del s
    if world == 1 and args.workload == "config2a" and not args.no_secondary:
        line["secondary"] = _secondary(tb, device, args.steps)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload, frames=args.cpu_frames)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_config4(args):
    """Config 4: args.episodes independent config-1 episodes, episode e on
    rank e mod N, all resident, every step one frame of each (tg_step_capture_many)."""
    import torch

    import paper_2301_08343_b200 as tb
    from paper_2301_08343_b200 import episodes

    rank, world, local = _dist_env()
    _init_dist(world, local)
    device = local
    torch.cuda.set_device(device)
    mine = episodes.shard(args.episodes, rank, world)
    eps = [episodes.make_episode(e) for e in mine]
    poses = np.array([[ep.offset_x_m, ep.offset_y_m, ep.z_rotation_rad] for ep in eps])
    t_build = time.perf_counter()
    sims = tb.sim.build_episodes({**CONFIG1, **FAST}, "", poses, device=device)
    build_s = time.perf_counter() - t_build
    rp = tb.render_params(CONFIG1, "")
    vel = np.tile(np.asarray(CONFIG1_V, np.float64), (len(sims), 1))
    n = sims[0].n if sims else 0

    def frame(want):
        # outputs straight into each handle's pinned host buffers (zero_copy)
        outs, _ = tb.sim.step_capture_many(sims, vel, SUBSTEPS_PER_FRAME, rp, want_depth=want,
                                           want_image=want, zero_copy=want)
        return outs

    def timed(steps, want):
        # every handle has its own stream: start event on the first handle's
        # stream with the device idle, end events on each stream, max span
        streams = [torch.cuda.ExternalStream(s.stream, device=device) for s in sims]
        torch.cuda.synchronize(device)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        outs = None
        for _ in range(steps):
            outs = frame(want)
        ends = []
        for st in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ends.append(e)
        torch.cuda.synchronize(device)
        return max(e0.elapsed_time(e) for e in ends), outs

    clocks = Clocks(device)
    for _ in range(args.warmup):
        frame(False)
    if world > 1:
        torch.distributed.barrier()
    k0 = sum(s.kernel_launches for s in sims)
    dev_ms, _ = timed(args.steps, False)
    launches = sum(s.kernel_launches for s in sims) - k0
    if world > 1:
        torch.distributed.barrier()
    e2e_ms, outs = timed(args.steps, True)
    clk = clocks.stop()
    d2h = sum(d.nbytes + im.nbytes for d, im in outs)
    grid_bytes = sum(s.stats()["grid_bytes"] for s in sims)
    free, total = torch.cuda.mem_get_info(device)
    if world > 1:
        dev_ms = episodes.max_over_ranks(dev_ms, device=f"cuda:{device}")
        e2e_ms = episodes.max_over_ranks(e2e_ms, device=f"cuda:{device}")
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    units = float(n) * args.episodes * SUBSTEPS_PER_FRAME * args.steps
    line = {
        "metric": METRIC, "value": units / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIG4_WORKLOAD.format(n=args.episodes),
                   "episodes": args.episodes, "episodes_per_gpu": len(sims),
                   "particles_per_episode": n, "substeps_per_step": SUBSTEPS_PER_FRAME,
                   "parallelism": f"episodes sharded e mod {world}, no collective",
                   "resident": "every episode of a rank resident in HBM",
                   "rank0_grid_node_arrays_bytes": grid_bytes,
                   "rank0_hbm_used_bytes": total - free, "rank0_build_s": build_s,
                   "l2": "no flush; a step streams every episode's state (>> 126 MB L2)"},
        "episode_frames_per_sec": args.episodes * args.steps / (dev_ms * 1e-3),
        "e2e": {"value": units / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": 3 * 8 * len(sims), "d2h_bytes_per_step": d2h,
                "api": "tb.sim.step_capture_many -> tg_step_capture_many (every episode's step + "
                       "capture submitted before any wait; depth f64 + RGB8 into each handle's "
                       "pinned host buffers each step)"},
        "gpu_launches": int(launches),
    }
    if clk:
        line["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline("config4", frames=args.cpu_frames)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _ref_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _harness_pattern(frames: int, n_episodes: int = 32):
    """The reference harness's batch pattern (harness.cpp:206-237): a pool of
    workers = host cores, each simulation on one thread (num_threads = 1),
    jobs = independent episodes. Times `frames` frames (10 substeps + capture)
    of n_episodes config-4 episodes; returns (particle-substeps/s, threads,
    episodes)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import refpy
    from paper_2301_08343_b200 import episodes

    threads = _ref_threads()
    eps = [episodes.make_episode(e) for e in range(n_episodes)]

    def build(ep):
        return refpy.RefSim.from_config(episodes.episode_config(CONFIG1, ep), "", ep.offset_x_m,
                                        ep.offset_y_m, threads=1)

    with ThreadPoolExecutor(threads) as pool:  # ctypes releases the GIL in the calls
        sims = list(pool.map(build, eps))

        def run(sim):
            for _ in range(frames):
                sim.step(CONFIG1_V, SUBSTEPS_PER_FRAME)
                sim.capture(CONFIG1)

        t0 = time.perf_counter()
        list(pool.map(run, sims))
        dt = time.perf_counter() - t0
    n = sims[0].n
    return n * n_episodes * SUBSTEPS_PER_FRAME * frames / dt, threads, n_episodes


def cpu_baseline(workload: str, frames: int = 2):
    """The reference's own CPU engine (oracle/_ref, unmodified sources, -O3
    -fopenmp) on a bounded sample of the same workload."""
    from oracle import refpy

    if not refpy.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref missing on this host"}
    if workload == "config4":
        value, threads, k = _harness_pattern(max(frames, 1))
        return {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                "cpu_model": _cpu_model(),
                "sample": f"harness pattern (harness.cpp:206-237): {threads} workers x 1 thread, "
                          f"{k} config-4 episodes x {max(frames, 1)} frames (10 substeps + "
                          "capture); per-episode work is independent, so the 1024-episode "
                          "throughput is this rate (extrapolated linearly)"}
    cfg, v, _ = WORKLOADS[workload]
    threads = _ref_threads()
    sim = refpy.RefSim.from_config(cfg, "", threads=threads)
    sim.step(v, 1)  # first touch of the dense 256^3 grid
    t0 = time.perf_counter()
    sim.step(v, SUBSTEPS_PER_FRAME * frames)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    sim.capture(cfg)
    cap = time.perf_counter() - t1
    n = sim.n
    del sim
    one = refpy.RefSim.from_config(cfg, "", threads=1)
    one.step(v, 1)
    t2 = time.perf_counter()
    one.step(v, 2)
    dt1 = time.perf_counter() - t2
    return {"value": n * SUBSTEPS_PER_FRAME * frames / dt, "unit": UNIT, "cores": threads,
            "kind": "reference", "capture_ms": cap * 1e3, "value_1_thread": n * 2 / dt1,
            "cpu_model": _cpu_model(),
            "sample": f"{frames * SUBSTEPS_PER_FRAME} substeps of {workload} ({n} particles), "
                      f"mpm::step wall time, OMP threads={threads}; value_1_thread: 2 substeps "
                      f"on one thread"}


REF_BUDGET_S = 90.0


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    from oracle import refpy

    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtacchi_ref.so not built"}))
        return
    threads = _ref_threads()
    if args.workload == "config4":
        value, threads, k = _harness_pattern(max(1, min(args.steps, 2)))
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": CONFIG4_WORKLOAD.format(n=args.episodes)},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                                 "kind": "reference", "cpu_model": _cpu_model(),
                                 "sample": f"harness pattern: {threads} workers x 1 thread over {k} "
                                           "episodes, extrapolated linearly to the batch"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    cfg, v, desc = WORKLOADS[args.workload]
    sim = refpy.RefSim.from_config(cfg, "", threads=threads)
    n = sim.n
    for _ in range(args.warmup):
        sim.step(v, SUBSTEPS_PER_FRAME)
        sim.capture(cfg)
    # A frame of the reference takes ~0.5 s on 16 threads: the timed sample
    # stops at K frames or REF_BUDGET_S seconds, whichever comes first.
    t0 = time.perf_counter()
    steps = 0
    while steps < args.steps:
        sim.step(v, SUBSTEPS_PER_FRAME)
        sim.capture(cfg)
        steps += 1
        if time.perf_counter() - t0 > REF_BUDGET_S:
            break
    dt = time.perf_counter() - t0
    value = n * SUBSTEPS_PER_FRAME * steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "particles_per_gpu": n, "substeps_per_step": SUBSTEPS_PER_FRAME},
        "frames_per_sec": steps / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu_model": _cpu_model(),
                         "sample": f"{steps} frames (10 substeps + capture) of {args.workload} "
                                   f"(of {args.steps} requested; {REF_BUDGET_S:.0f} s budget), "
                                   f"OMP threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): each rank
    takes its shard of the workload's episodes and reports a synthetic device
    time; rank 0 prints the plan and the max over ranks."""
    import torch.distributed as dist

    from paper_2301_08343_b200 import episodes

    rank, world, _ = _dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    n_eps = args.episodes if args.workload == "config4" else world
    mine = episodes.shard(n_eps, rank, world)
    fake_ms = 10.0 + rank
    worst = episodes.max_over_ranks(fake_ms)
    if world > 1:
        import torch

        sizes = [None] * world
        dist.all_gather_object(sizes, len(mine))
    else:
        sizes = [len(mine)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": args.workload,
                          "episodes_per_rank": sizes, "max_ms": worst}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(argv, n):
    """`bench.py --gpus N` outside torchrun: relaunch this script as N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2a",
                    choices=["config2a", "config1", "config2b", "config4"])
    ap.add_argument("--episodes", type=int, default=1024)
    ap.add_argument("--cpu-frames", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.workload == "config4":
        run_config4(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
