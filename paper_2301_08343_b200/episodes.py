"""Episode planning and sharding for batched / multi-GPU runs.

Indentation episodes are independent (harness.cpp:55-103: each owns its
SimState), so the multi-GPU layout is pure data parallelism over episodes:
episode e runs on rank e mod world, no data-path collective. The only
collective is the max-over-ranks of the device time used for reporting.

Config 4: per-episode seeds 1..N drive std::mt19937_64-style
draws of the lateral offset (uniform over [-1, 1] x [-1, 1] mm), the
z-rotation (uniform [0, 2 pi)) and the target depth (uniform [0.1, 1.0] mm).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Episode:
    index: int
    offset_x_m: float
    offset_y_m: float
    z_rotation_rad: float
    depth_m: float


def _u01(rng: np.random.Generator) -> float:
    return float(rng.random())


def make_episode(index: int, seed: int | None = None) -> Episode:
    """Pose and depth of episode `index` (seed defaults to index + 1)."""
    rng = np.random.default_rng(index + 1 if seed is None else seed)
    ox = -1e-3 + 2e-3 * _u01(rng)
    oy = -1e-3 + 2e-3 * _u01(rng)
    rot = 2.0 * math.pi * _u01(rng)
    depth = 0.1e-3 + 0.9e-3 * _u01(rng)
    return Episode(index, ox, oy, rot, depth)


def shard(n_episodes: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment: episode e -> rank e mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return list(range(rank, n_episodes, world))


def episode_config(base: dict, ep: Episode) -> dict:
    """SceneConfig overrides for one episode (z-rotation of the indenter)."""
    cfg = {k: (dict(v) if isinstance(v, dict) else v) for k, v in base.items()}
    ind = dict(cfg.get("indenter", {}))
    ind["z_rotation_rad"] = ep.z_rotation_rad
    cfg["indenter"] = ind
    return cfg


def press_substeps(cfg: dict, ep: Episode) -> int:
    """Substeps until the commanded travel reaches gap + depth
    (harness.cpp:66-72: llround(travel / (v dt)))."""
    dt = cfg.get("time", {}).get("dt_s", 1e-4)
    v = cfg.get("time", {}).get("press_speed_mm_s", 10.0) * 1e-3
    gap = cfg.get("indenter", {}).get("gap_mm", 0.1) * 1e-3
    return int(round((gap + ep.depth_m) / (v * dt)))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks of the default process group (the
    reporting collective; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
