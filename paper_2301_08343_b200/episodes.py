"""Episode planning and sharding for batched / multi-GPU runs.

Indentation episodes are independent (harness.cpp:55-103: each owns its
SimState), so the multi-GPU layout is pure data parallelism over episodes:
episode e runs on rank e mod world, no data-path collective. The only
collective is the max-over-ranks of the device time used for reporting.

Config 4: episode e (0-based) draws its pose from
std::mt19937_64 seeded with e + 1, in this order, each as the reference's
53-bit uniform (rng() >> 11) * 2^-53 (shapes.cpp:235):
  lateral offset x, y   uniform over [-1, 1] mm (the span of the paper's
                        +-1 mm press grid, harness.cpp:200-201),
  z-rotation            uniform [0, 2 pi) (scene_config.hpp:47),
  target depth          uniform [0.1, 1.0] mm.
The indenter cloud keeps its config seed (20230115).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of <random>): state
    size 312, shift 156, seeding f = 6364136223846793005. Pure Python; the
    episode planner draws four numbers per episode."""

    N, M = 312, 156
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [seed & _MASK64]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64)
        self.mt = mt
        self.i = self.N

    def _twist(self):
        mt, n, m = self.mt, self.N, self.M
        for k in range(n):
            y = (mt[k] & self.UPPER) | (mt[(k + 1) % n] & self.LOWER)
            mt[k] = mt[(k + m) % n] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform(self) -> float:
        """The reference's 53-bit uniform in [0, 1) (shapes.cpp:235)."""
        return (self() >> 11) * (1.0 / 9007199254740992.0)


@dataclass(frozen=True)
class Episode:
    index: int
    offset_x_m: float
    offset_y_m: float
    z_rotation_rad: float
    depth_m: float


def make_episode(index: int, seed: int | None = None) -> Episode:
    """Pose and target depth of config-4 episode `index` (seed = index + 1)."""
    rng = MT19937_64(index + 1 if seed is None else seed)
    ox = -1e-3 + 2e-3 * rng.uniform()
    oy = -1e-3 + 2e-3 * rng.uniform()
    rot = 2.0 * math.pi * rng.uniform()
    depth = 0.1e-3 + 0.9e-3 * rng.uniform()
    return Episode(index, ox, oy, rot, depth)


def shard(n_episodes: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment: episode e -> rank e mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return list(range(rank, n_episodes, world))


def waves(episodes: list[int], per_wave: int) -> list[list[int]]:
    """Splits a rank's episodes into waves of at most `per_wave` resident
    simulations (the memory budget of one GPU)."""
    if per_wave < 1:
        raise ValueError("per_wave must be >= 1")
    return [episodes[i:i + per_wave] for i in range(0, len(episodes), per_wave)]


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
