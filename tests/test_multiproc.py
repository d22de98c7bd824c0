"""Multi-process (world_size 2, gloo, CPU) coverage of the episode sharding
and the max-over-ranks reporting collective used by bench.py --gpus N."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2301_08343_b200 import episodes as E


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_episodes, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = E.shard(n_episodes, rank, world)
    # each rank reports a different "device time"; the job time is the max
    t = E.max_over_ranks(10.0 + rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    out[rank] = (mine, t, gathered)
    dist.destroy_process_group()


def test_sharding_over_two_ranks_with_gloo():
    world, n = 2, 1024
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, n, out), nprocs=world, join=True)
    shards = [out[r][0] for r in range(world)]
    assert sorted(sum(shards, [])) == list(range(n))  # disjoint, complete
    assert all(out[r][1] == 11.0 for r in range(world))  # max over ranks
    assert out[0][2] == out[1][2] == shards


def test_episode_draws_are_deterministic_and_in_range():
    a, b = E.make_episode(7), E.make_episode(7)
    assert a == b
    for i in range(200):
        ep = E.make_episode(i)
        assert -1e-3 <= ep.offset_x_m <= 1e-3 and -1e-3 <= ep.offset_y_m <= 1e-3
        assert 0 <= ep.z_rotation_rad < 6.2832
        assert 0.1e-3 <= ep.depth_m <= 1.0e-3
    cfg = E.episode_config({"time": {"dt_s": 2e-6}}, a)
    assert cfg["indenter"]["z_rotation_rad"] == a.z_rotation_rad
    # harness schedule: (gap + depth) / (v dt) substeps
    assert E.press_substeps({"time": {"dt_s": 2e-6}}, E.Episode(0, 0, 0, 0, 0.5e-3)) == 30000


def test_shard_rejects_bad_rank():
    with pytest.raises(ValueError):
        E.shard(8, 2, 2)


def test_mt19937_64_known_answer():
    """[rand.predef]: the 10000th output of a default-constructed
    std::mt19937_64 is 9981545732273789042; seed 1 as std::mt19937_64(1)."""
    r = E.MT19937_64()
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042
    r1 = E.MT19937_64(1)
    assert [r1(), r1()] == [2469588189546311528, 2516265689700432462]
    ep = E.make_episode(0)  # seed 1: the first four 53-bit uniforms
    assert ep.offset_x_m == -1e-3 + 2e-3 * ((2469588189546311528 >> 11) * 2.0**-53)


def test_waves_split_a_rank_share():
    eps = E.shard(1024, 3, 8)
    w = E.waves(eps, 50)
    assert [len(x) for x in w] == [50, 50, 28] and sum(w, []) == eps


def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun relaunches itself as two ranks
    (torch.distributed.run on 127.0.0.1); --dry-run runs the multi-rank
    plumbing on CPU (gloo): config-4 episodes sharded e mod 2 and the
    max-over-ranks device time."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--dry-run", "--workload", "config4", "--episodes", "1024"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["episodes_per_rank"] == [512, 512]
    assert line["max_ms"] == 11.0  # rank 1's synthetic time wins


def test_config4_cpu_baseline_harness_pattern():
    """bench.py's config-4 CPU baseline runs the reference's harness pattern
    (harness.cpp:206-237: a worker per host core, each simulation on one
    thread) over config-4 episodes; here on 2 episodes x 1 frame."""
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import refpy

    if not refpy.available():
        pytest.skip("oracle/_ref not built")
    import bench

    value, threads, k = bench._harness_pattern(1, 2)
    assert value > 0 and threads >= 1 and k == 2
