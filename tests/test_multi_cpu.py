"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: the shard plan
covers every episode exactly once, and the stats reduction equals the
single-process combination."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2505_06771_b200.multigpu import SUM_KEYS, Shard


def test_shard_plan_covers_episodes_once():
    world, B = 4, 1000
    seen = set()
    for wave in range(3):
        for r in range(world):
            s = Shard(r, world, B)
            for e in range(B):
                seen.add(s.first_episode + e + wave * s.episode_stride)
    assert seen == set(range(3 * world * B))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2505_06771_b200.multigpu import reduce_stats

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    part = {k: float(rank + 1) * (i + 1) for i, k in enumerate(SUM_KEYS)}
    part["min_pairwise_distance"] = 0.2 - 0.01 * rank
    out = reduce_stats(part)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_stats_reduction_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(30)
    for r in range(world):
        out = res[r]
        for i, k in enumerate(SUM_KEYS):
            assert out[k] == pytest.approx((1 + 2) * (i + 1))
        assert out["min_pairwise_distance"] == pytest.approx(0.19)
