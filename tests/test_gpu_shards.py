"""per-env results must be bit-identical for G in {1, 2, 4, 8}
GPUs. Simulated on one GPU with G independent contexts that each own the
contiguous slice a rank would own (Shard plan, auto-reset wave seeding);
contexts run one after another — nothing waits on another rank."""
import numpy as np
import pytest
import torch

import paper_2505_06771_b200 as m
from paper_2505_06771_b200.multigpu import Shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("task,n", [("navigation", 4), ("rware", 6), ("material_transport", 10)])
def test_per_env_results_independent_of_gpu_count(task, n):
    cfg = m.make_default_config(task)
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    cfg.max_steps = 30
    total = 512
    steps = 75  # crosses two auto-resets
    ref = None
    for G in (1, 2, 4, 8):
        per = total // G
        rows = []
        stats = []
        for r in range(G):
            sh = Shard(r, G, per)
            gb = m.CudaEnvBatch(cfg, per, fp64=True, auto_reset=True)
            gb.reset_episodes(root_seed=7, first_episode=sh.first_episode, episode_stride=sh.episode_stride)
            for _ in range(steps):
                gb.step(None, want_obs=False)
            torch.cuda.synchronize()
            gb.sync()
            st = gb.get_states()
            rows.append(np.array([(s.episode, s.step_index, s.collisions, *s.x[:n], *s.y[:n], *s.theta[:n])
                                  for s in st]))
            stats.append(gb.stats())
            gb.close()
        got = np.concatenate(rows)
        agg = {k: sum(s[k] for s in stats) for k in ("episodes", "env_steps", "sum_collisions", "sum_qp_infeasible",
                                                      "sum_success")}
        if ref is None:
            ref, ref_agg = got, agg
        else:
            assert np.array_equal(got, ref), G  # bit-identical per env
            assert agg == ref_agg


def test_permuting_or_deleting_instances_matches_reference(ref):
    """test_framework.cpp:140-158 on the device: permuting or deleting envs leaves every other
    env's step bit-identical, and equal to the reference's step of the same env."""
    cfg = m.make_default_config("foraging")
    gb = m.CudaEnvBatch(cfg, 3, fp64=True)
    gb.reset_seeds([1, 2, 3])
    st = list(gb.get_states())
    acts = np.array([1, 2, 3, 4, 0, 1, 2, 3, 4], dtype=np.int32)
    _, r0, _ = gb.step_host(acts)
    nxt = gb.get_states()
    gp = m.CudaEnvBatch(cfg, 3, fp64=True)
    gp.set_states([st[2], st[0], st[1]])
    _, rp, _ = gp.step_host(np.array([2, 3, 4, 1, 2, 3, 4, 0, 1], dtype=np.int32))
    pn = gp.get_states()
    assert list(pn[0].x[:3]) == list(nxt[2].x[:3]) and list(pn[1].y[:3]) == list(nxt[0].y[:3])
    assert rp[0] == r0[2]
    gs = m.CudaEnvBatch(cfg, 1, fp64=True)
    gs.set_states([st[1]])
    _, rs, _ = gs.step_host(np.array([4, 0, 1], dtype=np.int32))
    assert list(gs.get_states()[0].theta[:3]) == list(nxt[1].theta[:3]) and rs[0] == r0[1]
    rb = ref.RefBatch(ref.spec("foraging"))
    rb.reset([1, 2, 3])
    _, rr, _, _ = rb.step(acts)
    assert np.all(np.abs(rr - r0) <= 1e-9 * np.maximum(1, np.abs(rr)))


def test_scalar_equals_batched_on_device():
    """test_framework.cpp:114-138: 4 envs stepped as one batch equal 4 one-env batches bit-exactly."""
    cfg = m.make_default_config("random_waypoints")
    cfg.max_steps = 50
    seeds = [11, 22, 33, 44]
    gb = m.CudaEnvBatch(cfg, 4, fp64=True)
    gb.reset_seeds(seeds)
    ones = [m.CudaEnvBatch(cfg, 1, fp64=True) for _ in seeds]
    for o, s in zip(ones, seeds):
        o.reset_seeds([s])
    N = cfg.raw.num_robots
    for t in range(30):
        _, rb_, _ = gb.step_host(np.zeros((4, N), dtype=np.int32))
        bs = gb.get_states()
        for e, o in enumerate(ones):
            _, ro, _ = o.step_host(np.zeros((1, N), dtype=np.int32))
            s1 = o.get_states()[0]
            assert list(s1.x[:N]) == list(bs[e].x[:N]) and list(s1.theta[:N]) == list(bs[e].theta[:N])
            assert ro[0] == rb_[e]


@pytest.mark.parametrize("task,n", [("navigation", 4), ("discovery", 6), ("arctic_transport", 10)])
def test_random_permutation_of_a_large_batch_is_bit_identical(task, n):
    """Any env may land in any warp task of the persistent loop: a random permutation of 16,384
    envs (uploaded through the multi-threaded host state path) gives, per env, bit-identical
    states and rewards over 20 steps."""
    cfg = m.make_default_config(task)
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    if task == "arctic_transport":
        cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
    B = 16384
    perm = np.random.default_rng(7).permutation(B)
    a = m.CudaEnvBatch(cfg, B, fp64=True)
    a.reset_seeds([m.derive_episode_seed(3, e) for e in range(B)])
    st = list(a.get_states())
    b = m.CudaEnvBatch(cfg, B, fp64=True)
    b.set_states([st[i] for i in perm])
    rng = np.random.default_rng(1)
    for t in range(20):
        acts = rng.integers(0, 5, size=(B, n), dtype=np.int32)
        _, ra, _ = a.step_host(acts)
        _, rb_, _ = b.step_host(acts[perm])
        assert np.array_equal(ra[perm], rb_), t
    sa = np.ctypeslib.as_array(a.get_states())
    sb = np.ctypeslib.as_array(b.get_states())
    for f in ("x", "y", "theta", "step_index", "collisions", "scenario_metric", "min_pairwise_distance"):
        assert np.array_equal(sa[f][perm], sb[f]), f
