"""mrsim_rollout: num_steps fused steps in one launch (the harness random policy on device)
must equal num_steps calls of mrsim_step(actions = NULL) bit for bit -- states, per-step
obs / rewards / dones and episode statistics -- across episode boundaries (in-kernel
auto-reset), and a failing rollout is rolled back as a whole."""
import numpy as np
import pytest
import torch

import paper_2505_06771_b200 as m
from scale_parity import compare_arrays

pytestmark = pytest.mark.gpu


def _cfg(task, n):
    cfg = m.make_default_config(task)
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    if task == "arctic_transport" and n > 4:
        cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
    cfg.max_steps = 25
    return cfg


@pytest.mark.parametrize("task,n", [("navigation", 4), ("rware", 6), ("discovery", 6), ("material_transport", 10),
                                    ("arctic_transport", 10), ("predator_prey", 6)])
def test_rollout_equals_single_steps(task, n):
    cfg = _cfg(task, n)
    B, T = 3001, 60  # crosses two auto-resets; a partial last warp task
    a = m.CudaEnvBatch(cfg, B, fp64=True, auto_reset=True)
    b = m.CudaEnvBatch(cfg, B, fp64=True, auto_reset=True)
    a.reset_episodes(root_seed=4)
    b.reset_episodes(root_seed=4)
    obs, rew, done = [], [], []
    for _ in range(T):
        out = a.step(None)
        obs.append(out.obs.clone())
        rew.append(out.reward.clone())
        done.append(out.done.clone())
    ro = b.rollout(T)
    torch.cuda.synchronize()
    a.sync()
    b.sync()
    assert torch.equal(torch.stack(rew), ro.reward) and torch.equal(torch.stack(done), ro.done)
    assert torch.equal(torch.stack(obs), ro.obs)
    c = compare_arrays(a.get_states(), b.get_states(), n)
    assert not c["discrete_mismatch"] and c["pose"] == 0 and c["angle"] == 0 and c["real"] == 0, c
    sa, sb = a.stats(), b.stats()
    for k in ("episodes", "env_steps", "sum_collisions", "sum_return", "sum_metric", "sum_success"):
        assert sa[k] == sb[k], k


def test_rollout_in_chunks_and_mixed_with_steps():
    cfg = _cfg("navigation", 4)
    B = 1003  # a partial last warp task (ghost groups)
    a = m.CudaEnvBatch(cfg, B, fp64=True, auto_reset=True)
    b = m.CudaEnvBatch(cfg, B, fp64=True, auto_reset=True)
    a.reset_episodes(root_seed=9)
    b.reset_episodes(root_seed=9)
    a.rollout(40)
    for _ in range(7):
        b.step(None)
    b.rollout(20)
    for _ in range(13):
        b.step(None)
    a.sync()
    b.sync()
    c = compare_arrays(a.get_states(), b.get_states(), 4)
    assert not c["discrete_mismatch"] and c["pose"] == 0, c


def test_failing_rollout_rolls_back_and_policy_requirement():
    cfg = m.make_default_config("navigation")
    cfg.max_steps = 5
    gb = m.CudaEnvBatch(cfg, 16, auto_reset=True)
    gb.reset_episodes(root_seed=1)
    gb.rollout(12)  # two finished episodes per env
    gb.sync()
    before_stats = gb.stats()
    st = list(gb.get_states())
    st[7].x[1], st[7].y[1], st[7].theta[1] = st[7].x[0], st[7].y[0], st[7].theta[0]
    gb.set_states(st)
    gb.rollout(12)
    with pytest.raises(m.DomainError, match="environment 7"):
        gb.sync()
    after = gb.get_states()
    assert [list(s.x[:3]) for s in after] == [list(s.x[:3]) for s in st]
    assert gb.stats()["episodes"] == before_stats["episodes"]
    gb.set_policy(m.FeedforwardWeights.random([cfg.obs_dim, 8, 5], ["relu", "identity"], seed=1))
    with pytest.raises(m.Unsupported):
        gb.rollout(3)
