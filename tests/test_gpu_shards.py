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
