"""Small-B exercise of every device kernel, for compute-sanitizer (memcheck /
racecheck / synccheck; one tool per run): lane-group step kernels for L = 4 / 8
/ 16 (+ rware obstacle rows), the one-thread-per-env kernel, reset / observe /
random-actions, the feedforward and scripted policy kernels, trajectory
capture, auto-reset, the error / rollback path, and the QP unit kernel."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_06771_b200 as m  # noqa: E402

CASES = [("navigation", 4, {}), ("navigation", 4, {"env_per_thread": True}), ("rware", 4, {}),
         ("discovery", 6, {}), ("predator_prey", 6, {}), ("material_transport", 10, {}),
         ("arctic_transport", 10, {}), ("warehouse", 4, {"env_per_thread": True}),
         ("random_waypoints", 4, {})]
for task, n, kw in CASES:
    cfg = m.make_default_config(task)
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    if task == "arctic_transport" and n > 4:
        cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
    cfg.max_steps = 6
    B = 70  # several warps / warp tasks, a partial last warp
    gb = m.CudaEnvBatch(cfg, B, auto_reset=True, **kw)
    gb.reset_episodes(root_seed=1)
    for _ in range(8):  # crosses an auto-reset
        gb.step(None, want_next_obs=True)
    gb.sync()
    gb.observe()
    gb.random_actions()
    gb.set_policy(m.FeedforwardWeights.random([cfg.obs_dim, 32, 5], ["relu", "identity"], seed=1))
    gb.step(None)
    gb.set_policy("scripted_goal")
    gb.step(None)
    gb.sync()
    hb = m.CudaEnvBatch(cfg, 9, **kw)
    hb.reset_seeds(list(range(9)))
    acts = np.zeros((9, n), dtype=np.int32)
    hb.step_host(acts)
    acts[4, 0] = 9
    try:
        hb.step_host(acts)
    except m.InvalidArgument:
        pass
    hb.step_host(np.zeros((9, n), dtype=np.int32))
    print("ok", task, n, kw, flush=True)
cfg = m.make_default_config("navigation")
cb = m.CudaEnvBatch(cfg, 5)
cb.reset_seeds(list(range(5)))
lib = m.lib()
rc = lib.mrsim_capture_begin(cb._h, 4)
assert rc == 0
for _ in range(3):
    cb.step(None)
cb.sync()
lib.mrsim_capture_end(cb._h)
torch.cuda.synchronize()
print("sanitize smoke done")
