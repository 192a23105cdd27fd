"""Cost of zero-copy obs on the host-API step (nav N=4, 65,536 envs): host steps alternate between
writing obs to pinned host memory and writing none (same episode phase for both classes); CUDA
events on the legacy stream bracket each synchronous call (kernel + its launch gap), and the
host wall time of each call is taken too."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06771_b200 as m  # noqa: E402

cfg = m.make_default_config("navigation")
cfg.set_num_robots(4)
cfg.max_steps = 70
B = 65536
gb = m.CudaEnvBatch(cfg, B, auto_reset=True)
gb.reset_episodes(0)
acts = torch.from_numpy(np.random.default_rng(0).integers(0, 5, (B, 4), dtype=np.int32)).pin_memory().numpy()
obs = torch.empty((B, 4, cfg.obs_dim), dtype=torch.float32).pin_memory().numpy()
P = ctypes.POINTER(ctypes.c_int32)
import time
ev = {True: [], False: []}
wall = {True: [], False: []}
ap = acts.ctypes.data_as(P)
for i in range(80):
    with_obs = i % 2 == 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    m.lib().mrsim_step_host(gb._h, ap, obs.ctypes.data if with_obs else None, None, None, None)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    if i >= 10:
        ev[with_obs].append(a.elapsed_time(b) * 1e3)
        wall[with_obs].append((t1 - t0) * 1e6)
for k in (True, False):
    print("obs" if k else "none", "events %.1f us (median %.1f)" % (np.mean(ev[k]), np.median(ev[k])),
          "wall %.1f us (median %.1f)" % (np.mean(wall[k]), np.median(wall[k])))
