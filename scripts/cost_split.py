"""Where a navigation step's time goes: the same workload with the CBF filter
on / off and with / without observation output (device-resident, 65,536
envs, CUDA-event timed). Diagnostic only."""
import sys

import torch

import paper_2505_06771_b200 as m

task, n = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("navigation", 4)
for barrier in (1, 0):
    for want_obs in (True, False):
        cfg = m.make_default_config(task)
        if n != cfg.raw.num_robots:
            cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
        if task == "arctic_transport" and n > 4:
            cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
        cfg.max_steps = 70
        cfg.barrier_enabled = barrier
        gb = m.CudaEnvBatch(cfg, 65536, auto_reset=True)
        gb.reset_episodes(0)
        for _ in range(10):
            gb.step(None, want_obs=want_obs)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(200):
            gb.step(None, want_obs=want_obs)
        b.record()
        torch.cuda.synchronize()
        print(f"{task} N={n} barrier={barrier} obs={want_obs}: {a.elapsed_time(b) / 200 * 1000:.1f} us/step")
        gb.close()
