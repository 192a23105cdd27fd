"""Diagnostic (needs a -DMRSIM_TASK_STATS build in MRSIM_LIB_PATH): distribution of warp-task
durations (SM cycles) of the step kernel over a few steps of the bench workload."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06771_b200 as m  # noqa: E402

task, n, B, steps, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
cfg = m.make_default_config(task)
if n != cfg.raw.num_robots:
    cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
if task == "arctic_transport" and n > 4:
    cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])  # bench.py ARCTIC_SPAWN
cfg.max_steps = T
gb = m.CudaEnvBatch(cfg, B, auto_reset=True)
gb.reset_episodes(0)
for _ in range(5):
    gb.step(None)
gb.sync()
fn = getattr(m.lib(), f"mrsim_debug_task_hist_task{m.batch.TASKS.index(task)}")
out = (ctypes.c_ulonglong * 64)()
fn(out, 1)
for _ in range(steps):
    gb.step(None)
gb.sync()
fn(out, 0)
tot = sum(out[:48])
print(f"{task} N={n} B={B}: {tot} warp-tasks, mean {out[48] / max(tot, 1):.0f} cycles")
for b in range(48):
    if out[b]:
        print(f"  [{2**b:>9}, {2**(b+1):>9}) cycles: {out[b]:8d} ({out[b] / tot:.1%})")
