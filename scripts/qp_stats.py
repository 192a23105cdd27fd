"""Diagnostic (needs a -DMRSIM_QP_STATS build in MRSIM_LIB_PATH): QP solves, warm-start attempts
and fallbacks, and outer iterations per solve, for one task over a few steps of the bench workload."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06771_b200 as m  # noqa: E402

task, n, B, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = m.make_default_config(task)
if n != cfg.raw.num_robots:
    cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
if task == "arctic_transport" and n > 4:
    cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
gb = m.CudaEnvBatch(cfg, B, auto_reset=True)
gb.reset_episodes(0)
fn = getattr(m.lib(), f"mrsim_debug_qp_stats_task{m.batch.TASKS.index(task)}")
out = (ctypes.c_ulonglong * 8)()
fn(out, 1)
for _ in range(steps):
    gb.step(None)
gb.sync()
fn(out, 0)
solves, att, dep, neg, it = out[0], out[1], out[2], out[3], out[4]
print(f"{task} N={n}: solves {solves}, outer iterations {it} ({it / max(solves, 1):.2f}/solve), warm attempts {att} "
      f"({att / max(solves, 1):.2f}/solve), fallbacks dependent {dep}, negative multiplier {neg} "
      f"({(dep + neg) / max(att, 1):.1%} of attempts)")
