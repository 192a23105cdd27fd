"""Where a step launch's time goes, per warp (diagnostic -DMRSIM_TASK_STATS build): entry, first
task start, last task end and busy time from %globaltimer for every warp of one launch, after an
L2 flush like bench.py. Usage: MRSIM_LIB_PATH=build/ab/lib_taskstats.so python scripts/warp_timeline.py
[task N envs]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06771_b200 as m  # noqa: E402

task = sys.argv[1] if len(sys.argv) > 1 else "navigation"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
B = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
cfg = m.make_default_config(task)
if n != cfg.raw.num_robots:
    cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
if task == "arctic_transport" and n > 4:
    cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
cfg.max_steps = 70 if task == "navigation" else cfg.max_steps
gb = m.CudaEnvBatch(cfg, B, auto_reset=True)
gb.reset_episodes(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
fn = getattr(m.lib(), f"mrsim_debug_warp_log_task{m.batch.TASKS.index(task)}")
W = 8192
out = (ctypes.c_ulonglong * (5 * W))()
spans = []
for it in range(12):
    flush.fill_(it & 0xff)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gb.step(None)
    b.record()
    torch.cuda.synchronize()
    if it < 4:
        continue
    fn(out, W)
    L = np.frombuffer(out, dtype=np.uint64).reshape(W, 5).astype(np.float64)
    L = L[L[:, 0] > 0]
    t0 = L[:, 0].min()
    enter, first, last, busy, ntask = (L[:, 0] - t0) / 1e3, (L[:, 1] - t0) / 1e3, (L[:, 2] - t0) / 1e3, L[:, 3] / 1e3, L[:, 4]
    span = last.max()
    ev = a.elapsed_time(b) * 1e3
    spans.append((ev, span, enter.max(), np.median(first - enter), busy.sum() / (len(L) * span),
                  np.percentile(last, 5), np.percentile(last, 50), np.percentile(last, 95),
                  ((last - first) - busy).mean() / np.maximum(ntask - 1, 1).mean(), ntask.mean(), len(L)))
print(f"{task} N={n} B={B}")
print("event_us span_us enter_spread_us first_delay_us busy_frac exit_p5 exit_p50 exit_p95 gap_per_task_us tasks/warp warps")
for r in spans:
    print(" ".join(f"{x:.2f}" for x in r))
