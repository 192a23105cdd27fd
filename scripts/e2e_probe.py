"""Where the host-API step time goes (one GPU, nav N=4, 65,536 envs, random
actions that change every step): device step alone, host step without / with
outputs, raw pinned D2H of the obs block."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06771_b200 as m  # noqa: E402

cfg = m.make_default_config("navigation")
cfg.set_num_robots(4)
cfg.max_steps = 70
B, K = 65536, 16
gb = m.CudaEnvBatch(cfg, B, auto_reset=True)
gb.reset_episodes(0)
acts = torch.from_numpy(np.random.default_rng(0).integers(0, 5, (K, B, 4), dtype=np.int32)).pin_memory().numpy()
outs = (torch.empty((B, 4, cfg.obs_dim), dtype=torch.float32).pin_memory().numpy(),
        torch.empty(B, dtype=torch.float64).pin_memory().numpy(), torch.empty(B, dtype=torch.uint8).pin_memory().numpy())
da = [torch.from_numpy(a.astype(np.int8)).cuda() for a in acts]
P = ctypes.POINTER(ctypes.c_int32)
k = [0]


def nxt():
    k[0] = (k[0] + 1) % K
    return k[0]


def t(fn, n=64):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print("device step (policy)      %.1f us" % t(lambda: gb.step(None)))
print("device step (int8 acts)   %.1f us" % t(lambda: gb.step(da[nxt()])))
print("host step, no outputs     %.1f us" % t(lambda: m.lib().mrsim_step_host(
    gb._h, acts[nxt()].ctypes.data_as(P), None, None, None, None)))
print("host step, all outputs    %.1f us" % t(lambda: gb.step_host(acts[nxt()], out=outs)))
print("host step, obs only       %.1f us" % t(lambda: m.lib().mrsim_step_host(
    gb._h, acts[nxt()].ctypes.data_as(P), outs[0].ctypes.data, None, None, None)))
print("host step, reward+done    %.1f us" % t(lambda: m.lib().mrsim_step_host(
    gb._h, acts[nxt()].ctypes.data_as(P), None, outs[1].ctypes.data, outs[2].ctypes.data, None)))
src = torch.empty((B, 4, cfg.obs_dim), dtype=torch.float32, device="cuda")
dst = torch.empty((B, 4, cfg.obs_dim), dtype=torch.float32).pin_memory()
print("pinned D2H 5.2 MB         %.1f us" % t(lambda: (dst.copy_(src, non_blocking=True), torch.cuda.synchronize())))
print("sync only                 %.1f us" % t(lambda: gb.sync()))
print("device step + sync each   %.1f us" % t(lambda: (gb.step(da[nxt()]), gb.sync())))
print("device step, obs to dev, + 5.2 MB D2H + sync  %.1f us" % t(lambda: (gb.step(da[nxt()]), dst.copy_(gb._obs, non_blocking=True), gb.sync())))
