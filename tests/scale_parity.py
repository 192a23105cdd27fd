"""Parity at the benchmarked batch sizes (TEST INFRASTRUCTURE: the checker for
tests/test_gpu_scale.py and `bench.py --verify`; the reference runs from
oracle/_ref).

The reference makes results independent of how the batch is partitioned
(/root/reference/proj/include/mrsim/batch.hpp:3-6; test_framework.cpp:140-158,
200-230), so every env of the persistent kernel -- whichever warp or thread
takes it, in whichever iteration of the task loop -- must match the reference
stepping the same env. The device runs the exact bench workload (auto-reset,
harness random policy drawn on device, wave seeding of run_episodes,
harness.hpp:227-232); the reference steps the same envs with
policy_stream actions and re-seeds env e of wave w with
derive_episode_seed(root, w*B + e) at the horizon.

Comparison (fp64 product path): discrete fields bit-exact; poses within
1e-8 m / 1e-7 rad, reals within 1e-8; per-step done exact; per-step fp32
rewards within one fp32 rounding of the reference's double reward.
States are compared vectorised over numpy views of the mrsim_env_state arrays.
"""
from __future__ import annotations

import time

import numpy as np

import paper_2505_06771_b200 as m
from paper_2505_06771_b200 import _abi

DISCRETE = ("step_index", "collisions", "qp_infeasible", "success", "flash_timer", "sensed", "tagged",
            "slot_shelf", "carried", "requests", "levels", "foraged", "tiles", "loaded", "rng_key", "seed")
REALS = ("scenario_metric", "circle_remaining", "rect_remaining", "delivered", "total_initial", "loads",
         "goals", "landmarks", "resources", "prey", "targets", "target_headings",
         "min_pairwise_distance")


def compare_arrays(ga, ra, N: int) -> dict:
    """Vectorised state comparison of two mrsim_env_state ctypes arrays."""
    g = np.ctypeslib.as_array(ga)
    r = np.ctypeslib.as_array(ra)
    out = {"envs": int(g.shape[0])}
    out["pose"] = float(max(np.max(np.abs(g["x"][:, :N] - r["x"][:, :N])),
                            np.max(np.abs(g["y"][:, :N] - r["y"][:, :N]))))
    d = g["theta"][:, :N] - r["theta"][:, :N]
    out["angle"] = float(np.max(np.abs(np.remainder(d + np.pi, 2 * np.pi) - np.pi)))
    bad = {}
    for f in DISCRETE:
        a, b = g[f], r[f]
        neq = (a != b).reshape(a.shape[0], -1).any(axis=1)
        if neq.any():
            bad[f] = np.nonzero(neq)[0][:8].tolist()
    out["discrete_mismatch"] = bad
    rmax = 0.0
    for f in REALS:
        a, b = g[f].astype(np.float64), r[f].astype(np.float64)
        both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
        with np.errstate(invalid="ignore"):
            diff = np.where(both_inf, 0.0, np.abs(a - b))
        rmax = max(rmax, float(np.max(diff)) if diff.size else 0.0)
    out["real"] = rmax
    return out


def run_full_batch(ref, cfg, sp, B: int, steps: int, root: int = 0, every: int = 10, workers: int = 0,
                   device: int = 0) -> dict:
    """Every env of a B-env auto-reset device batch against the reference stepping all B envs."""
    N = cfg.raw.num_robots
    T = cfg.raw.max_steps
    gb = m.CudaEnvBatch(cfg, B, device=device, fp64=True, auto_reset=True)
    gb.reset_episodes(root_seed=root, first_episode=0, episode_stride=B)
    rb = ref.RefBatch(sp, workers=workers)
    rb.reset([m.derive_episode_seed(root, e) for e in range(B)])
    rep = {"B": B, "steps": steps, "checks": 0, "worst_pose": 0.0, "worst_angle": 0.0, "worst_real": 0.0,
           "discrete_mismatch": {}, "done_mismatch": 0, "reward_bad": 0, "waves": 0, "ok": True}
    t0 = time.time()
    import torch
    for t in range(steps):
        out = gb.step(None)
        acts = rb.random_actions()
        _, rrew, rdone, _ = rb.step(acts)
        torch.cuda.synchronize()
        gb.sync()
        gdone = out.done.cpu().numpy().astype(bool)
        grew = out.reward.cpu().numpy().astype(np.float64)
        rep["done_mismatch"] += int(np.sum(gdone != rdone.astype(bool)))
        tol = 1.2e-7 * np.maximum(1.0, np.abs(rrew))  # one fp32 rounding of the double reward
        rep["reward_bad"] += int(np.sum(np.abs(grew - rrew) > tol))
        wave_end = (t + 1) % T == 0
        if wave_end:  # run_episodes: the next wave re-seeds env e as episode w*B + e
            rep["waves"] += 1
            rb.reset([m.derive_episode_seed(root, rep["waves"] * B + e) for e in range(B)])
        if (t + 1) % every == 0 or wave_end or t == steps - 1:
            c = compare_arrays(gb.get_states(), rb.get_states(), N)
            rep["checks"] += 1
            rep["worst_pose"] = max(rep["worst_pose"], c["pose"])
            rep["worst_angle"] = max(rep["worst_angle"], c["angle"])
            rep["worst_real"] = max(rep["worst_real"], c["real"])
            for f, idx in c["discrete_mismatch"].items():
                rep["discrete_mismatch"].setdefault(f, (t, idx))
    st = gb.stats()
    rep["device_episodes"] = st["episodes"]
    rep["device_success"] = st["sum_success"]
    rep["device_collisions"] = st["sum_collisions"]
    rep["seconds"] = time.time() - t0
    rep["ok"] = (not rep["discrete_mismatch"] and rep["done_mismatch"] == 0 and rep["reward_bad"] == 0 and
                 rep["worst_pose"] <= 1e-8 and rep["worst_angle"] <= 1e-7 and rep["worst_real"] <= 1e-8 and
                 rep["device_episodes"] == rep["waves"] * B)
    gb.close()
    rb.close()
    return rep


def run_sampled(ref, cfg, sp, B: int, steps: int, ranges, root: int = 0, every: int = 10, device: int = 0) -> dict:
    """A B-env device batch; the reference steps only the envs in `ranges` (contiguous slices that
    span many warp tasks) with the same per-env seeds and policy_stream actions."""
    N = cfg.raw.num_robots
    T = cfg.raw.max_steps
    envs = np.concatenate([np.arange(a, b) for a, b in ranges])
    gb = m.CudaEnvBatch(cfg, B, device=device, fp64=True, auto_reset=True)
    gb.reset_episodes(root_seed=root, first_episode=0, episode_stride=B)
    rb = ref.RefBatch(sp, workers=0)
    rb.reset([m.derive_episode_seed(root, int(e)) for e in envs])
    rep = {"B": B, "sample": int(envs.size), "steps": steps, "checks": 0, "worst_pose": 0.0, "worst_angle": 0.0,
           "worst_real": 0.0, "discrete_mismatch": {}, "done_mismatch": 0, "reward_bad": 0, "waves": 0}
    import torch
    for t in range(steps):
        out = gb.step(None)
        _, rrew, rdone, _ = rb.step(rb.random_actions())
        torch.cuda.synchronize()
        gb.sync()
        gdone = out.done.cpu().numpy().astype(bool)[envs]
        grew = out.reward.cpu().numpy().astype(np.float64)[envs]
        rep["done_mismatch"] += int(np.sum(gdone != rdone.astype(bool)))
        rep["reward_bad"] += int(np.sum(np.abs(grew - rrew) > 1.2e-7 * np.maximum(1.0, np.abs(rrew))))
        wave_end = (t + 1) % T == 0
        if wave_end:
            rep["waves"] += 1
            rb.reset([m.derive_episode_seed(root, rep["waves"] * B + int(e)) for e in envs])
        if (t + 1) % every == 0 or wave_end or t == steps - 1:
            parts = [gb.get_states(a, b - a) for a, b in ranges]
            gs = [s for p in parts for s in p]
            garr = (_abi.EnvState * len(gs))(*gs)
            c = compare_arrays(garr, rb.get_states(), N)
            rep["checks"] += 1
            rep["worst_pose"] = max(rep["worst_pose"], c["pose"])
            rep["worst_angle"] = max(rep["worst_angle"], c["angle"])
            rep["worst_real"] = max(rep["worst_real"], c["real"])
            for f, idx in c["discrete_mismatch"].items():
                rep["discrete_mismatch"].setdefault(f, (t, [int(envs[i]) for i in idx]))
    rep["ok"] = (not rep["discrete_mismatch"] and rep["done_mismatch"] == 0 and rep["reward_bad"] == 0 and
                 rep["worst_pose"] <= 1e-8 and rep["worst_angle"] <= 1e-7 and rep["worst_real"] <= 1e-8)
    gb.close()
    rb.close()
    return rep
