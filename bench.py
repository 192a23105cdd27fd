#!/usr/bin/env python
"""bench.py — env-steps/s (CBF on) of the B200-native batched Robotarium step.

Workload (BASELINE.json configs[1]): navigation, 4 robots, 65,536 parallel
envs per GPU, 70-step episodes, CBF barrier certificates on, harness random
policy (policy_stream(seed, step, robot).uniform_int(5), drawn on device),
in-kernel auto-reset with the harness's wave seeding. One "step" = one
batched env-step of every env (10 physics ticks each).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--task navigation --robots 4 --envs 65536] [--fp32]

The product path computes in fp64 (bit-exact discrete outcomes vs the
reference); --fp32 selects the fast mode.

Under torchrun each rank drives one GPU with its own contiguous env slice
(weak scaling, no collective in the step); the only cross-GPU traffic is the
final all-reduce of the timing max and the episode statistics.

Timing: W warm-up steps, then K steps; each step is bracketed by CUDA events
on the launching stream and the 126 MB L2 is flushed (a 512 MiB write)
between steps, outside the events; the per-step device times are summed.
`e2e` is the same metric through the host-buffer C-ABI call
(mrsim_step_host: actions H2D from pinned memory, obs/reward/done D2H,
synchronous), wall-clock timed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ARCTIC_SPAWN = [-1.55, -1.05, -0.9, 0.9]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--task", default="navigation")
    ap.add_argument("--robots", type=int, default=4)
    ap.add_argument("--envs", type=int, default=65536, help="envs per GPU")
    ap.add_argument("--max-steps", type=int, default=70)
    ap.add_argument("--fp32", action="store_true",
                    help="opt-in fp32 fast mode (forks from the reference at hold-rule near-ties)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--dist-backend", default="nccl", help="nccl (GPUs) or gloo (multi-rank smoke test)")
    ap.add_argument("--controller", default="unicycle_position", choices=["unicycle_position", "unicycle_pose"],
                    help="ControllerKind (framework.hpp:126)")
    ap.add_argument("--policy", default="random", choices=["random", "mlp", "scripted_goal", "prey_chaser"],
                    help="on-device policy producing each step's actions (mlp: a random 64-32 relu network)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(a) -> str:
    ctl = "" if a.controller == "unicycle_position" else ", pose controller"
    acts = "stored random waypoints" if a.task == "random_waypoints" else (
        "random actions" if a.policy == "random" else f"on-device {a.policy} policy")
    return f"{a.task} N={a.robots}, {a.envs} envs/GPU, {a.max_steps}-step episodes, CBF on{ctl}, {acts}"


def build_cfg(a):
    import paper_2505_06771_b200 as m

    cfg = m.make_default_config(a.task)
    if a.robots != cfg.raw.num_robots:
        cfg.set_num_robots(a.robots, tile_roster=cfg.raw.het_rows > 0)
    if a.task == "arctic_transport" and a.robots > 4:
        cfg.set_layout("arctic.spawn_zone", ARCTIC_SPAWN)
    cfg.max_steps = a.max_steps
    cfg.set_controller(a.controller)
    cfg.validate()
    return cfg


def ref_spec(a):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refbind  # test infrastructure: the reference compiled under oracle/_ref

    layout = {"arctic.spawn_zone": ARCTIC_SPAWN} if a.task == "arctic_transport" and a.robots > 4 else {}
    tile = a.task in ("discovery", "foraging", "material_transport", "arctic_transport", "warehouse")
    return refbind, refbind.spec(a.task, num_robots=a.robots, tile_roster=tile, max_steps=a.max_steps,
                                 layout=layout, controller=0 if a.controller == "unicycle_position" else 1)


def cpu_reference_rate(a, seconds: float, max_envs: int):
    """The reference step_batch with WorkerPool(all host cores) on a bounded sample."""
    refbind, sp = ref_spec(a)
    if not refbind.available():
        return None
    rb = refbind.RefBatch(sp, workers=0)
    cores = refbind.lib().ref_pool_size(rb.h)
    import paper_2505_06771_b200 as m

    B = min(max_envs, 4096)
    rb.reset([m.derive_episode_seed(0, e) for e in range(B)])
    t = rb.time_steps(2)  # warm + estimate
    rate = 2 * B / max(t, 1e-6)
    B = int(min(max_envs, max(1024, rate * seconds / 8)))
    rb.reset([m.derive_episode_seed(0, e) for e in range(B)])
    steps = max(2, int(seconds * rate / B))
    t = rb.time_steps(steps)
    return {"value": B * steps / t, "unit": "env-steps/s", "cores": cores, "kind": "reference",
            "sample": f"{B} envs x {steps} steps of step_batch (oracle/_ref, WorkerPool({cores}))",
            "robot_steps_per_s": B * steps * a.robots / t, "seconds": t}


def algorithmic_bytes_per_env_step(cfg, fp64: bool) -> int:
    """HBM bytes one env-step must move: state read+write,
    obs/reward/done written; actions are drawn on device."""
    R = 8 if fp64 else 4
    N = cfg.raw.num_robots
    nf, ni = cfg.task_fields()
    state = 3 * N * R + 4 + 3 * 8 + 8 + 3 * 4 + 3 * R + nf * R + ni * 4
    return 2 * state + 4 * N * cfg.obs_dim + 4 + 1


def algorithmic_flops_per_env_step(cfg) -> int:
    """F_step = 10*(82N + 28P) (+ task, ~10N) excluding QP iterations."""
    N = cfg.raw.num_robots
    P = N * (N - 1) // 2
    return cfg.raw.sub_steps * (82 * N + 28 * P) + 10 * N


class ClockSampler:
    def __init__(self, gpu: int):
        self.path = f"/tmp/mrsim_clocks_{os.getpid()}.csv"
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.impl == "reference":
        return main_reference(a, rank, world)

    import torch

    import paper_2505_06771_b200 as m

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    rdev = "cuda"
    if world > 1:
        import torch.distributed as dist

        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(a.dist_backend)
            rdev = "cpu"
    cfg = build_cfg(a)
    B = a.envs
    batch = m.CudaEnvBatch(cfg, B, device=local, fp64=(not a.fp32), auto_reset=True)
    batch.reset_episodes(root_seed=0, first_episode=rank * B, episode_stride=world * B)
    if a.policy == "mlp":
        batch.set_policy(m.FeedforwardWeights.random([cfg.obs_dim, 64, 32, 5], ["relu", "relu", "identity"], seed=1))
    elif a.policy != "random":
        batch.set_policy(a.policy)
    launches_per_step = 1 if a.policy == "random" else 2  # the policy kernel, then the step
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    for _ in range(max(a.warmup, 3)):
        batch.step(None)
    batch.sync()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    clocks = ClockSampler(local) if rank == 0 else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for k in range(a.steps):
        flush.zero_()  # L2 flush outside the timed events
        starts[k].record(stream)
        batch.step(None)
        ends[k].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    if dist:
        dist.barrier()
    batch.sync()
    clk = clocks.stop() if clocks else None
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t_local = torch.tensor([dev_ms], dtype=torch.float64, device=rdev)
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    dev_ms = float(t_local.item())
    value = world * B * a.steps / (dev_ms / 1e3)
    kernel_ms = dev_ms / a.steps

    # episode statistics: the only cross-GPU reduction (sum + min)
    st = batch.stats()
    red = torch.tensor([st["episodes"], st["sum_return"], st["sum_collisions"], st["sum_success"],
                        st["sum_qp_infeasible"]], dtype=torch.float64, device=rdev)
    mn = torch.tensor([st["min_pairwise_distance"]], dtype=torch.float64, device=rdev)
    if dist:
        dist.all_reduce(red)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)

    # e2e through the host-buffer C-ABI call (one GPU's share, then scaled by world for the job)
    e2e = None
    if a.e2e_steps > 0:
        rng = np.random.default_rng(rank)
        # pinned host buffers: the step's inputs (the reference's int actions) and its outputs
        acts = torch.from_numpy(rng.integers(0, 5, size=(a.e2e_steps, B, a.robots), dtype=np.int32)).pin_memory()
        acts_np = acts.numpy()
        outs = (torch.empty((B, a.robots, cfg.obs_dim), dtype=torch.float32).pin_memory().numpy(),
                torch.empty((B,), dtype=torch.float64).pin_memory().numpy(),
                torch.empty((B,), dtype=torch.uint8).pin_memory().numpy())
        hb = m.CudaEnvBatch(cfg, B, device=local, fp64=(not a.fp32), auto_reset=True)
        hb.reset_episodes(root_seed=0, first_episode=rank * B, episode_stride=world * B)
        hb.step_host(acts_np[0], out=outs)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(a.e2e_steps):
            hb.step_host(acts_np[k], out=outs)
        t_e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=rdev)
        if dist:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        h2d = B * a.robots * 4  # int32 actions (std::vector<int>)
        d2h = B * a.robots * cfg.obs_dim * 4 + B * 8 + B
        e2e = {"value": world * B * a.e2e_steps / float(t_e2e.item()), "unit": "env-steps/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "api": "mrsim_step_host, synchronous, pinned host buffers: the step kernel reads the int32 actions "
                      "and writes obs / reward / done in place over the host link (zero-copy), then syncs"}
        hb.close()

    if rank == 0:
        peaks = {}
        pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(pk):
            peaks = json.load(open(pk))
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        bpe = algorithmic_bytes_per_env_step(cfg, (not a.fp32))
        fpe = algorithmic_flops_per_env_step(cfg)
        per_gpu = value / world
        achieved_gbs = per_gpu * bpe / 1e9
        fp64 = not a.fp32
        pipe_peak = m.lib().mrsim_probe_fma_peak(local, int(fp64)) / 1e12  # measured FMA-chain peak
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                traffic = json.load(open(tf)).get(f"{a.task}{a.robots}_{'fp64' if (not a.fp32) else 'fp32'}")
            except Exception:
                traffic = None
        cpu = None
        if not a.no_cpu_baseline:
            cpu = cpu_reference_rate(a, a.cpu_seconds, B)
        line = {
            "metric": "env-steps/sec (CBF on)",
            "value": value,
            "unit": "env-steps/s",
            "robot_steps_per_s": value * a.robots,
            "n_gpus": world,
            "steps": a.steps,
            "warmup": max(a.warmup, 3),
            "ms_per_step": kernel_ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64" if (not a.fp32) else "f32",
            "data": "synthetic: harness random policy on device, derive_episode_seed(0, e) resets",
            "config": {"workload": workload_name(a), "task": a.task, "robots": a.robots, "envs_per_gpu": B,
                       "global_envs": B * world, "max_steps": a.max_steps, "sub_steps": cfg.raw.sub_steps,
                       "barrier": True, "auto_reset": True, "parallelism": f"env-shard x{world}",
                       "l2": "flushed (512 MiB write) between timed steps; per-step CUDA events summed"},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                         "algorithmic_bytes_per_env_step": bpe, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                         "pipe": {"pipe": "fp64" if fp64 else "fp32",
                                  "achieved_tflops": per_gpu * fpe / 1e12, "peak_tflops": pipe_peak,
                                  "frac": per_gpu * fpe / 1e12 / pipe_peak,
                                  "algorithmic_flops_per_env_step": fpe,
                                  "peak_source": "measured FMA-chain probe (mrsim_probe_fma_peak) on this GPU"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": a.steps * launches_per_step,
            "clocks": clk,
            "wall_s_timed_region": wall,
            "episodes": {"completed": float(red[0].item()),
                         "mean_return": float(red[1].item() / max(red[0].item(), 1)),
                         "collisions": float(red[2].item()), "success": float(red[3].item()),
                         "qp_infeasible": float(red[4].item()), "min_pairwise_distance": float(mn.item())},
        }
        print(json.dumps(line), flush=True)
    batch.close()
    if dist:
        dist.destroy_process_group()


def main_reference(a, rank, world):
    if rank != 0:
        return
    refbind, sp = ref_spec(a)
    if not refbind.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmrsim_ref.so not built"}))
        return
    import paper_2505_06771_b200 as m  # noqa: F401  (seed derivation only)

    rb = refbind.RefBatch(sp, workers=0)
    cores = refbind.lib().ref_pool_size(rb.h)
    B = min(a.envs, 2048)
    rb.reset([m.derive_episode_seed(0, e) for e in range(B)])
    t = rb.time_steps(max(a.warmup, 1))
    rate = max(a.warmup, 1) * B / max(t, 1e-6)
    budget = 150.0  # seconds for the whole timed run
    B = int(min(a.envs, max(256, rate * budget / max(a.steps, 1))))
    rb.reset([m.derive_episode_seed(0, e) for e in range(B)])
    rb.time_steps(max(a.warmup, 1))
    t = rb.time_steps(a.steps)
    value = B * a.steps / t
    sample = f"{B} of {a.envs} envs per step x {a.steps} steps (step_batch, WorkerPool({cores}))"
    print(json.dumps({
        "impl": "reference", "metric": "env-steps/sec (CBF on)", "value": value, "unit": "env-steps/s",
        "robot_steps_per_s": value * a.robots, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": t / a.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: harness random policy, derive_episode_seed(0, e) resets",
        "config": {"workload": workload_name(a), "task": a.task, "robots": a.robots, "envs_per_gpu": a.envs,
                   "max_steps": a.max_steps, "barrier": True},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
