#!/usr/bin/env python
"""bench.py — env-steps/s (CBF on) of the B200-native batched Robotarium step.

Workload (BASELINE.json configs[1]): navigation, 4 robots, 65,536 parallel
envs per GPU, 70-step episodes, CBF barrier certificates on, harness random
policy (policy_stream(seed, step, robot).uniform_int(5), drawn on device),
in-kernel auto-reset with the harness's wave seeding. One "step" = one
batched env-step of every env (10 physics ticks each).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--task navigation --robots 4 --envs 65536] [--fp32] [--verify]

The product path computes in fp64 (bit-exact discrete outcomes vs the
reference); --fp32 selects the non-parity fast mode.

Multi-GPU (BASELINE metric "at 1/2/4/8 B200"): one process per
GPU, each with its own contiguous env slice (multigpu.Shard: weak scaling, no
collective in the step); the only cross-GPU traffic is the all-reduce of the
timing max and of the episode statistics (multigpu.reduce_stats). Under
torchrun the ranks come from the environment; `--gpus N` without torchrun
launches the N ranks itself (torch.distributed.run on 127.0.0.1). With fewer
visible GPUs than ranks the ranks share devices over gloo (a functional
check of the multi-rank path, not a scaling number).

Timing: W warm-up steps, then K steps; each step is bracketed by CUDA events
on the launching stream and the 126 MB L2 is flushed (a 512 MiB read, so no
dirty lines are written back inside the next step) between steps, outside
the events; the per-step device times are summed, max over ranks.
`e2e` is the same metric through the host-buffer C-ABI call
(mrsim_step_host: int32 actions from pinned host memory, obs / reward / done
to pinned host memory, synchronous), wall-clock timed, max over ranks.
`--verify` then checks every env of the bench batch against the reference
over 150 steps (tests/scale_parity.py; test infrastructure as the checker).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ARCTIC_SPAWN = [-1.55, -1.05, -0.9, 0.9]
METRIC = "env-steps/sec (CBF on)"


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
                    help="opt-in fp32 fast mode (not parity-grade: forks from the reference at hold-rule near-ties)")
    ap.add_argument("--env-per-thread", action="store_true",
                    help="teams of <= 4 robots: one thread per env instead of the lane-per-robot kernel (A/B)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--dist-backend", default="auto",
                    help="nccl | gloo | auto (nccl when every rank has its own GPU, else gloo)")
    ap.add_argument("--controller", default="unicycle_position", choices=["unicycle_position", "unicycle_pose"],
                    help="ControllerKind (framework.hpp:126)")
    ap.add_argument("--policy", default="random", choices=["random", "mlp", "scripted_goal", "prey_chaser"],
                    help="on-device policy producing each step's actions (mlp: a random 64-32 relu network)")
    ap.add_argument("--no-flush", action="store_true", help="no L2 flush between timed steps (traffic windows)")
    ap.add_argument("--rollout", type=int, default=10,
                    help="also time fused rollouts of this many steps per launch (mrsim_rollout; 0: skip)")
    ap.add_argument("--verify", action="store_true",
                    help="after the bench, check every env of the bench batch against the reference (150 steps)")
    ap.add_argument("--dump-states", default="", help="write each rank's final env states to PATH.rank<r>.npz")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def launch_ranks(a) -> int:
    """`--gpus N` without torchrun: start the N ranks (one process per GPU) on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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


def bench_config(a, cfg, world: int) -> dict:
    """The `config` object of both arms (same keys, same values)."""
    return {"workload": workload_name(a), "task": a.task, "robots": a.robots, "envs_per_gpu": a.envs,
            "global_envs": a.envs * world, "max_steps": a.max_steps, "sub_steps": int(cfg.raw.sub_steps),
            "barrier": True, "auto_reset": True, "controller": a.controller, "policy": a.policy,
            "parallelism": f"env-shard x{world}",
            "l2": "flushed (512 MiB read) between timed steps; per-step CUDA events summed"}


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


def measured_traffic(a, fp64: bool):
    """dram__bytes_read.sum + dram__bytes_write.sum per step-kernel launch, averaged over a window of
    consecutive launches of this bench loop (scripts/measure_traffic.sh, ncu; profiles/traffic_r02.json)."""
    path = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if not os.path.exists(path):
        return None
    try:
        rec = json.load(open(path)).get(f"{a.task}{a.robots}_{a.envs}_{'fp64' if fp64 else 'fp32'}")
    except Exception:
        return None
    return rec


def roofline(a, cfg, per_gpu: float, kernel_ms: float, fp64: bool, pipe_peak_tflops: float) -> dict:
    """The binding roof is chosen by arithmetic intensity against the ridge point."""
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    bpe = algorithmic_bytes_per_env_step(cfg, fp64)
    fpe = algorithmic_flops_per_env_step(cfg)
    ai = fpe / bpe
    ridge = pipe_peak_tflops * 1e12 / (hbm_peak * 1e9)
    gbs = per_gpu * bpe / 1e9
    tflops = per_gpu * fpe / 1e12
    pipe = "fp64" if fp64 else "fp32"
    tr = measured_traffic(a, fp64)
    envs_per_launch = a.envs
    hbm = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
           "algorithmic_bytes_per_env_step": bpe, "algorithmic_bytes_per_launch": bpe * envs_per_launch,
           "peak_source": hbm_src}
    comp = {"achieved": tflops, "peak": pipe_peak_tflops, "unit": "TFLOP/s", "frac": tflops / pipe_peak_tflops,
            "algorithmic_flops_per_env_step": fpe, "algorithmic_flops_per_launch": fpe * envs_per_launch,
            "peak_source": f"measured {pipe} FMA-chain probe (mrsim_probe_fma_peak) on this GPU"}
    bound_pipe = ai >= ridge
    out = dict(comp if bound_pipe else hbm)
    out["bound"] = f"{pipe}-pipe" if bound_pipe else "hbm"
    out["arithmetic_intensity"] = ai
    out["ridge_flop_per_byte"] = ridge
    out["traffic"] = tr["bytes_per_launch"] if tr else None
    out["traffic_window"] = tr
    out["hbm"] = hbm
    out[pipe] = comp
    out["kernel_ms"] = kernel_ms
    return out


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled from a thread
    every ~1 ms (the timed region of a short run lasts a few ms), nvidia-smi as the fallback."""
    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        import threading

        self.samples, self.mx, self.reasons = [], 0.0, set()
        self.stop_ev = threading.Event()
        self.proc = None
        self.thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop_ev.is_set():
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(k for k, v in bits.items() if r & v)
                    time.sleep(0.001)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.source = "nvml"
        except Exception:
            self.source = "nvidia-smi"
            self.path = f"/tmp/mrsim_clocks_{os.getpid()}.csv"
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except Exception:
                self.proc = None

    def wait_first(self, timeout: float = 2.0) -> None:
        t0 = time.time()
        while self.thread is not None and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.0005)

    def mark(self) -> int:
        return len(self.samples)

    def stop(self, since: int = 0):
        if self.thread is not None:
            self.stop_ev.set()
            self.thread.join()
            sm = self.samples[since:] or self.samples[-1:]
            if not sm:
                return None
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                    "samples": len(sm), "source": "nvml, 1 ms polling during the timed region"}
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0, set()
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(self.REASONS, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi -lms 50"}


def finite(v):
    return v if v is None or np.isfinite(v) else None


def dump_states(path: str, rank: int, shard, batch) -> None:
    from paper_2505_06771_b200 import _abi  # noqa: F401

    st = np.ctypeslib.as_array(batch.get_states())
    np.savez(f"{path}.rank{rank}.npz", first_episode=shard.first_episode,
             **{f: st[f] for f in ("x", "y", "theta", "step_index", "collisions", "rng_key", "episode",
                                   "scenario_metric", "success", "min_pairwise_distance")})


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(a))
    if a.impl == "reference":
        return main_reference(a, rank, world)

    import torch

    import paper_2505_06771_b200 as m
    from paper_2505_06771_b200.multigpu import Shard, reduce_stats

    ndev = max(torch.cuda.device_count(), 1)
    local = local % ndev
    torch.cuda.set_device(local)
    backend = a.dist_backend if a.dist_backend != "auto" else ("nccl" if world <= ndev else "gloo")
    dist = None
    rdev = "cuda"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / NVLS lines ...
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout is the JSON line
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
            rdev = "cpu"
    shard = Shard(rank, world, a.envs)
    cfg = build_cfg(a)
    B = a.envs
    batch = m.CudaEnvBatch(cfg, B, device=local, fp64=(not a.fp32), auto_reset=True, env_per_thread=a.env_per_thread)
    batch.reset_episodes(root_seed=0, first_episode=shard.first_episode, episode_stride=shard.episode_stride)
    if a.policy == "mlp":
        batch.set_policy(m.FeedforwardWeights.random([cfg.obs_dim, 64, 32, 5], ["relu", "relu", "identity"], seed=1))
    elif a.policy != "random":
        batch.set_policy(a.policy)
    launches_per_step = 1 if a.policy == "random" else 2  # the policy kernel, then the step
    stream = torch.cuda.current_stream()
    flush = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")

    for _ in range(max(a.warmup, 3)):
        batch.step(None)
    batch.sync()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.wait_first()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    mark = clocks.mark() if clocks else 0
    w0 = time.perf_counter()
    for k in range(a.steps):
        if not a.no_flush:
            torch.sum(flush, dim=0, out=sink)  # L2 flush (read-only) outside the timed events
        starts[k].record(stream)
        batch.step(None)
        ends[k].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    if dist:
        dist.barrier()
    batch.sync()
    clk = clocks.stop(mark) if clocks else None
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t_local = torch.tensor([dev_ms], dtype=torch.float64, device=rdev)
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    dev_ms = float(t_local.item())
    value = world * B * a.steps / (dev_ms / 1e3)
    kernel_ms = dev_ms / a.steps

    # fused rollouts (mrsim_rollout: T steps per launch, state kept on chip across them), reported
    # beside the per-step launches; same workload, same outputs per step, L2 flushed between launches
    rollout = None
    if a.rollout > 1 and a.policy == "random" and not a.env_per_thread:
        T = a.rollout
        launches = max(1, a.steps // T)
        ro_out = (None, torch.empty((T, B), dtype=torch.float32, device="cuda"),
                  torch.empty((T, B), dtype=torch.uint8, device="cuda"))
        ro_obs = torch.empty((T, B, a.robots, cfg.obs_dim), dtype=torch.float32, device="cuda")
        # a twin batch at the same episode phase as the per-step measurement: same reset, same warm-up
        rb = m.CudaEnvBatch(cfg, B, device=local, fp64=(not a.fp32), auto_reset=True)
        rb.reset_episodes(root_seed=0, first_episode=shard.first_episode, episode_stride=shard.episode_stride)
        for _ in range(max(a.warmup, 3)):
            rb.step(None)
        rs = [torch.cuda.Event(enable_timing=True) for _ in range(launches)]
        re_ = [torch.cuda.Event(enable_timing=True) for _ in range(launches)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(launches):
            if not a.no_flush:
                torch.sum(flush, dim=0, out=sink)
            rs[k].record(stream)
            rb.rollout(T, out=(ro_obs, ro_out[1], ro_out[2]))
            re_[k].record(stream)
        torch.cuda.synchronize()
        rb.sync()
        rb.close()
        r_ms = torch.tensor([sum(x.elapsed_time(y) for x, y in zip(rs, re_))], dtype=torch.float64, device=rdev)
        if dist:
            dist.all_reduce(r_ms, op=dist.ReduceOp.MAX)
        r_ms = float(r_ms.item())
        rollout = {"steps_per_launch": T, "launches": launches,
                   "value": world * B * T * launches / (r_ms / 1e3), "unit": "env-steps/s",
                   "ms_per_env_step_of_the_batch": r_ms / (T * launches),
                   "what": "mrsim_rollout: T fused steps per launch, bit-identical to T mrsim_step calls "
                           "(tests/test_gpu_rollout.py), on a twin batch over the same steps of the same "
                           "episodes as `value`; per-step obs / reward / done written; L2 flushed between "
                           "launches"}
        del ro_obs, ro_out

    # episode statistics: the only cross-GPU reduction (sum + min), multigpu.reduce_stats
    stats = reduce_stats(batch.stats(), device=rdev)
    if a.dump_states:
        dump_states(a.dump_states, rank, shard, batch)

    # e2e through the host-buffer C-ABI call (every rank, max over ranks)
    e2e = None
    if a.e2e_steps > 0:
        rng = np.random.default_rng(rank)
        # pinned host buffers: the step's inputs (the reference's int actions) and its outputs
        n_warm = max(3, a.warmup)  # untimed host steps first, like the device-timed loop
        acts = torch.from_numpy(rng.integers(0, 5, size=(a.e2e_steps + n_warm, B, a.robots),
                                             dtype=np.int32)).pin_memory()
        acts_np = acts.numpy()
        outs = (torch.empty((B, a.robots, cfg.obs_dim), dtype=torch.float32).pin_memory().numpy(),
                torch.empty((B,), dtype=torch.float64).pin_memory().numpy(),
                torch.empty((B,), dtype=torch.uint8).pin_memory().numpy())
        hb = m.CudaEnvBatch(cfg, B, device=local, fp64=(not a.fp32), auto_reset=True, env_per_thread=a.env_per_thread)
        hb.reset_episodes(root_seed=0, first_episode=shard.first_episode, episode_stride=shard.episode_stride)
        for k in range(n_warm):
            hb.step_host(acts_np[a.e2e_steps + k], out=outs)
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

    verify = None
    if a.verify and rank == 0:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import scale_parity  # test infrastructure: the checker (oracle/_ref)

        refbind, sp = ref_spec(a)
        verify = scale_parity.run_full_batch(refbind, cfg, sp, B, 150, device=local)
        verify = {k: v for k, v in verify.items() if k not in ("discrete_mismatch",)} | {
            "discrete_mismatch": {k: str(v) for k, v in verify["discrete_mismatch"].items()},
            "what": f"every env of a {B}-env auto-reset batch vs the reference, 150 steps, fp64"}

    if rank == 0:
        fp64 = not a.fp32
        per_gpu = value / world
        pipe_peak = m.lib().mrsim_probe_fma_peak(local, int(fp64)) / 1e12  # measured FMA-chain peak
        cpu = None
        if not a.no_cpu_baseline and world == 1:
            cpu = cpu_reference_rate(a, a.cpu_seconds, B)
        line = {
            "metric": METRIC,
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
            "dtype": "f64" if fp64 else "f32",
            "data": "synthetic: harness random policy on device, derive_episode_seed(0, e) resets",
            "config": bench_config(a, cfg, world),
            "kernel": "one thread per env (env_step_kernel)" if (a.env_per_thread and a.robots <= 4 and a.task != "rware")
                      else f"lane groups of {4 if a.robots <= 4 else (8 if a.robots <= 8 else 16)} (step_kernel)",
            "roofline": roofline(a, cfg, per_gpu, kernel_ms, fp64, pipe_peak),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": a.steps * launches_per_step,
            "rollout": rollout,
            "clocks": clk,
            "wall_s_timed_region": wall,
            "dist_backend": backend if world > 1 else None,
            "episodes": {"completed": stats["episodes"], "mean_return": stats["mean_return"],
                         "collisions": stats["sum_collisions"], "success": stats["sum_success"],
                         "qp_infeasible": stats["sum_qp_infeasible"],
                         "min_pairwise_distance": finite(stats["min_pairwise_distance"])},
        }
        if verify is not None:
            line["verify"] = verify
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
    import paper_2505_06771_b200 as m  # seed derivation and the config mirror (host-only calls)

    cfg = build_cfg(a)
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
        "impl": "reference", "metric": METRIC, "value": value, "unit": "env-steps/s",
        "robot_steps_per_s": value * a.robots, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": t / a.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: harness random policy, derive_episode_seed(0, e) resets",
        "config": bench_config(a, cfg, world),
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
