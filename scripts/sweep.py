"""Throughput sweep over the BASELINE configs (one GPU): device fp64 (product),
device fp32 (fast mode) and the reference CPU step_batch on the host cores.
Writes one JSON line per config to stdout."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [("navigation", 4, 65536), ("predator_prey", 6, 32768), ("discovery", 6, 32768), ("rware", 4, 65536),
           ("rware", 6, 65536), ("foraging", 4, 65536), ("foraging", 6, 65536), ("material_transport", 10, 131072),
           ("arctic_transport", 10, 131072), ("warehouse", 4, 65536), ("random_waypoints", 4, 65536)]


def run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1]) if lines else {"error": out.stderr[-500:]}


for task, n, envs in CONFIGS:
    base = ["--task", task, "--robots", str(n), "--envs", str(envs), "--steps", "100", "--warmup", "5",
            "--e2e-steps", "0"]
    d64 = run(base + ["--cpu-seconds", "8"])
    d32 = run(base + ["--fp32", "--no-cpu-baseline"])
    rec = {"task": task, "robots": n, "envs_per_gpu": envs,
           "fp64_env_steps_per_s": d64.get("value"), "fp64_robot_steps_per_s": d64.get("robot_steps_per_s"),
           "fp64_ms_per_step": d64.get("ms_per_step"),
           "fp32_env_steps_per_s": d32.get("value"), "fp32_robot_steps_per_s": d32.get("robot_steps_per_s"),
           "cpu_reference_env_steps_per_s": (d64.get("cpu_baseline") or {}).get("value"),
           "cpu_cores": (d64.get("cpu_baseline") or {}).get("cores"),
           "fp64_hbm_frac": (d64.get("roofline") or {}).get("frac"),
           "fp64_pipe_frac": ((d64.get("roofline") or {}).get("pipe") or {}).get("frac"),
           "episodes": d64.get("episodes")}
    if rec["fp64_env_steps_per_s"] and rec["cpu_reference_env_steps_per_s"]:
        rec["speedup_vs_cpu_reference"] = rec["fp64_env_steps_per_s"] / rec["cpu_reference_env_steps_per_s"]
    print(json.dumps(rec), flush=True)
