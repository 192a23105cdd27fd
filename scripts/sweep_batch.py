"""BASELINE configs[3]: RWARE / Level-Based Foraging, 4-6 robots, batch sweep
1K-1M envs (one GPU here; the driver's multi-GPU runs cover 2/4/8), plus
navigation N=4 for reference. Every point is a full bench.py run (fp64, CBF on,
auto-reset, on-device random policy) with its roofline object and the
reference CPU step_batch (WorkerPool(all host cores)) on a bounded sample of
the same workload. One JSON line per point on stdout."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [1024, 4096, 16384, 65536, 131072, 262144, 524288, 1048576]
CONFIGS = [("rware", 4, 100), ("rware", 6, 100), ("foraging", 4, 100), ("foraging", 6, 100), ("navigation", 4, 70)]


def run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=900)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else {"error": out.stderr[-500:]}


only = sys.argv[1:]  # optional task filter
for task, n, horizon in CONFIGS:
    if only and task not in only:
        continue
    for envs in SIZES:
        steps = max(10, min(200, int(2e7 // (envs * 10)) + 10))
        d = run(["--task", task, "--robots", str(n), "--envs", str(envs), "--max-steps", str(horizon),
                 "--steps", str(steps), "--warmup", "3", "--e2e-steps", "0", "--cpu-seconds", "4"])
        rf = d.get("roofline") or {}
        cpu = d.get("cpu_baseline") or {}
        rec = {"task": task, "robots": n, "envs_per_gpu": envs, "steps": steps,
               "env_steps_per_s": d.get("value"), "robot_steps_per_s": d.get("robot_steps_per_s"),
               "ms_per_step": d.get("ms_per_step"), "kernel": d.get("kernel"),
               "roofline_bound": rf.get("bound"), "roofline_frac": rf.get("frac"),
               "hbm_frac": (rf.get("hbm") or {}).get("frac"), "clocks": d.get("clocks"),
               "cpu_reference_env_steps_per_s": cpu.get("value"), "cpu_cores": cpu.get("cores"),
               "cpu_sample": cpu.get("sample"), "error": d.get("error")}
        if rec["env_steps_per_s"] and rec["cpu_reference_env_steps_per_s"]:
            rec["speedup_vs_cpu_reference"] = rec["env_steps_per_s"] / rec["cpu_reference_env_steps_per_s"]
        print(json.dumps(rec), flush=True)
