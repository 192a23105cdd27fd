"""bench.py plumbing on CPU: the reference arm's JSON contract (same `config` object as the
device arm), and the `--gpus N` self-launch through torch.distributed.run (rank 0 alone prints
the reference line; the other ranks exit 0)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, timeout=300):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]


def test_reference_arm_contract(ref):
    lines = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--envs", "256"])
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["metric"] == "env-steps/sec (CBF on)" and d["unit"] == "env-steps/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1

    import argparse

    import bench
    import paper_2505_06771_b200 as m  # noqa: F401

    a = argparse.Namespace(task="navigation", robots=4, envs=256, max_steps=70, controller="unicycle_position",
                           policy="random")
    assert d["config"] == bench.bench_config(a, bench.build_cfg(a), 1)  # the device arm's object


@pytest.mark.timeout(600)
def test_gpus_flag_launches_ranks(ref):
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--envs", "128"])
    assert len(lines) == 1  # rank 0 only
    assert lines[0]["n_gpus"] == 2 and lines[0]["config"]["global_envs"] == 256
    assert lines[0]["config"]["parallelism"] == "env-shard x2"
