"""The multi-GPU entry point of bench.py (BASELINE metric "at 1/2/4/8 B200",
SURVEY 8(e)) run as 2 ranks on the lease's GPU (gloo, since the ranks share a
device): one JSON line for the job with n_gpus = 2, and every env's final
state bit-identical to the 1-rank run over the same global episodes
(multigpu.Shard slices; results independent of partitioning, batch.hpp:3-6)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, tmp):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-cpu-baseline"] + args, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(900)
@pytest.mark.parametrize("task,n", [("navigation", 4), ("material_transport", 10)])
def test_two_ranks_equal_one_rank(task, n, tmp_path):
    B = 4096
    two = _bench(["--gpus", "2", "--envs", str(B), "--e2e-steps", "2", "--task", task, "--robots", str(n),
                  "--dump-states", str(tmp_path / "two")], tmp_path)
    assert two["n_gpus"] == 2 and two["config"]["global_envs"] == 2 * B
    assert two["config"]["parallelism"] == "env-shard x2" and two["dist_backend"] == "gloo"
    assert two["e2e"]["h2d_bytes_per_step"] > 0
    one = _bench(["--gpus", "1", "--envs", str(2 * B), "--e2e-steps", "0", "--task", task, "--robots", str(n),
                  "--dump-states", str(tmp_path / "one")], tmp_path)
    ref = np.load(tmp_path / "one.rank0.npz")
    for r in range(2):
        part = np.load(tmp_path / f"two.rank{r}.npz")
        assert int(part["first_episode"]) == r * B
        for f in ("x", "y", "theta", "step_index", "collisions", "rng_key", "episode", "scenario_metric",
                  "success", "min_pairwise_distance"):
            assert np.array_equal(part[f], ref[f][r * B:(r + 1) * B]), (r, f)
    assert two["episodes"]["completed"] == one["episodes"]["completed"]
