"""Randomised parity sweep: seeded random configurations -- task, team size, horizon, sub-steps,
barrier on/off, waypoint noise, position / pose controller, batch size -- each run through
scale_parity.run_full_batch: every env of an auto-reset device batch against the reference
stepping the same envs across two episode waves (discrete fields bit-exact, poses 1e-8 m).
Covers the combinations the targeted suites do not enumerate, on every lane-group variant
(L = 4 / 8 / 16, with and without obstacle slots)."""
import numpy as np
import pytest

from scale_parity import run_full_batch
from test_gpu_step import make_cfgs

pytestmark = pytest.mark.gpu

# team sizes that every task's default layout can spawn (arctic N > 4 uses the wider spawn zone)
N_RANGE = {"navigation": (1, 12), "predator_prey": (2, 8), "discovery": (2, 8), "rware": (1, 6),
           "foraging": (2, 6), "material_transport": (2, 10), "arctic_transport": (2, 10),
           "warehouse": (2, 6), "random_waypoints": (1, 12)}


def _draw(k: int):
    rng = np.random.default_rng(1000 + k)
    task = list(N_RANGE)[k % len(N_RANGE)]
    lo, hi = N_RANGE[task]
    return dict(task=task, n=int(rng.integers(lo, hi + 1)), max_steps=int(rng.integers(6, 25)),
                sub_steps=int(rng.choice([1, 4, 10])), barrier=int(rng.random() < 0.8),
                noise=float(rng.choice([0.0, 0.0, 0.25])), controller=int(rng.random() < 0.25),
                B=int(rng.integers(97, 700)))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("k", range(72))
def test_random_configuration_matches_reference(k, ref):
    d = _draw(k)
    cfg, sp = make_cfgs(ref, d["task"], d["n"], max_steps=d["max_steps"], controller=d["controller"])
    cfg.raw.sub_steps = d["sub_steps"]
    cfg.raw.barrier_enabled = d["barrier"]
    cfg.raw.action_noise_scale = d["noise"]
    sp.sub_steps = d["sub_steps"]
    sp.barrier = d["barrier"]
    sp.noise = d["noise"]
    rep = run_full_batch(ref, cfg, sp, d["B"], 2 * d["max_steps"] + 3, root=k, every=3)
    print(d, rep)
    assert rep["ok"], (d, rep)
    assert rep["waves"] == 2
