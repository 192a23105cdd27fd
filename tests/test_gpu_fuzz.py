"""Randomised parity sweep: seeded random configurations -- task, team size, horizon, sub-steps,
barrier on/off, waypoint noise, position / pose controller, batch size -- each run through
scale_parity.run_full_batch: every env of an auto-reset device batch against the reference
stepping the same envs across two episode waves (discrete fields bit-exact, poses 1e-8 m).
Covers the combinations the targeted suites do not enumerate, on every lane-group variant
(L = 4 / 8 / 16, with and without obstacle slots)."""
import os

import numpy as np
import pytest

from scale_parity import run_full_batch
from test_gpu_step import make_cfgs

pytestmark = pytest.mark.gpu
# MRSIM_FUZZ_SCALE=k multiplies the number of cases (long sweeps: profiles/r02/fuzz_long.log)
SCALE = int(os.environ.get("MRSIM_FUZZ_SCALE", "1"))

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
@pytest.mark.parametrize("k", range(72 * SCALE))
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


def _device_cfg(ref, d):
    cfg, _ = make_cfgs(ref, d["task"], d["n"], max_steps=d["max_steps"], controller=d["controller"])
    cfg.raw.sub_steps = d["sub_steps"]
    cfg.raw.barrier_enabled = d["barrier"]
    cfg.raw.action_noise_scale = d["noise"]
    return cfg


@pytest.mark.parametrize("k", range(24 * SCALE))
def test_random_configuration_rollout_equals_single_steps(k, ref):
    """mrsim_rollout (T fused steps) == T mrsim_step calls, bit for bit, on random configurations."""
    import torch

    import paper_2505_06771_b200 as m
    from scale_parity import compare_arrays
    d = _draw(5000 + k)
    cfg = _device_cfg(ref, d)
    T = 2 * d["max_steps"] + 3
    a = m.CudaEnvBatch(cfg, d["B"], fp64=True, auto_reset=True)
    b = m.CudaEnvBatch(cfg, d["B"], fp64=True, auto_reset=True)
    a.reset_episodes(root_seed=k)
    b.reset_episodes(root_seed=k)
    rew, obs = [], []
    for _ in range(T):
        out = a.step(None)
        rew.append(out.reward.clone())
        obs.append(out.obs.clone())
    ro = b.rollout(T)
    torch.cuda.synchronize()
    a.sync()
    b.sync()
    assert torch.equal(torch.stack(rew), ro.reward) and torch.equal(torch.stack(obs), ro.obs), d
    c = compare_arrays(a.get_states(), b.get_states(), d["n"])
    # Bit-identity of the two kernel instantiations (single step, MULTI) holds on the shipped build;
    # the device-checks build's asserts change FMA contraction in one of them, so there the fp64
    # poses may differ in the last bit (discrete fields and the fp32 outputs stay identical).
    ulp = 1e-14 if hasattr(m.lib(), "mrsim_debug_check_guards") else 0.0
    assert not c["discrete_mismatch"] and c["pose"] <= ulp and c["angle"] <= 10 * ulp and c["real"] <= ulp, (d, c)


@pytest.mark.parametrize("k", range(24 * SCALE))
def test_random_configuration_host_step_equals_device_step(k, ref):
    """The pinned host-buffer step (zero-copy, staged obs) == the device-buffer step."""
    import torch

    import paper_2505_06771_b200 as m
    d = _draw(9000 + k)
    cfg = _device_cfg(ref, d)
    B, n = d["B"], d["n"]
    ga, gb = m.CudaEnvBatch(cfg, B), m.CudaEnvBatch(cfg, B)
    seeds = [m.derive_episode_seed(k, e) for e in range(B)]
    ga.reset_seeds(seeds)
    gb.reset_seeds(seeds)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
    outs = (pin((B, n, cfg.obs_dim), torch.float32), pin((B,), torch.float64), pin((B,), torch.uint8))
    acts = pin((B, n), torch.int32)
    rng = np.random.default_rng(k)
    for _ in range(3):
        acts[:] = rng.integers(0, 5, size=(B, n), dtype=np.int32)
        o, r, dn = ga.step_host(acts, out=outs)
        out = gb.step(torch.from_numpy(acts.astype(np.int8)).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(o, out.obs.cpu().numpy()), d
        assert np.array_equal(r.astype(np.float32), out.reward.cpu().numpy()), d
        assert np.array_equal(dn, out.done.cpu().numpy()), d
