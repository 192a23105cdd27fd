"""GPU parity of the on-device feedforward policy (Policy::act with
PolicyKind::FeedforwardFile, policy.hpp:95-116, 445-480; seeded like
run_episodes, harness.hpp:238-252) against the UNMODIFIED reference.

Tolerance: relu/identity networks are bit-exact (same summation order, no
FMA contraction), so greedy actions must be identical. tanh and the softmax
exp use the device libm (<= 1 ulp from glibc): a decision can flip only at a
near-tie, bounded here at <= 1 in 1000 robot-steps.
"""
import numpy as np
import pytest
import torch

import paper_2505_06771_b200 as m
from test_gpu_step import compare_states, make_cfgs

pytestmark = pytest.mark.gpu

TASKS = [("navigation", 4), ("predator_prey", 6), ("discovery", 6), ("rware", 4), ("foraging", 6),
         ("material_transport", 10), ("arctic_transport", 10), ("warehouse", 4), ("random_waypoints", 4)]


def _weights(D, acts, seed):
    return m.FeedforwardWeights.random([D, 64, 32, 5], acts, seed=seed, scale=2.0)


@pytest.mark.parametrize("task,n", TASKS)
def test_greedy_relu_policy_bit_exact(task, n, ref, tmp_path):
    cfg, sp = make_cfgs(ref, task, n)
    w = _weights(cfg.obs_dim, ["relu", "relu", "identity"], seed=n)
    path = tmp_path / "w.txt"
    path.write_text(w.to_text())
    B = 96
    seeds = [m.derive_episode_seed(5, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    gb.set_policy(f"feedforward:{path}")
    for t in range(30):
        ra = rb.policy_actions(f"feedforward:{path}")
        ga = gb.policy_actions().cpu().numpy().astype(np.int32)
        assert np.array_equal(ga, ra), (t, np.argwhere(ga != ra)[:5])
        gb.step_host(ra)
        rb.step(ra)


@pytest.mark.parametrize("greedy", [True, False])
@pytest.mark.parametrize("task,n", [("navigation", 4), ("discovery", 6), ("arctic_transport", 10)])
def test_tanh_and_softmax_policy_match(task, n, greedy, ref, tmp_path):
    cfg, sp = make_cfgs(ref, task, n)
    w = _weights(cfg.obs_dim, ["tanh", "tanh", "identity"], seed=7 + n)
    path = tmp_path / "w.txt"
    path.write_text(w.to_text())
    spec = ("feedforward:" if greedy else "feedforward_sample:") + str(path)
    B = 96
    seeds = [m.derive_episode_seed(6, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    gb.set_policy(spec)
    flips = total = 0
    for t in range(30):
        ra = rb.policy_actions(spec)
        ga = gb.policy_actions().cpu().numpy().astype(np.int32)
        flips += int(np.sum(ga != ra))
        total += ga.size
        gb.step_host(ra)
        rb.step(ra)
    assert flips <= max(1, total // 1000), (flips, total)


def test_closed_loop_on_device_policy_matches_reference(ref, tmp_path):
    """mrsim_step(actions=NULL) runs the feedforward producer on device before
    the step; the trajectory equals the reference run_episodes loop."""
    cfg, sp = make_cfgs(ref, "navigation", 4)
    w = _weights(cfg.obs_dim, ["relu", "relu", "identity"], seed=11)
    path = tmp_path / "w.txt"
    path.write_text(w.to_text())
    B = 128
    seeds = [m.derive_episode_seed(8, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    gb.set_policy(w)
    for t in range(cfg.raw.max_steps):
        out = gb.step(None)
        ra = rb.policy_actions(f"feedforward:{path}")
        _, rrew, rdone, _ = rb.step(ra)
        torch.cuda.synchronize()
        gb.sync()
        assert np.array_equal(out.done.cpu().numpy().astype(bool), np.asarray(rdone).astype(bool)), t
        pe, ae, bad, re_ = compare_states(gb.get_states(), rb.get_states(), 4, 0, 0, 0)
        # free-running 100-step horizon: ulp-level QP arithmetic differences accumulate
        # (heading ~20x position through omega = (...)/l); discrete outputs stay identical
        assert not bad and pe <= 1e-7 and ae <= 2e-6, (t, pe, ae, bad[:3])


def test_policy_validation_errors():
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 4)
    gb.reset_seeds([1, 2, 3, 4])
    with pytest.raises(m.InvalidArgument, match="observation size"):
        gb.set_policy(m.FeedforwardWeights.random([7, 8, 5], ["relu", "identity"]))
    with pytest.raises(m.InvalidArgument, match="unknown policy"):
        gb.set_policy("scripted_bfs")
    with pytest.raises(m.Unsupported):
        gb.set_policy(m.FeedforwardWeights.random([5, 300, 5], ["relu", "identity"]))
    gb.set_policy("random")  # back to the harness random policy
    a = gb.policy_actions().cpu().numpy()
    assert a.shape == (4, 3) and a.min() >= 0 and a.max() <= 4


SCRIPTED = [("navigation", 4), ("predator_prey", 6), ("discovery", 6), ("rware", 4), ("foraging", 4),
            ("material_transport", 10), ("arctic_transport", 10), ("warehouse", 4), ("random_waypoints", 4)]


@pytest.mark.parametrize("task,n", SCRIPTED)
def test_scripted_goal_policy_matches_reference(task, n, ref):
    """PolicyKind::ScriptedGoal (policy.hpp:242-360): BFS planner on the device.
    Near-ties (device hypot vs glibc, <= 1 ulp) may flip a decision: <= 1 in 500."""
    cfg, sp = make_cfgs(ref, task, n)
    B = 48
    seeds = [m.derive_episode_seed(21, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    gb.set_policy("scripted_goal")
    flips = total = 0
    for t in range(12):
        ra = rb.policy_actions("scripted_goal")
        ga = gb.policy_actions().cpu().numpy().astype(np.int32)
        flips += int(np.sum(ga != ra))
        total += ga.size
        gb.step_host(ra)
        rb.step(ra)
    assert flips <= max(1, total // 500), (flips, total)


def test_prey_chaser_policy_matches_reference(ref):
    cfg, sp = make_cfgs(ref, "predator_prey", 6)
    B = 64
    seeds = [m.derive_episode_seed(22, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    gb.set_policy("prey_chaser")
    flips = total = 0
    for t in range(30):
        ra = rb.policy_actions("prey_chaser")
        ga = gb.policy_actions().cpu().numpy().astype(np.int32)
        flips += int(np.sum(ga != ra))
        total += ga.size
        gb.step_host(ra)
        rb.step(ra)
    assert flips <= max(1, total // 500), (flips, total)
    nav = m.CudaEnvBatch(m.make_default_config("navigation"), 2)
    with pytest.raises(m.InvalidArgument, match="prey_chaser policy only applies to predator_prey"):
        nav.set_policy("prey_chaser")


@pytest.mark.parametrize("spec", ["scripted_goal", "mlp"])
def test_policies_run_in_fp32_mode(spec, ref):
    """The fp32 fast mode drives the same device policies (observations / geometry in the state
    precision); actions stay in range and mostly agree with the fp64 path on identical states."""
    import torch
    cfg, _ = make_cfgs(ref, "navigation", 4)
    B = 64
    seeds = [m.derive_episode_seed(31, e) for e in range(B)]
    g32, g64 = m.CudaEnvBatch(cfg, B, fp64=False), m.CudaEnvBatch(cfg, B, fp64=True)
    g32.reset_seeds(seeds)
    g64.reset_seeds(seeds)
    pol = spec if spec != "mlp" else m.FeedforwardWeights.random([cfg.obs_dim, 32, 5], ["relu", "identity"], seed=2)
    g32.set_policy(pol)
    g64.set_policy(pol)
    a32 = g32.policy_actions().cpu().numpy()
    a64 = g64.policy_actions().cpu().numpy()
    assert a32.min() >= 0 and a32.max() <= 4
    assert np.mean(a32 == a64) >= 0.95
    g32.step(None)
    torch.cuda.synchronize()
    g32.sync()
