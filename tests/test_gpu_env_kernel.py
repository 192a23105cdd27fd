"""The one-thread-per-env step kernel (env_kernel.cuh, MRSIM_FLAG_ENV_PER_THREAD),
an opt-in alternative to the lane-per-robot kernel for teams of <= 4 robots
without obstacle rows: the same parity bar as the default kernel against the
UNMODIFIED reference (fp64: discrete bit-exact, poses 1e-9 per teacher-forced
step, 1e-8 m / 1e-7 rad free-running), and equal within 1e-12 to the default
kernel (the same method; rounding differs in the last places through the
summation order of the QP's dot products)."""
import numpy as np
import pytest

import paper_2505_06771_b200 as m
from scale_parity import compare_arrays, run_full_batch
from test_gpu_step import _teacher_forced, compare_states, make_cfgs

pytestmark = pytest.mark.gpu

SMALL = [("navigation", 4), ("navigation", 3), ("navigation", 1), ("foraging", 4), ("warehouse", 4),
         ("random_waypoints", 4), ("predator_prey", 3), ("discovery", 4), ("material_transport", 4),
         ("arctic_transport", 4)]


@pytest.mark.parametrize("task,n", SMALL)
def test_env_kernel_teacher_forced_matches_reference(task, n, ref):
    cfg0 = m.make_default_config(task)
    cfg, st = _teacher_forced(ref, task, n, True, 0, cfg0.raw.max_steps + 2, B=80, env_per_thread=True)
    assert st["discrete"] == [], st["discrete"][:5]
    assert st["pose"] <= 1e-9 and st["angle"] <= 1e-8, st
    assert st["real"] <= 1e-9 and st["reward_bad"] == 0, st


@pytest.mark.parametrize("task,n,controller", [("navigation", 4, 1), ("random_waypoints", 4, 1)])
def test_env_kernel_pose_controller(task, n, controller, ref):
    cfg, st = _teacher_forced(ref, task, n, True, 0, 120, B=40, max_steps=150, controller=controller,
                              env_per_thread=True)
    assert st["discrete"] == [] and st["pose"] <= 1e-9 and st["angle"] <= 1e-8, st


@pytest.mark.timeout(1200)
def test_env_kernel_bench_batch_every_env(ref):
    import paper_2505_06771_b200.batch as bm
    cfg, sp = make_cfgs(ref, "navigation", 4, max_steps=70)
    orig = bm.CudaEnvBatch.__init__

    def init(self, *a, **k):
        k["env_per_thread"] = True
        orig(self, *a, **k)
    bm.CudaEnvBatch.__init__ = init
    try:
        rep = run_full_batch(ref, cfg, sp, 65536, 80)
    finally:
        bm.CudaEnvBatch.__init__ = orig
    assert rep["ok"], rep


def test_env_kernel_equals_lane_groups_and_reports_errors():
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(4)
    B = 3000
    seeds = [m.derive_episode_seed(3, e) for e in range(B)]
    a, b = m.CudaEnvBatch(cfg, B), m.CudaEnvBatch(cfg, B, env_per_thread=True)
    a.reset_seeds(seeds)
    b.reset_seeds(seeds)
    rng = np.random.default_rng(1)
    for t in range(30):
        acts = rng.integers(0, 5, size=(B, 4), dtype=np.int32)
        oa, ra, da = a.step_host(acts)
        ob, rb, db = b.step_host(acts)
        assert np.array_equal(da, db)
        assert np.max(np.abs(ra - rb)) <= 1e-10 and np.max(np.abs(oa - ob)) <= 1e-5
    c = compare_arrays(a.get_states(), b.get_states(), 4)
    assert not c["discrete_mismatch"] and c["pose"] <= 1e-10, c
    acts = rng.integers(0, 5, size=(B, 4), dtype=np.int32)
    acts[1234, 3] = -2
    before = b.get_states(1234, 1)[0].x[0]
    with pytest.raises(m.InvalidArgument, match=r"invalid action -2 for environment 1234, robot 3"):
        b.step_host(acts)
    assert b.get_states(1234, 1)[0].x[0] == before
