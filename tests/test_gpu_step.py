"""GPU parity of the fused step (step_env, batch.hpp:165-224) and reset
(reset_env, batch.hpp:153-160) against the UNMODIFIED reference on
identical seeds, initial states and actions, for every benchmark task at
the BASELINE robot counts.

Tolerances (stated per SURVEY.md 8(d)):
  fp64 device path (the product default): discrete outputs bit-exact, poses
                     within 1e-9 per step and 1e-8 over the horizon, team
                     rewards within 1e-9*max(1,|r|).
  fp32 device path (opt-in fast mode): one teacher-forced physics tick:
                     poses 2e-6 m / 4e-5 rad. Over a 10-tick step the fp32
                     path can legitimately fork from the reference: the hold
                     rule (batch.hpp:187-188) compares the waypoint and the
                     pose for EXACT equality, and the reference's 1e-9 QP
                     tolerance produces sub-fp32-ulp displacements of held
                     robots that break that equality in fp64 but not in fp32
                     (then the robot "creeps" at 0.05 m/s). Those forks are
                     counted and bounded, not treated as failures.
"""
import numpy as np
import pytest

import paper_2505_06771_b200 as m
from util import wrap_diff

pytestmark = pytest.mark.gpu

# BASELINE.json configs 2-5 (+ warehouse at default N)
CONFIGS = [("navigation", 4), ("predator_prey", 6), ("discovery", 6), ("rware", 4), ("rware", 6),
           ("foraging", 4), ("foraging", 6), ("material_transport", 10), ("arctic_transport", 10),
           ("warehouse", 4), ("random_waypoints", 4)]
# ControllerKind::UnicyclePose (controllers.hpp:68-82) on a subset, horizon capped at 150 steps
POSE_CONFIGS = [("navigation", 4), ("random_waypoints", 4), ("random_waypoints", 10), ("rware", 4),
                ("material_transport", 10)]
ARCTIC_SPAWN = [-1.55, -1.05, -0.9, 0.9]  # default zone fails 1.4% of N=10 resets


def make_cfgs(ref, task, n, max_steps=0, controller=-1):
    cfg = m.make_default_config(task)
    tile = cfg.raw.het_rows > 0
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=tile)
    layout = {}
    if task == "arctic_transport" and n > 4:
        cfg.set_layout("arctic.spawn_zone", ARCTIC_SPAWN)
        layout["arctic.spawn_zone"] = ARCTIC_SPAWN
    if max_steps:
        cfg.max_steps = max_steps
    if controller >= 0:
        cfg.controller = controller
    sp = ref.spec(task, num_robots=n, tile_roster=tile, layout=layout, max_steps=max_steps, controller=controller)
    return cfg, sp


DISCRETE = ["step_index", "collisions", "qp_infeasible", "success", "flash_timer", "sensed", "tagged",
            "slot_shelf", "carried", "requests", "levels", "foraged", "tiles", "loaded"]


def compare_states(a, b, N, pos_tol, ang_tol, real_tol):
    """Returns (max pose err, max angle err, list of discrete mismatches, max real err)."""
    pe = ae = re_ = 0.0
    bad = []
    for e, (sa, sb) in enumerate(zip(a, b)):
        x = np.array(sa.x[:N]) - np.array(sb.x[:N])
        y = np.array(sa.y[:N]) - np.array(sb.y[:N])
        pe = max(pe, float(np.max(np.abs(x))), float(np.max(np.abs(y))))
        ae = max(ae, float(np.max(wrap_diff(sa.theta[:N], sb.theta[:N]))))
        for f in DISCRETE:
            va, vb = getattr(sa, f), getattr(sb, f)
            if hasattr(va, "__len__"):
                va, vb = list(va), list(vb)
            if va != vb:
                bad.append((e, f, va, vb))
        for f in ("scenario_metric", "circle_remaining", "rect_remaining", "delivered", "total_initial"):
            re_ = max(re_, abs(getattr(sa, f) - getattr(sb, f)))
        re_ = max(re_, float(np.max(np.abs(np.array(sa.loads[:N]) - np.array(sb.loads[:N])))))
        for arr in ("goals", "landmarks", "resources", "prey", "targets", "target_headings"):
            re_ = max(re_, float(np.max(np.abs(np.array(getattr(sa, arr)) - np.array(getattr(sb, arr))))))
    return pe, ae, bad, re_


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("task,n", CONFIGS)
def test_reset_matches_reference(task, n, fp64, ref):
    cfg, sp = make_cfgs(ref, task, n)
    B = 256
    seeds = [m.derive_episode_seed(0, e) for e in range(B)]
    gb = m.CudaEnvBatch(cfg, B, fp64=fp64)
    gobs = gb.reset_seeds(seeds).cpu().numpy()
    rb = ref.RefBatch(sp)
    robs = rb.reset(seeds)
    gs, rs = gb.get_states(), rb.get_states()
    if fp64:
        pe, ae, bad, re_ = compare_states(gs, rs, n, 0, 0, 0)
        assert pe == 0.0 and ae == 0.0 and re_ == 0.0 and not bad
    else:
        pe, ae, bad, re_ = compare_states(gs, rs, n, 0, 0, 0)
        assert pe < 1e-6 and ae < 1e-6 and re_ < 1e-5 and not bad
        for sa, sb in zip(gs, rs):  # fp32 poses are exactly the rounded reference poses
            assert np.array_equal(np.float32(sa.x[:n]), np.float32(sb.x[:n]))
    np.testing.assert_allclose(gobs, robs, atol=2e-6, rtol=1e-6)
    for sa, sb in zip(gs, rs):
        assert sa.rng_key == sb.rng_key


def _teacher_forced(ref, task, n, fp64, sub_steps, T, B=48, max_steps=0, controller=-1, **batch_kw):
    cfg, sp = make_cfgs(ref, task, n, max_steps=max_steps, controller=controller)
    if sub_steps:
        cfg.sub_steps = sub_steps
        sp.sub_steps = sub_steps
    seeds = [m.derive_episode_seed(1, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=fp64, **batch_kw)
    stats = {"pose": 0.0, "angle": 0.0, "real": 0.0, "discrete": [], "reward_bad": 0, "obs": 0.0}
    for t in range(T):
        st = rb.get_states()
        acts = rb.random_actions()
        gb.set_states(list(st))
        gobs, grew, gdone = gb.step_host(acts)
        robs, rrew, rdone, _ = rb.step(acts)
        gs, rs = gb.get_states(), rb.get_states()
        pe, ae, bad, re_ = compare_states(gs, rs, n, 0, 0, 0)
        assert np.array_equal(gdone, rdone), t
        stats["pose"] = max(stats["pose"], pe)
        stats["angle"] = max(stats["angle"], ae)
        stats["real"] = max(stats["real"], re_)
        stats["discrete"] += [(t,) + b for b in bad]
        ok = np.abs(grew - rrew) <= (1e-9 if fp64 else 1e-4) * np.maximum(1.0, np.abs(rrew))
        stats["reward_bad"] += int((~ok).sum())
        stats["obs"] = max(stats["obs"], float(np.max(np.abs(gobs - robs))))
    return cfg, stats


@pytest.mark.parametrize("task,n", CONFIGS)
def test_teacher_forced_steps_match_reference_fp64(task, n, ref):
    """Upload the reference state of every step to the device, step both with
    the same actions, compare one step. Covers the whole horizon incl.
    done/finalize and two steps past it (done stays true, batch.hpp:218-220)."""
    cfg0 = m.make_default_config(task)
    cfg, st = _teacher_forced(ref, task, n, True, 0, cfg0.raw.max_steps + 2)
    assert st["discrete"] == [], st["discrete"][:5]
    assert st["pose"] <= 1e-9 and st["angle"] <= 1e-8, st
    assert st["real"] <= 1e-9, st
    assert st["reward_bad"] == 0
    assert st["obs"] <= 2e-6 * 16  # fp32 obs of values up to |16|


@pytest.mark.parametrize("task,n", POSE_CONFIGS)
def test_teacher_forced_pose_controller_fp64(task, n, ref):
    cfg, st = _teacher_forced(ref, task, n, True, 0, 152, max_steps=150, controller=1)
    assert st["discrete"] == [], st["discrete"][:5]
    assert st["pose"] <= 1e-9 and st["angle"] <= 1e-8, st
    assert st["real"] <= 1e-9, st
    assert st["reward_bad"] == 0


@pytest.mark.parametrize("task,n", POSE_CONFIGS)
def test_free_running_pose_controller_fp64(task, n, ref):
    cfg, sp = make_cfgs(ref, task, n, max_steps=150, controller=1)
    B = 64
    seeds = [m.derive_episode_seed(4, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    for t in range(150):
        acts = rb.random_actions()
        _, grew, gdone = gb.step_host(acts)
        _, rrew, rdone, _ = rb.step(acts)
        assert np.array_equal(gdone, rdone)
        pe, ae, bad, re_ = compare_states(gb.get_states(), rb.get_states(), n, 0, 0, 0)
        assert not bad and pe <= 1e-8 and ae <= 1e-7 and re_ <= 1e-8, (t, pe, ae, bad[:3], re_)
        assert np.all(np.abs(grew - rrew) <= 1e-9 * np.maximum(1.0, np.abs(rrew)))


@pytest.mark.parametrize("task,n", CONFIGS)
def test_teacher_forced_ticks_match_reference_fp32(task, n, ref):
    """fp32 mode, one physics tick per step (sub_steps=1): the per-tick
    controller + CBF-QP + Euler + task logic agree to fp32 accuracy."""
    cfg, st = _teacher_forced(ref, task, n, False, 1, 60)
    assert st["pose"] <= 2e-6 and st["angle"] <= 4e-5, st
    assert len(st["discrete"]) <= 1, st["discrete"][:5]


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("task,n", CONFIGS)
def test_free_running_horizon_matches_reference(task, n, fp64, ref):
    """Both sides reset from the same seeds and step the full horizon with the
    harness random policy; compare per-step poses, rewards and discrete outputs."""
    cfg, sp = make_cfgs(ref, task, n)
    B = 64
    seeds = [m.derive_episode_seed(2, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=fp64)
    gb.reset_seeds(seeds)
    pos_tol, ang_tol = (1e-8, 1e-7) if fp64 else (1e-3, 1e-2)
    worst = 0.0
    diverged = set()
    for t in range(cfg.raw.max_steps):
        acts = rb.random_actions()
        gobs, grew, gdone = gb.step_host(acts)
        robs, rrew, rdone, _ = rb.step(acts)
        assert np.array_equal(gdone, rdone)
        gs, rs = gb.get_states(), rb.get_states()
        for e in range(B):
            if e in diverged:
                continue
            pe, ae, bad, re_ = compare_states([gs[e]], [rs[e]], n, 0, 0, 0)
            rew_ok = abs(grew[e] - rrew[e]) <= (1e-9 if fp64 else 1e-4) * max(1.0, abs(rrew[e]))
            if fp64:
                assert not bad and rew_ok, (t, e, bad, grew[e], rrew[e])
                assert pe <= pos_tol and ae <= ang_tol, (t, e, pe, ae)
            else:
                if bad or not rew_ok or pe > pos_tol or ae > ang_tol:
                    diverged.add(e)  # hold-rule fork (module docstring): the trajectory legitimately forks here
                    continue
            worst = max(worst, pe)
    if not fp64:  # hold-rule forks (see module docstring): bounded, reported
        print(f"fp32 {task} N={n}: {len(diverged)}/{B} envs forked from the reference within the horizon")
        assert len(diverged) <= (3 * B) // 4, sorted(diverged)


@pytest.mark.parametrize("env_per_thread", [False, True])
def test_invalid_action_reports_env_and_robot_and_rolls_back(env_per_thread):
    # test_framework.cpp:171-185. The lane-group kernel's last warp hands the error word to the
    # host step in pinned memory; the env kernel has no such epilogue (the host copies the word).
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 2, env_per_thread=env_per_thread)
    gb.reset_seeds([5, 6])
    before = gb.get_states()
    with pytest.raises(m.InvalidArgument, match=r"environment 0, robot 1"):
        gb.step_host([0, 7, 0, 0, 0, 0])
    after = gb.get_states()
    assert [s.x[0] for s in before] == [s.x[0] for s in after]
    gb.step_host([0] * 6)  # context stays usable


@pytest.mark.parametrize("env_per_thread", [False, True])
def test_host_step_reports_an_earlier_queued_failure(env_per_thread):
    """A failing asynchronous device step, then a host step: the host step's launch is a no-op
    (sticky word) whose last warp still hands the word over; the error of the earlier step is
    raised and the state rolled back to that step's input."""
    import torch
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 40, env_per_thread=env_per_thread)
    gb.reset_seeds(list(range(40)))
    before = gb.get_states()
    bad = torch.zeros((40, 3), dtype=torch.int8, device="cuda")
    bad[23, 2] = 6
    gb.step(bad)
    with pytest.raises(m.InvalidArgument, match=r"environment 23, robot 2"):
        gb.step_host([0] * 120)
    after = gb.get_states()
    assert [list(s.x[:3]) for s in before] == [list(s.x[:3]) for s in after]
    assert [s.step_index for s in before] == [s.step_index for s in after]
    gb.step_host([0] * 120)  # usable again
    assert gb.get_states(0, 1)[0].step_index == before[0].step_index + 1


def test_device_invalid_action_is_sticky_then_rolled_back():
    import torch
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 4)
    gb.reset_seeds([1, 2, 3, 4])
    before = gb.get_states()
    a = torch.zeros((4, 3), dtype=torch.int8, device="cuda")
    a[2, 1] = 9
    gb.step(a)
    with pytest.raises(m.InvalidArgument, match=r"environment 2, robot 1"):
        gb.sync()
    after = gb.get_states()
    assert [s.x[0] for s in before] == [s.x[0] for s in after]


def test_all_stay_freezes_world():
    # test_framework.cpp:187-198 (barrier on: spawn separation keeps rows slack)
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 1, fp64=True)
    gb.reset_seeds([3])
    s0 = gb.get_states()[0]
    _, r1, _ = gb.step_host([0, 0, 0])
    _, r2, _ = gb.step_host([0, 0, 0])
    s2 = gb.get_states()[0]
    assert list(s0.x[:3]) == list(s2.x[:3]) and list(s0.y[:3]) == list(s2.y[:3])
    assert r1[0] == r2[0]


def test_identical_instances_and_purity():
    # test_framework.cpp:100-112
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 3)
    gb.reset_seeds([7, 7, 9])
    obs, rew, _ = gb.step_host([1, 4, 0, 1, 4, 0, 2, 3, 1])
    s = gb.get_states()
    assert list(s[0].x[:3]) == list(s[1].x[:3])
    assert rew[0] == rew[1] and rew[2] != rew[0]
    assert np.array_equal(obs[0], obs[1])


@pytest.mark.parametrize("pinned", [False, True])
def test_host_api_matches_device_step(pinned):
    """mrsim_step_host with pageable buffers (staged copies) or pinned ones (the
    kernel reads actions / writes outputs in place over the host link) equals
    the device-buffer step."""
    import torch
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(4)
    B = 50000
    seeds = [m.derive_episode_seed(12, e) for e in range(B)]
    ga, gb = m.CudaEnvBatch(cfg, B), m.CudaEnvBatch(cfg, B)
    ga.reset_seeds(seeds)
    gb.reset_seeds(seeds)
    rng = np.random.default_rng(0)

    def buf(shape, dt):
        t = torch.empty(shape, dtype=dt)
        return (t.pin_memory() if pinned else t).numpy()

    outs = (buf((B, 4, cfg.obs_dim), torch.float32), buf((B,), torch.float64), buf((B,), torch.uint8))
    act_buf = buf((B, 4), torch.int32)
    for t in range(3):
        act_buf[:] = rng.integers(0, 5, size=(B, 4), dtype=np.int32)
        acts = act_buf
        obs, rew, done = ga.step_host(acts, out=outs)
        out = gb.step(torch.from_numpy(acts.astype(np.int8)).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(obs, out.obs.cpu().numpy())
        assert np.array_equal(rew.astype(np.float32), out.reward.cpu().numpy())
        assert np.array_equal(done, out.done.cpu().numpy())
    sa, sb = ga.get_states(), gb.get_states()
    for e in (0, 18943, 18944, 37888, B - 1):
        assert list(sa[e].x[:4]) == list(sb[e].x[:4]) and sa[e].step_index == sb[e].step_index
    act_buf[:] = rng.integers(0, 5, size=(B, 4), dtype=np.int32)
    act_buf[40000, 2] = 300  # reported with its full value, the step rolled back
    before = ga.get_states(40000, 1)[0].x[0]
    with pytest.raises(m.InvalidArgument, match=r"invalid action 300 for environment 40000, robot 2"):
        ga.step_host(act_buf, out=outs)
    assert ga.get_states(40000, 1)[0].x[0] == before


@pytest.mark.parametrize("task,n", [("navigation", 4), ("discovery", 6), ("rware", 6), ("material_transport", 10),
                                    ("arctic_transport", 10)])
def test_host_step_obs_staging_matches_device_step(task, n):
    """Every obs path of the pinned host step equals the device-buffer step: the warp stage when it
    is free (navigation), when it costs a resident block (discovery, rware N=6, MT N=10: smaller
    grid) and the QP-workspace stage (arctic N=10); B odd, so the last warp task is partial."""
    import torch
    cfg = m.make_default_config(task)
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    if task == "arctic_transport":
        cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9])
    B = 3001
    seeds = [m.derive_episode_seed(5, e) for e in range(B)]
    ga, gb = m.CudaEnvBatch(cfg, B), m.CudaEnvBatch(cfg, B)
    ga.reset_seeds(seeds)
    gb.reset_seeds(seeds)
    rng = np.random.default_rng(1)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
    outs = (pin((B, n, cfg.obs_dim), torch.float32), pin((B,), torch.float64), pin((B,), torch.uint8))
    acts = pin((B, n), torch.int32)
    for _ in range(4):
        acts[:] = rng.integers(0, 5, size=(B, n), dtype=np.int32)
        obs, rew, done = ga.step_host(acts, out=outs)
        out = gb.step(torch.from_numpy(acts.astype(np.int8)).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(obs, out.obs.cpu().numpy())
        assert np.array_equal(rew.astype(np.float32), out.reward.cpu().numpy())
        assert np.array_equal(done, out.done.cpu().numpy())
    sa, sb = ga.get_states(), gb.get_states()
    for e in (0, 1, B // 2, B - 2, B - 1):
        assert list(sa[e].x[:n]) == list(sb[e].x[:n]) and sa[e].step_index == sb[e].step_index


# Every kernel variant and the extremes of the team size: N = 1 (no pair rows), 2, 7 (L=8, 4 pair
# slots per lane), 9 (L=16, 3 pair slots: the 4-blocks-per-SM build), 13 and 16 (L=16, 8 pair
# slots; 16 = MRSIM_MAX_ROBOTS), and rware with 8 slots (the 16-obstacle-slot variant).
@pytest.mark.parametrize("n", [1, 2, 7, 9, 13, 16])
def test_team_size_extremes_match_reference(n, ref):
    cfg, st = _teacher_forced(ref, "navigation", n, True, 0, 40, B=24)
    assert st["discrete"] == [], st["discrete"][:5]
    assert st["pose"] <= 1e-9 and st["angle"] <= 1e-8, st
    assert st["reward_bad"] == 0


def test_rware_wide_layout_variant_matches_reference(ref):
    slots = [-1.2, -0.4, -0.8, -0.4, -0.4, -0.4, 0.0, -0.4, -1.2, 0.4, -0.8, 0.4, -0.4, 0.4, 0.0, 0.4]
    cfg = m.make_default_config("rware")
    cfg.set_num_robots(4)
    cfg.set_layout("rware.slots", slots)
    sp = ref.spec("rware", num_robots=4, layout={"rware.slots": slots})
    B = 32
    seeds = [m.derive_episode_seed(9, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    for t in range(cfg.raw.max_steps):
        st0 = rb.get_states()
        acts = rb.random_actions()
        gb.set_states(list(st0))
        gobs, grew, gdone = gb.step_host(acts)
        robs, rrew, rdone, _ = rb.step(acts)
        pe, ae, bad, re_ = compare_states(gb.get_states(), rb.get_states(), 4, 0, 0, 0)
        assert not bad and pe <= 1e-9 and ae <= 1e-8, (t, pe, ae, bad[:3])
        assert np.array_equal(gdone, rdone)
        assert np.all(np.abs(grew - rrew) <= 1e-9 * np.maximum(1.0, np.abs(rrew)))


@pytest.mark.parametrize("task,n", [("navigation", 4), ("arctic_transport", 10)])
def test_action_noise_matches_reference(task, n, ref):
    """framework.hpp:96-108: waypoint noise drawn from the step stream (2 draws per robot)."""
    cfg, sp = make_cfgs(ref, task, n)
    cfg.action_noise_scale = 0.3
    sp.noise = 0.3
    B = 32
    seeds = [m.derive_episode_seed(13, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    for t in range(40):
        acts = rb.random_actions()
        _, grew, gdone = gb.step_host(acts)
        _, rrew, rdone, _ = rb.step(acts)
        pe, ae, bad, re_ = compare_states(gb.get_states(), rb.get_states(), n, 0, 0, 0)
        assert not bad and pe <= 1e-8 and ae <= 1e-7, (t, pe, ae, bad[:3])
        assert np.all(np.abs(grew - rrew) <= 1e-9 * np.maximum(1.0, np.abs(rrew)))


def test_auto_reset_continues_with_the_next_wave(ref):
    """In-kernel auto-reset: a done env restarts as episode + B, i.e. exactly
    the reference's next run_episodes wave (harness.hpp:227-232)."""
    cfg, sp = make_cfgs(ref, "navigation", 4, max_steps=12)
    B = 32
    gb = m.CudaEnvBatch(cfg, B, fp64=True, auto_reset=True)
    gb.reset_episodes(root_seed=5, first_episode=0, episode_stride=B)
    for wave in range(2):
        rb = ref.RefBatch(sp)
        seeds = [m.derive_episode_seed(5, wave * B + e) for e in range(B)]
        rb.reset(seeds)
        for t in range(12):
            acts = rb.random_actions()
            _, grew, gdone = gb.step_host(acts)
            _, rrew, rdone, _ = rb.step(acts)
            assert np.array_equal(gdone, rdone)
            assert np.all(np.abs(grew - rrew) <= 1e-9 * np.maximum(1.0, np.abs(rrew)))
            if t < 11:  # the done step's state is already the next episode's reset
                pe, ae, bad, _ = compare_states(gb.get_states(), rb.get_states(), 4, 0, 0, 0)
                assert not bad and pe <= 1e-8, (wave, t, pe, bad[:3])
    st = gb.get_states()
    assert [s.episode for s in st] == [2 * B + e for e in range(B)]
    assert all(s.step_index == 0 for s in st)
    assert gb.stats()["episodes"] == 2 * B


@pytest.mark.parametrize("task,n,controller", [("random_waypoints", 4, 1), ("navigation", 4, 1),
                                               ("random_waypoints", 4, 0)])
def test_fp32_fast_mode_new_paths_track_reference(task, n, controller, ref):
    """fp32 opt-in mode on the pose controller / random_waypoints paths: one teacher-forced tick
    agrees to fp32 accuracy (same bound as the benchmark tasks)."""
    cfg, st = _teacher_forced(ref, task, n, False, 1, 40, max_steps=60, controller=controller)
    assert st["pose"] <= 2e-6 and st["angle"] <= 4e-5, st
    assert len(st["discrete"]) <= 1, st["discrete"][:5]


@pytest.mark.parametrize("env_per_thread", [False, True])
def test_rollback_after_more_than_64_queued_steps(env_per_thread):
    """A failing device step followed by 70 queued (no-op) steps before the sync: the state is
    rolled back to the failing step's input (step_batch is pure, batch.hpp:267-290)."""
    import torch
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 64, env_per_thread=env_per_thread)
    gb.reset_seeds(list(range(64)))
    good = torch.zeros((64, 3), dtype=torch.int8, device="cuda")
    gb.step(good)
    gb.sync()
    before = gb.get_states()
    bad = good.clone()
    bad[17, 2] = 5
    gb.step(bad)
    for _ in range(70):
        gb.step(good)
    with pytest.raises(m.InvalidArgument, match=r"environment 17, robot 2"):
        gb.sync()
    after = gb.get_states()
    assert [list(s.x[:3]) for s in before] == [list(s.x[:3]) for s in after]
    assert [s.step_index for s in before] == [s.step_index for s in after]
    gb.step(good)  # the context stays usable
    gb.sync()
    assert gb.get_states(0, 1)[0].step_index == before[0].step_index + 1


@pytest.mark.parametrize("env_per_thread", [False, True])
def test_failed_step_rolls_back_episode_stats(env_per_thread):
    """Every env finishes its episode on the failing step; the envs that completed before the
    error was noticed must not keep their EpisodeStats update (no double count on retry)."""
    cfg = m.make_default_config("navigation")
    B = 200
    gb = m.CudaEnvBatch(cfg, B, env_per_thread=env_per_thread)
    gb.reset_seeds([m.derive_episode_seed(0, e) for e in range(B)])
    st = list(gb.get_states())
    for s in st:
        s.step_index = cfg.raw.max_steps - 1
    gb.set_states(st)
    acts = np.zeros((B, 3), dtype=np.int32)
    acts[150, 0] = 9
    with pytest.raises(m.InvalidArgument):
        gb.step_host(acts)
    assert gb.stats()["episodes"] == 0
    acts[150, 0] = 0
    gb.step_host(acts)
    assert gb.stats()["episodes"] == B


@pytest.mark.parametrize("env_per_thread", [False, True])
def test_invalid_action_outranks_a_physics_error_in_a_lower_env(env_per_thread):
    """validate_actions runs over every env before any env steps (batch.hpp:271): an invalid
    action in env 5 is reported even though env 3 has coincident robots (domain_error)."""
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 8, env_per_thread=env_per_thread)
    gb.reset_seeds(list(range(8)))
    st = list(gb.get_states())
    st[3].x[1], st[3].y[1], st[3].theta[1] = st[3].x[0], st[3].y[0], st[3].theta[0]
    gb.set_states(st)
    acts = np.zeros((8, 3), dtype=np.int32)
    with pytest.raises(m.DomainError, match=r"environment 3"):
        gb.step_host(acts)
    acts[5, 1] = 7
    with pytest.raises(m.InvalidArgument, match=r"invalid action 7 for environment 5, robot 1"):
        gb.step_host(acts)
