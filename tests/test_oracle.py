"""CPU: pin the C restatement (oracle/mrsim_oracle.c) before trusting it.

1. Bit-exact against the reference itself (oracle/_ref): RNG streams, the
   reference's 1000 random QPs, apply_barrier on random teams, and full
   reset + random-action rollouts of every benchmark config over the horizon
   (every pose, reward, obs value and discrete field identical).
2. The reference's own golden values (test_scenario_rules.cpp, test_qp.cpp,
   test_framework.cpp) restated against the oracle.
"""
import ctypes

import numpy as np
import pytest

import paper_2505_06771_b200 as m
from util import diff_structs

CONFIGS = [("navigation", 3), ("navigation", 4), ("predator_prey", 3), ("predator_prey", 6), ("discovery", 4),
           ("discovery", 6), ("rware", 3), ("rware", 4), ("rware", 6), ("foraging", 3), ("foraging", 4),
           ("foraging", 6), ("material_transport", 4), ("material_transport", 10), ("arctic_transport", 4),
           ("arctic_transport", 10), ("warehouse", 4), ("random_waypoints", 4)]
ARCTIC_SPAWN = [-1.55, -1.05, -0.9, 0.9]


@pytest.fixture(scope="module")
def orc():
    import oraclebind

    if not oraclebind.available():
        pytest.skip("oracle/_build/libmrsim_oracle.so not built")
    return oraclebind


def cfg_and_spec(ref, task, n, **kw):
    cfg = m.make_default_config(task)
    tile = cfg.raw.het_rows > 0
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=tile)
    layout = {}
    if task == "arctic_transport" and n > 4:
        cfg.set_layout("arctic.spawn_zone", ARCTIC_SPAWN)
        layout["arctic.spawn_zone"] = ARCTIC_SPAWN
    for k, v in kw.items():
        setattr(cfg.raw, k, v)
    sp = ref.spec(task, num_robots=n, tile_roster=tile, layout=layout,
                  max_steps=kw.get("max_steps", 0), barrier=kw.get("barrier_enabled", -1),
                  noise=kw.get("action_noise_scale", -1.0), controller=kw.get("controller", -1))
    return cfg, sp


def test_rng_streams_bit_exact(orc, ref):
    for seed in (0, 1, 42, 2**63 + 5):
        for kind, n in ((0, 0), (1, 0), (2, 0), (3, 5), (3, 7)):
            fo, uo = np.zeros(64), np.zeros(64, dtype=np.uint64)
            fr, ur = np.zeros(64), np.zeros(64, dtype=np.uint64)
            orc.lib().orc_rng_draws(seed, 7, kind, n, 64, orc.dptr(fo), uo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
            ref.lib().ref_rng_draws(seed, 7, kind, n, 64, ref.dptr(fr), ur.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
            assert np.array_equal(fo, fr) and np.array_equal(uo, ur)
    for root in (0, 3):
        for ep in (0, 1, 999, 123456):
            assert orc.lib().orc_derive_episode_seed(root, ep) == ref.lib().ref_derive_episode_seed(root, ep)
            for step in (0, 69):
                for r in range(4):
                    s = orc.lib().orc_derive_episode_seed(root, ep)
                    assert orc.lib().orc_policy_action(s, step, r) == ref.lib().ref_policy_action(s, step, r)


def test_qp_bit_exact_on_reference_random_qps(orc, ref):
    # generator and seed of test_qp.cpp:91-107
    n, mm, A, b, u = ref.random_qps(2024, 1000)
    for t in range(1000):
        At, bt, ut = A[t, :mm[t], :n[t]], b[t, :mm[t]], u[t, :n[t]]
        lo, hi = np.full(n[t], -1e30), np.full(n[t], 1e30)
        so, uo, io = orc.solve_qp(At, bt, lo, hi, ut)
        sr, ur, ir, _ = ref.solve_qp(At, bt, lo, hi, ut)
        assert so == sr == 0 and io == ir and np.array_equal(uo, ur), t
        en = ref.qp_enumeration(At, bt, ut)  # the reference test's brute-force oracle
        assert abs(0.5 * np.sum((uo - ut) ** 2) - en[1]) <= 1e-6


def test_qp_closed_forms(orc):
    # test_qp.cpp:9-72
    inf = 1e30
    s, u, _ = orc.solve_qp(np.zeros((0, 2)), [], [-inf, -inf], [inf, inf], [0.1, -0.05])
    assert s == 0 and u[0] == 0.1 and u[1] == -0.05
    s, u, _ = orc.solve_qp([[1.0, 0.0]], [0.0], [-inf, -inf], [inf, inf], [0.1, 0.0])
    assert s == 0 and abs(u[0]) < 1e-12 and abs(u[1]) < 1e-12
    s, u, _ = orc.solve_qp(np.zeros((0, 3)), [], [-1, -1, -1], [1, 1, 1], [2.0, -3.0, 0.25])
    assert s == 0 and np.allclose(u, [1, -1, 0.25])
    assert orc.solve_qp([[1.0], [-1.0]], [0.0, -1.0], [-inf], [inf], [0.0])[0] == 1
    assert orc.solve_qp([[-1.0, -1.0]], [-3.0], [-1, -1], [1, 1], [0.0, 0.0])[0] == 1


@pytest.mark.parametrize("N", [2, 4, 10])
def test_apply_barrier_bit_exact(N, orc, ref):
    rng = np.random.default_rng(N)
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(N)
    rb = ref.RefBatch(ref.spec("navigation", num_robots=N))
    for t in range(150):
        poses = []
        while len(poses) < N:
            p = (rng.uniform(-1.4, 1.4), rng.uniform(-0.8, 0.8), rng.uniform(-np.pi, np.pi))
            if all(np.hypot(p[0] - q[0], p[1] - q[1]) >= 0.15 for q in poses):
                poses.append(p)
        poses = np.array(poses)
        nom = np.stack([rng.uniform(-0.3, 0.3, N), rng.uniform(-4, 4, N)], axis=1)
        nob = int(rng.integers(0, 4))
        obs = np.stack([rng.uniform(-1, 1, nob), rng.uniform(-0.6, 0.6, nob), np.full(nob, 0.12)], axis=1) \
            if nob else None
        masks = rng.integers(0, 2**N, nob).astype(np.uint64) if nob else None
        co, io = orc.apply_barrier(cfg.raw, poses, nom, obs, masks)
        cr, ir, _ = ref.apply_barrier(rb, poses, nom, obs, masks)
        assert io == ir and np.array_equal(co, cr), t


@pytest.mark.parametrize("task,n", CONFIGS)
def test_rollouts_bit_exact_against_reference(task, n, orc, ref):
    cfg, sp = cfg_and_spec(ref, task, n)
    B = 6
    T = cfg.raw.max_steps + 3
    seeds = [m.derive_episode_seed(11, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    robs = rb.reset(seeds)
    envs = [orc.OracleEnv(cfg.raw) for _ in range(B)]
    for e, env in enumerate(envs):
        assert np.array_equal(env.reset(seeds[e]), robs[e])
    for t in range(T):
        acts = rb.random_actions()
        robs, rrew, rdone, _ = rb.step(acts)
        rs = rb.get_states()
        for e, env in enumerate(envs):
            obs, rew, done = env.step(acts[e])
            assert rew == rrew[e] and done == bool(rdone[e]) and np.array_equal(obs, robs[e]), (t, e)
            d = diff_structs(env.state, rs[e])
            d.pop("episode_return", None)
            assert d == {}, (t, e, d)


@pytest.mark.parametrize("task,n", [("navigation", 4), ("rware", 4), ("random_waypoints", 4),
                                    ("random_waypoints", 8), ("material_transport", 4)])
def test_pose_controller_rollouts_bit_exact(task, n, orc, ref):
    # ControllerKind::UnicyclePose (controllers.hpp:68-82, batch.hpp:169-195)
    cfg, sp = cfg_and_spec(ref, task, n, controller=1, max_steps=120)
    rb = ref.RefBatch(sp)
    seeds = [m.derive_episode_seed(3, e) for e in range(4)]
    robs = rb.reset(seeds)
    envs = [orc.OracleEnv(cfg.raw) for _ in seeds]
    for e, env in enumerate(envs):
        assert np.array_equal(env.reset(seeds[e]), robs[e])
    for t in range(120):
        acts = rb.random_actions()
        robs, rrew, rdone, _ = rb.step(acts)
        rs = rb.get_states()
        for e, env in enumerate(envs):
            obs, rew, done = env.step(acts[e])
            assert rew == rrew[e] and np.array_equal(obs, robs[e]), (t, e)
            d = diff_structs(env.state, rs[e])
            d.pop("episode_return", None)
            assert d == {}, (t, e, d)


def test_random_waypoints_reassignment_and_noise(orc, ref):
    # test_scenario_rules.cpp:545-566: seed 99, all-stay, targets change within 100 steps
    cfg = m.make_default_config("random_waypoints")
    cfg.max_steps = 200
    env = orc.OracleEnv(cfg.raw)
    env.reset(99)
    changes = 0
    for _ in range(100):
        before = np.array(env.state.targets)[:4].copy()
        env.step([0] * 4)
        changes += int(np.sum(np.any(np.array(env.state.targets)[:4] != before, axis=1)))
    assert changes > 0
    # waypoint noise must not consume draws for this task (its waypoints ignore the rng)
    cfg2, sp = cfg_and_spec(ref, "random_waypoints", 4, action_noise_scale=0.3, max_steps=60)
    rb = ref.RefBatch(sp)
    rb.reset([1, 2])
    envs = [orc.OracleEnv(cfg2.raw) for _ in range(2)]
    for env, sd in zip(envs, [1, 2]):
        env.reset(sd)
    for t in range(60):
        acts = rb.random_actions()
        robs, rrew, _, _ = rb.step(acts)
        rs = rb.get_states()
        for e, env in enumerate(envs):
            obs, rew, _ = env.step(acts[e])
            assert np.array_equal(obs, robs[e]) and diff_structs(env.state, rs[e]).keys() <= {"episode_return"}


def test_rollouts_with_noise_and_barrier_off(orc, ref):
    for kw in ({"action_noise_scale": 0.25}, {"barrier_enabled": 0}):
        cfg, sp = cfg_and_spec(ref, "rware", 4, **kw)
        rb = ref.RefBatch(sp)
        seeds = [5, 6, 7]
        rb.reset(seeds)
        envs = [orc.OracleEnv(cfg.raw) for _ in seeds]
        for env, s in zip(envs, seeds):
            env.reset(s)
        for t in range(40):
            acts = rb.random_actions()
            robs, rrew, _, _ = rb.step(acts)
            for e, env in enumerate(envs):
                obs, rew, _ = env.step(acts[e])
                assert rew == rrew[e] and np.array_equal(obs, robs[e])


# ---- the reference's golden episodes (test_scenario_rules.cpp), restated on the oracle ----

class Golden:
    """test_scenario_rules.cpp:13-36: barrier off, hand-placed poses, all-stay steps."""

    def __init__(self, orc, task, seed=1234):
        self.cfg = m.make_default_config(task)
        self.cfg.raw.barrier_enabled = 0
        self.env = orc.OracleEnv(self.cfg.raw)
        self.env.reset(seed)
        self.cum = 0.0

    @property
    def s(self):
        return self.env.state

    def place(self, r, x, y, th=0.0):
        self.s.x[r], self.s.y[r], self.s.theta[r] = x, y, th

    def stay(self):
        _, rew, _ = self.env.step([0] * self.cfg.raw.num_robots)
        self.cum += rew
        return rew


def test_golden_navigation(orc):  # test_scenario_rules.cpp:74-86
    g = Golden(orc, "navigation")
    for i, gl in enumerate([(-1.0, 0.6), (0.0, 0.6), (1.0, 0.6)]):
        g.s.goals[i][0], g.s.goals[i][1] = gl
    g.place(0, -1.0, -0.4, np.pi / 2)
    g.place(1, 0.0, 0.1, np.pi / 2)
    g.place(2, 1.0, 0.35, np.pi / 2)
    for _ in range(3):
        assert g.stay() == pytest.approx(-1.75, abs=1e-9)
    assert g.cum == pytest.approx(-5.25, abs=1e-9)


def test_golden_warehouse(orc):  # :88-103
    g = Golden(orc, "warehouse")
    g.place(0, 1.35, 0.5); g.place(1, 0.0, 0.8); g.place(2, 0.0, -0.8); g.place(3, 0.6, 0.0)
    assert g.stay() == pytest.approx(1.0, abs=1e-9)
    g.place(0, -1.35, 0.5)
    assert g.stay() == pytest.approx(3.0, abs=1e-9)
    assert g.s.scenario_metric == 1.0
    assert g.stay() == pytest.approx(0.0, abs=1e-9)
    assert g.cum == pytest.approx(4.0, abs=1e-9)


def test_golden_material_transport(orc):  # :118-162
    g = Golden(orc, "material_transport")
    g.s.circle_remaining, g.s.rect_remaining, g.s.total_initial = 75, 15, 90
    g.place(0, 0.2, 0.0); g.place(1, -0.6, 0.8); g.place(2, -0.6, -0.8); g.place(3, 0.8, -0.8)
    assert g.stay() == pytest.approx(1.15, abs=1e-9)
    assert g.s.circle_remaining == 70
    g.place(0, -1.3, 0.0)
    assert g.stay() == pytest.approx(3.65, abs=1e-9)
    assert g.stay() == pytest.approx(-0.1, abs=1e-9)
    g = Golden(orc, "material_transport")
    g.s.circle_remaining, g.s.rect_remaining, g.s.total_initial = 0, 15, 15
    g.place(0, -0.6, 0.8); g.place(1, -0.6, -0.8); g.place(2, 1.3, 0.0); g.place(3, 0.5, 0.8)
    assert g.stay() == pytest.approx(3.75, abs=1e-9)
    g.place(2, -1.3, 0.0)
    assert g.stay() == pytest.approx(11.25, abs=1e-9)
    assert g.s.delivered == 15
    assert g.stay() == 0.0


def test_golden_foraging(orc):  # :164-196
    g = Golden(orc, "foraging")
    g.s.resources[0][0], g.s.resources[0][1] = 0.0, 0.0
    g.s.resources[1][0], g.s.resources[1][1] = 1.0, 0.5
    g.s.levels[0], g.s.levels[1] = 3, 2
    g.s.foraged[0] = g.s.foraged[1] = 0
    g.place(0, 0.25, 0.0); g.place(1, -0.25, 0.0); g.place(2, 0.0, -0.8)
    assert g.stay() == pytest.approx(3.0, abs=1e-9)
    g.place(2, 1.0, 0.25)
    assert g.stay() == pytest.approx(2.0, abs=1e-9)
    assert g.stay() == 0.0
    assert g.cum == pytest.approx(5.0, abs=1e-9)


def test_golden_discovery(orc):  # :198-255
    g = Golden(orc, "discovery")
    lms = [(0.3, 0.0), (1, 1), (1, -1), (-1, 1), (-1, -1), (0, 1)]
    for k, (x, y) in enumerate(lms):
        g.s.landmarks[k][0], g.s.landmarks[k][1] = x, y
        g.s.sensed[k] = 0
        g.s.tagged[k] = 0 if k == 0 else 1
    g.place(0, -1.2, 0.8); g.place(1, -1.2, 0.3); g.place(2, -1.2, -0.3); g.place(3, -1.2, -0.8)
    assert g.stay() == pytest.approx(-0.05, abs=1e-9)
    g.place(0, 0.0, 0.0)
    assert g.stay() == pytest.approx(0.95, abs=1e-9)
    g.place(2, 0.3, 0.2)
    assert g.stay() == pytest.approx(5.0, abs=1e-9)
    assert g.s.scenario_metric == 1.0
    assert g.stay() == pytest.approx(0.0, abs=1e-9)


def test_golden_arctic(orc):  # :257-306
    g = Golden(orc, "arctic_transport")
    g.place(0, -1.0, 0.8); g.place(1, -1.0, -0.8); g.place(2, 0.2, 0.4); g.place(3, 0.2, -0.4)
    assert g.stay() == pytest.approx(-0.2, abs=1e-9)
    g.place(2, 1.4, 0.3); g.place(3, 1.4, -0.3)
    assert g.stay() == pytest.approx(0.0, abs=1e-9)
    assert g.stay() == pytest.approx(0.0, abs=1e-9)


def test_golden_predator_prey(orc):  # :308-326
    g = Golden(orc, "predator_prey")
    g.s.prey[0], g.s.prey[1] = 1.45, 0.85
    g.place(0, 1.21, 0.85)
    g.place(1, 1.2662 + 0.0141421356, 0.6662 + 0.0141421356)
    g.place(2, 1.45, 0.61)
    for _ in range(3):
        assert g.stay() == pytest.approx(10.0, abs=1e-9)
        assert g.s.prey[0] == 1.45 and g.s.prey[1] == 0.85
    assert g.s.scenario_metric == 3.0


def test_golden_rware(orc):  # :328-387
    g = Golden(orc, "rware")
    g.s.requests[0], g.s.requests[1], g.s.requests[2] = 1, 2, 3
    g.place(0, -0.2, -0.3); g.place(1, 0.9, 0.8); g.place(2, 0.9, -0.8)
    assert g.stay() == 0.0
    assert g.s.carried[0] == 1 and g.s.slot_shelf[0] == 0
    g.place(0, -1.35, 0.0)
    assert g.stay() == pytest.approx(1.0, abs=1e-9)
    reqs = list(g.s.requests[:3])
    assert 1 not in reqs and len(set(reqs)) == 3 and all(1 <= r <= 6 for r in reqs)
    assert g.s.carried[0] == 1
    g.place(0, -0.2, -0.3)
    assert g.stay() == 0.0
    assert g.s.carried[0] == 0 and g.s.slot_shelf[0] == 1


def test_all_stay_freezes_world(orc):  # test_framework.cpp:187-198
    cfg = m.make_default_config("navigation")
    env = orc.OracleEnv(cfg.raw)
    env.reset(3)
    x0 = list(env.state.x[:3])
    _, r1, _ = env.step([0, 0, 0])
    _, r2, _ = env.step([0, 0, 0])
    assert list(env.state.x[:3]) == x0 and r1 == r2


@pytest.mark.parametrize("name", ["navigation", "discovery", "material_transport"])
def test_barrier_on_rollouts_never_collide(name, orc):  # test_scenario_rules.cpp:499-513
    cfg = m.make_default_config(name)
    arng_key = 45 ^ 0x5EED
    env = orc.OracleEnv(cfg.raw)
    env.reset(45)
    # the reference test draws actions from SplitRng::from_seed(seed ^ 0x5eed) (no fork); emulate in python
    key = m.batch.mix64((arng_key + 0x9E3779B97F4A7C15) & (2**64 - 1))
    ctr = 0
    for t in range(1000):
        acts = []
        for r in range(cfg.raw.num_robots):
            ctr += 1
            z = m.batch.mix64((key + ctr * 0x9E3779B97F4A7C15) & (2**64 - 1))
            acts.append((z * 5) >> 64)
        _, _, done = env.step(acts)
        assert env.state.collisions == 0
        assert env.state.min_pairwise_distance >= cfg.raw.safety_radius - 1e-3
        if done:
            env.reset(45 + t + 1)


# ---- feedforward policy (policy.hpp:95-116, 445-480) ----

@pytest.mark.parametrize("greedy", [True, False])
@pytest.mark.parametrize("task,n", [("navigation", 4), ("discovery", 6), ("rware", 4), ("arctic_transport", 10)])
def test_policy_actions_bit_exact_against_reference(task, n, greedy, orc, ref, tmp_path):
    cfg, sp = cfg_and_spec(ref, task, n)
    D = cfg.obs_dim
    w = m.FeedforwardWeights.random([D, 32, 16, 5], ["relu", "tanh", "identity"], seed=n, scale=2.0)
    path = tmp_path / "w.txt"
    path.write_text(w.to_text())
    spec = ("feedforward:" if greedy else "feedforward_sample:") + str(path)
    rb = ref.RefBatch(sp)
    seeds = [m.derive_episode_seed(9, e) for e in range(4)]
    rb.reset(seeds)
    envs = [orc.OracleEnv(cfg.raw) for _ in seeds]
    for env, s in zip(envs, seeds):
        env.reset(s)
    for t in range(25):
        ra = rb.policy_actions(spec)
        for e, env in enumerate(envs):
            oa = [orc.policy_act(cfg.raw, env.state, r, w, greedy) for r in range(n)]
            assert oa == list(ra[e]), (t, e)
        rb.step(ra)
        for e, env in enumerate(envs):
            env.step(ra[e])


def test_weights_text_round_trip_and_errors(tmp_path):
    w = m.FeedforwardWeights.random([5, 8, 5], ["tanh", "identity"], seed=3)
    w2 = m.FeedforwardWeights.from_text(w.to_text())
    for a, b in zip(w.layers, w2.layers):
        assert a[:3] == b[:3] and np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    with pytest.raises(m.InvalidArgument, match="magic"):
        m.FeedforwardWeights.from_text("nope 1")
    with pytest.raises(m.InvalidArgument, match="5 logits"):
        m.FeedforwardWeights.random([5, 4], ["identity"])
    with pytest.raises(m.InvalidArgument, match="activation"):
        m.FeedforwardWeights.random([5, 5], ["gelu"])
    with pytest.raises(RuntimeError, match="cannot open"):
        m.FeedforwardWeights.load(str(tmp_path / "missing.txt"))
