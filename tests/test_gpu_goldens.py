"""The reference's own golden episodes and invariant suites
(/root/reference/proj/tests/test_scenario_rules.cpp), run on the CUDA kernel
through the C-ABI, and closed-loop rollouts that fire every discrete branch
of the scenario transitions, compared field by field with the UNMODIFIED
reference (oracle/_ref) on identical states and actions.

Goldens (test_scenario_rules.cpp:13-36): barrier off, hand-placed poses,
all-stay steps, so the expected rewards are exact hand-computed constants.
Each golden runs in B = 40 identical envs (several warp tasks, later
iterations of the persistent loop) and every env must agree with the
reference: discrete fields bit-exact, poses and reals within 1e-12 (the
stay action is an exact fixed point of the controller), rewards within
1e-9 of the golden constant (the reference test uses Catch::Approx margins).

Branch-firing rollouts: the reference's scripted policies (policy.hpp:242-416)
drive both sides with the same actions; each test asserts the branch it pins
fired at least once and prints how often:
  rware.hpp:79-95         dropoff + request resample on the step stream
  predator_prey.hpp:80-89 tag (+10), flash timer
  warehouse.hpp:43-50     pickup / delivery
  navigation.hpp:53-61    success at done (finalize)
Tolerances: fp64 product path, discrete bit-exact, poses 1e-8 m / 1e-7 rad
over the horizon, rewards 1e-9 * max(1, |r|).
"""
import numpy as np
import pytest

import paper_2505_06771_b200 as m
from test_gpu_step import compare_states, make_cfgs

pytestmark = pytest.mark.gpu

GB = 40  # envs per golden: 10 warp tasks of the L = 4 kernel, 40 threads of the env-per-thread kernel


class DevGolden:
    """Golden (test_scenario_rules.cpp:13-36) on the device, mirrored on the reference."""

    def __init__(self, ref, task, seed=1234, B=GB):
        self.cfg = m.make_default_config(task)
        self.cfg.raw.barrier_enabled = 0
        self.N = self.cfg.raw.num_robots
        self.B = B
        self.gb = m.CudaEnvBatch(self.cfg, B, fp64=True)
        self.gb.reset_seeds([seed] * B)
        self.rb = ref.RefBatch(ref.spec(task, barrier=0))
        self.rb.reset([seed] * B)
        self.states = list(self.gb.get_states())
        pe, ae, bad, re_ = compare_states(self.states, self.rb.get_states(), self.N, 0, 0, 0)
        assert pe == 0 and ae == 0 and re_ == 0 and not bad  # reset_env is bit-exact
        self.dirty = False
        self.cum = 0.0

    @property
    def s(self):
        """An editable view: edits apply to every env's state."""
        self.dirty = True
        return _Fan(self.states)

    def place(self, r, x, y, th=0.0):
        for st in self.states:
            st.x[r], st.y[r], st.theta[r] = x, y, th
        self.dirty = True

    def get(self, field):
        vals = [getattr(st, field) for st in self.states]
        v0 = vals[0]
        if hasattr(v0, "__len__"):
            vals = [list(v) for v in vals]
            v0 = vals[0]
        assert all(v == v0 for v in vals), field
        return v0

    def stay(self):
        if self.dirty:
            self.gb.set_states(self.states)
            self.rb.set_states(self.states)
            self.dirty = False
        acts = np.zeros((self.B, self.N), dtype=np.int32)
        _, grew, gdone = self.gb.step_host(acts)
        _, rrew, rdone, _ = self.rb.step(acts)
        gs, rs = self.gb.get_states(), self.rb.get_states()
        pe, ae, bad, re_ = compare_states(gs, rs, self.N, 0, 0, 0)
        assert not bad, bad[:4]
        assert pe <= 1e-12 and ae <= 1e-12 and re_ <= 1e-12, (pe, ae, re_)
        assert np.array_equal(gdone, rdone)
        assert np.all(grew == grew[0]), "identical envs must give identical rewards"
        assert abs(grew[0] - rrew[0]) <= 1e-12 * max(1.0, abs(rrew[0]))
        self.states = list(gs)
        self.cum += float(grew[0])
        return float(grew[0])


class _Fan:
    """Attribute fan-out over a list of ctypes states (g.s.field[i] = v writes every env)."""

    def __init__(self, states):
        object.__setattr__(self, "_states", states)

    def __getattr__(self, name):
        vals = [getattr(st, name) for st in self._states]
        if hasattr(vals[0], "__len__"):
            return _FanArr(vals)
        return vals[0]

    def __setattr__(self, name, value):
        for st in self._states:
            setattr(st, name, value)


class _FanArr:
    def __init__(self, arrs):
        self.arrs = arrs

    def __getitem__(self, i):
        v = self.arrs[0][i]
        if hasattr(v, "__len__"):
            return _FanArr([a[i] for a in self.arrs])
        return v

    def __setitem__(self, i, value):
        for a in self.arrs:
            a[i] = value


def test_golden_navigation(ref):  # test_scenario_rules.cpp:74-86
    g = DevGolden(ref, "navigation")
    for i, gl in enumerate([(-1.0, 0.6), (0.0, 0.6), (1.0, 0.6)]):
        g.s.goals[i][0] = gl[0]
        g.s.goals[i][1] = gl[1]
    g.place(0, -1.0, -0.4, np.pi / 2)
    g.place(1, 0.0, 0.1, np.pi / 2)
    g.place(2, 1.0, 0.35, np.pi / 2)
    for _ in range(3):
        assert g.stay() == pytest.approx(-1.75, abs=1e-9)
    assert g.cum == pytest.approx(-5.25, abs=1e-9)


def test_golden_navigation_success_at_done(ref):  # navigation.hpp:53-61 (finalize)
    g = DevGolden(ref, "navigation")
    for st in g.states:
        st.step_index = g.cfg.raw.max_steps - 1
        for i in range(3):
            st.goals[i][0], st.goals[i][1] = st.x[i] + 0.05, st.y[i]  # within the 0.1 m on-goal radius
    g.dirty = True
    g.stay()
    assert g.get("success") == 1 and g.get("scenario_metric") == 1.0


def test_golden_warehouse(ref):  # :88-103
    g = DevGolden(ref, "warehouse")
    g.place(0, 1.35, 0.5); g.place(1, 0.0, 0.8); g.place(2, 0.0, -0.8); g.place(3, 0.6, 0.0)
    assert g.stay() == pytest.approx(1.0, abs=1e-9)
    assert g.get("loaded")[0] == 1
    g.place(0, -1.35, 0.5)
    assert g.stay() == pytest.approx(3.0, abs=1e-9)
    assert g.get("scenario_metric") == 1.0 and g.get("loaded")[0] == 0
    assert g.stay() == pytest.approx(0.0, abs=1e-9)
    assert g.cum == pytest.approx(4.0, abs=1e-9)


def test_golden_material_transport(ref):  # :118-162
    g = DevGolden(ref, "material_transport")
    g.s.circle_remaining = 75
    g.s.rect_remaining = 15
    g.s.total_initial = 90
    g.place(0, 0.2, 0.0); g.place(1, -0.6, 0.8); g.place(2, -0.6, -0.8); g.place(3, 0.8, -0.8)
    assert g.stay() == pytest.approx(1.15, abs=1e-9)
    assert g.get("circle_remaining") == 70
    g.place(0, -1.3, 0.0)
    assert g.stay() == pytest.approx(3.65, abs=1e-9)
    assert g.stay() == pytest.approx(-0.1, abs=1e-9)
    g = DevGolden(ref, "material_transport")
    g.s.circle_remaining = 0
    g.s.rect_remaining = 15
    g.s.total_initial = 15
    g.place(0, -0.6, 0.8); g.place(1, -0.6, -0.8); g.place(2, 1.3, 0.0); g.place(3, 0.5, 0.8)
    assert g.stay() == pytest.approx(3.75, abs=1e-9)
    g.place(2, -1.3, 0.0)
    assert g.stay() == pytest.approx(11.25, abs=1e-9)
    assert g.get("delivered") == 15
    assert g.stay() == 0.0


def test_golden_foraging(ref):  # :164-196
    g = DevGolden(ref, "foraging")
    g.s.resources[0][0] = 0.0
    g.s.resources[0][1] = 0.0
    g.s.resources[1][0] = 1.0
    g.s.resources[1][1] = 0.5
    g.s.levels[0] = 3
    g.s.levels[1] = 2
    g.s.foraged[0] = 0
    g.s.foraged[1] = 0
    g.place(0, 0.25, 0.0); g.place(1, -0.25, 0.0); g.place(2, 0.0, -0.8)
    assert g.stay() == pytest.approx(3.0, abs=1e-9)
    assert g.get("foraged")[:2] == [1, 0]
    g.place(2, 1.0, 0.25)
    assert g.stay() == pytest.approx(2.0, abs=1e-9)
    assert g.stay() == 0.0
    assert g.cum == pytest.approx(5.0, abs=1e-9)


def test_golden_discovery(ref):  # :198-255
    g = DevGolden(ref, "discovery")
    lms = [(0.3, 0.0), (1, 1), (1, -1), (-1, 1), (-1, -1), (0, 1)]
    for k, (x, y) in enumerate(lms):
        g.s.landmarks[k][0] = x
        g.s.landmarks[k][1] = y
        g.s.sensed[k] = 0
        g.s.tagged[k] = 0 if k == 0 else 1
    g.place(0, -1.2, 0.8); g.place(1, -1.2, 0.3); g.place(2, -1.2, -0.3); g.place(3, -1.2, -0.8)
    assert g.stay() == pytest.approx(-0.05, abs=1e-9)
    g.place(0, 0.0, 0.0)
    assert g.stay() == pytest.approx(0.95, abs=1e-9)
    assert g.get("sensed")[0] == 1
    g.place(2, 0.3, 0.2)
    assert g.stay() == pytest.approx(5.0, abs=1e-9)
    assert g.get("scenario_metric") == 1.0 and g.get("tagged")[0] == 1
    assert g.stay() == pytest.approx(0.0, abs=1e-9)


def test_golden_arctic(ref):  # :257-306
    g = DevGolden(ref, "arctic_transport")
    g.place(0, -1.0, 0.8); g.place(1, -1.0, -0.8); g.place(2, 0.2, 0.4); g.place(3, 0.2, -0.4)
    assert g.stay() == pytest.approx(-0.2, abs=1e-9)
    g.place(2, 1.4, 0.3); g.place(3, 1.4, -0.3)
    assert g.stay() == pytest.approx(0.0, abs=1e-9)
    assert g.stay() == pytest.approx(0.0, abs=1e-9)


def test_golden_arctic_success_at_done(ref):  # arctic_transport.hpp:88-97 (finalize)
    g = DevGolden(ref, "arctic_transport")
    g.place(0, -1.0, 0.8); g.place(1, -1.0, -0.8); g.place(2, 1.4, 0.3); g.place(3, 1.4, -0.3)
    for st in g.states:
        st.step_index = g.cfg.raw.max_steps - 1
    g.stay()
    assert g.get("success") == 1 and g.get("scenario_metric") == 1.0


def test_golden_predator_prey_cornered(ref):  # :308-326
    g = DevGolden(ref, "predator_prey")
    g.s.prey[0] = 1.45
    g.s.prey[1] = 0.85
    g.place(0, 1.21, 0.85)
    g.place(1, 1.2662 + 0.0141421356, 0.6662 + 0.0141421356)
    g.place(2, 1.45, 0.61)
    for _ in range(3):
        assert g.stay() == pytest.approx(10.0, abs=1e-9)
        assert g.get("prey")[:2] == [1.45, 0.85]
        assert g.get("flash_timer") == g.cfg.get_layout("pp.flash_steps")[0]
    assert g.get("scenario_metric") == 3.0


def test_golden_predator_prey_contained(ref):  # :424-443
    g = DevGolden(ref, "predator_prey")
    g.s.prey[0] = 1.5
    g.s.prey[1] = 0.9
    g.place(0, 1.28, 0.9)
    g.place(1, 1.34, 0.74)
    g.place(2, 1.5, 0.68)
    tags = sum(1 for _ in range(5) if g.stay() > 0)
    assert tags == 5


def test_golden_predator_prey_flash_decays(ref):  # predator_prey.hpp:80-89: timer counts down untagged
    g = DevGolden(ref, "predator_prey")
    g.s.prey[0] = 0.0
    g.s.prey[1] = 0.0
    g.s.flash_timer = 3
    g.place(0, -1.4, 0.8); g.place(1, -1.4, -0.8); g.place(2, 1.4, 0.8)
    for want in (2, 1, 0, 0):
        assert g.stay() == 0.0
        assert g.get("flash_timer") == want


def test_golden_rware(ref):  # :328-387
    g = DevGolden(ref, "rware")
    g.s.requests[0] = 1
    g.s.requests[1] = 2
    g.s.requests[2] = 3
    g.place(0, -0.2, -0.3); g.place(1, 0.9, 0.8); g.place(2, 0.9, -0.8)
    assert g.stay() == 0.0
    assert g.get("carried")[0] == 1 and g.get("slot_shelf")[0] == 0
    g.place(0, -1.35, 0.0)
    assert g.stay() == pytest.approx(1.0, abs=1e-9)  # dropoff: request 1 resampled on the step stream
    reqs = g.get("requests")[:3]
    assert 1 not in reqs and len(set(reqs)) == 3 and all(1 <= r <= 6 for r in reqs)
    assert g.get("carried")[0] == 1
    g.place(0, -0.2, -0.3)
    assert g.stay() == 0.0
    assert g.get("carried")[0] == 0 and g.get("slot_shelf")[0] == 1


def test_golden_rware_non_requested_dropoff_is_noop(ref):  # :363-387
    g = DevGolden(ref, "rware")
    g.s.requests[0] = 2
    g.s.requests[1] = 3
    g.s.requests[2] = 4
    g.place(0, -0.2, -0.3); g.place(1, 0.9, 0.8); g.place(2, 0.9, -0.8)
    g.stay()
    assert g.get("carried")[0] == 1
    g.place(0, -1.35, 0.0)
    assert g.stay() == 0.0
    assert g.get("requests")[:3] == [2, 3, 4] and g.get("scenario_metric") == 0.0


# ---- invariant suites (test_scenario_rules.cpp:445-526), device vs reference ----

def _arng_actions(seed, n, steps):
    """SplitRng::from_seed(seed ^ 0x5eed).uniform_int(5) per robot (test_scenario_rules.cpp:47-53)."""
    key = m.batch.mix64(((seed ^ 0x5EED) + 0x9E3779B97F4A7C15) & (2**64 - 1))
    out = np.zeros((steps, n), dtype=np.int32)
    ctr = 0
    for t in range(steps):
        for r in range(n):
            ctr += 1
            z = m.batch.mix64((key + ctr * 0x9E3779B97F4A7C15) & (2**64 - 1))
            out[t, r] = (z * 5) >> 64
    return out


def _run_random_steps(ref, name, total, seed, check):
    cfg = m.make_default_config(name)
    N = cfg.raw.num_robots
    gb = m.CudaEnvBatch(cfg, 1, fp64=True)
    rb = ref.RefBatch(ref.spec(name))
    gb.reset_seeds([seed])
    rb.reset([seed])
    acts = _arng_actions(seed, N, total)
    last = None
    for t in range(total):
        _, grew, gdone = gb.step_host(acts[t][None])
        _, rrew, rdone, _ = rb.step(acts[t][None])
        gs, rs = gb.get_states(), rb.get_states()
        pe, ae, bad, re_ = compare_states(gs, rs, N, 0, 0, 0)
        assert not bad and pe <= 1e-8 and ae <= 1e-7 and re_ <= 1e-8, (name, t, pe, ae, bad[:3])
        assert abs(grew[0] - rrew[0]) <= 1e-9 * max(1.0, abs(rrew[0])) and gdone[0] == rdone[0]
        check(cfg, gs[0], last)
        last = gs[0]
        if gdone[0]:
            gb.reset_seeds([seed + t + 1])
            rb.reset([seed + t + 1])
            last = None


def test_invariant_material_transport_conserves_units(ref):  # :445-459
    def check(cfg, st, last):
        carried = sum(st.loads[: cfg.raw.num_robots])
        assert st.circle_remaining + st.rect_remaining + carried + st.delivered == pytest.approx(
            st.total_initial, abs=1e-9)
        assert st.circle_remaining >= 0 and st.rect_remaining >= 0
    _run_random_steps(ref, "material_transport", 1000, 42, check)


def test_invariant_rware_shelves_and_requests(ref):  # :461-485
    def check(cfg, st, last):
        total = int(cfg.get_layout("rware.num_shelves")[0])
        ids = [v for v in list(st.slot_shelf[: st.num_slots]) + list(st.carried[: cfg.raw.num_robots]) if v]
        assert sorted(ids) == list(range(1, total + 1))
        reqs = list(st.requests[: st.num_requests])
        assert len(reqs) == int(cfg.get_layout("rware.request_size")[0]) and len(set(reqs)) == len(reqs)
        assert all(1 <= r <= total for r in reqs)
    _run_random_steps(ref, "rware", 1000, 43, check)


@pytest.mark.parametrize("name", ["discovery", "foraging", "warehouse", "predator_prey", "rware"])
def test_invariant_counters_never_decrease(name, ref):  # :487-497
    def check(cfg, st, last):
        if last is not None:
            assert st.scenario_metric >= last.scenario_metric and st.collisions >= last.collisions
        th = np.array(st.theta[: cfg.raw.num_robots])
        assert np.all(th > -np.pi) and np.all(th <= np.pi)
    _run_random_steps(ref, name, 1000, 44, check)


@pytest.mark.parametrize("name", ["navigation", "discovery", "material_transport"])
def test_invariant_barrier_on_never_collides(name, ref):  # :499-513
    def check(cfg, st, last):
        N = cfg.raw.num_robots
        assert st.collisions == 0
        assert st.min_pairwise_distance >= cfg.raw.safety_radius - 1e-3
        hw, hh = cfg.raw.arena_half_width, cfg.raw.arena_half_height
        assert np.all(np.abs(st.x[:N]) <= hw) and np.all(np.abs(st.y[:N]) <= hh)
    _run_random_steps(ref, name, 1000, 45, check)


def test_random_waypoints_reassignment(ref):  # :547-567
    cfg = m.make_default_config("random_waypoints")
    cfg.max_steps = 200
    gb = m.CudaEnvBatch(cfg, 2, fp64=True)
    gb.reset_seeds([99, 99])
    rb = ref.RefBatch(ref.spec("random_waypoints", max_steps=200))
    rb.reset([99, 99])
    re = 0
    for t in range(100):
        t0 = [list(v) for v in gb.get_states()[0].targets[:4]]
        gb.step_host(np.zeros((2, 4), dtype=np.int32))
        rb.step(np.zeros((2, 4), dtype=np.int32))
        a, b = gb.get_states()
        assert [list(v) for v in a.targets[:4]] == [list(v) for v in b.targets[:4]]
        pe, ae, bad, re_ = compare_states([a], rb.get_states(0, 1), 4, 0, 0, 0)
        assert not bad and pe <= 1e-8 and re_ <= 1e-8, (t, pe, bad[:3])
        re += sum(1 for i in range(4) if list(a.targets[i]) != t0[i])
    assert re > 0


# ---- closed-loop rollouts that fire the discrete branches ----

def _closed_loop(ref, task, n, policy, steps, B, seed_root, fired, max_steps=0):
    cfg, sp = make_cfgs(ref, task, n, max_steps=max_steps)
    seeds = [m.derive_episode_seed(seed_root, e) for e in range(B)]
    rb = ref.RefBatch(sp)
    rb.reset(seeds)
    gb = m.CudaEnvBatch(cfg, B, fp64=True)
    gb.reset_seeds(seeds)
    counts = {}
    prev = list(rb.get_states())
    for t in range(steps):
        acts = rb.policy_actions(policy)
        _, grew, gdone = gb.step_host(acts)
        _, rrew, rdone, _ = rb.step(acts)
        gs, rs = gb.get_states(), rb.get_states()
        pe, ae, bad, re_ = compare_states(gs, rs, n, 0, 0, 0)
        assert not bad, (t, bad[:4])
        assert pe <= 1e-8 and ae <= 1e-7 and re_ <= 1e-8, (t, pe, ae, re_)
        assert np.array_equal(gdone, rdone), t
        assert np.all(np.abs(grew - rrew) <= 1e-9 * np.maximum(1.0, np.abs(rrew))), t
        for k, v in fired(cfg, prev, list(rs), rrew, rdone).items():
            counts[k] = counts.get(k, 0) + v
        prev = list(rs)
    print(f"{task} N={n} {policy}: {counts}")
    return counts


@pytest.mark.parametrize("n", [4, 6])
def test_rware_dropoff_and_request_resample_fire(n, ref):  # rware.hpp:79-95
    def fired(cfg, prev, cur, rew, done):
        res = sum(1 for a, b in zip(prev, cur) if list(a.requests[: a.num_requests]) != list(b.requests[: b.num_requests]))
        pick = sum(1 for a, b in zip(prev, cur) for i in range(n) if a.carried[i] == 0 and b.carried[i] != 0)
        return {"resamples": res, "pickups": pick, "dropoff_reward": int(np.sum(rew > 0))}
    c = _closed_loop(ref, "rware", n, "scripted_goal", 100, 64, 2, fired)
    assert c["resamples"] > 0 and c["pickups"] > 0 and c["dropoff_reward"] > 0


def test_predator_prey_tags_fire(ref):  # predator_prey.hpp:80-89
    def fired(cfg, prev, cur, rew, done):
        tags = sum(1 for a, b in zip(prev, cur) if b.scenario_metric > a.scenario_metric)
        flash = sum(1 for a, b in zip(prev, cur) if 0 < b.flash_timer < a.flash_timer)
        return {"tags": tags, "flash_decays": flash}
    c = _closed_loop(ref, "predator_prey", 6, "prey_chaser", 30, 64, 22, fired)
    assert c["tags"] > 0 and c["flash_decays"] > 0


def test_navigation_success_fires(ref):  # navigation.hpp:53-61
    def fired(cfg, prev, cur, rew, done):
        return {"success": sum(1 for b, d in zip(cur, done) if d and b.success), "done": int(np.sum(done))}
    c = _closed_loop(ref, "navigation", 4, "scripted_goal", 70, 64, 3, fired, max_steps=70)
    assert c["success"] > 0 and c["done"] == 64


def test_warehouse_delivery_fires(ref):  # warehouse.hpp:43-50
    def fired(cfg, prev, cur, rew, done):
        dl = sum(1 for a, b in zip(prev, cur) if b.scenario_metric > a.scenario_metric)
        ld = sum(1 for a, b in zip(prev, cur) for i in range(4) if not a.loaded[i] and b.loaded[i])
        return {"deliveries": dl, "loads": ld}
    c = _closed_loop(ref, "warehouse", 4, "scripted_goal", 100, 64, 4, fired)
    assert c["loads"] > 0 and c["deliveries"] > 0


def test_foraging_and_discovery_fire(ref):  # foraging.hpp:51-68, discovery.hpp:40-67
    def fired(cfg, prev, cur, rew, done):
        return {"metric_up": sum(1 for a, b in zip(prev, cur) if b.scenario_metric > a.scenario_metric)}
    for task, n in (("foraging", 4), ("discovery", 6)):
        c = _closed_loop(ref, task, n, "scripted_goal", 100, 48, 5, fired)
        assert c["metric_up"] > 0, task


def test_material_transport_load_and_drop_fire(ref):  # material_transport.hpp:49-69
    def fired(cfg, prev, cur, rew, done):
        loads = sum(1 for a, b in zip(prev, cur) for i in range(10) if a.loads[i] == 0 and b.loads[i] > 0)
        drops = sum(1 for a, b in zip(prev, cur) if b.delivered > a.delivered)
        return {"loads": loads, "drops": drops}
    c = _closed_loop(ref, "material_transport", 10, "scripted_goal", 70, 32, 6, fired)
    assert c["loads"] > 0 and c["drops"] > 0
