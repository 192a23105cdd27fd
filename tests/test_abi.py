"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every
symbol include/mrsim_cuda.h declares, its struct sizes match the ctypes
mirror, and its host-side ScenarioConfig resolution equals the reference's
own (make_default_config / resolve_scenario_config, flattened by the
oracle/_ref shim) field by field."""
import ctypes

import pytest

import paper_2505_06771_b200 as m
from paper_2505_06771_b200 import _abi
from util import diff_structs

TASKS = m.TASKS


def test_library_exports_every_declared_symbol():
    lib = m.lib()
    declared = _abi.declared_functions()
    assert len(declared) >= 20
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing
    assert set(declared) == set(_abi.FUNCTIONS), "ctypes signature table out of date"


def test_struct_sizes_match_header_mirror():
    lib = m.lib()
    for which, st in enumerate((_abi.Cfg, _abi.Layout, _abi.EnvState, _abi.Stats, _abi.TrajRecord)):
        assert lib.mrsim_sizeof(which) == ctypes.sizeof(st)
    assert lib.mrsim_sizeof(9) == -1


@pytest.mark.parametrize("task", TASKS)
def test_default_config_matches_reference(task, ref):
    mine = m.make_default_config(task).raw
    theirs = ref.resolve_config(ref.spec(task))
    assert diff_structs(mine, theirs) == {}


@pytest.mark.parametrize("task,n", [
    ("navigation", 4), ("discovery", 6), ("predator_prey", 6), ("rware", 4), ("rware", 6),
    ("foraging", 4), ("foraging", 6), ("material_transport", 10), ("arctic_transport", 10),
    ("warehouse", 6), ("navigation", 16), ("random_waypoints", 8),
])
def test_num_robots_and_roster_tiling_match_reference(task, n, ref):
    cfg = m.make_default_config(task)
    tile = cfg.raw.het_rows > 0
    cfg.set_num_robots(n, tile_roster=tile)
    cfg.validate()
    theirs = ref.resolve_config(ref.spec(task, num_robots=n, tile_roster=tile))
    assert diff_structs(cfg.raw, theirs) == {}


def test_fixed_roster_refuses_num_robots_like_reference(ref):
    cfg = m.make_default_config("discovery")
    with pytest.raises(m.InvalidArgument, match="fixed robot roster"):
        cfg.set_num_robots(6)
    with pytest.raises(ref.RefError, match="fixed robot roster"):
        ref.resolve_config(ref.spec("discovery", num_robots=6))


@pytest.mark.parametrize("key,vals", [
    ("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9]),
    ("rware.slots", [-0.2, -0.3, 0.25, -0.3, 0.7, -0.3, -0.2, 0.3]),
    ("rware.num_shelves", [4]),
    ("discovery.num_landmarks", [3]),
    ("mt.circle_zone", [0.1, 0.2, 0.25]),
    ("pp.flash_steps", [3.7]),
    ("spawn.margin", [0.3]),
])
def test_layout_overrides_match_reference(key, vals, ref):
    task = {"arctic": "arctic_transport", "rware": "rware", "discovery": "discovery", "mt": "material_transport",
            "pp": "predator_prey", "spawn": "navigation"}[key.split(".")[0]]
    cfg = m.make_default_config(task)
    cfg.set_layout(key, vals)
    theirs = ref.resolve_config(ref.spec(task, layout={key: vals}))
    assert diff_structs(cfg.raw, theirs) == {}


def test_pose_controller_config_matches_reference(ref):
    for task in ("navigation", "random_waypoints", "rware"):
        cfg = m.make_default_config(task).set_controller("unicycle_pose")
        cfg.validate()
        theirs = ref.resolve_config(ref.spec(task, controller=1))
        assert diff_structs(cfg.raw, theirs) == {}


def test_overrides_max_steps_barrier_noise(ref):
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(4)
    cfg.max_steps = 70
    cfg.barrier_enabled = 0
    cfg.action_noise_scale = 0.25
    cfg.sub_steps = 5
    theirs = ref.resolve_config(ref.spec("navigation", num_robots=4, max_steps=70, barrier=0, noise=0.25,
                                         sub_steps=5))
    assert diff_structs(cfg.raw, theirs) == {}


def test_validation_errors_mirror_reference():
    with pytest.raises(m.InvalidArgument):
        m.make_default_config("not_a_scenario")
    cfg = m.make_default_config("navigation")
    cfg.max_steps = 0
    with pytest.raises(m.InvalidArgument, match="max_steps"):
        cfg.validate()
    cfg = m.make_default_config("navigation")
    cfg.safety_radius = 0.1
    with pytest.raises(m.InvalidArgument, match="safety_radius"):
        cfg.validate()
    cfg = m.make_default_config("navigation")
    cfg.k_beta = 0.5
    with pytest.raises(m.InvalidArgument, match="stability"):
        cfg.validate()
    cfg = m.make_default_config("rware")
    cfg.set_layout("rware.num_shelves", [7])
    with pytest.raises(m.InvalidArgument, match="fewer slots than shelves"):
        cfg.validate()
    cfg = m.make_default_config("navigation")
    with pytest.raises(m.Unsupported):
        cfg.set_num_robots(17)
    cfg = m.make_default_config("navigation")
    cfg.controller = 2
    with pytest.raises(m.InvalidArgument, match="controller"):
        cfg.validate()
    with pytest.raises(m.InvalidArgument, match="unknown controller"):
        m.make_default_config("navigation").set_controller("pid")
    with pytest.raises(m.InvalidArgument):
        m.make_default_config("navigation").set_layout("no.such.key", [1.0])


@pytest.mark.parametrize("task", TASKS)
def test_obs_dims_match_reference(task, ref):
    # test_framework.cpp:232-259 pins the default-N dimensions
    expected = {"arctic_transport": 31, "discovery": 29, "foraging": 16, "material_transport": 20,
                "navigation": 5, "predator_prey": 9, "rware": 29, "warehouse": 12, "random_waypoints": 5}
    assert m.make_default_config(task).obs_dim == expected[task]
    rb = ref.RefBatch(ref.spec(task))
    assert rb.D == expected[task]


@pytest.mark.parametrize("task,n,dim", [("navigation", 4, 5), ("discovery", 6, 37), ("predator_prey", 6, 15),
                                        ("rware", 4, 31), ("rware", 6, 35), ("foraging", 4, 19),
                                        ("foraging", 6, 25), ("material_transport", 10, 44),
                                        ("arctic_transport", 10, 79)])
def test_baseline_obs_dims(task, n, dim, ref):
    cfg = m.make_default_config(task)
    cfg.set_num_robots(n, tile_roster=cfg.raw.het_rows > 0)
    assert cfg.obs_dim == dim
    rb = ref.RefBatch(ref.spec(task, num_robots=n, tile_roster=True))
    assert rb.D == dim


def test_harness_seed_derivation_matches_reference(ref):
    for root in (0, 1, 12345):
        for ep in (0, 1, 7, 65535, 1 << 20):
            assert m.derive_episode_seed(root, ep) == ref.lib().ref_derive_episode_seed(root, ep)
