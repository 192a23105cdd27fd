"""Episode runs with on-device trajectory capture, the trajectory file format
and replay verification — the caller side of the hot path (SURVEY.md 8(f)
row 1), mirroring the reference:

  run_episodes          harness.hpp:216-300 (waves of `batch` envs, seeds
                        derive_episode_seed(seed, episode), one row per
                        (episode, step, robot), rows ordered env-major)
  build_header / RunConfig / resolve_scenario_config
                        harness.hpp:37-67, 71-103, 105-148
  write / read_trajectory, TrajectoryRow, fnv1a
                        trajectory.hpp:20-180 (same bytes: '#'-header with
                        FNV-1a config hash, %.17g floats)
  verify_trajectory     harness.hpp:444-518

The rows are recorded on the GPU by the step itself (mrsim_capture_*: one
record per (env, robot) per step, written next to the state in HBM) and
rendered by the library's host writer (mrsim_trajectory_write).

Verification replays the header's configuration on the GPU. The device path
is bit-exact on every discrete column against the reference but its poses
agree to ~1e-9 m, not to the last %.17g digit, so rows are compared with
stated tolerances (discrete columns exact; x, y within pos_tol; theta within
ang_tol mod 2 pi; reward and metric within real_tol * max(1, |v|)) instead of
the reference's byte equality. Files written here are byte-compatible with the
reference's read_trajectory (same header, hash and row format).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._lib import InvalidArgument, lib, raise_for
from .batch import CudaEnvBatch, ScenarioConfig, make_default_config

FORMAT_VERSION = 1  # kTrajectoryFormatVersion (trajectory.hpp:20)
COLUMNS = "env,step,robot,x,y,theta,action,reward,done,collisions,metric"  # trajectory.hpp:84-85

RECORD_DTYPE = np.dtype([("x", "<f8"), ("y", "<f8"), ("theta", "<f8"), ("reward", "<f8"), ("metric", "<f8"),
                         ("collisions", "<i8"), ("action", "<i4"), ("done", "<i4")])
ROW_DTYPE = np.dtype([("env", "<i8"), ("step", "<i8"), ("robot", "<i4"), ("x", "<f8"), ("y", "<f8"),
                      ("theta", "<f8"), ("action", "<i4"), ("reward", "<f8"), ("done", "<i4"),
                      ("collisions", "<i8"), ("metric", "<f8")])
assert RECORD_DTYPE.itemsize == ctypes.sizeof(_abi.TrajRecord)


def format_double(v: float) -> str:  # trajectory.hpp:22-26
    return "%.17g" % v


def fnv1a(text: str) -> int:  # trajectory.hpp:28-36
    h = 0xCBF29CE484222325
    for c in text.encode():
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


class TrajectoryHeader:
    """Ordered key = value fields; the hash covers the canonical text (trajectory.hpp:87-112)."""

    def __init__(self, fields=None):
        self.fields: list[tuple[str, str]] = list(fields or [])

    def get(self, key: str) -> str:
        for k, v in self.fields:
            if k == key:
                return v
        raise InvalidArgument(f"trajectory header: missing field '{key}'")

    def has(self, key: str) -> bool:
        return any(k == key for k, _ in self.fields)

    def set(self, key: str, value: str) -> None:
        self.fields.append((key, value))

    def canonical_text(self) -> str:
        return "".join(f"{k} = {v}\n" for k, v in self.fields)

    def hash(self) -> int:
        return fnv1a(self.canonical_text())

    def block(self) -> str:
        """Everything write_trajectory emits before the first row (trajectory.hpp:116-125)."""
        lines = [f"# mrsim-trajectory {FORMAT_VERSION}", f"# config-hash {self.hash():016x}"]
        lines += [f"# {k} = {v}" for k, v in self.fields]
        lines.append(COLUMNS)
        return "\n".join(lines) + "\n"


@dataclass
class RunConfig:
    """RunConfig (harness.hpp:37-67), the fields a GPU run uses."""

    scenario: str = "navigation"
    seed: int = 0
    batch: int = 1
    episodes: int = 1
    policy: str = "random"
    max_steps: int = -1
    num_robots: int = -1
    sub_steps: int = -1
    noise_scale: float = -1.0
    barriers: int = -1
    controller: str = ""
    layout_overrides: dict = field(default_factory=dict)

    def validate(self) -> None:  # harness.hpp:60-67
        if self.batch < 1:
            raise InvalidArgument("run: batch must be >= 1")
        if self.episodes < 1:
            raise InvalidArgument("run: episodes must be >= 1")
        parse_policy(self.policy)
        if self.controller not in ("", "unicycle_position", "unicycle_pose"):
            raise InvalidArgument("run: controller must be unicycle_position or unicycle_pose")


def parse_policy(text: str) -> tuple[str, str, bool]:
    """PolicySpec::parse (policy.hpp:24-47) for the policies the device runs:
    returns (kind, path, greedy); to_string() is the canonical spelling."""
    if text == "random":
        return "random", "", True
    for prefix, greedy in (("feedforward:", True), ("feedforward_sample:", False)):
        if text.startswith(prefix):
            if not text[len(prefix):]:
                raise InvalidArgument("feedforward policy needs a weights file path")
            return "feedforward", text[len(prefix):], greedy
    if text in ("scripted_goal", "scripted"):
        return "scripted_goal", "", True
    if text == "prey_chaser":
        return "prey_chaser", "", True
    raise InvalidArgument(f"unknown policy '{text}'")


def resolve_scenario_config(run: RunConfig) -> ScenarioConfig:
    """harness.hpp:71-103."""
    run.validate()
    cfg = make_default_config(run.scenario)
    for key in sorted(run.layout_overrides):
        cfg.set_layout(key, list(run.layout_overrides[key]))
    if run.num_robots > 0 and run.num_robots != cfg.raw.num_robots:
        cfg.set_num_robots(run.num_robots)  # fixed rosters raise like the reference
    if run.max_steps > 0:
        cfg.max_steps = run.max_steps
    if run.sub_steps > 0:
        cfg.sub_steps = run.sub_steps
    if run.noise_scale >= 0:
        cfg.action_noise_scale = run.noise_scale
    if run.barriers >= 0:
        cfg.barrier_enabled = int(run.barriers != 0)
    if run.controller:
        cfg.set_controller(run.controller)
    cfg.validate()
    return cfg


def build_header(run: RunConfig, cfg: ScenarioConfig) -> TrajectoryHeader:
    """harness.hpp:105-129: layout keys that differ from the defaults, sorted (std::map order)."""
    h = TrajectoryHeader()
    h.set("scenario", cfg.scenario_name)
    h.set("seed", str(run.seed))
    h.set("episodes", str(run.episodes))
    h.set("batch", str(run.batch))
    h.set("num_robots", str(cfg.raw.num_robots))
    h.set("max_steps", str(cfg.raw.max_steps))
    h.set("sub_steps", str(cfg.raw.sub_steps))
    h.set("dt", format_double(cfg.raw.dt))
    h.set("controller", "unicycle_pose" if cfg.raw.controller == _abi.MRSIM_CONTROLLER_UNICYCLE_POSE
          else "unicycle_position")
    h.set("barriers", "1" if cfg.raw.barrier_enabled else "0")
    h.set("noise_scale", format_double(cfg.raw.action_noise_scale))
    kind, path, greedy = parse_policy(run.policy)
    h.set("policy", kind if kind in ("random", "scripted_goal", "prey_chaser")
          else ("feedforward:" if greedy else "feedforward_sample:") + path)
    defaults = make_default_config(run.scenario)
    for key in sorted(run.layout_overrides):
        vals = [float(v) for v in run.layout_overrides[key]]
        if vals == defaults.get_layout(key):
            continue
        h.set("layout." + key, " ".join(format_double(v) for v in vals))
    return h


def run_config_from_header(h: TrajectoryHeader) -> RunConfig:  # harness.hpp:131-148
    run = RunConfig(scenario=h.get("scenario"), seed=int(h.get("seed")), episodes=int(h.get("episodes")),
                    batch=int(h.get("batch")), num_robots=int(h.get("num_robots")),
                    max_steps=int(h.get("max_steps")), sub_steps=int(h.get("sub_steps")),
                    controller=h.get("controller"), barriers=1 if h.get("barriers") == "1" else 0,
                    noise_scale=float(h.get("noise_scale")), policy=h.get("policy"))
    for k, v in h.fields:
        if k.startswith("layout."):
            run.layout_overrides[k[7:]] = [float(x) for x in v.split()]
    return run


@dataclass
class EpisodeStats:  # harness.hpp:150-157
    total_reward: float = 0.0
    final_metric: float = 0.0
    collisions: int = 0
    success: bool = False
    min_pairwise_distance: float = math.inf
    qp_infeasible: int = 0


@dataclass
class RunSummary:  # harness.hpp:159-186
    scenario: str
    episodes: list
    rows: np.ndarray
    trajectory_path: str = ""


def run_episodes(run: RunConfig, out: str | None = None, device: int = 0, max_wave: int = 1 << 16) -> RunSummary:
    """harness.hpp:216-300 on the GPU: waves of min(batch, max_wave) envs, each
    stepped max_steps times with the run's policy on device, every step
    recorded on device. Row content depends only on (config, seed, episode)."""
    cfg = resolve_scenario_config(run)
    kind, path, greedy = parse_policy(run.policy)
    N, T = cfg.raw.num_robots, cfg.raw.max_steps
    wave_size = max(1, min(run.batch, max_wave))
    header = build_header(run, cfg)
    rows = []
    stats = []
    first_write = True
    for wave_start in range(0, run.episodes, wave_size):
        wave = min(wave_size, run.episodes - wave_start)
        gb = CudaEnvBatch(cfg, wave, device=device, fp64=True)
        if kind != "random":
            gb.set_policy(run.policy)
        gb.reset_episodes(root_seed=run.seed, first_episode=wave_start, episode_stride=wave)
        gb._check(lib().mrsim_capture_begin(gb._h, T))
        ret = np.zeros(wave)
        for _ in range(T):
            gb.step(None, want_obs=False)
        recs = np.empty((T, wave, N), dtype=RECORD_DTYPE)
        gb._check(lib().mrsim_capture_read(gb._h, 0, wave, recs.ctypes.data_as(ctypes.c_void_p)))
        if out is not None:
            rc = lib().mrsim_trajectory_write(out.encode(), header.block().encode(), recs.ctypes.data_as(ctypes.c_void_p),
                                              T, wave, N, wave_start, 0 if first_write else 1)
            raise_for(rc, f"cannot write '{out}'")
            first_write = False
        states = gb.get_states()
        ret = recs["reward"][:, :, 0].sum(axis=0)
        for e in range(wave):
            s = states[e]
            stats.append(EpisodeStats(total_reward=float(ret[e]), final_metric=s.scenario_metric,
                                      collisions=s.collisions, success=bool(s.success),
                                      min_pairwise_distance=s.min_pairwise_distance, qp_infeasible=s.qp_infeasible))
        rows.append(_rows_of(recs, wave_start))
        gb._check(lib().mrsim_capture_end(gb._h))
        gb.close()
    return RunSummary(cfg.scenario_name, stats, np.concatenate(rows), out or "")


def _rows_of(recs: np.ndarray, env_offset: int) -> np.ndarray:
    T, E, N = recs.shape
    r = np.empty((E, T, N), dtype=ROW_DTYPE)
    rt = recs.transpose(1, 0, 2)  # env-major like the reference's episode_rows
    r["env"] = (env_offset + np.arange(E))[:, None, None]
    r["step"] = np.arange(T)[None, :, None]
    r["robot"] = np.arange(N)[None, None, :]
    for f in ("x", "y", "theta", "action", "reward", "done", "collisions", "metric"):
        r[f] = rt[f]
    return r.reshape(-1)


@dataclass
class TrajectoryFile:
    header: TrajectoryHeader
    row_lines: list
    rows: np.ndarray


def read_trajectory(path: str) -> TrajectoryFile:
    """trajectory.hpp:136-180 (same errors, same hash check)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open '{path}'") from None
    with f:
        lines = f.read().decode().split("\n")
    it = iter(lines)
    line = next(it, None)
    if line is None or not line.startswith("# mrsim-trajectory"):
        raise InvalidArgument("trajectory: missing magic line")
    parts = line[2:].split()
    if len(parts) < 2 or parts[1] != str(FORMAT_VERSION):
        raise InvalidArgument("trajectory: unsupported format version")
    line = next(it, None)
    if line is None or not line.startswith("# config-hash "):
        raise InvalidArgument("trajectory: missing config-hash")
    stored = line[14:]
    header = TrajectoryHeader()
    for line in it:
        if line.startswith("# "):
            if " = " not in line:
                raise InvalidArgument("trajectory: malformed header line: " + line)
            k, v = line[2:].split(" = ", 1)
            header.set(k, v)
            continue
        if line == COLUMNS:
            break
        raise InvalidArgument("trajectory: unexpected line before columns: " + line)
    if stored != f"{header.hash():016x}":
        raise InvalidArgument("trajectory: config-hash mismatch (file corrupt or edited)")
    row_lines = [ln for ln in it if ln]
    rows = np.empty(len(row_lines), dtype=ROW_DTYPE)
    for k, ln in enumerate(row_lines):
        t = ln.split(",")
        if len(t) < 11:
            raise InvalidArgument("trajectory: short row")
        rows[k] = (int(t[0]), int(t[1]), int(t[2]), float(t[3]), float(t[4]), float(t[5]), int(t[6]),
                   float(t[7]), int(t[8]) != 0, int(t[9]), float(t[10]))
    return TrajectoryFile(header, row_lines, rows)


@dataclass
class VerifyReport:  # harness.hpp:446-450
    ok: bool = True
    message: str = "ok"
    first_divergent_row: int = -1


def verify_trajectory(path: str, pos_tol: float = 1e-7, ang_tol: float = 1e-6, real_tol: float = 1e-7,
                      device: int = 0) -> VerifyReport:
    """harness.hpp:444-518: replay the header configuration (on the GPU),
    compare row by row (tolerances in the module docstring), then re-check the
    collision counter and the safety invariant from the recorded poses."""
    rep = VerifyReport()
    try:
        file = read_trajectory(path)
    except Exception as e:  # noqa: BLE001 - report, like the reference
        return VerifyReport(False, str(e))
    run = run_config_from_header(file.header)
    try:
        replay = run_episodes(run, out=None, device=device)
    except Exception as e:  # noqa: BLE001
        return VerifyReport(False, f"replay failed: {e}")
    a, b = file.rows, replay.rows
    if len(a) != len(b):
        return VerifyReport(False, f"row count mismatch: file has {len(a)}, replay produced {len(b)}")
    exact = np.ones(len(a), dtype=bool)
    for f in ("env", "step", "robot", "action", "done", "collisions"):
        exact &= a[f] == b[f]
    dth = np.abs(np.remainder(a["theta"] - b["theta"] + np.pi, 2 * np.pi) - np.pi)
    close = (np.abs(a["x"] - b["x"]) <= pos_tol) & (np.abs(a["y"] - b["y"]) <= pos_tol) & (dth <= ang_tol)
    for f in ("reward", "metric"):
        close &= np.abs(a[f] - b[f]) <= real_tol * np.maximum(1.0, np.abs(b[f]))
    bad = np.flatnonzero(~(exact & close))
    if bad.size:
        i = int(bad[0])
        return VerifyReport(False, f"replay diverges at data row {i + 1}:\n  file:   {file.row_lines[i]}\n"
                                   f"  replay: {_csv(b[i])}", i + 1)
    # independent checks from the recorded poses (harness.hpp:488-516)
    n = int(file.header.get("num_robots"))
    barriers = file.header.get("barriers") == "1"
    cfg = resolve_scenario_config(run)
    if len(a) % n:
        return VerifyReport(False, "rows not ordered by (env, step, robot)")
    g = a.reshape(-1, n)
    if np.any(g["robot"] != np.arange(n)[None, :]):
        return VerifyReport(False, "rows not ordered by (env, step, robot)")
    if n > 1:
        dx = g["x"][:, :, None] - g["x"][:, None, :]
        dy = g["y"][:, :, None] - g["y"][:, None, :]
        d = np.hypot(dx, dy)
        d[:, np.arange(n), np.arange(n)] = np.inf
        mind = d.min(axis=(1, 2))
    else:
        mind = np.full(len(g), np.inf)
    env = g["env"][:, -1]
    coll = g["collisions"][:, -1]
    hit = (mind < cfg.raw.collision_radius).astype(np.int64)
    for e in np.unique(env):
        sel = env == e
        recount = np.cumsum(hit[sel])
        if np.any(coll[sel] < recount):
            k = int(np.flatnonzero(coll[sel] < recount)[0])
            return VerifyReport(False, f"collision counter at env {e} step {g['step'][sel][k, -1]} is below the "
                                       "pose-level recount")
    if barriers:
        viol = np.flatnonzero(mind < cfg.raw.safety_radius - 1e-3)
        if viol.size:
            k = int(viol[0])
            return VerifyReport(False, f"safety invariant violated at env {env[k]} step {g['step'][k, -1]}: "
                                       f"min pairwise distance {format_double(mind[k])}")
    return rep


def _csv(r) -> str:  # TrajectoryRow::to_csv
    return (f"{r['env']},{r['step']},{r['robot']},{format_double(r['x'])},{format_double(r['y'])},"
            f"{format_double(r['theta'])},{r['action']},{format_double(r['reward'])},{int(r['done'] != 0)},"
            f"{r['collisions']},{format_double(r['metric'])}")
