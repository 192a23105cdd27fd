"""Host-side mirror of the reference batch engine, on top of the C ABI.

Reference interface (paths relative to /root/reference/proj/include/mrsim):
  ScenarioConfig / make_default_config   framework.hpp:129-166, scenario.hpp:230-236
  reset_batch(cfg, seeds)                batch.hpp:240-259
  step_batch(state, actions, cfg)        batch.hpp:268-290
  derive_episode_seed / policy_stream    harness.hpp:25-34

`CudaEnvBatch` owns one device context (one per GPU) and keeps the batch
state in HBM; `reset_batch` / `step_batch` keep the reference's call shape
(host arrays in, host arrays out). Errors raise the same exception kinds as
the reference (InvalidArgument ~ std::invalid_argument, DomainError ~
std::domain_error, SimRuntimeError ~ std::runtime_error).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._lib import InvalidArgument, lib, raise_for

TASKS = ("navigation", "predator_prey", "discovery", "rware", "foraging", "material_transport",
         "arctic_transport", "warehouse", "random_waypoints")
COEF_NAMES = ("violation", "dist", "tag", "sense", "step", "dropoff", "forage", "load", "delivery")


class ScenarioConfig:
    """mrsim::ScenarioConfig (framework.hpp:129-166), flattened as mrsim_cfg."""

    def __init__(self, raw: _abi.Cfg):
        self.raw = raw

    @classmethod
    def default(cls, name: str) -> "ScenarioConfig":
        raw = _abi.Cfg()
        rc = lib().mrsim_config_default(name.encode(), ctypes.byref(raw))
        if rc != 0:
            raise InvalidArgument(f"unknown scenario '{name}' (available: {', '.join(sorted(TASKS))})")
        return cls(raw)

    def copy(self) -> "ScenarioConfig":
        raw = _abi.Cfg()
        ctypes.memmove(ctypes.byref(raw), ctypes.byref(self.raw), ctypes.sizeof(raw))
        return ScenarioConfig(raw)

    @property
    def scenario_name(self) -> str:
        return TASKS[self.raw.task]

    def __getattr__(self, item):
        raw = self.__dict__.get("raw")
        if raw is not None and item in {f for f, _ in _abi.Cfg._fields_}:
            return getattr(raw, item)
        raise AttributeError(item)

    def __setattr__(self, key, value):
        if key != "raw" and key in {f for f, _ in _abi.Cfg._fields_}:
            setattr(self.raw, key, value)
        else:
            object.__setattr__(self, key, value)

    CONTROLLERS = ("unicycle_position", "unicycle_pose")  # ControllerKind names (harness.hpp:95-96, 117)

    def set_controller(self, name: str) -> "ScenarioConfig":
        if name not in self.CONTROLLERS:
            raise InvalidArgument(f"unknown controller '{name}' (available: {', '.join(self.CONTROLLERS)})")
        self.raw.controller = self.CONTROLLERS.index(name)
        return self

    def coefficient(self, name: str) -> float:  # ScenarioConfig::coefficient (framework.hpp:145-151)
        k = COEF_NAMES.index(name)
        if not (self.raw.coef_present >> k) & 1:
            raise InvalidArgument(f"ScenarioConfig: missing reward coefficient '{name}' for scenario "
                                  f"{self.scenario_name}")
        return self.raw.coef[k]

    def set_num_robots(self, n: int, tile_roster: bool = False) -> "ScenarioConfig":
        rc = lib().mrsim_config_set_num_robots(ctypes.byref(self.raw), int(n), int(bool(tile_roster)))
        if rc == 1 and n >= 1:
            raise InvalidArgument(f"scenario '{self.scenario_name}' has a fixed robot roster; "
                                  "num_robots cannot change")
        raise_for(rc, f"num_robots={n} not supported")
        return self

    def set_layout(self, key: str, values) -> "ScenarioConfig":
        vals = (ctypes.c_double * len(values))(*values)
        rc = lib().mrsim_config_set_layout(ctypes.byref(self.raw), key.encode(), vals, len(values))
        raise_for(rc, f"layout: bad key or value count for '{key}'")
        return self

    def get_layout(self, key: str) -> list:
        buf = (ctypes.c_double * 64)()
        n = lib().mrsim_config_get_layout(ctypes.byref(self.raw), key.encode(), buf, 64)
        if n < 0:
            raise InvalidArgument(f"layout: unknown key '{key}'")
        return list(buf[:n])

    def validate(self) -> None:
        buf = ctypes.create_string_buffer(256)
        rc = lib().mrsim_config_validate(ctypes.byref(self.raw), buf, 256)
        raise_for(rc, buf.value.decode())

    @property
    def obs_dim(self) -> int:
        return lib().mrsim_obs_dim(ctypes.byref(self.raw))

    def task_fields(self) -> tuple[int, int]:
        nf, ni = ctypes.c_int(), ctypes.c_int()
        lib().mrsim_task_fields(ctypes.byref(self.raw), ctypes.byref(nf), ctypes.byref(ni))
        return nf.value, ni.value

    def heterogeneity(self) -> np.ndarray:
        return np.array([[self.raw.het[i][k] for k in range(self.raw.het_cols)]
                         for i in range(self.raw.het_rows)], dtype=np.float64)

    def step_sizes(self) -> np.ndarray:
        return np.array(self.raw.step_sizes[: self.raw.num_robots], dtype=np.float64)


def make_default_config(name: str) -> ScenarioConfig:
    """make_default_config (scenario.hpp:230-236)."""
    cfg = ScenarioConfig.default(name)
    cfg.validate()
    return cfg


@dataclass
class StepOutputs:
    obs: object        # torch.float32 [B, N, D] or None
    reward: object     # torch.float32 [B]
    done: object       # torch.uint8 [B]
    next_obs: object   # torch.float32 [B, N, D] or None (written where done, auto-reset only)


def _torch():
    import torch  # device buffers and streams only

    return torch


def _stream_handle(stream) -> ctypes.c_void_p:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class CudaEnvBatch:
    """B environments stepped in lockstep on one GPU (one mrsim_ctx)."""

    def __init__(self, cfg: ScenarioConfig, num_envs: int, device: int = 0, fp64: bool = True,
                 auto_reset: bool = False, env_per_thread: bool = False):
        cfg.validate()
        self.cfg = cfg.copy()
        self.num_envs = int(num_envs)
        self.device = int(device)
        self.fp64 = bool(fp64)
        self.auto_reset = bool(auto_reset)
        self.N = cfg.raw.num_robots
        self.D = cfg.obs_dim
        flags = (_abi.MRSIM_FLAG_FP64 if fp64 else 0) | (_abi.MRSIM_FLAG_AUTO_RESET if auto_reset else 0) | \
            (_abi.MRSIM_FLAG_ENV_PER_THREAD if env_per_thread else 0)
        handle = ctypes.c_void_p()
        rc = lib().mrsim_create(ctypes.byref(self.cfg.raw), self.device, self.num_envs, flags,
                                ctypes.byref(handle))
        raise_for(rc, "mrsim_create failed (see stderr)")
        self._h = handle
        torch = _torch()
        dev = torch.device("cuda", self.device)
        self._obs = torch.empty((self.num_envs, self.N, self.D), dtype=torch.float32, device=dev)
        self._next_obs = torch.empty_like(self._obs)
        self._reward = torch.empty((self.num_envs,), dtype=torch.float32, device=dev)
        self._done = torch.empty((self.num_envs,), dtype=torch.uint8, device=dev)
        self._actions = torch.empty((self.num_envs, self.N), dtype=torch.int8, device=dev)

    # -- plumbing --
    def _check(self, rc: int) -> None:
        if rc != 0:
            raise_for(rc, lib().mrsim_last_error(self._h).decode())

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().mrsim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reset (batch.hpp:240-259; harness.hpp:227-232) --
    def reset_seeds(self, seeds, stream=None):
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        if seeds.size != self.num_envs:
            raise InvalidArgument("reset_batch: seed list size != batch size")
        ptr = seeds.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        self._check(lib().mrsim_reset_seeds(self._h, ptr, ctypes.c_void_p(self._obs.data_ptr()),
                                            _stream_handle(stream)))
        return self._obs

    def reset_episodes(self, root_seed: int = 0, first_episode: int = 0, episode_stride: int | None = None,
                       stream=None):
        stride = self.num_envs if episode_stride is None else int(episode_stride)
        self._check(lib().mrsim_reset_episodes(self._h, int(root_seed), int(first_episode), stride,
                                               ctypes.c_void_p(self._obs.data_ptr()), _stream_handle(stream)))
        return self._obs

    # -- step (batch.hpp:268-290) --
    def step(self, actions=None, want_obs: bool = True, want_next_obs: bool = False, stream=None,
             obs_out=None, reward_out=None, done_out=None) -> StepOutputs:
        """Asynchronous device step. `actions`: int8 cuda tensor [B, N] or None (on-device random policy)."""
        a = ctypes.c_void_p(actions.data_ptr()) if actions is not None else None
        obs = obs_out if obs_out is not None else (self._obs if want_obs else None)
        rew = reward_out if reward_out is not None else self._reward
        done = done_out if done_out is not None else self._done
        nxt = self._next_obs if want_next_obs else None
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        self._check(lib().mrsim_step(self._h, a, ptr(obs), ptr(rew), ptr(done), ptr(nxt), _stream_handle(stream)))
        return StepOutputs(obs, rew, done, nxt)

    def rollout(self, num_steps: int, want_obs: bool = True, stream=None, out=None) -> StepOutputs:
        """num_steps fused steps with the on-device random policy in one launch (mrsim_rollout):
        step-major outputs obs [T, B, N, D], reward [T, B], done [T, B]; bit-identical to
        calling step(None) num_steps times."""
        torch = _torch()
        dev = torch.device("cuda", self.device)
        T = int(num_steps)
        if out is not None:
            obs, rew, done = out
        else:
            obs = torch.empty((T, self.num_envs, self.N, self.D), dtype=torch.float32, device=dev) if want_obs else None
            rew = torch.empty((T, self.num_envs), dtype=torch.float32, device=dev)
            done = torch.empty((T, self.num_envs), dtype=torch.uint8, device=dev)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        self._check(lib().mrsim_rollout(self._h, T, ptr(obs), ptr(rew), ptr(done), _stream_handle(stream)))
        return StepOutputs(obs, rew, done, None)

    def step_host(self, actions, out=None):
        """Synchronous step with host buffers (the reference's std::vector<int> actions).
        `out` = (obs float32 [B,N,D], reward float64 [B], done uint8 [B]) reuses caller
        buffers (pinned ones make the copies run at full link speed)."""
        a = actions
        if not (isinstance(a, np.ndarray) and a.dtype == np.int32 and a.flags.c_contiguous and
                a.size == self.num_envs * self.N):
            a = np.ascontiguousarray(np.asarray(actions, dtype=np.int32).reshape(self.num_envs, self.N))
        if out is None:
            obs = np.empty((self.num_envs, self.N, self.D), dtype=np.float32)
            rew = np.empty((self.num_envs,), dtype=np.float64)
            done = np.empty((self.num_envs,), dtype=np.uint8)
            ptrs = (obs.ctypes.data, rew.ctypes.data, done.ctypes.data)
        else:
            obs, rew, done = out
            key = (id(obs), id(rew), id(done))
            cached = getattr(self, "_out_ptrs", None)
            if cached is None or cached[0] != key:  # the caller's reused buffers: addresses looked up once
                self._out_ptrs = (key, (obs.ctypes.data, rew.ctypes.data, done.ctypes.data), out)
            ptrs = self._out_ptrs[1]
        self._check(lib().mrsim_step_host(self._h, a.ctypes.data, ptrs[0], ptrs[1], ptrs[2], None))
        return obs, rew, done

    def observe(self):
        """assemble_observations of the current state (host float32 [B, N, D])."""
        obs = np.empty((self.num_envs, self.N, self.D), dtype=np.float32)
        self._check(lib().mrsim_observe_host(self._h, obs.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return obs

    def random_actions(self, stream=None):
        self._check(lib().mrsim_random_actions(self._h, ctypes.c_void_p(self._actions.data_ptr()),
                                               _stream_handle(stream)))
        return self._actions

    # -- on-device policy (Policy, policy.hpp:432-486) --
    def set_policy(self, spec):
        """PolicySpec forms (policy.hpp:24-47): "random", "scripted_goal" (or "scripted"),
        "prey_chaser", "feedforward:<path>", "feedforward_sample:<path>", or a
        FeedforwardWeights (greedy)."""
        if isinstance(spec, FeedforwardWeights):
            return self.set_feedforward(spec, greedy=True)
        if spec == "random":
            self._check(lib().mrsim_set_policy_random(self._h))
            return self
        if spec in ("scripted_goal", "scripted"):
            self._check(lib().mrsim_set_policy_scripted(self._h, _abi.MRSIM_POLICY_SCRIPTED_GOAL))
            return self
        if spec == "prey_chaser":
            self._check(lib().mrsim_set_policy_scripted(self._h, _abi.MRSIM_POLICY_PREY_CHASER))
            return self
        for prefix, greedy in (("feedforward:", True), ("feedforward_sample:", False)):
            if spec.startswith(prefix):
                path = spec[len(prefix):]
                if not path:
                    raise InvalidArgument("feedforward policy needs a weights file path")
                return self.set_feedforward(FeedforwardWeights.load(path), greedy=greedy)
        raise InvalidArgument(f"unknown policy '{spec}'")

    def set_feedforward(self, weights: "FeedforwardWeights", greedy: bool = True):
        dims, acts, flat = weights.packed()
        self._check(lib().mrsim_set_policy_feedforward(
            self._h, len(acts), dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            acts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            int(bool(greedy))))
        return self

    def policy_actions(self, stream=None):
        """The context policy's actions for the current state (int8 cuda tensor [B, N])."""
        self._check(lib().mrsim_policy_actions(self._h, ctypes.c_void_p(self._actions.data_ptr()),
                                               _stream_handle(stream)))
        return self._actions

    def sync(self, stream=None) -> None:
        self._check(lib().mrsim_sync(self._h, _stream_handle(stream)))

    # -- state I/O (parity / checkpoint) --
    def get_states(self, first: int = 0, count: int | None = None):
        count = self.num_envs - first if count is None else int(count)
        arr = (_abi.EnvState * count)()
        self._check(lib().mrsim_get_env_states(self._h, int(first), count, arr))
        return arr

    def set_states(self, states, first: int = 0) -> None:
        arr = (_abi.EnvState * len(states))(*states)
        self._check(lib().mrsim_set_env_states(self._h, int(first), len(states), arr))

    def stats(self) -> dict:
        s = _abi.Stats()
        self._check(lib().mrsim_get_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _abi.Stats._fields_}


class FeedforwardWeights:
    """FeedforwardWeights (policy.hpp:69-195): dense layers (in, out, activation,
    W out x in row-major, b). Text I/O follows the reference's self-describing
    format (from_text / to_text, policy.hpp:134-195) so weight files written for
    the reference load here unchanged."""

    ACTIVATIONS = ("relu", "tanh", "identity")  # Activation order (policy.hpp:60)

    def __init__(self, layers):
        self.layers = [(int(i), int(o), str(a), np.asarray(w, dtype=np.float64).reshape(int(o), int(i)),
                        np.asarray(b, dtype=np.float64).reshape(int(o))) for i, o, a, w, b in layers]
        self.validate()

    def validate(self) -> None:  # policy.hpp:77-93
        if not self.layers:
            raise InvalidArgument("weights: no layers")
        for k, (i, o, a, w, b) in enumerate(self.layers):
            if i <= 0 or o <= 0:
                raise InvalidArgument("weights: bad layer dimensions")
            if a not in self.ACTIVATIONS:
                raise InvalidArgument(f"weights: unknown activation '{a}'")
            if k > 0 and self.layers[k - 1][1] != i:
                raise InvalidArgument("weights: layer dimensions do not chain")
        if self.layers[-1][1] != 5:
            raise InvalidArgument("weights: final layer must emit 5 logits")

    @property
    def input_dim(self) -> int:
        return self.layers[0][0]

    def packed(self):
        dims = np.array([d for i, o, *_ in self.layers for d in (i, o)], dtype=np.int32)
        acts = np.array([self.ACTIVATIONS.index(a) for _, _, a, _, _ in self.layers], dtype=np.int32)
        flat = np.concatenate([np.concatenate([w.ravel(), b]) for *_, w, b in self.layers]).astype(np.float64)
        return dims, acts, np.ascontiguousarray(flat)

    @classmethod
    def from_text(cls, text: str) -> "FeedforwardWeights":
        tok = text.split()
        pos = 0

        def take():
            nonlocal pos
            if pos >= len(tok):
                raise InvalidArgument("weights: truncated file")
            pos += 1
            return tok[pos - 1]

        if take() != "mrsim-weights":
            raise InvalidArgument("weights: missing 'mrsim-weights' magic")
        if take() != "1":
            raise InvalidArgument("weights: unsupported format version")
        if take() != "layers":
            raise InvalidArgument("weights: bad layer count")
        n = int(take())
        layers = []
        for _ in range(n):
            if take() != "layer":
                raise InvalidArgument("weights: bad layer header")
            take()  # index
            i, o, a = int(take()), int(take()), take()
            w = [float(take()) for _ in range(i * o)]
            b = [float(take()) for _ in range(o)]
            layers.append((i, o, a, w, b))
        return cls(layers)

    @classmethod
    def load(cls, path: str) -> "FeedforwardWeights":
        try:
            with open(path) as f:
                return cls.from_text(f.read())
        except OSError:
            raise RuntimeError(f"weights: cannot open '{path}'") from None

    def to_text(self) -> str:
        out = ["mrsim-weights 1", f"layers {len(self.layers)}"]
        for k, (i, o, a, w, b) in enumerate(self.layers):
            out.append(f"layer {k} {i} {o} {a}")
            out += [" ".join(f"{v:.17g}" for v in row) for row in w]
            out.append(" ".join(f"{v:.17g}" for v in b))
        return "\n".join(out) + "\n"

    @classmethod
    def random(cls, dims, activations, seed: int = 0, scale: float = 1.0) -> "FeedforwardWeights":
        rng = np.random.default_rng(seed)
        layers = []
        for (i, o), a in zip(zip(dims[:-1], dims[1:]), activations):
            layers.append((i, o, a, rng.normal(0, scale / np.sqrt(i), (o, i)), rng.normal(0, 0.1, o)))
        return cls(layers)


def reset_batch(cfg: ScenarioConfig, seeds, device: int = 0, fp64: bool = True):
    """reset_batch (batch.hpp:240-259): returns (batch, obs [B, N, D] host float32)."""
    seeds = list(seeds)
    if not seeds:
        raise InvalidArgument("reset_batch: seed list is empty")
    b = CudaEnvBatch(cfg, len(seeds), device=device, fp64=fp64)
    obs = b.reset_seeds(seeds)
    return b, obs.cpu().numpy()


def step_batch(batch: CudaEnvBatch, actions):
    """step_batch (batch.hpp:268-290) with host buffers; transactional on error."""
    return batch.step_host(actions)


# ---- harness seeds / random policy (harness.hpp:25-34, rng.hpp) in integer arithmetic ----
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def fork(key: int, tag: int) -> int:
    return mix64(key ^ mix64((tag * _GAMMA + 0x632BE59BD9B4E019) & _M64))


def derive_episode_seed(root: int, episode: int) -> int:
    return fork(fork(mix64(root + _GAMMA), 0xE915E915E915E915), episode & _M64)
