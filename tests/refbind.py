"""ctypes binding of oracle/_ref/libmrsim_ref.so — the UNMODIFIED reference
(/root/reference/proj/include, compiled by oracle/Makefile). TEST
INFRASTRUCTURE: used only as the checker by tests/, smoke() and bench.py's
cpu_baseline / --impl reference legs.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2505_06771_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libmrsim_ref.so")

P = ctypes.POINTER


class RefSpec(ctypes.Structure):
    _fields_ = [("scenario", ctypes.c_char_p), ("num_robots", ctypes.c_int32), ("tile_roster", ctypes.c_int32),
                ("max_steps", ctypes.c_int32), ("sub_steps", ctypes.c_int32), ("barrier", ctypes.c_int32),
                ("controller", ctypes.c_int32), ("noise", ctypes.c_double), ("layout", ctypes.c_char_p)]


_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_LIB)
        sig = {
            "ref_resolve_config": (ctypes.c_int, [P(RefSpec), P(_abi.Cfg), ctypes.c_char_p, ctypes.c_int]),
            "ref_create": (ctypes.c_void_p, [P(RefSpec), ctypes.c_int, ctypes.c_char_p, ctypes.c_int]),
            "ref_destroy": (None, [ctypes.c_void_p]),
            "ref_flatten": (ctypes.c_int, [ctypes.c_void_p, P(_abi.Cfg)]),
            "ref_num_robots": (ctypes.c_int, [ctypes.c_void_p]),
            "ref_obs_dim": (ctypes.c_int, [ctypes.c_void_p]),
            "ref_pool_size": (ctypes.c_int, [ctypes.c_void_p]),
            "ref_reset": (ctypes.c_int, [ctypes.c_void_p, P(ctypes.c_uint64), ctypes.c_int, P(ctypes.c_double),
                                         ctypes.c_char_p, ctypes.c_int]),
            "ref_step": (ctypes.c_int, [ctypes.c_void_p, P(ctypes.c_int32), P(ctypes.c_double), P(ctypes.c_double),
                                        P(ctypes.c_uint8), P(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]),
            "ref_batch_size": (ctypes.c_int, [ctypes.c_void_p]),
            "ref_get_states": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, P(_abi.EnvState)]),
            "ref_set_states": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, P(_abi.EnvState), ctypes.c_char_p,
                                              ctypes.c_int]),
            "ref_observe": (ctypes.c_int, [ctypes.c_void_p, P(ctypes.c_double)]),
            "ref_random_actions": (ctypes.c_int, [ctypes.c_void_p, P(ctypes.c_int32)]),
            "ref_run_episodes_file": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                                     ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p,
                                                     ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                                     ctypes.c_int]),
            "ref_verify_trajectory": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                                     P(ctypes.c_longlong)]),
            "ref_read_trajectory": (ctypes.c_long, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]),
            "ref_policy_actions": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, P(ctypes.c_int32),
                                                  ctypes.c_char_p, ctypes.c_int]),
            "ref_time_steps": (ctypes.c_double, [ctypes.c_void_p, ctypes.c_int]),
            "ref_derive_episode_seed": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_int]),
            "ref_policy_action": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int]),
            "ref_rng_draws": (None, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                     P(ctypes.c_double), P(ctypes.c_uint64)]),
            "ref_solve_qp": (ctypes.c_int, [ctypes.c_int, ctypes.c_int] + [P(ctypes.c_double)] * 5 +
                             [ctypes.c_double, ctypes.c_int, P(ctypes.c_double), P(ctypes.c_int), P(ctypes.c_double)]),
            "ref_qp_enumeration": (ctypes.c_int, [ctypes.c_int, ctypes.c_int] + [P(ctypes.c_double)] * 3 +
                                   [P(ctypes.c_double), P(ctypes.c_double)]),
            "ref_random_qps": (None, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_int),
                                      P(ctypes.c_int), P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double)]),
            "ref_apply_barrier": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, P(ctypes.c_double),
                                                 P(ctypes.c_double), ctypes.c_int, P(ctypes.c_double),
                                                 P(ctypes.c_uint64), P(ctypes.c_double), P(ctypes.c_int),
                                                 P(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]),
            "ref_run_episodes": (ctypes.c_long, [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_double),
                                                 ctypes.c_long, ctypes.c_char_p, ctypes.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def dptr(a: np.ndarray):
    return a.ctypes.data_as(P(ctypes.c_double))


def spec(scenario: str, num_robots: int = 0, tile_roster: bool = False, max_steps: int = 0, sub_steps: int = 0,
         barrier: int = -1, noise: float = -1.0, layout: dict | None = None, controller: int = -1) -> RefSpec:
    text = ";".join(f"{k} " + " ".join(repr(float(v)) for v in vals) for k, vals in (layout or {}).items())
    s = RefSpec(scenario.encode(), num_robots, int(tile_roster), max_steps, sub_steps, barrier, controller, noise,
                text.encode())
    s._keep = text  # noqa: keep the buffer alive
    return s


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def resolve_config(sp: RefSpec) -> _abi.Cfg:
    out = _abi.Cfg()
    err = ctypes.create_string_buffer(512)
    rc = lib().ref_resolve_config(ctypes.byref(sp), ctypes.byref(out), err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return out


class RefBatch:
    """The reference BatchWorldState + step_batch, driven through the shim."""

    def __init__(self, sp: RefSpec, workers: int = 1):
        err = ctypes.create_string_buffer(512)
        self.h = lib().ref_create(ctypes.byref(sp), workers, err, 512)
        if not self.h:
            raise RefError(1, err.value.decode())
        self.N = lib().ref_num_robots(self.h)
        self.D = lib().ref_obs_dim(self.h)
        self.B = 0

    def close(self):
        if self.h:
            lib().ref_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def cfg(self) -> _abi.Cfg:
        out = _abi.Cfg()
        lib().ref_flatten(self.h, ctypes.byref(out))
        return out

    def reset(self, seeds):
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        self.B = seeds.size
        obs = np.zeros((self.B, self.N, self.D))
        err = ctypes.create_string_buffer(512)
        rc = lib().ref_reset(self.h, seeds.ctypes.data_as(P(ctypes.c_uint64)), self.B, dptr(obs), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.int32).reshape(self.B, self.N))
        obs = np.zeros((self.B, self.N, self.D))
        rew = np.zeros(self.B)
        done = np.zeros(self.B, dtype=np.uint8)
        met = np.zeros((self.B, 6))
        err = ctypes.create_string_buffer(512)
        rc = lib().ref_step(self.h, a.ctypes.data_as(P(ctypes.c_int32)), dptr(obs), dptr(rew),
                            done.ctypes.data_as(P(ctypes.c_uint8)), dptr(met), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return obs, rew, done, met

    def get_states(self, first: int = 0, count: int | None = None):
        count = self.B - first if count is None else count
        arr = (_abi.EnvState * count)()
        lib().ref_get_states(self.h, first, count, arr)
        return arr

    def set_states(self, states):
        arr = (_abi.EnvState * len(states))(*states)
        err = ctypes.create_string_buffer(512)
        rc = lib().ref_set_states(self.h, len(states), arr, err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        self.B = len(states)

    def observe(self):
        obs = np.zeros((self.B, self.N, self.D))
        lib().ref_observe(self.h, dptr(obs))
        return obs

    def random_actions(self):
        out = np.zeros((self.B, self.N), dtype=np.int32)
        lib().ref_random_actions(self.h, out.ctypes.data_as(P(ctypes.c_int32)))
        return out

    def policy_actions(self, spec: str):
        out = np.zeros((self.B, self.N), dtype=np.int32)
        err = ctypes.create_string_buffer(512)
        rc = lib().ref_policy_actions(self.h, spec.encode(), out.ctypes.data_as(P(ctypes.c_int32)), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return out

    def time_steps(self, steps: int) -> float:
        return lib().ref_time_steps(self.h, steps)


def apply_barrier(batch: RefBatch, poses, nominal, obstacles=None, masks=None):
    poses = np.ascontiguousarray(poses, dtype=np.float64)
    nominal = np.ascontiguousarray(nominal, dtype=np.float64)
    n = poses.shape[0]
    nob = 0 if obstacles is None else len(obstacles)
    ob = np.ascontiguousarray(obstacles if nob else np.zeros((1, 3)), dtype=np.float64)
    mk = np.ascontiguousarray(masks if masks is not None else np.zeros(max(nob, 1)), dtype=np.uint64)
    cmds = np.zeros((n, 2))
    inf = ctypes.c_int()
    kkt = ctypes.c_double()
    err = ctypes.create_string_buffer(512)
    rc = lib().ref_apply_barrier(batch.h, n, dptr(poses), dptr(nominal), nob, dptr(ob),
                                 mk.ctypes.data_as(P(ctypes.c_uint64)), dptr(cmds), ctypes.byref(inf),
                                 ctypes.byref(kkt), err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return cmds, bool(inf.value), kkt.value


def random_qps(seed: int, count: int, max_n: int = 8, max_m: int = 12):
    n = np.zeros(count, dtype=np.int32)
    m = np.zeros(count, dtype=np.int32)
    A = np.zeros((count, max_m, max_n))
    b = np.zeros((count, max_m))
    u = np.zeros((count, max_n))
    lib().ref_random_qps(seed, count, max_n, max_m, n.ctypes.data_as(P(ctypes.c_int)),
                         m.ctypes.data_as(P(ctypes.c_int)), dptr(A), dptr(b), dptr(u))
    return n, m, A, b, u


def solve_qp(A, b, lo, hi, u_nom, tol=1e-9, max_iter=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    u = np.zeros(n)
    it = ctypes.c_int()
    kkt = ctypes.c_double()
    st = lib().ref_solve_qp(n, m, dptr(A), dptr(np.ascontiguousarray(b, dtype=np.float64)),
                            dptr(np.ascontiguousarray(lo, dtype=np.float64)),
                            dptr(np.ascontiguousarray(hi, dtype=np.float64)),
                            dptr(np.ascontiguousarray(u_nom, dtype=np.float64)), tol, max_iter, dptr(u),
                            ctypes.byref(it), ctypes.byref(kkt))
    return st, u, it.value, kkt.value


def qp_enumeration(A, b, u_nom):
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    u = np.zeros(n)
    obj = ctypes.c_double()
    ok = lib().ref_qp_enumeration(n, m, dptr(A), dptr(np.ascontiguousarray(b, dtype=np.float64)),
                                  dptr(np.ascontiguousarray(u_nom, dtype=np.float64)), dptr(u), ctypes.byref(obj))
    return (u, obj.value) if ok else None


def run_episodes(scenario: str, seed: int, episodes: int, batch: int, max_steps: int, num_robots: int = -1,
                 workers: int = 1) -> np.ndarray:
    max_rows = episodes * max_steps * 16
    rows = np.zeros((max_rows, 11))
    err = ctypes.create_string_buffer(512)
    k = lib().ref_run_episodes(scenario.encode(), seed, episodes, batch, workers, num_robots, max_steps,
                               dptr(rows), max_rows, err, 512)
    if k < 0:
        raise RefError(-k, err.value.decode())
    return rows[:k]


def run_episodes_file(path: str, scenario: str, seed: int, episodes: int, batch: int, num_robots: int = -1,
                      max_steps: int = -1, policy: str = "random", controller: str = "",
                      layout: dict | None = None) -> None:
    text = ";".join(f"{k} " + " ".join(repr(float(v)) for v in vals) for k, vals in (layout or {}).items())
    err = ctypes.create_string_buffer(512)
    rc = lib().ref_run_episodes_file(scenario.encode(), seed, episodes, batch, num_robots, max_steps,
                                     policy.encode(), controller.encode(), text.encode(), path.encode(), err, 512)
    if rc:
        raise RefError(rc, err.value.decode())


def verify_trajectory(path: str):
    msg = ctypes.create_string_buffer(2048)
    row = ctypes.c_longlong()
    ok = lib().ref_verify_trajectory(path.encode(), msg, 2048, ctypes.byref(row))
    return bool(ok), msg.value.decode(), row.value


def read_trajectory_rows(path: str) -> int:
    err = ctypes.create_string_buffer(512)
    k = lib().ref_read_trajectory(path.encode(), err, 512)
    if k < 0:
        raise RefError(-k, err.value.decode())
    return k
