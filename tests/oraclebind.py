"""ctypes binding of oracle/_build/libmrsim_oracle.so — the plain-C fp64
restatement of the reference hot path (TEST INFRASTRUCTURE, checker only)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2505_06771_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "libmrsim_oracle.so")
P = ctypes.POINTER
_lib = None


def available() -> bool:
    return os.path.exists(ORACLE_LIB)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(ORACLE_LIB)
        d = P(ctypes.c_double)
        sig = {
            "orc_derive_episode_seed": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_int]),
            "orc_policy_action": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int]),
            "orc_rng_draws": (None, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                     d, P(ctypes.c_uint64)]),
            "orc_solve_qp": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, d, d, d, d, d, ctypes.c_double, ctypes.c_int,
                                            d, P(ctypes.c_int)]),
            "orc_apply_barrier": (ctypes.c_int, [P(_abi.Cfg), ctypes.c_int, d, d, ctypes.c_int, d,
                                                 P(ctypes.c_uint64), d, P(ctypes.c_int)]),
            "orc_obs_dim": (ctypes.c_int, [P(_abi.Cfg)]),
            "orc_reset_env": (ctypes.c_int, [P(_abi.Cfg), ctypes.c_uint64, P(_abi.EnvState), ctypes.c_char_p,
                                             ctypes.c_int]),
            "orc_step_env": (ctypes.c_int, [P(_abi.Cfg), P(_abi.EnvState), P(ctypes.c_int32), d, d, P(ctypes.c_int),
                                            ctypes.c_char_p, ctypes.c_int]),
            "orc_observe": (ctypes.c_int, [P(_abi.Cfg), P(_abi.EnvState), d]),
            "orc_policy_act": (ctypes.c_int, [P(_abi.Cfg), P(_abi.EnvState), ctypes.c_int, ctypes.c_int,
                                              P(ctypes.c_int32), P(ctypes.c_int32), d, ctypes.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def dptr(a):
    return a.ctypes.data_as(P(ctypes.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleEnv:
    """One environment stepped by the C restatement (reset_env / step_env)."""

    def __init__(self, cfg: _abi.Cfg):
        self.cfg = cfg
        self.N = cfg.num_robots
        self.D = lib().orc_obs_dim(ctypes.byref(cfg))
        self.state = _abi.EnvState()

    def reset(self, seed: int):
        err = ctypes.create_string_buffer(256)
        rc = lib().orc_reset_env(ctypes.byref(self.cfg), seed, ctypes.byref(self.state), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return self.observe()

    def observe(self):
        obs = np.zeros((self.N, self.D))
        lib().orc_observe(ctypes.byref(self.cfg), ctypes.byref(self.state), dptr(obs))
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.int32))
        obs = np.zeros((self.N, self.D))
        rew = ctypes.c_double()
        done = ctypes.c_int()
        err = ctypes.create_string_buffer(256)
        rc = lib().orc_step_env(ctypes.byref(self.cfg), ctypes.byref(self.state), a.ctypes.data_as(P(ctypes.c_int32)),
                                dptr(obs), ctypes.byref(rew), ctypes.byref(done), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return obs, rew.value, bool(done.value)


def policy_act(cfg: _abi.Cfg, state: _abi.EnvState, robot: int, weights, greedy: bool = True) -> int:
    dims, acts, flat = weights.packed()
    return lib().orc_policy_act(ctypes.byref(cfg), ctypes.byref(state), robot, len(acts),
                                dims.ctypes.data_as(P(ctypes.c_int32)), acts.ctypes.data_as(P(ctypes.c_int32)),
                                dptr(flat), int(bool(greedy)))


def solve_qp(A, b, lo, hi, u_nom, tol=1e-9, max_iter=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    u = np.zeros(n)
    it = ctypes.c_int()
    st = lib().orc_solve_qp(n, m, dptr(A), dptr(np.ascontiguousarray(b, dtype=np.float64)),
                            dptr(np.ascontiguousarray(lo, dtype=np.float64)),
                            dptr(np.ascontiguousarray(hi, dtype=np.float64)),
                            dptr(np.ascontiguousarray(u_nom, dtype=np.float64)), tol, max_iter, dptr(u),
                            ctypes.byref(it))
    return st, u, it.value


def apply_barrier(cfg: _abi.Cfg, poses, nominal, obstacles=None, masks=None):
    poses = np.ascontiguousarray(poses, dtype=np.float64)
    nominal = np.ascontiguousarray(nominal, dtype=np.float64)
    n = poses.shape[0]
    nob = 0 if obstacles is None else len(obstacles)
    ob = np.ascontiguousarray(obstacles if nob else np.zeros((1, 3)), dtype=np.float64)
    mk = np.ascontiguousarray(masks if masks is not None else np.zeros(max(nob, 1)), dtype=np.uint64)
    cmds = np.zeros((n, 2))
    inf = ctypes.c_int()
    rc = lib().orc_apply_barrier(ctypes.byref(cfg), n, dptr(poses), dptr(nominal), nob, dptr(ob),
                                 mk.ctypes.data_as(P(ctypes.c_uint64)), dptr(cmds), ctypes.byref(inf))
    if rc:
        raise OracleError(rc, "coincident robot positions")
    return cmds, bool(inf.value)
