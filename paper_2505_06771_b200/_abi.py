"""ctypes mirror of include/mrsim_cuda.h, generated from the header itself.

The C structs (mrsim_layout, mrsim_cfg, mrsim_env_state, mrsim_stats) are
parsed out of the header at import time so the Python mirror cannot drift
from the ABI; `check_sizes()` cross-checks against the library's own
sizeof().
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mrsim_cuda.h")

_CTYPES = {
    "double": ctypes.c_double,
    "float": ctypes.c_float,
    "int32_t": ctypes.c_int32,
    "uint32_t": ctypes.c_uint32,
    "int64_t": ctypes.c_int64,
    "uint64_t": ctypes.c_uint64,
    "int8_t": ctypes.c_int8,
    "uint8_t": ctypes.c_uint8,
}


def _strip_comments(text: str) -> str:
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.sub(r"//[^\n]*", "", text)


def _parse(text: str):
    defines = {}
    for m in re.finditer(r"#define\s+(MRSIM_\w+)\s+([^\n]+)", _strip_comments(text)):
        val = m.group(2).strip()
        if re.fullmatch(r"[0-9xXa-fA-F]+u?", val):
            defines[m.group(1)] = int(val.rstrip("u"), 0)
    body = _strip_comments(text)

    def evaluate(expr: str) -> int:
        for k, v in sorted(defines.items(), key=lambda kv: -len(kv[0])):
            expr = expr.replace(k, str(v))
        return int(eval(expr, {"__builtins__": {}}, {}))  # arithmetic only (e.g. 2 * 16)

    structs = {}
    for m in re.finditer(r"typedef\s+struct\s+(\w+)\s*\{(.*?)\}\s*(\w+)\s*;", body, flags=re.S):
        name = m.group(3)
        fields = []
        for decl in m.group(2).split(";"):
            decl = " ".join(decl.split())
            if not decl:
                continue
            typ, rest = decl.split(" ", 1)
            base = _CTYPES.get(typ) or structs.get(typ)
            if base is None:
                raise TypeError(f"unknown field type {typ} in {name}")
            for item in rest.split(","):
                item = item.strip()
                dims = [evaluate(d) for d in re.findall(r"\[([^\]]+)\]", item)]
                fname = item.split("[")[0].strip()
                t = base
                for d in reversed(dims):
                    t = t * d
                fields.append((fname, t))
        structs[name] = type(name, (ctypes.Structure,), {"_fields_": fields})
    return defines, structs


with open(HEADER) as _f:
    DEFINES, STRUCTS = _parse(_f.read())

Layout = STRUCTS["mrsim_layout"]
Cfg = STRUCTS["mrsim_cfg"]
EnvState = STRUCTS["mrsim_env_state"]
Stats = STRUCTS["mrsim_stats"]
TrajRecord = STRUCTS["mrsim_traj_record"]
globals().update(DEFINES)

# Every function the header declares (name -> (restype, argtypes)).
P = ctypes.POINTER
c_void_p = ctypes.c_void_p
FUNCTIONS = {
    "mrsim_abi_version": (ctypes.c_int, []),
    "mrsim_sizeof": (ctypes.c_int, [ctypes.c_int]),
    "mrsim_config_default": (ctypes.c_int, [ctypes.c_char_p, P(Cfg)]),
    "mrsim_config_set_num_robots": (ctypes.c_int, [P(Cfg), ctypes.c_int, ctypes.c_int]),
    "mrsim_config_set_layout": (ctypes.c_int, [P(Cfg), ctypes.c_char_p, P(ctypes.c_double), ctypes.c_int]),
    "mrsim_config_get_layout": (ctypes.c_int, [P(Cfg), ctypes.c_char_p, P(ctypes.c_double), ctypes.c_int]),
    "mrsim_config_validate": (ctypes.c_int, [P(Cfg), ctypes.c_char_p, ctypes.c_int]),
    "mrsim_obs_dim": (ctypes.c_int, [P(Cfg)]),
    "mrsim_task_name": (ctypes.c_char_p, [ctypes.c_int]),
    "mrsim_task_fields": (ctypes.c_int, [P(Cfg), P(ctypes.c_int), P(ctypes.c_int)]),
    "mrsim_create": (ctypes.c_int, [P(Cfg), ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, P(c_void_p)]),
    "mrsim_destroy": (None, [c_void_p]),
    "mrsim_last_error": (ctypes.c_char_p, [c_void_p]),
    "mrsim_num_envs": (ctypes.c_int64, [c_void_p]),
    "mrsim_reset_seeds": (ctypes.c_int, [c_void_p, P(ctypes.c_uint64), c_void_p, c_void_p]),
    "mrsim_reset_episodes": (ctypes.c_int, [c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                            c_void_p, c_void_p]),
    "mrsim_step": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mrsim_rollout": (ctypes.c_int, [c_void_p, ctypes.c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    # raw addresses (the host path is the e2e hot call: no per-call ctypes pointer objects)
    "mrsim_step_host": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mrsim_observe": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
    "mrsim_observe_host": (ctypes.c_int, [c_void_p, P(ctypes.c_float)]),
    "mrsim_random_actions": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
    "mrsim_set_policy_feedforward": (ctypes.c_int, [c_void_p, ctypes.c_int, P(ctypes.c_int32), P(ctypes.c_int32),
                                                    P(ctypes.c_double), ctypes.c_int]),
    "mrsim_set_policy_random": (ctypes.c_int, [c_void_p]),
    "mrsim_set_policy_scripted": (ctypes.c_int, [c_void_p, ctypes.c_int]),
    "mrsim_policy_actions": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
    "mrsim_sync": (ctypes.c_int, [c_void_p, c_void_p]),
    "mrsim_capture_begin": (ctypes.c_int, [c_void_p, ctypes.c_int64]),
    "mrsim_capture_steps": (ctypes.c_int64, [c_void_p]),
    "mrsim_capture_read": (ctypes.c_int, [c_void_p, ctypes.c_int64, ctypes.c_int64, c_void_p]),
    "mrsim_capture_end": (ctypes.c_int, [c_void_p]),
    "mrsim_trajectory_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, c_void_p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int]),
    "mrsim_get_env_states": (ctypes.c_int, [c_void_p, ctypes.c_int64, ctypes.c_int64, P(EnvState)]),
    "mrsim_set_env_states": (ctypes.c_int, [c_void_p, ctypes.c_int64, ctypes.c_int64, P(EnvState)]),
    "mrsim_get_stats": (ctypes.c_int, [c_void_p, P(Stats)]),
    "mrsim_qp_solve_batch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double),
                                            P(ctypes.c_double), P(ctypes.c_double), ctypes.c_double,
                                            P(ctypes.c_double), P(ctypes.c_int32), P(ctypes.c_int32)]),
    "mrsim_probe_fma_peak": (ctypes.c_double, [ctypes.c_int, ctypes.c_int]),
    "mrsim_apply_barrier_batch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, P(Cfg), ctypes.c_int,
                                                 P(ctypes.c_double), P(ctypes.c_double), ctypes.c_int,
                                                 P(ctypes.c_double), P(ctypes.c_uint64), P(ctypes.c_double),
                                                 P(ctypes.c_int32)]),
}


def declared_functions() -> list[str]:
    """Function names declared in include/mrsim_cuda.h (for the export test)."""
    body = _strip_comments(open(HEADER).read())
    return sorted(set(re.findall(r"\b(mrsim_\w+)\s*\(", body)) - {"mrsim_ctx"})
