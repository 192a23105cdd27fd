"""Shared helpers for the parity tests."""
import ctypes

import numpy as np


def struct_dict(s, prefix=""):
    """Flatten a ctypes struct into {path: python value} for field-by-field diffs."""
    out = {}
    for name, typ in s._fields_:
        v = getattr(s, name)
        key = prefix + name
        if isinstance(v, ctypes.Structure):
            out.update(struct_dict(v, key + "."))
        elif isinstance(v, ctypes.Array):
            out[key] = np.array(np.ctypeslib.as_array(v)).tolist()
        else:
            out[key] = v
    return out


def diff_structs(a, b):
    da, db = struct_dict(a), struct_dict(b)
    return {k: (da[k], db[k]) for k in da if not k.startswith("_") and da[k] != db[k]}


def wrap_diff(a, b):
    d = np.asarray(a) - np.asarray(b)
    return np.abs(np.remainder(d + np.pi, 2 * np.pi) - np.pi)
