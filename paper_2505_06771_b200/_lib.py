"""Loader of the in-tree sm_100a library (libmrsim_cuda.so).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises. Build it with `make -j` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os

from . import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MRSIM_LIB_PATH") or os.path.join(_HERE, "libmrsim_cuda.so")  # override: A/B builds

_lib = None


class MrsimError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""

    code = -1


class InvalidArgument(MrsimError, ValueError):  # std::invalid_argument
    code = 1


class DomainError(MrsimError, ArithmeticError):  # std::domain_error
    code = 2


class SimRuntimeError(MrsimError):  # std::runtime_error (spawn failures)
    code = 3


class CudaError(MrsimError):
    code = 4


class Unsupported(MrsimError, NotImplementedError):
    code = 5


_BY_CODE = {c.code: c for c in (InvalidArgument, DomainError, SimRuntimeError, CudaError, Unsupported)}


def raise_for(code: int, message: str) -> None:
    if code == 0:
        return
    raise _BY_CODE.get(code, MrsimError)(message)


def lib() -> ctypes.CDLL:
    """The loaded library with every header-declared signature bound."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension (make -j) first")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _abi.FUNCTIONS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.mrsim_abi_version() != _abi.MRSIM_ABI_VERSION:
            raise ImportError("libmrsim_cuda.so ABI version does not match include/mrsim_cuda.h")
        for which, st in enumerate((_abi.Cfg, _abi.Layout, _abi.EnvState, _abi.Stats, _abi.TrajRecord)):
            if handle.mrsim_sizeof(which) != ctypes.sizeof(st):
                raise ImportError(f"ctypes mirror of {st.__name__} has the wrong size")
        _lib = handle
    return _lib
