"""Negative control of the -DMRSIM_DEVICE_CHECKS build (scripts/device_checks.sh runs the whole GPU
suite against it as the compute-sanitizer substitute): a guard overwritten behind a state field or
an allocation is reported. Skipped with the shipped library, which has no debug exports."""
import ctypes

import pytest

import paper_2505_06771_b200 as m

pytestmark = pytest.mark.gpu


def _checks_lib():
    lib = m.lib()
    if not hasattr(lib, "mrsim_debug_check_guards"):
        pytest.skip("not a -DMRSIM_DEVICE_CHECKS build")
    lib.mrsim_debug_check_guards.argtypes = [ctypes.c_void_p]
    lib.mrsim_debug_poke_guard.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    return lib


@pytest.mark.parametrize("which", [0, 1])
def test_overwritten_guard_is_reported(which):
    lib = _checks_lib()
    cfg = m.make_default_config("navigation")
    gb = m.CudaEnvBatch(cfg, 300, auto_reset=True)
    gb.reset_episodes(3)
    for _ in range(5):
        gb.step(None)
    gb.sync()
    assert lib.mrsim_debug_check_guards(gb._h) == 0
    assert lib.mrsim_debug_poke_guard(gb._h, which, 0) == 0
    assert lib.mrsim_debug_check_guards(gb._h) == 3  # MRSIM_E_RUNTIME
    assert "guard overwritten" in lib.mrsim_last_error(gb._h).decode()
    assert lib.mrsim_debug_poke_guard(gb._h, which, 0xA5) == 0  # restore, or close() aborts the run
    assert lib.mrsim_debug_check_guards(gb._h) == 0
    gb.close()
