"""Device bounds checks (compute-sanitizer is closed on the GPU pool).

`make CHECKS=1` builds libtac_b200_checks.so: every shared-memory and global
index of the stream blur, shade, epilogue splat and tiled shadow march is
checked (TAC_CHECK, csrc/tac_internal.cuh) and a violation traps the kernel.
tools/sanitize_case.py runs every kernel family (sigma 1,2,4 stream blur,
small and ragged frames, column strips with padded shade rows, shadows on the
tiled and L1 marches, the fp16 LUT, the z-buffer) under that library in a
fresh process; a trap surfaces as a CUDA error and a non-zero exit."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKS_LIB = os.path.join(ROOT, "paper_2411_04776_b200", "libtac_b200_checks.so")


@pytest.mark.gpu
def test_every_kernel_family_under_bounds_checks():
    if not os.path.exists(CHECKS_LIB):
        pytest.skip("libtac_b200_checks.so not built (make CHECKS=1)")
    env = dict(os.environ, TAC_B200_LIB=CHECKS_LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize case ok" in r.stdout


def test_checks_library_is_the_checked_build():
    """CPU: the checks build differs from the default one (the checks are
    compiled in) and exports the same C ABI."""
    if not os.path.exists(CHECKS_LIB):
        pytest.skip("libtac_b200_checks.so not built (make CHECKS=1)")
    import ctypes

    lib = ctypes.CDLL(CHECKS_LIB)
    for sym in ("tac_ctx_create", "tac_ctx_destroy", "tac_pipeline", "tac_last_error"):
        assert hasattr(lib, sym)
    default = os.path.join(ROOT, "paper_2411_04776_b200", "libtac_b200.so")
    if os.path.exists(default):
        assert open(default, "rb").read() != open(CHECKS_LIB, "rb").read()
