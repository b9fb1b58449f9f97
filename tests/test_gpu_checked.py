"""Bounds-checked run (SURVEY.md §4/§5 race / memory checking; compute-sanitizer is closed on the GPU
pool - its runs left GPUs needing a reset - so the library checks itself): tools/checked_case.py under
librmx_checked.so (-DRMX_CHECKS: device-side traps on out-of-range workspace / output indices), with
guard bands around every output buffer and oracle parity. A trap shows up as a CUDA error and a
non-zero exit of the subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_workload():
    lib = os.path.join(ROOT, "paper_1403_5524_b200", "librmx_checked.so")
    if not os.path.exists(lib):
        from paper_1403_5524_b200 import build
        build.build_checked()
    env = dict(os.environ, RMX_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_case.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    assert "RMX_CHECK" not in log and "CHECKED_CASE_OK" in out.stdout, log[-3000:]


def test_checked_build_traps_out_of_range():
    """The checks are live: in librmx_checked.so an index one row past a 4 x 4 view traps (the kernel
    fails with a CUDA error), while an in-range index passes."""
    lib = os.path.join(ROOT, "paper_1403_5524_b200", "librmx_checked.so")
    code = ("import ctypes, sys; l = ctypes.CDLL(sys.argv[1]); "
            "print('RC', l.rmx_debug_checks_selftest(int(sys.argv[2])))")
    ok = subprocess.run([sys.executable, "-c", code, lib, "3"], capture_output=True, text=True, timeout=300)
    assert "RC 0" in ok.stdout, ok.stdout + ok.stderr
    bad = subprocess.run([sys.executable, "-c", code, lib, "4"], capture_output=True, text=True, timeout=300)
    assert "RMX_CHECK" in bad.stdout + bad.stderr and "RC 0" not in bad.stdout, bad.stdout + bad.stderr
