"""CPU-side checks of the C-ABI boundary (no GPU compute): librmx.so builds for sm_100a, loads,
exports every function include/rmx.h declares, and carries sm_100a SASS with the FP64 tensor-core
(DMMA) and TMA instructions the design relies on."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rmx.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1403_5524_b200 import build
    build.build()
    import paper_1403_5524_b200 as rmx
    return rmx.load_library()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rmx_[a-zA-Z0-9_]+)\s*\(", src)))


def test_header_declares_expected_api():
    import paper_1403_5524_b200 as rmx
    names = header_functions()
    assert set(names) == set(rmx.EXPORTED), names
    for n in ("rmx_build_R", "rmx_match_K", "rmx_collision_strength"):  # BASELINE.json:5
        assert n in names


def test_library_exports_every_header_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_version_and_target(lib):
    assert lib.rmx_version() >= 100
    assert lib.rmx_sm_target() == 100


def test_null_ctx_is_einval(lib):
    import ctypes
    assert lib.rmx_destroy(None) == 1
    assert lib.rmx_build_R(None, None, 0, None, 0, 0, 1.0, None, 0, None, None) == 1
    assert lib.rmx_last_error(None) == b"null ctx"
    # every other entry point rejects a null context synchronously, before touching CUDA
    assert lib.rmx_match_K(None, None, None, None, None, None, 1.0, 1, 1, None, None, None) == 1
    assert lib.rmx_collision_strength(None, None, 1, 1, None, None, None, None) == 1
    assert lib.rmx_collision_strength_levels(None, None, 1, 1, None, None, 1, 1.0, None, None) == 1
    assert lib.rmx_sweep_levels(None, None, 2, None, 1, 1, 1.0, None, 1, None, None, None, None, None, 0,
                                None, 1, 1.0, None, None, None) == 1
    assert lib.rmx_dipole_amplitude(None, None, 2, None, None, 1, 1, None, 1, None, None) == 1
    assert lib.rmx_photoionization(None, None, None, None, None, None, 1, 1, None, 0.0, 1.0, None, None,
                                   None) == 1
    assert lib.rmx_sweep_photo(None, None, 2, None, None, 1, 1, 1.0, None, 1, None, None, None, None,
                               None, 0, 0.0, 1.0, None, None, None) == 1
    assert lib.rmx_inner_region(None, None, 1, None, 1, None, None, 1) == 1
    assert lib.rmx_convolve_gaussian(None, None, 1, None, 1, 1.0, 3.0, None) == 1
    assert lib.rmx_maxwell_average(None, None, 1, 1, None, None, None, 1, None) == 1


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump missing")
def test_sass_is_sm100a_with_dmma_and_tma(lib):
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "DMMA.8x8x4" in sass          # FP64 tensor-core MMA in R formation / LU / Cholesky
    assert "UTMALDG" in sass             # TMA tile loads (cp.async.bulk.tensor) in R formation
    assert "UBLKCP" in sass              # cp.async.bulk C-tile copies in the per-energy dense LA


def test_workspace_slot_layout(lib):
    """Host-only layout query: every per-energy slot base must stay 16-byte aligned for the TMA
    tensor maps built on it (an odd slot size broke rmx_match_K at nch = 37), and a slot must hold
    what the kernels write - the matching [A | B_open] block (n x 2n) and the five T planes."""
    f = lib.rmx_workspace_doubles_per_energy
    assert f(0) == -1 and f(-5) == -1 and f((1 << 16) + 1) == -1
    prev = 0
    for n in list(range(1, 300)) + [511, 512, 513, 1200, 2000, 2944, 2945, 3500, 8192]:
        d = f(n)
        assert d % 16 == 0, (n, d)
        assert d >= 2 * n * n + 9 * n and d >= 5 * n * n, (n, d)
        assert d >= prev  # monotone in nch: a context grown for n serves every smaller n
        prev = d
