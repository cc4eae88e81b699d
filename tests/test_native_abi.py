"""The C-ABI library loads without a GPU and exports every entry point
include/pdz.h declares; host-only entry points answer correctly."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "pdz.h")
LIB = os.path.join(REPO, "paper_2506_08793_b200", "libpdz.so")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdz_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    from paper_2506_08793_b200 import _native

    return _native.lib()


def test_header_declares_the_binding_table():
    from paper_2506_08793_b200 import _native

    assert header_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_header_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_solve_params_layout():
    from paper_2506_08793_b200._native import SolveParams

    assert ctypes.sizeof(SolveParams) == 64
    assert SolveParams.sigma.offset == 32 and SolveParams.rel_tol.offset == 56


def test_host_only_entry_points(lib):
    assert lib.pdz_version() >= 1
    taps = np.empty(13)
    assert lib.pdz_gaussian_taps(2.0, 13, taps.ctypes.data) == 0
    d = np.arange(13) - 6
    g = np.exp(-(d * d) / 8.0)
    np.testing.assert_allclose(taps, g / g.sum(), rtol=1e-15)
    assert lib.pdz_gaussian_taps(2.0, 4, taps.ctypes.data) == 1
    assert b"odd" in lib.pdz_last_error()
    assert lib.pdz_airlight_count(1024, 1024, 0.001) == 1049
    assert lib.pdz_airlight_count(4320, 7680, 0.001) == 33178
    assert lib.pdz_airlight_count(480, 640, 0.001) == 308
    assert lib.pdz_airlight_workspace_bytes(64, 64, 0.01) > 0
    assert lib.pdz_dark_channel_workspace_bytes(64, 64) >= 3 * 64 * 64 * 8


def test_workspace_queries_validate(lib):
    from paper_2506_08793_b200._native import SolveParams

    p = SolveParams(height=1024, width=1024, planes=3, channels=3, kernel_size=19,
                    edge_preserving=1, max_iters=200, sigma=3.0, epsilon=1e-3,
                    tau=2.25e-4, rel_tol=1e-4)
    need = lib.pdz_solve_workspace_bytes(ctypes.byref(p))
    assert need >= 2 * 3 * 1024 * 1024 * 4
    bad = SolveParams(height=1, width=5, planes=1, channels=1, kernel_size=5, max_iters=1,
                      sigma=2.0, epsilon=1e-3)
    assert lib.pdz_solve_workspace_bytes(ctypes.byref(bad)) == 0


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2506_08793_b200 as pkg

    with pytest.raises(RuntimeError, match="CUDA"):
        pkg.dark_channel(np.zeros((4, 4, 3)), np.ones(3), 1)
