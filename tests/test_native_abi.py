"""The C-ABI library: loads on a CPU-only box and exports every symbol include/pipefill.h declares."""

import ctypes
import os

import pytest

from paper_2410_07192_b200 import native


def test_library_built():
    assert os.path.exists(native.LIB_PATH), "run `make` (or __graft_entry__.build())"


def test_every_declared_symbol_is_exported():
    lib = native.load()
    declared = native.declared_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_every_declared_symbol_is_typed_in_binding():
    declared = set(native.declared_symbols())
    assert declared == set(native._SIGNATURES), declared ^ set(native._SIGNATURES)


def test_abi_version_and_error_plumbing_without_gpu():
    lib = native.load()
    assert lib.pf_abi_version() == 1
    out = ctypes.c_uint32(0)
    # pure host-side entry points work without a device
    assert lib.pf_gemm_units(4096, 3072, 768, ctypes.byref(out)) == native.PF_OK
    assert out.value > 0
    assert lib.pf_copy_units(1 << 20, ctypes.byref(out)) == native.PF_OK and out.value == 4
    assert lib.pf_gemm_units(0, 1, 1, ctypes.byref(out)) == native.PF_ERR_INVALID
    assert "pf_gemm_units" in native.last_error()


def test_compute_entry_points_fail_loudly_without_a_device():
    """No CPU fallback: with no GPU the kernels refuse with a status, never compute."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.NativeUnavailable):
        native.require_device()
    lib = native.load()
    rc = lib.pf_gemm(ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, ctypes.c_void_p(16),
                     128, 128, 64, 0, None, None)
    assert rc != native.PF_OK


def test_sass_contains_tcgen05_and_tma():
    """The GEMM / attention are tcgen05 + TMA kernels (SASS UTCHMMA / UTMALDG / LDTM)."""
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not installed")
    sass = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path
