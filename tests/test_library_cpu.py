"""CPU-side checks of the C ABI library: it loads, exports every symbol that
include/osbf_gpu.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "osbf_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(osbf_gpu_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("osbf_gpu_iterate", "osbf_gpu_osbf_host", "osbf_gpu_filter_multichannel_host",
              "osbf_gpu_osbf_step_host", "osbf_gpu_sat", "osbf_gpu_subwindow_means"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2108_05021_b200 import _native

    lib = _native.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in osbf_gpu.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (osbf_gpu_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_bindings_cover_the_header():
    from paper_2108_05021_b200 import _native

    assert sorted(n for n, _, _ in _native.SIGNATURES) == declared_symbols()


def test_library_is_sm100a_code():
    from paper_2108_05021_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_no_fallback():
    import torch

    import paper_2108_05021_b200 as ob
    from paper_2108_05021_b200 import _native

    lib = _native.lib()
    assert lib.osbf_gpu_abi_version() == 1
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu suite")
    assert lib.osbf_gpu_device_available() == 0
    h = ctypes.c_void_p()
    assert lib.osbf_gpu_ctx_create(0, ctypes.byref(h)) == _native.OSBF_ERR_NO_DEVICE
    assert b"no CUDA device" in lib.osbf_gpu_last_error()
    with pytest.raises(ob.NoDevice):
        ob.osbf(np.zeros((4, 4)), 2, 1)


def test_null_context_is_invalid_argument():
    from paper_2108_05021_b200 import _native

    lib = _native.lib()
    st = lib.osbf_gpu_iterate(None, 2, None, 4, 16, None, 4, 16, 4, 4, 1, 2, 1, 0, None)
    assert st == _native.OSBF_ERR_INVALID_ARGUMENT
    assert lib.osbf_gpu_last_error() == b"null context"


def test_kernel_family_overrides_validate_names():
    """The diagnostic family switches are host-side state: known names (and
    None / "" to clear) are accepted without a device, unknown ones rejected."""
    import paper_2108_05021_b200 as ob

    lib = ob.lib()
    try:
        for fam in ("strip", "gwalk", "twalk", "stencil"):
            assert lib.osbf_gpu_set_exact_kernel(fam.encode()) == 0
        assert lib.osbf_gpu_set_exact_kernel(b"no-such-family") != 0
        assert b"unknown exact kernel family" in lib.osbf_gpu_last_error()
        assert lib.osbf_gpu_set_fast_kernel(b"walk") == 0
        assert lib.osbf_gpu_set_fast_kernel(b"no-such-family") != 0
    finally:
        assert lib.osbf_gpu_set_exact_kernel(None) == 0
        assert lib.osbf_gpu_set_fast_kernel(b"") == 0


def test_python_value_types_mirror_reference():
    import paper_2108_05021_b200 as ob

    wins = ob.sub_windows(2)
    assert [(w.u0, w.u1, w.v0, w.v1) for w in wins[:2]] == [(-2, 0, 0, 2), (0, 2, 0, 2)]
    with pytest.raises(ob.InvalidArgument):
        ob.sub_windows(0)
    cfg = ob.FilterConfig()
    assert (cfg.radius, cfg.iterations, cfg.variant, cfg.sigma) == (2, 10, ob.FilterVariant.OsbfExact, 3.0)
    cfg.radius = 0
    with pytest.raises(ob.InvalidArgument):
        cfg.validate()
    cfg = ob.FilterConfig(iterations=-1)
    with pytest.raises(ValueError):
        cfg.validate()


def test_dropin_headers_compile_and_link():
    """include/osbf/*.hpp (the reference's declarations) compile and the C++
    drop-in test links against libosbf_gpu.so (run on the GPU by test_dropin_gpu)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-D", exe], capture_output=True, text=True, check=True).stdout
    assert "osbf_gpu_osbf_host" in out and "oracle_osbf" in out
