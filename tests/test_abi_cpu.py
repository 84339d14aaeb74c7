"""CPU-side checks of the C ABI: the library builds, loads, exports every symbol include/sketch.h
declares, and its synchronous host-side validation behaves as documented (no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2603_20966_b200 as sk
from tests.conftest import ROOT


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "sketch.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sk_status_t|const char\*|uint64_t)\s+(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_expected_entry_points():
    decl = _declared_functions()
    assert set(decl) == set(sk.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = sk.load_library()
    for name in _declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {sk.library_path()}").read()
    assert "sm_100a" in out


def test_host_validation_without_gpu():
    lib = sk.load_library()
    h = ctypes.c_void_p()
    assert lib.sketch_create(1, 0, 0, 16, ctypes.byref(h)) == 1  # n2 < 1
    assert lib.sketch_create(1, 7, 10, 16, ctypes.byref(h)) == 1  # bad dist
    assert lib.sketch_create(1, 0, 1000, 64, ctypes.byref(h)) == 0
    try:
        assert lib.sketch_set_mode(h, 9) == 1
        assert lib.sketch_set_split_k(h, 65) == 1
        # CTA grouping override: 0 / 1 / 2 / 4 / 6 / 8 (clusters of 0..4 pairs), anything else rejected
        for cg in (0, 1, 2, 4, 6, 8):
            assert lib.sketch_set_cta_group(h, cg) == 0
        for cg in (3, 5, 7, 16, -1):
            assert lib.sketch_set_cta_group(h, cg) == 1
        n = ctypes.c_size_t()
        assert lib.sketch_workspace_size(h, 5000, ctypes.byref(n)) == 0
        # degenerate sizes plan without faulting (empty A, one row), in every mode
        for mode in (0, 1, 2):
            assert lib.sketch_set_mode(h, mode) == 0
            for n1 in (0, 1, 7, 129, 5000, 2048):
                assert lib.sketch_workspace_size(h, n1, ctypes.byref(n)) == 0
        assert lib.sketch_workspace_size(h, -1, ctypes.byref(n)) == 1
        # shape mismatch is reported before any device work
        st = lib.sketch_apply(h, None, 10, 999, 999, None, 64, None, 0, None)
        assert lib.sketch_status_string(st) == b"SK_ERR_SHAPE_MISMATCH"
        assert b"n2" in lib.sketch_last_error()
        # misaligned lda
        st = lib.sketch_apply(h, 16, 10, 1000, 1001, 32, 64, None, 1 << 30, None)
        assert lib.sketch_status_string(st) == b"SK_ERR_ALIGNMENT"
        # out-of-range Omega block
        st = lib.sketch_generate(h, 0, 4, 60, 8, 16, 8, None)
        assert lib.sketch_status_string(st) == b"SK_ERR_INVALID_VALUE"
    finally:
        lib.sketch_destroy(h)


def test_python_layer_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    s = sk.Sketch(1, "gaussian", 100, 8)
    with pytest.raises(sk.SketchError):
        s.apply(torch.zeros((4, 100)))
