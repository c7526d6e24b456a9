"""CPU-side checks of the C-ABI library: it loads and exports every symbol include/c0ip.h declares;
argument errors are reported synchronously (no device work is issued on these paths)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "c0ip.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(c0ip_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2412_05082_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2412_05082_b200.build import build
        build()
    return _lib.load()


def test_header_declares_expected_calls():
    names = _declared()
    for n in ["c0ip_create", "c0ip_destroy", "c0ip_apply", "c0ip_residual", "c0ip_smooth", "c0ip_restrict",
              "c0ip_prolongate_add", "c0ip_vcycle", "c0ip_pcg", "c0ip_patch_dofs", "c0ip_color_patches",
              "c0ip_get_fdm", "c0ip_rhs", "c0ip_level_info", "c0ip_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2412_05082_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(c0ip_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= exported


def test_sm100a_code_present(lib):
    from paper_2412_05082_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("field,value", [("dim", 4), ("degree", 1), ("degree", 8), ("finest_level", 0),
                                         ("cells_override", 1), ("penalty_scale", -1.0)])
def test_create_rejects_bad_config(lib, field, value):
    from paper_2412_05082_b200 import _lib
    cfg = _lib.Config(2, 3, 3, 0, 1.0, 0)
    setattr(cfg, field, value)
    h = C.c_void_p()
    assert lib.c0ip_create(C.byref(cfg), C.byref(h)) == _lib.ERR_ARG
    assert h.value is None
    assert len(lib.c0ip_last_error()) > 0


def test_null_context_errors(lib):
    from paper_2412_05082_b200 import _lib
    assert lib.c0ip_destroy(None) == _lib.ERR_ARG
    assert lib.c0ip_apply(None, 1, 0, None, None, None) == _lib.ERR_ARG
    assert lib.c0ip_set_path(None, 0) == _lib.ERR_ARG
