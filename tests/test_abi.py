"""The C-ABI library loads without a GPU and exports every symbol that
include/wino.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wino.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wino_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_surface():
    from paper_1509_09308_b200 import _lib
    assert set(declared_functions()) == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    from paper_1509_09308_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_version_and_error_string():
    from paper_1509_09308_b200 import _lib
    assert "sm_100a" in _lib.version()
    h = ctypes.c_void_p()
    desc = _lib.LayerDesc(1, 1, 6, 6, 1, 3, 3, 1)
    rc = _lib.lib.wino_plan_create(ctypes.byref(desc), 5, 0, 0, ctypes.byref(h))
    assert rc == _lib.WINO_EUNSUPPORTED
    assert b"F(5,3)" in _lib.lib.wino_last_error()


def test_null_arguments_rejected():
    from paper_1509_09308_b200 import _lib
    assert _lib.lib.wino_plan_create(None, 2, 0, 0, None) == _lib.WINO_EINVAL
    assert _lib.lib.wino_forward(None, None, None, None, None, None, 0, None) == _lib.WINO_EINVAL


def test_compiled_for_sm100a_with_tcgen05():
    from paper_1509_09308_b200 import _lib
    try:
        sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                              text=True, timeout=120).stdout
    except (FileNotFoundError, subprocess.TimeoutExpired):
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in sass
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
