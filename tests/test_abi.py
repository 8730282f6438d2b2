"""C-ABI library checks that need no GPU: it builds, loads, exports every
symbol include/bm.h declares, and the Python binding refuses to run without it."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_01405_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("bm_cover_build", "bm_cover_build_ex", "bm_cover_build_host", "bm_free",
              "bm_last_error", "bm_version"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in header_functions():
        assert hasattr(lib, f), f"{f} declared in include/bm.h but not exported"


def test_binding_lists_match_header():
    from paper_2601_01405_b200 import bm
    assert sorted(bm.EXPORTED) == header_functions()


def test_version_and_error_string(lib):
    lib.bm_version.restype = ctypes.c_int32
    assert lib.bm_version() == (0 << 16) | 1
    lib.bm_last_error.restype = ctypes.c_char_p
    assert lib.bm_last_error() == b""
    lib.bm_free(None)  # NULL-safe, no device work


def test_invalid_arguments_rejected_before_device_work(lib):
    """Argument validation happens on the host before any CUDA call."""
    from paper_2601_01405_b200 import bm
    L = bm.load()
    out = ctypes.POINTER(bm._Cover)()
    rc = L.bm_cover_build(None, 0, 10, 2, 0, 1.0, None, ctypes.byref(out))
    assert rc == bm.BM_EINVAL and not out
    buf = (ctypes.c_float * 8)()
    for n, d, eps in [(0, 2, 1.0), (4, 0, 1.0), (4, 2, 0.0), (4, 2, -1.0), (4, 2, float("nan"))]:
        assert L.bm_cover_build(ctypes.addressof(buf), 0, n, d, 0, eps, None,
                                ctypes.byref(out)) == bm.BM_EINVAL
    assert L.bm_cover_build(ctypes.addressof(buf), 1, 4, 2, 2, 1.0, None,
                            ctypes.byref(out)) == bm.BM_EUNSUPPORTED
    assert L.bm_cover_build(ctypes.addressof(buf), 0, 2**31, 2, 0, 1.0, None,
                            ctypes.byref(out)) == bm.BM_EOVERFLOW
    assert b"INT32" in L.bm_last_error()


def test_sm100a_only_cubin(lib):
    """The fatbin carries sm_100a SASS only (no PTX, no other arch)."""
    import subprocess
    from paper_2601_01405_b200 import build
    r = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert archs == {"100a"}, archs
    r = subprocess.run(["cuobjdump", "--list-ptx", build.LIB], capture_output=True, text=True)
    assert ".ptx" not in r.stdout
