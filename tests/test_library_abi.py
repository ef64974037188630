"""CPU tests of the boundary: libfmm_b200.so loads and exports every function that
include/fmm_b200.h declares; configuration validation happens before any CUDA call;
the product package never imports the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "fmm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(fmm_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def so():
    from paper_1204_3105_b200 import _build

    path = _build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    names = declared_functions()
    for need in ["fmm_build_tree", "fmm_evaluate", "fmm_export", "fmm_free", "fmm_status", "fmm_error_string"]:
        assert need in names


def test_every_declared_symbol_is_exported(so):
    for name in declared_functions():
        assert hasattr(so, name), name


def test_version_and_error_strings(so):
    so.fmm_error_string.restype = ctypes.c_char_p
    assert so.fmm_version() >= 1
    assert so.fmm_error_string(2) == b"point outside the root domain"


def test_bad_config_rejected_without_gpu():
    from paper_1204_3105_b200 import Config, lib

    L = lib()
    h = ctypes.c_void_p()
    for bad in [Config.make("quad", 0, 8, 0, 0, 1), Config.make("quad", 3, 0, 0, 0, 1),
                Config.make("quad", 3, 32, 0, 0, 1), Config.make("sept", 11, 8, 0, 0, 1),
                Config.make("triq", 3, 8, 0, 0, -1.0), Config.make("quad", 3, 8, 0, 0, 1, rank=2, nranks=2)]:
        assert L.fmm_build_tree(ctypes.byref(bad), None, None, 0, None, 0, None, ctypes.byref(h)) == 1


def test_product_package_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_1204_3105_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "fmm_oracle" not in txt and "liboracle" not in txt, f


def test_build_limits_refused_up_front():
    """Depths and point counts beyond the build's device scans are refused before any CUDA call
    with FMM_EBADCFG and a message (no GPU needed: the checks precede the device work)."""
    import ctypes as C

    from paper_1204_3105_b200 import Config, lib

    L = lib()
    L.fmm_build_tree.restype = C.c_int
    L.fmm_last_error_message.restype = C.c_char_p
    for tiling, depth, n in (("quad", 13, 16), ("sept", 10, 16), ("triq", 12, (1 << 27) + 1)):
        cfg = Config.make(tiling, depth, 8, 0.0, 0.0, 1.0, True)
        out = C.c_void_p()
        xy = (C.c_double * 2)()
        u = (C.c_double * 1)()
        rc = L.fmm_build_tree(C.byref(cfg), xy, u, C.c_int64(n), None, C.c_int64(0), None, C.byref(out))
        assert rc == 1 and not out.value, (tiling, depth, rc)  # FMM_EBADCFG
        msg = L.fmm_last_error_message().decode()
        assert ("depth" in msg) if n < (1 << 27) else ("points" in msg), msg
