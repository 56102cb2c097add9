"""CPU-side checks of the C ABI: the shared library loads and exports every symbol that
include/lf_b200.h declares (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lf_b200.h")
LIB = os.path.join(ROOT, "paper_2512_11269_b200", "libcerium_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("lf_ctx_create", "lf_ntt_fwd", "lf_ntt_inv", "lf_ewise", "lf_automorph", "lf_bconv",
              "lf_keyswitch", "lf_hom_mul", "lf_rotate", "lf_rescale", "lf_ks_decompose"):
        assert s in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.lf_abi_version.restype = ctypes.c_int
    assert lib.lf_abi_version() == 1


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_python_binding_signatures_cover_the_header():
    from paper_2512_11269_b200 import _native
    _native.lib()
    assert set(declared_symbols()) <= set(_native.EXPORTS)


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_errors_without_gpu_are_loud():
    """Calls that would touch the GPU fail with an error code, never silently."""
    lib = ctypes.CDLL(LIB)
    lib.lf_last_error.restype = ctypes.c_char_p
    lib.lf_ntt_fwd.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int] + [ctypes.c_void_p] * 2
    rc = lib.lf_ntt_fwd(None, None, 1, None, None)
    assert rc != 0
    assert lib.lf_last_error()


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2512_11269_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b|import_module\(.oracle", src, re.M), f
