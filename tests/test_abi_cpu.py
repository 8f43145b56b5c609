"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol that
include/mpb.h declares (no compute calls -- there is no GPU here), host-only helpers
behave, and the product path never reaches the oracle."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpb.h")
LIB = os.path.join(ROOT, "paper_2410_18129_b200", "libmpb.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["mp_batch_mul", "mp_batch_sqr", "mont_batch_mul", "mont_batch_sqr", "mont_batch_redc",
                     "mont_batch_modexp_ct", "mont_batch_setup", "mpb_layout_expand", "mpb_layout_contract",
                     "mpb_last_error"]:
        assert required in names


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__ as g

        g.build_cuda()
    return ctypes.CDLL(LIB)


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_host_only_helpers(lib):
    lib.mpb_limbs.restype = ctypes.c_int
    lib.mpb_supported.restype = ctypes.c_int
    assert [lib.mpb_limbs(b) for b in (0, 1, 512, 1024, 2048, 3072, 4096, 4108, 4154)] == \
        [0, 4, 16, 32, 64, 96, 128, 132, 132]
    assert lib.mpb_supported(2048) == 1 and lib.mpb_supported(700) == 1 and lib.mpb_supported(20000) == 0
    lib.mont_batch_modexp_ct_workspace.restype = ctypes.c_size_t
    lib.mont_batch_modexp_ct_workspace.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    # warp-tiled exponentiation workspace: count rounded up to 32 operands, 2^w + 7 arrays of L limbs
    assert lib.mont_batch_modexp_ct_workspace(10, 2048, 5, 0) == 32 * 64 * (32 + 7) * 4
    assert lib.mont_batch_modexp_ct_workspace(64, 2048, 5, 0) == 64 * 64 * (32 + 7) * 4
    assert lib.mont_batch_modexp_ct_workspace(10, 2048, 7, 0) == 0
    # radix-2^52 path (algo 4): D = 40 digits at 2048 bits as doubles, 2^w + 8 numbers per operand
    assert lib.mont_batch_modexp_ct_workspace(10, 2048, 5, 4) == 32 * 20 * 16 * (32 + 8)
    assert lib.mont_batch_modexp_ct_workspace(10, 700, 5, 4) == 0  # no radix-2^52 instance
    # hybrid (algo 5): the 32-bit tiled workspace and the radix-2^52 one, side by side
    assert lib.mont_batch_modexp_ct_workspace(10, 2048, 5, 5) == 32 * 64 * (32 + 7) * 4 + 32 * 20 * 16 * (32 + 8) + 256
    assert lib.mont_batch_modexp_ct_workspace(10, 4096, 5, 5) == 0
    lib.mont_batch_setup_workspace.restype = ctypes.c_size_t
    lib.mont_batch_setup_workspace.argtypes = [ctypes.c_size_t, ctypes.c_int]
    assert lib.mont_batch_setup_workspace(10, 2048) == 10 * 6 * 64 * 4
    lib.mp_batch_workspace.restype = ctypes.c_size_t
    lib.mp_batch_workspace.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
    assert lib.mp_batch_workspace(10, 4096, 1) == 0  # schoolbook needs none
    # 1 level at L = 128 (C = 16, 8 blocks): 4 * 4 blocks of 16 limbs
    assert lib.mp_batch_workspace(10, 4096, 2) == 10 * 16 * 16 * 4
    # 2 levels at 4154 bits (L = 132, C = 12, 11 blocks): 4*6 + 4*3 blocks of 12 limbs
    assert lib.mp_batch_workspace(10, 4154, 3) == 10 * 36 * 12 * 4


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_18129_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert "oracle.h" not in txt, f


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    """The binding has no CPU fallback: with the .so absent, import raises."""
    import importlib.util

    src = os.path.join(ROOT, "paper_2410_18129_b200", "mpb.py")
    fake_pkg = tmp_path / "fakepkg"
    fake_pkg.mkdir()
    (fake_pkg / "mpb.py").write_text(open(src).read())
    spec = importlib.util.spec_from_file_location("fakepkg_mpb", fake_pkg / "mpb.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_host_side_argument_checks(lib):
    """Argument errors are reported before any device work (no GPU needed): count beyond 2^27,
    bits beyond 16384, window / redc / algo out of range, null pointers; count 0 is a no-op."""
    vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    lib.mont_batch_mul.argtypes = [vp, vp, vp, vp, vp, sz, i, i, vp, sz, vp]
    lib.mont_batch_modexp_ct.argtypes = [vp, vp, vp, vp, vp, vp, sz, i, i, i, i, vp, sz, vp]
    lib.mpb_last_error.restype = ctypes.c_char_p
    EINVAL, EUNSUPPORTED = -1, -2
    big = (1 << 27) + 1
    assert lib.mont_batch_mul(None, None, None, None, None, big, 1024, 1, None, 0, None) == EUNSUPPORTED
    assert b"2^27" in lib.mpb_last_error()
    assert lib.mont_batch_mul(None, None, None, None, None, 4, 20000, 1, None, 0, None) == EUNSUPPORTED
    assert lib.mont_batch_mul(None, None, None, None, None, 4, 1024, 7, None, 0, None) == EINVAL
    assert lib.mont_batch_mul(None, None, None, None, None, 4, 1024, 1, None, 0, None) == EINVAL  # null
    assert lib.mont_batch_mul(None, None, None, None, None, 0, 1024, 1, None, 0, None) == 0  # no-op
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 1024, 7, 1, 0, None, 0, None) == EINVAL
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 1024, 5, 1, 9, None, 0, None) == EINVAL
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, big, 1024, 5, 1, 0, None, 0, None) \
        == EUNSUPPORTED
    # radix-2^52 exponentiation: truncated / full REDC only, sizes with an instance only, not a product
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 2048, 5, 2, 4, None, 0, None) \
        == EUNSUPPORTED
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 700, 5, 1, 4, None, 0, None) \
        == EUNSUPPORTED
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 2048, 5, 1, 6, None, 0, None) == EINVAL
    assert lib.mont_batch_modexp_ct(None, None, None, None, None, None, 4, 4096, 5, 1, 5, None, 0, None) \
        == EUNSUPPORTED  # the hybrid serves 2048-bit operands only
    lib.mp_batch_mul.argtypes = [vp, vp, vp, sz, i, i, vp, sz, vp]
    assert lib.mp_batch_mul(None, None, None, 4, 2048, 4, None, 0, None) == EUNSUPPORTED
    # CRT-RSA runs 2 * count half-size operands in one exponentiation: at most 2^26 per call
    lib.rsa_batch_crt_ct.argtypes = [vp, vp, vp, vp, vp, vp, vp, sz, i, i, i, vp, sz, vp]
    crt_big = (1 << 26) + 1
    assert lib.rsa_batch_crt_ct(None, None, None, None, None, None, None, crt_big, 2048, 5, 1, None, 0, None) \
        == EUNSUPPORTED
    assert b"2^26" in lib.mpb_last_error()
