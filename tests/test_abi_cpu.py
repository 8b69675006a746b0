"""CPU-side checks of the C ABI: the in-tree library loads, exports every symbol
include/anyprec_b200.h declares, and its host-side validation returns the
reference's error classes before any device work (engine.py:263-281 style
raise-before-compute).  No kernel is launched here."""

import ctypes
import os
import re

import pytest

from paper_2402_10517_b200 import _lib
from paper_2402_10517_b200.errors import (
    CodeRangeError,
    DeviceError,
    LayoutError,
    ParameterError,
    ShapeError,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "anyprec_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apb_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_version_and_strings(lib):
    assert lib.apb_version() == 100
    assert lib.apb_status_string(0) == b"ok"
    assert lib.apb_status_string(2) == b"parameter error"


def test_pad_columns(lib):
    # bitplane.py:72-73 / test_bitplane.py:90-93
    assert lib.apb_pad_columns(1) == 1024
    assert lib.apb_pad_columns(1024) == 1024
    assert lib.apb_pad_columns(1025) == 2048
    assert lib.apb_pad_columns(11008) == 11264


def test_host_validation_before_launch(lib):
    nul = ctypes.c_void_p(0)
    fake = ctypes.c_void_p(0x1000)
    # k outside [2, 8]
    assert lib.apb_gemv(fake, 8, 16, 1024, 1024, 9, fake, fake, 1, 1024, 0, fake, 0, 16, 0, nul) == 2
    # padded columns inconsistent
    assert lib.apb_gemv(fake, 8, 16, 1024, 2048, 4, fake, fake, 1, 1024, 0, fake, 0, 16, 0, nul) == 1
    # misaligned activations (ldx % 8)
    assert lib.apb_gemv(fake, 8, 16, 1000, 1024, 4, fake, fake, 1, 1001, 0, fake, 0, 16, 0, nul) == 2
    # k > n_max
    assert lib.apb_gemv(fake, 4, 16, 1024, 1024, 5, fake, fake, 1, 1024, 0, fake, 0, 16, 0, nul) == 2
    # odd hi/lo activation count
    assert lib.apb_gemv(fake, 8, 16, 1024, 1024, 4, fake, fake, 3, 1024, 1, fake, 0, 16, 0, nul) == 1
    # pack: n_max out of range, empty matrix
    assert lib.apb_pack(fake, 4, 4, 4, 9, 1, fake, nul, nul) == 2
    assert lib.apb_pack(fake, 0, 4, 4, 3, 1, fake, nul, nul) == 1
    # unpack: k = 0
    assert lib.apb_unpack(fake, 3, 4, 4, 1024, 1, 0, fake, 4, nul) == 2
    # transpose width
    assert lib.apb_transpose_words(fake, 1, 4, fake, nul) == 2
    # permute in place is rejected
    assert lib.apb_permute(fake, fake, 1, 1, 1024, 0, nul) == 2
    # dequant dtype
    assert lib.apb_dequant(fake, 8, 4, 1024, 1024, 1, 3, fake, fake, 7, 1024, nul) == 2
    # fused tcgen05 dense path (engine.py:343-354): activation prep and GEMM validate first
    F32, F16 = 0, 1
    assert lib.apb_dense_prep_x(fake, F32, 4, 1000, 1000, fake, 1000, fake, nul) == 1  # padded % 1024
    assert lib.apb_dense_prep_x(fake, F32, 4, 1000, 999, fake, 1024, fake, nul) == 1   # ldx < cols
    assert lib.apb_dense_prep_x(fake, F32, 4, 1000, 1000, fake, 1024, nul, nul) == 2   # fp32 needs inv
    assert lib.apb_dense_prep_x(fake, 7, 4, 1000, 1000, fake, 1024, fake, nul) == 2    # dtype
    assert lib.apb_dense_prep_x(fake, F16, 0, 1000, 1000, fake, 1024, nul, nul) == 1   # empty batch
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1024, 9, fake, fake, 64, 1, fake, fake, 16, nul, 0, nul) == 2  # k
    assert lib.apb_gemm_dense_tc(fake, 4, 16, 1024, 1024, 5, fake, fake, 64, 1, fake, fake, 16, nul, 0, nul) == 2  # k > n_max
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1000, 4, fake, fake, 64, 1, fake, fake, 16, nul, 0, nul) == 1  # padded
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1024, 4, fake, fake, 63, 1, fake, fake, 16, nul, 0, nul) == 1  # odd pairs
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1024, 4, fake, fake, 64, 1, nul, fake, 16, nul, 0, nul) == 2  # pairs need inv
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1024, 4, fake, fake, 64, 0, nul, fake, 8, nul, 0, nul) == 1   # ldy < rows
    odd = ctypes.c_void_p(0x1008)  # not 16-byte aligned: a TMA operand
    assert lib.apb_gemm_dense_tc(odd, 8, 16, 1024, 1024, 4, fake, fake, 64, 0, nul, fake, 16, nul, 0, nul) == 2
    assert lib.apb_gemm_dense_tc(fake, 8, 16, 1024, 1024, 4, fake, odd, 64, 0, nul, fake, 16, nul, 0, nul) == 2


def test_status_mapping():
    with pytest.raises(ShapeError):
        _lib.check(1, "x")
    with pytest.raises(ParameterError):
        _lib.check(2, "x")
    with pytest.raises(LayoutError):
        _lib.check(3, "x")
    with pytest.raises(CodeRangeError):
        _lib.check(4, "x")
    with pytest.raises(DeviceError):
        _lib.check(5, "x")
    _lib.check(0, "x")


def test_reference_error_hierarchy():
    # errors.py:4-35: ShapeError/ParameterError/CodeRangeError are ValueErrors,
    # LayoutError is a RuntimeError, all derive from AnyPrecError
    from paper_2402_10517_b200.errors import AnyPrecError

    assert issubclass(ShapeError, ValueError) and issubclass(ShapeError, AnyPrecError)
    assert issubclass(ParameterError, ValueError)
    assert issubclass(CodeRangeError, ValueError)
    assert issubclass(LayoutError, RuntimeError)
