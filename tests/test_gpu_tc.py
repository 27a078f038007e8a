"""The tensor-core (tcgen05, kind::tf32) operand layout used by the binned
scan: one 128x256x16 product through the C-ABI diagnostic, checked on the host
against float64 dot products of the same tf32 values."""

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")


def test_tc_selftest():
    from paper_2406_02807_b200 import _lib
    err = C.c_double(-1.0)
    _lib.check(_lib.lib().capt_tc_selftest(_lib.default_device(), C.byref(err)), "tc selftest")
    # fp32 accumulation of 16 exact tf32 products
    assert 0.0 <= err.value < 1e-6, err.value
