"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/convtact_b200.h declares, and argument validation maps to the
reference's ValueError cases without touching the device."""

import ctypes
import os
import re

import pytest

from paper_1612_08825_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "convtact_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|size_t|char\s*\*|const char\s*\*)\s*\*?\s*(ct_\w+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS), (set(names) ^ set(_lib.EXPORTS))


def test_library_exports_every_declared_symbol():
    L = _lib.load(require_gpu=False)
    for name in declared_functions():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.ct_version()


def test_validation_errors_without_device():
    L = _lib.load(require_gpu=False)
    shp = _lib.i64_array([3])
    kshp = _lib.i64_array([5])
    # VALID with kernel larger than signal -> CT_EINVAL before any launch (conv.py:93-98)
    rc = L.ct_direct(_lib.CT_F64, 1, None, shp, 1, None, None, kshp, _lib.CT_VALID, _lib.CT_ZERO, 1, None, None)
    assert rc == _lib.CT_EINVAL
    assert b"VALID" in L.ct_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    # zero rank
    assert L.ct_direct(_lib.CT_F64, 0, None, shp, 1, None, None, kshp, 0, 0, 0, None, None) == _lib.CT_EINVAL
    # run_sequence guards (ttc.py:235-241, ttc.py:294-297)
    assert L.ct_run_sequence(_lib.CT_F64, None, 1, 1, 8, 8, 0, -1, 1e-9, None, None, 0, None) == _lib.CT_EINVAL
    assert L.ct_run_sequence(_lib.CT_F64, None, 1, 4, 16, 16, 3, -1, 1e-9, None, None, 0, None) == _lib.CT_EINVAL
    assert L.ct_run_sequence(_lib.CT_F64, None, 1, 4, 16, 16, -1, -1, 1e-9, None, None, 0, None) == _lib.CT_EINVAL
    # normal system border / interior (ttc.py:103-109)
    assert L.ct_normal_system(_lib.CT_F64, None, None, None, None, 4, 4, 0, None, None, 0, None) == _lib.CT_EINVAL
    assert L.ct_normal_system(_lib.CT_F64, None, None, None, None, 4, 4, 2, None, None, 0, None) == _lib.CT_EINVAL
    # downsample (ttc.py:200-201)
    assert L.ct_pyramid_down(_lib.CT_F64, None, 1, 1, 8, None, None) == _lib.CT_EINVAL
    # bad dtype
    assert L.ct_ttc_derivatives(7, None, None, 4, 4, None, None, None, None) == _lib.CT_EINVAL


def test_workspace_queries_are_pure():
    L = _lib.load(require_gpu=False)
    a = L.ct_run_sequence_workspace_bytes(_lib.CT_F64, 4, 64, 256, 256, 0, -1)
    b = L.ct_run_sequence_workspace_bytes(_lib.CT_F64, 4, 64, 256, 256, 0, -1)
    assert a == b and a > 0
    ms = L.ct_run_sequence_workspace_bytes(_lib.CT_F32, 1, 16, 1080, 1920, 0, 3)
    # pyramid levels 1..3 of 16 f32 frames plus sums: at least the level-1 frames
    assert ms >= 16 * 540 * 960 * 4
    assert L.ct_ttc_moments_workspace_bytes(_lib.CT_F64, 1, 1, 8, 8) == 0
