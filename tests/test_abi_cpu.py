"""CPU-side checks of the native boundary and the host mirror of the tick API.

No compute calls: the library must load and export every symbol declared in
include/tickjoin_b200.h; config validation and result containers follow the
reference's semantics.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tickjoin_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(tj_\w+)\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tj_create", "tj_destroy", "tj_tick", "tj_get_index", "tj_get_subqueries", "tj_get_directory",
              "tj_get_bitmaps", "tj_last_error"):
        assert s in syms


def test_library_loads_and_exports_every_symbol():
    import __graft_entry__

    __graft_entry__.build()
    from paper_1411_3212_b200 import _native

    lib = _native.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(_native.EXPORTED) == set(declared_symbols())
    assert lib.tj_abi_version() == 4
    # loading the .so must not need a GPU; creating a context must fail loudly without one
    n = ctypes.c_int(-1)
    lib.tj_device_count(ctypes.byref(n))
    assert n.value >= 0


def test_engine_fails_loudly_without_device():
    from paper_1411_3212_b200 import Engine, MethodConfig, _native
    from paper_1411_3212_b200.errors import DeviceError

    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceError):
        Engine(MethodConfig())


def test_method_config_validation():
    from paper_1411_3212_b200 import MethodConfig
    from paper_1411_3212_b200.errors import BadConfig

    MethodConfig().validate()
    MethodConfig(method="ug").validate()  # split factor swept on the first tick
    MethodConfig(method="ug", split_factor=37, th_quad=0).validate()  # th_quad is a quad-only field
    MethodConfig(method="ug_baseline", split_factor=12).validate()
    for bad in (dict(method="rtree"), dict(method="ug_baseline", split_factor=0), dict(method="ug", split_factor=0),
                dict(method="ug", split_factor=5000), dict(th_quad=0), dict(l_max=13), dict(schedule="lifo"),
                dict(rebuild="never"), dict(n_workers=0)):
        with pytest.raises(BadConfig):
            MethodConfig(**bad).validate()


def test_qos_formulas():
    from paper_1411_3212_b200 import QosParams, check_latency, min_bandwidth
    from paper_1411_3212_b200.errors import BadQos

    assert check_latency(1.0, QosParams(1.0, 2.0, 1))  # test_acceptance.py:466-494
    assert not check_latency(1.5, QosParams(1.0, 2.0, 1))
    assert min_bandwidth(QosParams(1.0, 3.0, 500)) == 250.0
    with pytest.raises(BadQos):
        min_bandwidth(QosParams(1.0, 1.0, 10))


def test_result_set_lines_and_merge():
    from paper_1411_3212_b200 import ColumnarResult, ResultSet
    from paper_1411_3212_b200.errors import DuplicateResult

    assert ResultSet({3: [1, 2], 1: []}).lines() == ["1:", "3: 1,2"]  # test_decode.py:114-116
    r = ColumnarResult(np.array([7, 8, 7]), np.array([0, 1, 1, 3]), np.array([5, 2, 9]))
    assert r.to_result_set().by_query == {7: [2, 5, 9], 8: []}
    r = ColumnarResult(np.array([1, 1]), np.array([0, 1, 2]), np.array([4, 4]))
    with pytest.raises(DuplicateResult):
        r.to_result_set()


def test_rect_validation():
    from paper_1411_3212_b200 import Rect

    with pytest.raises(ValueError):
        Rect(1.0, 0.0, 0.0, 1.0)


def test_multi_gpu_entry_points_without_a_device():
    """NCCL is loaded at run time (no link-time dependency): a unique id can be made on any
    host, and the in-process group used for one-device runs of the sharded tick is plain host
    state."""
    from paper_1411_3212_b200 import _native

    uid = _native.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    assert uid != _native.nccl_unique_id()  # a fresh id per call
    g = _native.LocalGroup(3)
    assert g.nranks == 3
    g.close()
