"""Outputs of host-array calls without ``out=`` come from the library's page-locked pool
(batch._PinnedPool): they are page-locked (the D2H copies land in them directly), blocks
are recycled once a result is dropped, and the results are bit-identical to the
caller-allocated ``out=`` route."""

import numpy as np
import pytest

import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _lib, batch, workloads

pytestmark = pytest.mark.gpu


def _locked(a) -> bool:
    return _lib.lib().fn_host_is_page_locked(a.ctypes.data) == 1


def _bits(a):
    return np.asarray(a).view(np.uint64 if np.asarray(a).dtype == np.float64 else np.uint32)


def test_default_outputs_are_page_locked_and_recycled():
    p = fn.preset("double")
    x = workloads.host_rows(5, 0, 1 << 20)
    r0 = np.empty(1 << 20)
    u0 = np.empty((1 << 20, 3))
    fn.normalize3(p, x, out=(r0, u0))
    res = fn.normalize3(p, x)
    assert _locked(res.unit) and _locked(res.length)
    assert np.array_equal(_bits(res.length), _bits(r0)) and np.array_equal(_bits(res.unit), _bits(u0))
    del res
    pool = batch.pinned_pool
    allocs = pool.allocs
    reuses = pool.reuses
    for _ in range(5):
        res = fn.normalize3(p, x)
        assert np.array_equal(_bits(res.unit), _bits(u0))
        del res
    assert pool.allocs == allocs and pool.reuses == reuses + 10  # r and unit, five times


def test_views_keep_blocks_alive():
    p = fn.preset("double")
    x = workloads.host_rows(5, 0, 1 << 18)
    res = fn.normalize3(p, x)
    view = res.unit[:, 1]
    want = view.copy()
    del res
    for _ in range(3):  # other calls must not reuse the block the view still points into
        fn.normalize3(p, x + 1.0)
    assert np.array_equal(_bits(view), _bits(want))


def test_pool_off_gives_pageable_outputs():
    p = fn.preset("single")
    x = workloads.host_rows(4, 0, 1 << 18)
    pool = batch.pinned_pool
    saved = pool._limit
    try:
        pool._limit = 0
        res = fn.normalize3(p, x)
        assert not _locked(res.unit)
    finally:
        pool._limit = saved
    res2 = fn.normalize3(p, x)
    assert _locked(res2.unit)
    assert np.array_equal(_bits(res.unit), _bits(res2.unit)) and np.array_equal(_bits(res.length), _bits(res2.length))


def test_soa_and_rotation_outputs_from_pool():
    p = fn.preset("double")
    x = workloads.host_rows(5, 0, 1 << 17)
    cols = [np.ascontiguousarray(x[:, k]) for k in range(3)]
    soa = fn.normalize3(p, *cols)
    aos = fn.normalize3(p, x)
    assert _locked(soa.length)
    assert np.array_equal(_bits(soa.length), _bits(aos.length))
    for k in range(3):
        assert np.array_equal(_bits(soa.unit[k]), _bits(aos.unit[:, k]))
