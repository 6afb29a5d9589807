"""numpy <-> device transfers of the drop-in API (_native.to_device / to_host):
large vectors go through the pinned staging path in chunks; results must be
bitwise the input, whatever the size (chunk remainders) or the call order."""

import numpy as np
import pytest

from paper_2006_12883_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [N._STAGE_MIN_BYTES // 8 - 1, N._STAGE_MIN_BYTES // 8,
                               3 * N._STAGE_CHUNK + 17])
def test_staged_round_trip_bitwise(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n)
    d = N.to_device(a)
    assert d.is_cuda and d.numel() == n
    back = N.to_host(d)
    assert isinstance(back, np.ndarray)
    np.testing.assert_array_equal(back, a)
    # the staging buffer is reused: a second, different vector must not see the first
    b = -a[::-1].copy()
    np.testing.assert_array_equal(N.to_host(N.to_device(b)), b)
    np.testing.assert_array_equal(back, a)


def test_staged_path_matches_pageable(monkeypatch):
    a = np.random.default_rng(1).standard_normal(2 * N._STAGE_CHUNK + 5)
    staged = N.to_host(N.to_device(a))
    monkeypatch.setenv("PD_STAGED_IO", "0")
    np.testing.assert_array_equal(N.to_host(N.to_device(a)), staged)
