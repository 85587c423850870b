"""Accuracy of the kernels' XU-light elementary functions (fastmath.cuh) against numpy."""

import numpy as np
import pytest
import torch

from paper_2408_10731_b200 import _lib

pytestmark = pytest.mark.gpu


def ev(fn, x, y=None):
    lib = _lib.load()
    dx = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")
    dy = torch.as_tensor(np.ascontiguousarray(y, dtype=np.float64), device="cuda") if y is not None else None
    out = torch.empty_like(dx)
    rc = lib.tro_fastmath_eval(fn, dx.data_ptr(), dy.data_ptr() if dy is not None else None, dx.numel(),
                               out.data_ptr(), _lib.stream_handle())
    _lib.check(rc, "tro_fastmath_eval")
    return out.cpu().numpy()


def ulps(a, b):
    return np.max(np.abs(a - b) / np.spacing(np.maximum(np.abs(b), 1e-300)))


def test_sincos_on_angle_range():
    x = np.concatenate([np.linspace(-np.pi, np.pi, 200001), [0.0, -0.0, np.pi, -np.pi, np.pi / 2, 1e-300, 3e4]])
    assert np.max(np.abs(ev(0, x) - np.sin(x))) <= 2.3e-16
    assert np.max(np.abs(ev(1, x) - np.cos(x))) <= 2.3e-16
    big = np.array([2e5, -7.5e6, 1e300])
    np.testing.assert_allclose(ev(0, big), np.sin(big), atol=1e-15)


def test_atan2_quadrants_and_zeros():
    rng = np.random.default_rng(0)
    y = rng.normal(size=200000) * np.exp(rng.normal(size=200000) * 3)
    x = rng.normal(size=200000) * np.exp(rng.normal(size=200000) * 3)
    assert np.max(np.abs(ev(2, x, y) - np.arctan2(y, x))) <= 4.5e-16
    zs = np.array([0.0, -0.0, 0.0, -0.0, 1.0, -1.0, 0.0, -0.0])
    zx = np.array([0.0, 0.0, -0.0, -0.0, 0.0, 0.0, 1.0, -1.0])
    np.testing.assert_array_equal(ev(2, zx, zs), np.arctan2(zs, zx))


def test_reciprocal_sqrt_family():
    rng = np.random.default_rng(1)
    v = np.exp(rng.uniform(-30, 30, size=200000))
    assert ulps(ev(3, v), 1.0 / v) <= 1.0
    assert ulps(ev(4, v), 1.0 / np.sqrt(v)) <= 2.0
    assert ulps(ev(5, v), np.sqrt(v)) <= 1.0


def test_unit_direction_matches_cos_sin_of_atan2():
    rng = np.random.default_rng(2)
    c, s = rng.normal(size=100000), rng.normal(size=100000)
    a = np.arctan2(s, c)
    assert np.max(np.abs(ev(6, c, s) - np.cos(a))) <= 4.5e-16
    assert np.max(np.abs(ev(7, c, s) - np.sin(a))) <= 4.5e-16


def test_los_scale_clamps():
    q = np.array([0.0, 0.25, 1.0, 1.0 + 1e-15, 4.0, 1e12, 2e12, 1e20])
    ref = np.minimum(np.maximum(1.0, np.sqrt(q)), 1e6)
    np.testing.assert_array_equal(ev(8, q), ref)
