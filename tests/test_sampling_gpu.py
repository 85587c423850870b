"""Throughput-mode sampling for PRIEST / CEM (SURVEY.md §8(e) "per-sample Philox counters keyed by global
index") and the refit's numpy edge-case semantics.

Philox normals are not numpy's stream (parity mode keeps the Generator draws, tests/test_priest_gpu.py), so
they are checked statistically and structurally: moments, determinism, shard independence (sample s is the
same whichever shard draws it), round independence; the Cholesky draw factor reproduces the covariance; a
throughput-mode priest_optimize / cem_optimize is deterministic and reaches the parity-mode cost level.
"""

import numpy as np
import pytest
import torch

from oracle import priest as OP
from paper_2408_10731_b200 import _lib
from paper_2408_10731_b200 import solver_priest as SP
from test_priest_gpu import setup_from

pytestmark = pytest.mark.gpu


def test_philox_normals_moments_determinism_and_shards():
    n, d = 16384, 33
    z = SP.device_normals(7, 0, n, d).cpu().numpy()
    assert z.shape == (n, d) and np.isfinite(z).all()
    assert abs(z.mean()) < 5.0 / np.sqrt(n * d)
    assert abs(z.var() - 1.0) < 0.01
    # kurtosis of a normal is 3; tail mass beyond 3 sigma 0.27 %
    assert abs(np.mean(z**4) - 3.0) < 0.05
    assert abs(np.mean(np.abs(z) > 3.0) - 0.0027) < 0.0006
    # pairs (Box-Muller siblings) are uncorrelated
    assert abs(np.corrcoef(z[:, 0], z[:, 1])[0, 1]) < 0.03
    np.testing.assert_array_equal(z, SP.device_normals(7, 0, n, d).cpu().numpy())
    # shard [5000, 9000) draws exactly rows 5000..8999 of the full batch
    np.testing.assert_array_equal(SP.device_normals(7, 0, 4000, d, first=5000).cpu().numpy(), z[5000:9000])
    other = SP.device_normals(7, 1, n, d).cpu().numpy()
    assert abs(np.corrcoef(z.ravel(), other.ravel())[0, 1]) < 0.01  # another round: another stream


def test_cholesky_draw_factor():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((33, 40))
    S = A @ A.T / 40 + 1e-3 * np.eye(33)
    dev = torch.device("cuda")
    L = torch.empty((33, 33), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().tro_cholesky_f64(torch.as_tensor(S, device=dev).data_ptr(), 33, L.data_ptr(), None), "chol")
    Lh = L.cpu().numpy()
    assert np.allclose(np.triu(Lh, 1), 0.0)
    np.testing.assert_allclose(Lh @ Lh.T, S, rtol=0, atol=1e-13 * np.abs(S).max())
    np.testing.assert_allclose(Lh, np.linalg.cholesky(S), rtol=1e-12, atol=1e-14)
    # rank-deficient PSD: zero columns, L L' still equals the matrix
    B = rng.standard_normal((33, 10))
    S2 = B @ B.T
    _lib.check(_lib.load().tro_cholesky_f64(torch.as_tensor(S2, device=dev).data_ptr(), 33, L.data_ptr(), None),
               "chol")
    L2 = L.cpu().numpy()
    assert np.isfinite(L2).all()
    np.testing.assert_allclose(L2 @ L2.T, S2, atol=1e-9 * np.abs(S2).max())


def test_priest_throughput_mode(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    params = SP.PriestParams(n_outer=3, n_batch=512, n_constraint_elite=256, n_elite=32, n_inner=30, seed=3)
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    r1 = SP.priest_optimize(st, c1, dist, params, sampler="philox")
    r2 = SP.priest_optimize(st, c1, dist, params, sampler="philox")
    np.testing.assert_array_equal(r1.mu, r2.mu)
    np.testing.assert_array_equal(r1.sigma_mat, r2.sigma_mat)
    assert len(r1.history) == 3 and all(np.isfinite(h["best_aug_cost"]) for h in r1.history)
    rn = SP.priest_optimize(st, c1, dist, params)  # parity mode, same recipe
    # same distribution of samples: the rounds reach the same cost level (within 25 %)
    a, b = r1.history[-1]["best_aug_cost"], rn.history[-1]["best_aug_cost"]
    assert abs(a - b) <= 0.25 * abs(b) + 1e-9
    assert np.all(np.linalg.eigvalsh(r1.sigma_mat) > -1e-12)
    with pytest.raises(ValueError):
        SP.priest_optimize(st, c1, dist, params, sampler="mt19937")


def test_cem_throughput_mode(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    params = SP.CemParams(iterations=3, n_batch=512, n_elite=32, seed=1)
    r1 = SP.cem_optimize(st, c1, dist, params, sampler="philox")
    r2 = SP.cem_optimize(st, c1, dist, params, sampler="philox")
    np.testing.assert_array_equal(r1.mu, r2.mu)
    assert np.isfinite(r1.best_cost)


@pytest.mark.parametrize("gamma", [-1.0, 0.0, 2.5])
def test_update_distribution_edge_cases_follow_numpy(gamma):
    """gamma == 0 is numpy's exp(x / 0) (inf / NaN weights), not a CEM switch; a NaN cost propagates through
    min() like np.min."""
    rng = np.random.default_rng(4)
    mu, S = rng.standard_normal(9), np.eye(9)
    X, c = rng.standard_normal((16, 9)), rng.uniform(0, 3, 16)
    with np.errstate(all="ignore"):
        ref_mu, ref_S = OP.update_distribution(mu, S, X, c, 0.7, gamma)
        got_mu, got_S = SP.update_distribution(mu, S, X, c, 0.7, gamma)
    np.testing.assert_allclose(got_mu, ref_mu, rtol=1e-12, atol=1e-14, equal_nan=True)
    np.testing.assert_array_equal(np.isnan(got_S), np.isnan(ref_S))
    c2 = c.copy()
    c2[5] = np.nan
    with np.errstate(all="ignore"):
        ref_mu, _ = OP.update_distribution(mu, S, X, c2, 0.7, gamma)
        got_mu, _ = SP.update_distribution(mu, S, X, c2, 0.7, gamma)
    np.testing.assert_array_equal(np.isnan(got_mu), np.isnan(ref_mu))
