"""PRIEST / CEM device kernels vs golden rounds of the live reference (teacher-forced per round).

Contract (SURVEY.md §8(c) tiers 1 and 4): the projection is fed the reference round's own
standard normals z, mean and covariance; projected coefficients match to 1e-10 relative and
scores to 1e-9 relative (absolute 1e-11 for feasible samples, whose reference scores are
rounding noise ~1e-15 while the device's trig-free targets give exact zeros); costs, elite
selection and the refit are checked given identical inputs (top-k bit-exact).
"""

import numpy as np
import pytest
import torch

from oracle import priest as OP
from paper_2408_10731_b200 import solver_priest as SP
from paper_2408_10731_b200.basis import AxisBoundary, BasisSet, TimeGrid
from paper_2408_10731_b200.geometry import EllipsoidShape, ObstacleTrack

pytestmark = pytest.mark.gpu


def setup_from(g, tag):
    P = g[f"{tag}_P"]
    ts = np.linspace(0.0, 10.0, P.shape[0])
    basis = BasisSet(grid=TimeGrid(0.0, 10.0, P.shape[0], ts), degree=P.shape[1] - 1, P=P, Pdot=g[f"{tag}_Pd"],
                     Pddot=g[f"{tag}_Pdd"])
    bv = g[f"{tag}_bvals"]
    bnd = tuple(AxisBoundary(*bv[k]) for k in range(bv.shape[0]))
    tr = g[f"{tag}_tracks"]
    obs = [ObstacleTrack(tr[j], EllipsoidShape(float(g[f"{tag}_a"][j]), float(g[f"{tag}_b"][j])))
           for j in range(tr.shape[0])]
    lims = g[f"{tag}_lims"]
    return SP.ProjectionSetup(basis, bnd, obs, float(lims[0]), float(lims[1]), g[f"{tag}_smin"], g[f"{tag}_smax"],
                              float(lims[2]))


def close_scores(dev, ref):
    np.testing.assert_allclose(dev, ref, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("tag,rounds", [("p3", 3), ("p2", 2)])
def test_projection_teacher_forced(golden, tag, rounds):
    g = golden("priest.npz")
    st = setup_from(g, tag)
    for r in range(rounds):
        mu, S = g[f"{tag}_r{r}_mu_in"], g[f"{tag}_r{r}_sigma_in"]
        samples = mu + g[f"{tag}_r{r}_z"] @ OP.draw_transform(mu, S).T
        out = SP.project(st, samples, n_inner=30)
        xi = np.stack([p.projected for p in out])
        ref = g[f"{tag}_r{r}_xi"]
        assert np.max(np.abs(xi - ref)) <= 1e-10 * np.max(np.abs(ref))
        close_scores(np.array([p.residual for p in out]), g[f"{tag}_r{r}_scores"])


def test_fused_draw_matches_numpy_sampler(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    d = st.device()
    mu, S = g["p3_r1_mu_in"], g["p3_r1_sigma_in"]
    d["L"].copy_(torch.as_tensor(SP._draw_factor(S)))
    d["mu"].copy_(torch.as_tensor(mu))
    z = torch.as_tensor(g["p3_r1_z"], device="cuda")
    xi, _, _, _ = SP._run_project(st, z=z, n_inner=-1)
    ref = mu + g["p3_r1_z"] @ OP.draw_transform(mu, S).T
    np.testing.assert_allclose(xi.cpu().numpy(), ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_residual_history_and_scores_only(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    ref = g["p3_r0_xi"]
    close_scores(SP.residual_scores(st, ref), g["p3_r0_scores"])
    mu, S = g["p3_r0_mu_in"], g["p3_r0_sigma_in"]
    samples = mu + g["p3_r0_z"][:16] @ OP.draw_transform(mu, S).T
    hist = []
    SP.project(st, samples, n_inner=5, residual_history=hist)
    oh = []
    OP.project(OP.make_setup(g["p3_P"], g["p3_Pd"], g["p3_Pdd"], g["p3_bvals"], g["p3_tracks"], g["p3_a"], g["p3_b"],
                             3.0, 3.0, g["p3_smin"], g["p3_smax"], 1.0), samples, 5, history=oh)
    assert len(hist) == 5
    for a, b in zip(hist, oh):
        close_scores(a, b)


@pytest.mark.parametrize("tag", ["p3", "p2"])
def test_costs_selection_and_refit_given_reference_inputs(golden, tag):
    g = golden("priest.npz")
    st = setup_from(g, tag)
    N, n_ce, n_el, n_inner, sigma, gamma, w = g[f"{tag}_params"]
    dev = torch.device("cuda")
    xi = torch.as_tensor(g[f"{tag}_r0_xi"], device=dev)
    scores = torch.as_tensor(g[f"{tag}_r0_scores"], device=dev)
    # keep = stable argsort of the reference scores: bit-exact given identical keys
    keep = SP._topk(scores, int(n_ce))
    np.testing.assert_array_equal(keep.cpu().numpy(), g[f"{tag}_r0_keep"])
    # aug costs of the reference keep set: barn cost + residual weight * score
    dim = 3 if tag == "p3" else 2
    c1 = SP.BarnCost(np.zeros(dim), np.r_[12.0, np.zeros(dim - 1)])
    aug = SP._run_cost(st, xi, keep, scores, 1.0, float(w), 0.0, c1.line(dev))
    np.testing.assert_allclose(aug.cpu().numpy(), g[f"{tag}_r0_aug"], rtol=1e-11)
    # elites: stable top-k over the reference aug costs (residual-rank order on ties)
    ref_aug = torch.as_tensor(g[f"{tag}_r0_aug"], device=dev)
    erank = SP._topk(ref_aug, int(n_el))
    np.testing.assert_array_equal(keep[erank].cpu().numpy(), g[f"{tag}_r0_elites"])
    # weighted refit given the reference elites and costs
    mu, S = SP.update_distribution(g[f"{tag}_r0_mu_in"], g[f"{tag}_r0_sigma_in"], g[f"{tag}_r0_xi"][g[f"{tag}_r0_elites"]],
                                   ref_aug[erank].cpu().numpy(), sigma, gamma)
    np.testing.assert_allclose(mu, g[f"{tag}_r0_mu"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(S, g[f"{tag}_r0_sigma"], rtol=1e-10, atol=1e-14)


def test_cem_penalty_matches_reference(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    xi = torch.as_tensor(g["p3_r0_xi"], device="cuda")
    pen = SP._run_cost(st, xi, None, None, 0.0, 0.0, 1.0, st.device()["line"])
    np.testing.assert_allclose(pen.cpu().numpy(), g["p3_cem_penalty0"], rtol=1e-11, atol=1e-12)


def test_priest_optimize_end_to_end_is_deterministic_and_feasible(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    params = SP.PriestParams(n_outer=3, n_batch=96, n_constraint_elite=48, n_elite=12, n_inner=30, seed=0)
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    r1 = SP.priest_optimize(st, c1, dist, params)
    r2 = SP.priest_optimize(st, c1, dist, params)
    np.testing.assert_array_equal(r1.mu, r2.mu)
    np.testing.assert_array_equal(r1.sigma_mat, r2.sigma_mat)
    assert len(r1.history) == 3
    # round 0 sees the reference's exact samples: the best feasible sample's cost level agrees
    ref0 = g["p3_best_hist"][0]
    assert abs(r1.history[0]["min_residual"] - ref0[2]) <= 1e-9 * max(ref0[2], 1.0) + 1e-11
    assert r1.best.residual <= max(g["p3_best_hist"][:, 1].max(), 1e-6) * 10
    # a plain-callable c1 takes the host path and must agree with the device cost object
    r3 = SP.priest_optimize(st, lambda tr: c1(tr), dist, SP.PriestParams(n_outer=1, n_batch=96, n_constraint_elite=48,
                                                                        n_elite=12, n_inner=30, seed=0))
    np.testing.assert_allclose(r3.history[0]["best_aug_cost"], r1.history[0]["best_aug_cost"], rtol=1e-10)


def test_cem_optimize_runs_and_refits(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    res = SP.cem_optimize(st, c1, dist, SP.CemParams(n_batch=96, n_elite=12, iterations=2, seed=3))
    # same standard normals, same costs up to rounding -> same first-iteration best
    np.testing.assert_allclose(res.history[0]["best_cost"], g["p3_cem_hist"][0][0], rtol=1e-9)
    np.testing.assert_allclose(res.history[0]["mean_cost"], g["p3_cem_hist"][0][1], rtol=1e-9)


@pytest.mark.parametrize("degree,dim", [(7, 3), (8, 2), (10, 2)])
def test_generic_paths_vs_oracle(degree, dim):
    """Runtime-m (degree 7), M=9 and moving obstacles (non-static tracks) against the oracle."""
    from paper_2408_10731_b200.basis import build_basis

    n_p = 50
    basis = build_basis(0.0, 8.0, n_p, degree)
    rng = np.random.default_rng(degree)
    ts = basis.grid.timestamps
    obs = []
    for _ in range(6):
        c = np.r_[rng.uniform(2, 6), rng.uniform(-1, 1), rng.uniform(-0.5, 0.5)][:dim]
        v = np.r_[rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 0.0][:dim]
        obs.append(ObstacleTrack(c[None, :] + v[None, :] * ts[:, None], EllipsoidShape(0.7, 0.5)))
    bnd = tuple(AxisBoundary(p0=0.0, v0=1.0, p1=8.0) if k == 0 else AxisBoundary(p0=0.0, p1=0.0) for k in range(dim))
    smin, smax = np.full(dim, -3.0), np.full(dim, 10.0)
    st = SP.ProjectionSetup(basis, bnd, obs, 2.5, 3.0, smin, smax, 1.0)
    assert not st.static_tracks
    ost = OP.make_setup(basis.P, basis.Pdot, basis.Pddot, np.stack([b.values() for b in bnd]),
                        np.stack([o.centers for o in obs]), np.full(6, 0.7), np.full(6, 0.5), 2.5, 3.0, smin, smax,
                        1.0)
    samples = rng.normal(size=(40, dim * (degree + 1))) * 2.0
    out = SP.project(st, samples, n_inner=12)
    xi_ref, sc_ref = OP.project(ost, samples, 12, mode="kinv")
    xi = np.stack([p.projected for p in out])
    assert np.max(np.abs(xi - xi_ref)) <= 1e-10 * np.max(np.abs(xi_ref))
    close_scores(np.array([p.residual for p in out]), sc_ref)


@pytest.mark.parametrize("n_ce", [48, 20])
def test_sharded_rounds_are_bitwise_the_single_gpu_rounds(golden, n_ce):
    """Multi-GPU PRIEST semantics on one GPU: 3 sample shards run their local phase (projection + local
    stable top-k), their candidate rows are concatenated in rank order exactly as the all-gather
    delivers them, and the replicated global phase (keep set, costs, elites, refit) reproduces the
    single-GPU priest_optimize bit for bit.  n_ce 20 < shard size exercises the local pre-selection."""
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    params = SP.PriestParams(n_outer=3, n_batch=96, n_constraint_elite=n_ce, n_elite=12, n_inner=30, seed=0)
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    ref = SP.priest_optimize(st, c1, dist, params)
    rng = np.random.default_rng(params.seed)
    z_rounds = [rng.standard_normal((params.n_batch, dist.mu.size)) for _ in range(params.n_outer)]
    d = st.device()
    mu = torch.as_tensor(dist.mu.copy(), device="cuda")
    sig = torch.as_tensor(dist.sigma_mat.copy(), device="cuda")
    rnd = SP.ShardedRound(st, c1, params)
    hist = []
    for r in range(params.n_outer):
        d["L"].copy_(torch.as_tensor(SP._draw_factor(sig.cpu().numpy())))
        d["mu"].copy_(mu)
        parts = [rnd.local(torch.as_tensor(z_rounds[r][lo:lo + 32], device="cuda").contiguous(), lo)
                 for lo in (0, 32, 64)]
        out = rnd.global_(torch.cat(parts), mu, sig)
        hist.append(out["entry"])
    np.testing.assert_array_equal(mu.cpu().numpy(), ref.mu)
    np.testing.assert_array_equal(sig.cpu().numpy(), ref.sigma_mat)
    np.testing.assert_array_equal(np.array(hist), np.array([[h["best_aug_cost"], h["best_residual"],
                                                             h["min_residual"]] for h in ref.history]))
    one = SP.priest_optimize_sharded(st, c1, dist, params)  # the entry point, world size 1
    np.testing.assert_array_equal(one.mu, ref.mu)
    np.testing.assert_array_equal(one.best.projected, ref.best.projected)
    np.testing.assert_array_equal(one.best.original, ref.best.original)


def test_pinned_host_normals_match_device_normals(golden):
    """z_rounds from pinned host memory (asynchronous per-round upload, solver_priest._z_round), from
    numpy and from the device give the same rounds bit for bit."""
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    dist = SP.SamplingDistribution(g["p3_mu0"], g["p3_sigma0"])
    params = SP.PriestParams(n_outer=3, n_batch=96, n_constraint_elite=48, n_elite=12, n_inner=30, seed=0)
    c1 = SP.BarnCost(np.zeros(3), np.array([12.0, 0.0, 0.0]))
    z = np.random.default_rng(7).standard_normal((params.n_outer, params.n_batch, dist.mu.size))
    runs = [SP.priest_optimize(st, c1, dist, params, z_rounds=zr)
            for zr in (torch.as_tensor(z, device="cuda"), torch.as_tensor(z).pin_memory(), z)]
    for r in runs[1:]:
        np.testing.assert_array_equal(r.mu, runs[0].mu)
        np.testing.assert_array_equal(r.sigma_mat, runs[0].sigma_mat)
        np.testing.assert_array_equal(r.best.projected, runs[0].best.projected)
        assert r.history == runs[0].history
