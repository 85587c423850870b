"""Pin the PRIEST / CEM oracle (oracle/priest.py) against golden vectors of the live reference."""

import numpy as np
import pytest

from oracle import priest as OP


def setup_from(g, tag):
    lims = g[f"{tag}_lims"]
    return OP.make_setup(g[f"{tag}_P"], g[f"{tag}_Pd"], g[f"{tag}_Pdd"], g[f"{tag}_bvals"], g[f"{tag}_tracks"],
                         g[f"{tag}_a"], g[f"{tag}_b"], float(lims[0]), float(lims[1]), g[f"{tag}_smin"],
                         g[f"{tag}_smax"], float(lims[2]))


def barn_c1(dim):
    start = np.zeros(dim)
    goal = np.zeros(dim)
    goal[0] = 12.0
    return lambda pos, vel, acc: OP.barn_cost(pos, vel, acc, start, goal)


@pytest.mark.parametrize("tag,dim,rounds", [("p3", 3, 3), ("p2", 2, 2)])
def test_priest_rounds_bitexact(golden, tag, dim, rounds):
    g = golden("priest.npz")
    st = setup_from(g, tag)
    N, n_ce, n_el, n_inner, sigma, gamma, w = g[f"{tag}_params"]
    for r in range(rounds):
        out = OP.priest_round(st, g[f"{tag}_r{r}_z"], g[f"{tag}_r{r}_mu_in"], g[f"{tag}_r{r}_sigma_in"], int(n_ce),
                              int(n_el), int(n_inner), sigma, gamma, w, barn_c1(dim))
        np.testing.assert_array_equal(out["xi_bar"], g[f"{tag}_r{r}_xi"])
        np.testing.assert_array_equal(out["scores"], g[f"{tag}_r{r}_scores"])
        np.testing.assert_array_equal(out["keep"], g[f"{tag}_r{r}_keep"])
        np.testing.assert_array_equal(out["aug"], g[f"{tag}_r{r}_aug"])
        np.testing.assert_array_equal(out["elites"], g[f"{tag}_r{r}_elites"])
        np.testing.assert_array_equal(out["mu"], g[f"{tag}_r{r}_mu"])
        np.testing.assert_array_equal(out["sigma_mat"], g[f"{tag}_r{r}_sigma"])


def test_cem_penalty_matches(golden):
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    np.testing.assert_array_equal(OP.cem_penalty(st, g["p3_r0_xi"]), g["p3_cem_penalty0"])


def test_kinv_projection_twin_is_close(golden):
    """The device's K^-1 contraction vs the reference LU: 1e-12 over 30 inner iterations."""
    g = golden("priest.npz")
    st = setup_from(g, "p3")
    samples = g["p3_r0_mu_in"] + g["p3_r0_z"] @ OP.draw_transform(g["p3_r0_mu_in"], g["p3_r0_sigma_in"]).T
    xi_k, _ = OP.project(st, samples, 30, mode="kinv")
    assert np.max(np.abs(xi_k - g["p3_r0_xi"])) <= 1e-11 * np.max(np.abs(g["p3_r0_xi"]))
