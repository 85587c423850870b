"""The receding-horizon oracle (oracle/mpc.py) against the live reference's receding_horizon_run
(tests/golden/mpc.npz).  CPU only."""

import os

import numpy as np
import pytest

from oracle import mpc as omp
from paper_2408_10731_b200.basis import build_basis
from paper_2408_10731_b200.bench.scenarios import gen_scenario, obstacle_arrays

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mpc.npz")

CASES = {  # tag: (kind, params, seed, receding_horizon_run kwargs) — as make_golden.make_mpc
    "s3": ("random-static", {"dim": 3, "n_o": 6}, 2, dict(step_budget=25, n_steps=12)),
    "f2": ("dynamic-flow", {"n_o": 6}, 4, dict(step_budget=20, n_steps=14, exec_fraction=0.3, goal_radius=1.0)),
    "r2": ("random-static", {"n_o": 5}, 1, dict(step_budget=30, n_steps=10, exec_fraction=0.5, goal_radius=3.0)),
}


def oracle_run(tag, starts=None, goals=None):
    kind, params, seed, kw = CASES[tag]
    sc = gen_scenario(kind, params, seed=seed)
    b = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
    c, v, a, bb = obstacle_arrays(sc)
    starts = [sc.boundary.start] if starts is None else starts
    goals = [sc.boundary.goal] if goals is None else goals
    return sc, omp.run(b.P, b.Pdot, b.Pddot, b.grid.timestamps, c, v, a, bb, starts, goals, **kw)


@pytest.mark.parametrize("tag", sorted(CASES))
def test_oracle_mpc_matches_reference(tag):
    g = np.load(GOLD)
    _, out = oracle_run(tag)
    flags = g[f"{tag}_flags"]  # success, reached, collided
    assert bool(out.flags[0] == 2) == bool(flags[1]) and bool(out.flags[0] == 1) == bool(flags[2])
    np.testing.assert_array_equal(out.traces[0], g[f"{tag}_pos"])
    np.testing.assert_array_equal(out.times[0], g[f"{tag}_t"])
    rec = g[f"{tag}_records"]
    assert len(out.metrics[0]) == rec.shape[0]
    m = np.array(out.metrics[0])
    np.testing.assert_array_equal(m[:, [0, 1, 2, 4]], rec[:, :4])  # smoothness, tracking, arc, clearance
    np.testing.assert_array_equal(np.array(out.residuals[0]), rec[:, 4])


def test_oracle_mpc_fleet_members_independent():
    """A fleet of robots equals each robot driven alone (lockstep clock, shared tracks)."""
    sc = gen_scenario("random-static", {"dim": 3, "n_o": 6}, seed=2)
    rng = np.random.default_rng(0)
    starts = np.array(sc.boundary.start)[None] + rng.uniform(-0.3, 0.3, (3, 3)) * np.array([0, 1, 1])
    goals = np.array(sc.boundary.goal)[None] + rng.uniform(-0.3, 0.3, (3, 3)) * np.array([0, 1, 1])
    _, fleet = oracle_run("s3", starts, goals)
    for i in range(3):
        _, one = oracle_run("s3", starts[i:i + 1], goals[i:i + 1])
        np.testing.assert_array_equal(fleet.traces[i], one.traces[0])
        np.testing.assert_array_equal(np.array(fleet.metrics[i]), np.array(one.metrics[0]))
