"""Scenario -> solver-problem adapters (reference bench/runner.py:59-161).

Each adapter builds this package's device-backed problem from a ``Scenario``: the straight start->goal desired
path, the scenario's boundary points, and the obstacle tracks predicted on the basis grid with the semi-axes
inflated by the 5 cm planning margin.  ``fleet_batch_from_scenario`` is the batched form: B robots in one
obstacle field as ONE ``SingleBatch`` (tracks shared, boundaries and desired lines per robot).
"""

from __future__ import annotations

import numpy as np

from .. import solver_batch, solver_multiagent, solver_priest, solver_single
from ..basis import AxisBoundary, straight_line_coeffs
from ..geometry import EllipsoidShape, ObstacleTrack
from .scenarios import Scenario, agent_boundaries, predict_obstacles

__all__ = ["PLAN_MARGIN", "desired_line", "planning_tracks", "single_problem_from_scenario",
           "fleet_batch_from_scenario", "batch_problem_from_scenario", "priest_setup_from_scenario",
           "multiagent_problem_from_scenario", "default_sampling_distribution", "barn_cost_fn"]

PLAN_MARGIN = 0.05


def _ends(scenario: Scenario):
    return np.asarray(scenario.boundary.start, dtype=float), np.asarray(scenario.boundary.goal, dtype=float)


def desired_line(start, goal, n_p: int) -> np.ndarray:
    """start + s (goal - start) at s = linspace(0, 1, n_p) (runner.py:59-63, 369-370)."""
    start, goal = np.asarray(start, dtype=float), np.asarray(goal, dtype=float)
    return start[None, :] + np.linspace(0.0, 1.0, n_p)[:, None] * (goal - start)[None, :]


def _point_boundary(scenario: Scenario) -> tuple:
    s, g = scenario.boundary.start, scenario.boundary.goal
    return tuple(AxisBoundary(p0=s[k], p1=g[k]) for k in range(scenario.dim))


def planning_tracks(scenario: Scenario, timestamps, margin: float = PLAN_MARGIN, t_now: float = 0.0) -> list:
    """Predicted tracks, semi-axes inflated by the planning margin so converged plans clear the raw
    geometry strictly (runner.py:88-101)."""
    tracks = predict_obstacles(scenario, timestamps, t_now=t_now)
    if margin == 0.0:
        return tracks
    grow = lambda sh: EllipsoidShape(sh.a + margin, sh.b + margin)  # noqa: E731
    return [ObstacleTrack(centers=tr.centers, shape=grow(tr.shape)) for tr in tracks]


def single_problem_from_scenario(scenario: Scenario, basis, plan_margin: float = PLAN_MARGIN):
    s, g = _ends(scenario)
    return solver_single.SingleProblem(basis=basis, boundary=_point_boundary(scenario),
                                       desired=desired_line(s, g, basis.n_p),
                                       obstacles=planning_tracks(scenario, basis.grid.timestamps, plan_margin))


def fleet_batch_from_scenario(scenario: Scenario, basis, starts, goals, plan_margin: float = PLAN_MARGIN):
    """B robots (starts / goals (B, dim)) in one scenario's obstacle field -> one SingleBatch; solve it with
    solver_single.solve_single_batch."""
    starts = np.atleast_2d(np.asarray(starts, dtype=float))
    goals = np.atleast_2d(np.asarray(goals, dtype=float))
    bvals = np.zeros(starts.shape + (6,))
    bvals[..., 0], bvals[..., 3] = starts, goals
    return solver_single.SingleBatch(basis=basis, bvals=bvals,
                                     obstacles=planning_tracks(scenario, basis.grid.timestamps, plan_margin))


def batch_problem_from_scenario(scenario: Scenario, basis, n_batch: int = 100, plan_margin: float = PLAN_MARGIN):
    """Alg. 2 problem: heading boundary = the start->goal direction, the robot's footprint circles."""
    if scenario.dim != 2:
        raise ValueError("the batch solver is planar")
    s, g = _ends(scenario)
    psi = float(np.arctan2(g[1] - s[1], g[0] - s[0]))
    robot = scenario.robot
    return solver_batch.BatchProblem(
        basis=basis, boundary=_point_boundary(scenario), psi_boundary=(psi, psi),
        desired=desired_line(s, g, basis.n_p),
        obstacles=planning_tracks(scenario, basis.grid.timestamps, plan_margin),
        footprint=solver_batch.FootprintSpec(offsets=tuple(robot.footprint_offsets) or (0.0,)),
        v_max=robot.v_max, a_max=robot.a_max, n_batch=n_batch)


def priest_setup_from_scenario(scenario: Scenario, basis, rho: float = 1.0, plan_margin: float = PLAN_MARGIN):
    """PRIEST projection: workspace box = the bounding box of start, goal and obstacle centres, padded 4 m."""
    pts = np.asarray([scenario.boundary.start, scenario.boundary.goal] + [o.center for o in scenario.obstacles],
                     dtype=float)
    return solver_priest.ProjectionSetup(basis=basis, boundary=_point_boundary(scenario),
                                         obstacles=planning_tracks(scenario, basis.grid.timestamps, plan_margin),
                                         v_max=scenario.robot.v_max, a_max=scenario.robot.a_max,
                                         s_min=pts.min(axis=0) - 4.0, s_max=pts.max(axis=0) + 4.0, rho=rho)


def multiagent_problem_from_scenario(scenario: Scenario, basis):
    if scenario.kind != "square-antipodal":
        raise ValueError("the multiagent solver expects a square-antipodal scenario")
    roster = [tuple(AxisBoundary(p0=float(s[k]), p1=float(g[k])) for k in range(3))
              for s, g in agent_boundaries(scenario)]
    a, b = scenario.robot.shape[:2]
    return solver_multiagent.MultiAgentProblem(basis=basis, boundaries=roster, agent_shape=EllipsoidShape(a=a, b=b))


def default_sampling_distribution(scenario: Scenario, basis, spread: float = 0.6):
    """N(straight-line coefficients, spread^2 I) (runner.py:155-161)."""
    s, g = _ends(scenario)
    mu = straight_line_coeffs(basis, s, g).ravel()
    return solver_priest.SamplingDistribution(mu=mu, sigma_mat=np.eye(mu.size) * spread**2)


def barn_cost_fn(scenario: Scenario):
    """The BARN cost of a trajectory against the scenario's start->goal line (runner.py:78-85)."""
    s, g = _ends(scenario)
    return lambda traj: solver_priest.barn_cost(traj.pos, traj.vel, traj.acc, s, g)
