"""Seeded benchmark problems for the hot path (host-side setup, not timed).

* ``random_static``: the reference's "random-static" generator
  (bench/scenarios.py:186-216) — the C1 configuration
  (3-D, 10 static spheres, n_p 100).
* ``flow3d_*``: the 3-D dynamic-obstacle recipe of SURVEY.md §8(d) used for
  C2 (n_o 50, B 1024) and C5 (n_o 100, B 131072): obstacles drawn from
  ``default_rng(seed)`` (per obstacle, in order: cx~U(1.2,10.8), cy~U(-3,3),
  cz~U(-1.5,1.5), vx~U(-0.4,0), vy~U(-0.05,0.05); vz = 0; a = 0.4, b = 0.3),
  member i from ``default_rng(1000 + i)``: start (0, U(-1,1), U(-0.5,0.5)),
  goal (12, U(-1,1), U(-0.5,0.5)); straight-line desired path.
* Tracks are constant-velocity extrapolations on the grid
  (bench/scenarios.py:118-127) and shapes are inflated by the runner's 5 cm
  planning margin (bench/runner.py:88-110).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import AxisBoundary, BasisSet, build_basis
from .geometry import EllipsoidShape, ObstacleTrack

PLAN_MARGIN = 0.05


@dataclass
class ObstacleSpec:
    a: float
    b: float
    center: np.ndarray
    velocity: np.ndarray


def tracks_on_grid(specs: list[ObstacleSpec], timestamps: np.ndarray, margin: float = PLAN_MARGIN,
                   t_now: float = 0.0) -> list[ObstacleTrack]:
    """Constant-velocity tracks, shapes inflated by `margin`."""
    rel = t_now + timestamps - timestamps[0]
    out = []
    for o in specs:
        centers = np.asarray(o.center, float)[None, :] + np.asarray(o.velocity, float)[None, :] * rel[:, None]
        out.append(ObstacleTrack(centers=centers, shape=EllipsoidShape(o.a + margin, o.b + margin)))
    return out


def random_static(dim: int = 3, n_o: int = 10, seed: int = 0, length: float = 12.0, radius: float = 0.5,
                  clearance: float = 1.5):
    """(obstacle specs, start, goal) of the reference's random-static scenario."""
    rng = np.random.default_rng(seed)
    start = np.zeros(dim)
    goal = np.zeros(dim)
    goal[0] = length
    lo = np.full(dim, -3.0)
    hi = np.full(dim, 3.0)
    lo[0], hi[0] = 0.1 * length, 0.9 * length
    if dim == 3:
        lo[2], hi[2] = -1.5, 1.5
    specs: list[ObstacleSpec] = []
    while len(specs) < n_o:
        c = rng.uniform(lo, hi)
        if np.linalg.norm(c - start) < clearance or np.linalg.norm(c - goal) < clearance:
            continue
        specs.append(ObstacleSpec(radius, radius, c, np.zeros(dim)))
    return specs, start, goal


def c1_problem(n_p: int = 100, seed: int = 0):
    """C1: single quadrotor, 3-D, 10 static ellipsoids, horizon 100 -> SingleProblem."""
    from .solver_single import SingleProblem

    basis = build_basis(0.0, 10.0, n_p, 10)
    specs, start, goal = random_static(3, 10, seed)
    frac = np.linspace(0.0, 1.0, n_p)[:, None]
    desired = start[None] + frac * (goal - start)[None]
    bnd = tuple(AxisBoundary(p0=float(start[k]), p1=float(goal[k])) for k in range(3))
    return SingleProblem(basis, bnd, desired, tracks_on_grid(specs, basis.grid.timestamps))


def flow3d_obstacles(n_o: int, seed: int = 0) -> list[ObstacleSpec]:
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_o):
        cx = rng.uniform(1.2, 10.8)
        cy = rng.uniform(-3.0, 3.0)
        cz = rng.uniform(-1.5, 1.5)
        vx = rng.uniform(-0.4, 0.0)
        vy = rng.uniform(-0.05, 0.05)
        out.append(ObstacleSpec(0.4, 0.3, np.array([cx, cy, cz]), np.array([vx, vy, 0.0])))
    return out


def flow3d_scenario(n_o: int, member: int = 0, seed: int = 0):
    """The C2/C5 recipe as a bench Scenario (raw obstacle geometry, member's boundary): what the reference's
    metrics (check_collision_free, metrics.py:60-82) evaluate a member's trajectory against."""
    from .bench.scenarios import Boundary, Horizon, RobotSpec, Scenario, ScenarioObstacle

    starts, goals = flow3d_endpoints([member])
    return Scenario(kind="dynamic-flow", dim=3, horizon=Horizon(0.0, 10.0, 100),
                    robot=RobotSpec(shape=[0.0, 0.0], v_max=3.0, a_max=3.0),
                    obstacles=[ScenarioObstacle(a=o.a, b=o.b, center=[float(v) for v in o.center],
                                                velocity=[float(v) for v in o.velocity])
                               for o in flow3d_obstacles(n_o, seed)],
                    boundary=Boundary(start=[float(v) for v in starts[0]], goal=[float(v) for v in goals[0]]),
                    seed=seed)


def flow3d_endpoints(members) -> tuple[np.ndarray, np.ndarray]:
    """(starts, goals), each (len(members), 3), member i seeded by default_rng(1000 + i)."""
    members = list(members)
    starts = np.empty((len(members), 3))
    goals = np.empty((len(members), 3))
    for k, i in enumerate(members):
        rng = np.random.default_rng(1000 + int(i))
        starts[k] = (0.0, rng.uniform(-1.0, 1.0), rng.uniform(-0.5, 0.5))
        goals[k] = (12.0, rng.uniform(-1.0, 1.0), rng.uniform(-0.5, 0.5))
    return starts, goals


def flow3d_batch(n_o: int, members, n_p: int = 100, seed: int = 0, basis: BasisSet | None = None):
    """C2/C5 members [lo, hi) -> solver_single.SingleBatch (shared basis + tracks)."""
    from .solver_single import SingleBatch

    basis = basis or build_basis(0.0, 10.0, n_p, 10)
    obstacles = tracks_on_grid(flow3d_obstacles(n_o, seed), basis.grid.timestamps)
    starts, goals = flow3d_endpoints(members)
    bvals = np.zeros((starts.shape[0], 3, 6))
    bvals[:, :, 0] = starts
    bvals[:, :, 3] = goals
    return SingleBatch(basis=basis, bvals=bvals, obstacles=obstacles, desired=None)


def priest_c4_centers(n_o: int = 100, seed: int = 1) -> np.ndarray:
    """C4 obstacle centres: default_rng(1), per obstacle cx~U(1.5,10.5),
    cy~U(-3,3), cz~U(-1.5,1.5); static spheres a = b = 0.4 (+5 cm planning margin)."""
    rng = np.random.default_rng(seed)
    out = np.empty((n_o, 3))
    for k in range(n_o):
        out[k] = (rng.uniform(1.5, 10.5), rng.uniform(-3.0, 3.0), rng.uniform(-1.5, 1.5))
    return out


def square_antipodal(n_agents: int = 8, side: float = 6.0, radius: float = 0.4, seed: int = 0, z: float = 1.0,
                     jitter: float = 0.05):
    """(starts, goals) of the reference's "square-antipodal" roster (bench/scenarios.py:248-288 and
    agent_boundaries :130-143): agents evenly spaced on the square's perimeter with jitter, goals
    antipodal through the layout centre."""
    rng = np.random.default_rng(seed)
    perim = 4.0 * side
    starts = []
    for k in range(n_agents):
        s = (k / n_agents) * perim
        edge, off = int(s // side), s % side
        if edge == 0:
            p = (-side / 2 + off, -side / 2)
        elif edge == 1:
            p = (side / 2, -side / 2 + off)
        elif edge == 2:
            p = (side / 2 - off, side / 2)
        else:
            p = (-side / 2, side / 2 - off)
        starts.append(np.array([p[0], p[1], z]) + np.array([rng.uniform(-jitter, jitter), rng.uniform(-jitter, jitter),
                                                            0.0]))
    centre = np.array([0.0, 0.0, z])
    goal0 = 2.0 * centre - starts[0]
    mid = 0.5 * (starts[0] + goal0)
    goals = [goal0] + [2.0 * mid - s for s in starts[1:]]
    return np.stack(starts), np.stack(goals)


def dynamic_flow(n_o: int = 10, seed: int = 0, length: float = 12.0, speed: float = 0.4, radius: float = 0.4):
    """(obstacle specs, start, goal) of the reference's 2-D "dynamic-flow" scenario
    (bench/scenarios.py:219-245): per obstacle x~U(0.3 L, 1.1 L), y~U(-2, 2),
    v = (-speed U(0.5, 1), U(-0.05, 0.05))."""
    rng = np.random.default_rng(seed)
    specs = []
    for _ in range(n_o):
        x = rng.uniform(0.3 * length, 1.1 * length)
        y = rng.uniform(-2.0, 2.0)
        v = np.array([-speed * rng.uniform(0.5, 1.0), rng.uniform(-0.05, 0.05)])
        specs.append(ObstacleSpec(radius, radius, np.array([x, y]), v))
    return specs, np.zeros(2), np.array([length, 0.0])


def batch2d_problem(n_o: int = 50, n_batch: int = 1024, n_p: int = 100, seed: int = 0, offsets=(0.0,),
                    v_max: float = 3.0, a_max: float = 3.0, basis: BasisSet | None = None):
    """Alg. 2 benchmark problem (SURVEY.md §8 a9 "C2-alt"): the dynamic-flow scenario through the
    reference runner's batch_problem_from_scenario (bench/runner.py:113-129): heading boundary =
    start->goal direction, straight-line desired path, 5 cm inflated tracks."""
    from .solver_batch import BatchProblem, FootprintSpec

    basis = basis or build_basis(0.0, 10.0, n_p, 10)
    specs, start, goal = dynamic_flow(n_o, seed)
    heading = float(np.arctan2(goal[1] - start[1], goal[0] - start[0]))
    frac = np.linspace(0.0, 1.0, basis.n_p)[:, None]
    desired = start[None, :] + frac * (goal - start)[None, :]
    return BatchProblem(
        basis=basis,
        boundary=(AxisBoundary(p0=start[0], p1=goal[0]), AxisBoundary(p0=start[1], p1=goal[1])),
        psi_boundary=(heading, heading),
        desired=desired,
        obstacles=tracks_on_grid(specs, basis.grid.timestamps),
        footprint=FootprintSpec(offsets=tuple(offsets)),
        v_max=v_max,
        a_max=a_max,
        n_batch=n_batch,
    )
