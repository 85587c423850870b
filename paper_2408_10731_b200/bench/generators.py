"""Seeded scenario generators (reference bench/scenarios.py:146-366).

Every kind draws from ``np.random.default_rng(seed)`` in the reference's draw order, so a (kind, params, seed)
triple gives the identical scenario (pinned: ``tests/golden/scenarios.json`` holds the reference's JSON text
for every kind with default and custom parameters).
"""

from __future__ import annotations

import numpy as np

from .scenarios import KINDS, Boundary, Horizon, RobotSpec, Scenario, ScenarioObstacle

__all__ = ["gen_scenario"]


# Every kind draws from default_rng(seed) in the reference's order; `_p` reads a parameter with the
# reference's default and type.
def _p(params, key, default, kind=float):
    return kind(params.get(key, default))


def _horizon(params) -> Horizon:
    return Horizon(t0=_p(params, "t0", 0.0), tf=_p(params, "tf", 10.0), n_p=_p(params, "n_p", 100, int))


def _point_robot(params, vmax: float) -> RobotSpec:
    return RobotSpec(shape=[0.0, 0.0], v_max=_p(params, "v_max", vmax), a_max=_p(params, "a_max", vmax))


def _static(r: float, c) -> ScenarioObstacle:
    c = [float(x) for x in c]
    return ScenarioObstacle(a=r, b=r, center=c, velocity=[0.0] * len(c))


def _planar(kind, params, seed, obstacles, length, vmax=3.0, horizon=None) -> Scenario:
    return Scenario(kind=kind, dim=2, horizon=horizon or _horizon(params), robot=_point_robot(params, vmax),
                    obstacles=obstacles, boundary=Boundary(start=[0.0, 0.0], goal=[length, 0.0]), seed=seed)


def _corridor(params, seed) -> Scenario:
    """:154-183 — staggered blockers near the centre line (weaving), the rest as wall posts."""
    rng = np.random.default_rng(seed)
    L, n_o = _p(params, "length", 12.0), _p(params, "n_o", 10, int)
    hw, r = _p(params, "half_width", 1.6), _p(params, "obstacle_radius", 0.45)
    n_blk = min(n_o, (n_o + 1) // 2)
    obs = []
    for k, x in enumerate(np.linspace(0.18 * L, 0.82 * L, n_blk)):
        y = 0.55 * r * (-1 if k % 2 else 1) + rng.uniform(-0.08, 0.08)
        obs.append(_static(r, (x + rng.uniform(-0.2, 0.2), y)))
    n_wall = n_o - n_blk
    for k in range(n_wall):
        x = (0.25 + 0.5 * (k / max(n_wall - 1, 1))) * L + rng.uniform(-0.3, 0.3)
        obs.append(_static(r, (x, (-1 if k % 2 else 1) * hw)))
    return _planar("corridor", params, seed, obs, L)


def _random_static(params, seed) -> Scenario:
    """:186-216 — uniform centres in a box, rejected within `clearance` of start / goal."""
    rng = np.random.default_rng(seed)
    dim, n_o = _p(params, "dim", 2, int), _p(params, "n_o", 10, int)
    L, r, clear = _p(params, "length", 12.0), _p(params, "obstacle_radius", 0.5), _p(params, "clearance", 1.5)
    start, goal = np.zeros(dim), np.zeros(dim)
    goal[0] = L
    lo, hi = np.full(dim, -3.0), np.full(dim, 3.0)
    lo[0], hi[0] = 0.1 * L, 0.9 * L
    if dim == 3:
        lo[2], hi[2] = -1.5, 1.5
    obs = []
    while len(obs) < n_o:
        c = rng.uniform(lo, hi)
        if min(np.linalg.norm(c - start), np.linalg.norm(c - goal)) >= clear:
            obs.append(_static(r, c))
    return Scenario(kind="random-static", dim=dim, horizon=_horizon(params), robot=_point_robot(params, 3.0),
                    obstacles=obs, boundary=Boundary(start=[float(x) for x in start], goal=[float(x) for x in goal]),
                    seed=seed)


def _dynamic_flow(params, seed) -> Scenario:
    """:219-245 — obstacles drifting against the robot (x~U(0.3L, 1.1L), y~U(-2, 2))."""
    rng = np.random.default_rng(seed)
    n_o, L = _p(params, "n_o", 10, int), _p(params, "length", 12.0)
    speed, r = _p(params, "obstacle_speed", 0.4), _p(params, "obstacle_radius", 0.4)
    obs = []
    for _ in range(n_o):
        x, y = rng.uniform(0.3 * L, 1.1 * L), rng.uniform(-2.0, 2.0)
        vx = -speed * rng.uniform(0.5, 1.0)
        obs.append(ScenarioObstacle(a=r, b=r, center=[float(x), float(y)],
                                    velocity=[float(vx), float(rng.uniform(-0.05, 0.05))]))
    return _planar("dynamic-flow", params, seed, obs, L)


def _square_antipodal(params, seed) -> Scenario:
    """:248-288 — agents evenly spaced on a square's perimeter (jittered), goals antipodal through the
    centre; agent 0 in the boundary block, agents 1.. as stationary pseudo-obstacles."""
    rng = np.random.default_rng(seed)
    n_a, side = _p(params, "n_agents", 8, int), _p(params, "side", 6.0)
    rad, z, jit = _p(params, "agent_radius", 0.4), _p(params, "z", 1.0), _p(params, "jitter", 0.05)
    h = side / 2
    starts = []
    for k in range(n_a):
        s = (k / n_a) * (4.0 * side)
        edge, off = int(s // side), s % side
        xy = [(-h + off, -h), (h, -h + off), (h - off, h), (-h, h - off)][min(edge, 3)]
        jx, jy = rng.uniform(-jit, jit), rng.uniform(-jit, jit)
        starts.append(np.array([xy[0], xy[1], z]) + np.array([jx, jy, 0.0]))
    goal0 = 2.0 * np.array([0.0, 0.0, z]) - starts[0]
    obs = [ScenarioObstacle(a=rad, b=rad, center=[float(x) for x in s], velocity=[0.0, 0.0, 0.0])
           for s in starts[1:]]
    return Scenario(kind="square-antipodal", dim=3, horizon=_horizon(params),
                    robot=RobotSpec(shape=[rad, rad], v_max=_p(params, "v_max", 4.0), a_max=_p(params, "a_max", 4.0)),
                    obstacles=obs, boundary=Boundary(start=[float(x) for x in starts[0]],
                                                     goal=[float(x) for x in goal0]), seed=seed)


def _barn_like(params, seed) -> Scenario:
    """:291-321 — cluttered field with minimum spacing, at most 2000 draws."""
    rng = np.random.default_rng(seed)
    n_o, L = _p(params, "n_o", 16, int), _p(params, "length", 10.0)
    r, spacing, clear = _p(params, "obstacle_radius", 0.3), _p(params, "min_spacing", 1.0), _p(params, "clearance", 1.2)
    start, goal = np.array([0.0, 0.0]), np.array([L, 0.0])
    cs: list = []
    for _ in range(2000):
        if len(cs) >= n_o:
            break
        c = np.array([rng.uniform(0.15 * L, 0.85 * L), rng.uniform(-2.5, 2.5)])
        if np.linalg.norm(c - start) < clear or np.linalg.norm(c - goal) < clear:
            continue
        if all(np.linalg.norm(c - o) >= spacing for o in cs):
            cs.append(c)
    return _planar("barn-like", params, seed, [_static(r, c) for c in cs], L, vmax=2.0)


def _all_infeasible_probe(params, seed) -> Scenario:
    """:324-349 — a big blocker on the straight start-goal line (the default sampling mean starts inside
    it), flanked by two smaller obstacles; n_p defaults to 50."""
    rng = np.random.default_rng(seed)
    L, big = _p(params, "length", 10.0), _p(params, "blocker_radius", 1.6)
    mx = 0.5 * L + rng.uniform(-0.5, 0.5)
    obs = [_static(big, (mx, 0.0))]
    for sgn in (1.0, -1.0):
        obs.append(ScenarioObstacle(a=0.6, b=0.6, center=[float(mx + rng.uniform(-1.5, 1.5)), float(sgn * (big + 1.4))],
                                    velocity=[0.0, 0.0]))
    hz = Horizon(t0=0.0, tf=_p(params, "tf", 10.0), n_p=_p(params, "n_p", 50, int))
    return _planar("all-infeasible-probe", params, seed, obs, L, horizon=hz)


_GEN = {"corridor": _corridor, "random-static": _random_static, "dynamic-flow": _dynamic_flow,
        "square-antipodal": _square_antipodal, "barn-like": _barn_like, "all-infeasible-probe": _all_infeasible_probe}


def gen_scenario(kind: str, params: dict | None = None, seed: int = 0) -> Scenario:
    """Deterministic scenario of a kind (bench/scenarios.py:362-366)."""
    gen = _GEN.get(kind)
    if gen is None:
        raise ValueError(f"unknown scenario kind {kind!r}; choose from {KINDS}")
    return gen(params or {}, int(seed))
