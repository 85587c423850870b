"""Scenario model, seeded generators, JSON wire format and obstacle prediction.

Drop-in for the reference ``trajopt.bench.scenarios`` (bench/scenarios.py:1-366): the same dataclasses
(field order fixes the JSON key order), the same six kinds drawn from ``np.random.default_rng(seed)`` in
the reference's draw order (so a seed gives the identical scenario, pinned by ``tests/golden/scenarios.json``),
``to_json`` / ``from_json`` byte-compatible with the reference's files, and ``predict_obstacles``.

B200 additions for batched use:

* ``predict_obstacles_device`` — the constant-velocity extrapolation of every obstacle of S scenarios (or one
  scenario at S times) on the device in one launch of ``tro_predict_tracks_f64`` (csrc/mpc.cu), bit-exact
  with ``predict_obstacles`` (same operation order, no FMA contraction), written either in the reference's
  (obstacle, sample, axis) order or in the Alg. 1 engine's track layout (obstacle, axis, sample);
* ``obstacle_arrays`` — a scenario's obstacle table as flat arrays (what the device kernels read).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import asdict, dataclass, field

import numpy as np

from ..geometry import EllipsoidShape, ObstacleTrack

__all__ = ["KINDS", "Horizon", "RobotSpec", "ScenarioObstacle", "Boundary", "Scenario", "to_json", "from_json",
           "save_scenario", "load_scenario", "predict_obstacles", "agent_boundaries", "gen_scenario",
           "obstacle_arrays", "predict_obstacles_device"]

KINDS = ("corridor", "random-static", "dynamic-flow", "square-antipodal", "barn-like", "all-infeasible-probe")


# ---------------------------------------------------------------- model (bench/scenarios.py:35-87)
@dataclass
class Horizon:
    t0: float
    tf: float
    n_p: int


@dataclass
class RobotSpec:
    shape: list  # [a, b] agent half-dims; [0, 0] for point robots
    v_max: float
    a_max: float
    footprint_offsets: list = field(default_factory=list)


@dataclass
class ScenarioObstacle:
    a: float
    b: float
    center: list
    velocity: list


@dataclass
class Boundary:
    start: list
    goal: list


@dataclass
class Scenario:
    kind: str
    dim: int
    horizon: Horizon
    robot: RobotSpec
    obstacles: list
    boundary: Boundary
    seed: int

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown scenario kind {self.kind!r}")
        if self.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        if any(len(o.center) != self.dim or len(o.velocity) != self.dim for o in self.obstacles):
            raise ValueError("obstacle center/velocity must match the scenario dimension")
        if len(self.boundary.start) != self.dim or len(self.boundary.goal) != self.dim:
            raise ValueError("boundary vectors must match the scenario dimension")

    @property
    def scenario_id(self) -> str:
        return f"{self.kind}-{self.seed}"


# ---------------------------------------------------------------- JSON wire format (bench/scenarios.py:90-115)
def to_json(scenario: Scenario) -> str:
    """The reference's file body: ``json.dumps(asdict(s), indent=2)`` (keys in dataclass field order)."""
    return json.dumps(asdict(scenario), indent=2)


def from_json(text: str) -> Scenario:
    d = json.loads(text)
    return Scenario(kind=d["kind"], dim=d["dim"], horizon=Horizon(**d["horizon"]), robot=RobotSpec(**d["robot"]),
                    obstacles=[ScenarioObstacle(**o) for o in d["obstacles"]], boundary=Boundary(**d["boundary"]),
                    seed=d["seed"])


def save_scenario(scenario: Scenario, path) -> None:
    with open(path, "w") as fh:
        fh.write(to_json(scenario) + "\n")


def load_scenario(path) -> Scenario:
    with open(path) as fh:
        return from_json(fh.read())


# ---------------------------------------------------------------- obstacle prediction
def obstacle_arrays(scenario: Scenario):
    """(centers (n_o, dim), velocities (n_o, dim), a (n_o,), b (n_o,)) as fp64 arrays."""
    dim = int(scenario.dim)
    obs = list(scenario.obstacles)
    if not obs:
        z = np.zeros((0, dim))
        return z, z.copy(), np.zeros(0), np.zeros(0)
    return (np.array([o.center for o in obs], dtype=float), np.array([o.velocity for o in obs], dtype=float),
            np.array([o.a for o in obs], dtype=float), np.array([o.b for o in obs], dtype=float))


def predict_obstacles(scenario: Scenario, timestamps, t_now: float = 0.0) -> list:
    """Constant-velocity tracks c + v (t_now + t - t[0]) on the grid (bench/scenarios.py:118-127)."""
    ts = np.asarray(timestamps, dtype=float)
    rel = (t_now + ts - ts[0])[:, None]
    c, v, a, b = obstacle_arrays(scenario)
    return [ObstacleTrack(centers=c[j][None, :] + v[j][None, :] * rel, shape=EllipsoidShape(a=a[j], b=b[j]))
            for j in range(a.size)]


def predict_obstacles_device(scenarios, timestamps, t_now=0.0, *, layout: str = "reference", device=None):
    """Tracks of S scenarios with the same obstacle count (or one scenario at S values of ``t_now``) in ONE
    launch.  ``scenarios``: a Scenario, a list of them, or a tuple (centers (S, n_o, dim), velocities) of
    arrays / device tensors.  ``t_now``: scalar or (S,).  Returns an fp64 device tensor
    (S, n_o, n_p, dim) for layout "reference" (``predict_obstacles`` order) or (S, n_o, dim, n_p) for
    "engine" (the Alg. 1 ``tro_alg1_consts.tracks`` layout)."""
    import torch

    from .. import _lib

    _lib.require_cuda()
    lib = _lib.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    if isinstance(scenarios, tuple):
        c, v = (torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x, **f64) for x in scenarios)
    else:
        scs = [scenarios] if isinstance(scenarios, Scenario) else list(scenarios)
        arrs = [obstacle_arrays(s) for s in scs]
        if len({a[0].shape for a in arrs}) != 1:
            raise ValueError("scenarios must have the same obstacle count and dimension")
        c = torch.as_tensor(np.stack([a[0] for a in arrs]), **f64)
        v = torch.as_tensor(np.stack([a[1] for a in arrs]), **f64)
    ts = torch.as_tensor(np.array(timestamps, dtype=float).reshape(-1), **f64)
    tn = np.asarray(t_now, dtype=float).reshape(-1)
    S = max(int(c.shape[0]), tn.size)
    if c.shape[0] not in (1, S) or tn.size not in (1, S):
        raise ValueError("scenario count and t_now count disagree")
    c, v = c.contiguous(), v.contiguous()
    n_o, dim, n_p = int(c.shape[1]), int(c.shape[2]), int(ts.numel())
    tn_d = torch.as_tensor(np.broadcast_to(tn, (S,)).copy(), **f64)
    eng = layout == "engine"
    if layout not in ("reference", "engine"):
        raise ValueError("layout must be 'reference' or 'engine'")
    out = torch.empty((S, n_o, dim, n_p) if eng else (S, n_o, n_p, dim), **f64)
    if out.numel() == 0:
        return out
    dims = _lib.TrackDims(n_scen=S, n_obs=n_o, n_p=n_p, dim=dim, layout=int(eng),
                          shared_obstacles=int(c.shape[0] == 1 and S > 1))
    with torch.cuda.device(dev):
        rc = lib.tro_predict_tracks_f64(ctypes.byref(dims), _lib.ptr(c), _lib.ptr(v), _lib.ptr(ts), _lib.ptr(tn_d),
                                        _lib.ptr(out), _lib.stream_handle())
    _lib.check(rc, "tro_predict_tracks_f64")
    return out


def agent_boundaries(scenario: Scenario) -> list:
    """(start, goal) per agent of a square-antipodal scenario (bench/scenarios.py:130-143): agent 0 in the
    boundary block, the others as pseudo-obstacles whose goals mirror through the start/goal midpoint."""
    s0 = np.asarray(scenario.boundary.start, dtype=float)
    g0 = np.asarray(scenario.boundary.goal, dtype=float)
    mid2 = 2.0 * (0.5 * (s0 + g0))
    out = [(s0, g0)]
    for o in scenario.obstacles:
        s = np.asarray(o.center, dtype=float)
        out.append((s, mid2 - s))
    return out


# ---------------------------------------------------------------- generators (bench/scenarios.py:146-366)
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
