"""Scenario model, seeded generators, JSON wire format and obstacle prediction.

Drop-in for the reference ``trajopt.bench.scenarios`` (bench/scenarios.py:1-366): the same dataclasses
(field order fixes the JSON key order), ``gen_scenario`` for the six kinds (``bench.generators``: the
reference's seeded draw order, pinned by ``tests/golden/scenarios.json``), ``to_json`` / ``from_json``
byte-compatible with the reference's files, and ``predict_obstacles``.

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


def gen_scenario(kind: str, params: dict | None = None, seed: int = 0) -> Scenario:
    """Deterministic scenario of a kind (bench/scenarios.py:362-366); the generators are in bench.generators."""
    from .generators import gen_scenario as _gen

    return _gen(kind, params, seed)


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
