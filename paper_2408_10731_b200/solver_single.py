"""Single-robot AM/AL trajectory optimizer on B200 (drop-in for ``trajopt.solver_single``).

Same public surface as the reference module (solver_single.py:30-450):
``SingleProblem``, ``SingleParams``, ``SingleState``, ``SingleSolution``,
``init_state``, ``am_iteration``, ``solve_single``, ``equality_residuals``,
``residual_report``, ``augmented_lagrangian`` — plus the batched entry point
``solve_single_batch`` (B independent members sharing a basis and an
obstacle set, the C2/C5 configurations), whose members behave exactly like
separate ``solve_single`` calls.

Every AM iteration runs as one fused sm_100a kernel launch
(``tro_alg1_iterate``); the numpy ``SingleState`` is only the host-side view
used at solve boundaries.  There is no CPU fallback.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import hashlib
import threading

import numpy as np
import torch

from . import _lib, qpcore
from ._alg1 import Alg1Engine
from .basis import AxisBoundary, BasisSet, Trajectory
from .geometry import ObstacleTrack  # noqa: F401

__all__ = [
    "SingleProblem",
    "SingleParams",
    "SingleState",
    "SingleSolution",
    "SingleBatch",
    "BatchSolution",
    "BatchResult",
    "make_batch_engine",
    "init_state",
    "am_iteration",
    "solve_single",
    "solve_single_batch",
    "equality_residuals",
    "residual_report",
    "augmented_lagrangian",
]


@dataclass
class SingleProblem:
    basis: BasisSet
    boundary: tuple
    desired: np.ndarray
    obstacles: list = field(default_factory=list)
    w_smooth: float = 1.0
    w_track: float = 1.0

    def __post_init__(self):
        self.desired = np.asarray(self.desired, dtype=float)
        if self.desired.shape != (self.basis.n_p, self.dim):
            raise ValueError(f"desired trajectory must be (n_p, {self.dim})")
        if self.w_smooth < 0 or self.w_track < 0 or self.w_smooth + self.w_track == 0:
            raise ValueError("need w_smooth, w_track >= 0 and not both zero")
        for obs in self.obstacles:
            if obs.centers.shape != (self.basis.n_p, self.dim):
                raise ValueError("obstacle track must cover the full grid in problem dimension")

    @property
    def dim(self) -> int:
        return len(self.boundary)

    @property
    def n_o(self) -> int:
        return len(self.obstacles)


@dataclass
class SingleParams:
    max_iter: int = 300
    tol: float = 1e-3
    rho_start: float = 1.0
    rho_growth: float = 1.4
    rho_cap: float = 1e3
    stall_window: int = 5
    stall_improvement: float = 0.01


@dataclass
class SingleState:
    xi: np.ndarray
    d: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray | None
    cos_a: np.ndarray
    sin_a: np.ndarray
    cos_b: np.ndarray | None
    sin_b: np.ndarray | None
    lam_pos: np.ndarray
    lam_cos_a: np.ndarray
    lam_sin_a: np.ndarray
    lam_cos_b: np.ndarray | None
    lam_sin_b: np.ndarray | None
    rho: float
    rho_o: float
    iteration: int = 0
    _factor: qpcore.KKTFactor | None = field(default=None, repr=False)
    _factor_rho_o: float | None = field(default=None, repr=False)
    n_factorizations: int = 0


@dataclass
class SingleSolution:
    trajectory: Trajectory
    converged: bool
    iterations: int
    residual_norm: float
    residual_max: float
    residual_history: list
    smoothness_cost: float
    tracking_cost: float
    n_factorizations: int
    state: SingleState


# ---------------------------------------------------------------- problem -> device arrays
def _tracks(problem: SingleProblem) -> np.ndarray:
    if not problem.obstacles:
        return np.zeros((0, problem.basis.n_p, problem.dim))
    return np.stack([o.centers for o in problem.obstacles]).astype(float)


def _shapes(problem: SingleProblem):
    return (np.array([o.shape.a for o in problem.obstacles], dtype=float),
            np.array([o.shape.b for o in problem.obstacles], dtype=float))


def _linear_term(basis: BasisSet, desired: np.ndarray, w_track: float) -> np.ndarray:
    """-2 w_track (P' desired)' (solver_single.py:173); desired (n_p, dim) -> (dim, m) or
    (B, n_p, dim) -> (B, dim, m), one GEMM per member so every member's bits match a single solve."""
    if desired.ndim == 2:
        return -2.0 * w_track * (basis.P.T @ desired).T
    return -2.0 * w_track * np.transpose(np.matmul(basis.P.T[None], desired), (0, 2, 1))


def _engine_for(problem: SingleProblem, params: SingleParams, *, rho0=None, export=True, max_hist=0,
                dtype=torch.float64) -> Alg1Engine:
    a, b = _shapes(problem)
    bvals = np.stack([bc.values() for bc in problem.boundary])[None]
    return Alg1Engine(problem.basis, _tracks(problem), a, b, bvals, desired=problem.desired[None], params=params,
                      rho0=rho0, w_smooth=problem.w_smooth, w_track=problem.w_track, dtype=dtype, max_hist=max_hist,
                      export=export, keep_d=True)


def _owner_key():
    """Cached engines are single-owner: one per (thread, device, stream), so concurrent solver
    calls from different threads or streams never share device buffers or captured graphs."""
    dev = torch.cuda.current_device()
    return (threading.get_ident(), dev, torch.cuda.current_stream(dev).cuda_stream)


_ENGINE_CACHE: dict = {}


def _cached_engine(problem: SingleProblem, params: SingleParams, *, max_hist: int) -> Alg1Engine:
    """Cold-start engines reused across solve_single calls on the same problem content and parameters:
    the device buffers, constants and level table are built once (one solver per stream)."""
    h = hashlib.blake2b(digest_size=20)
    b = problem.basis
    for arr in (b.P, b.Pdot, b.Pddot, problem.desired, _tracks(problem), *_shapes(problem),
                np.stack([bc.values() for bc in problem.boundary])):
        h.update(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
    key = (h.digest(), problem.w_smooth, problem.w_track, params.rho_start, params.rho_growth, params.rho_cap,
           params.tol, params.stall_window, params.stall_improvement, int(max_hist), _owner_key())
    eng = _ENGINE_CACHE.get(key)
    if eng is None:
        if len(_ENGINE_CACHE) > 16:
            _ENGINE_CACHE.clear()
        eng = _ENGINE_CACHE[key] = _engine_for(problem, params, max_hist=max_hist)
    return eng


def _upload(eng: Alg1Engine, state: SingleState):
    dim = eng.dim
    if eng.n_o:
        planes = [state.lam_pos[k] for k in range(dim)] + [state.lam_cos_a, state.lam_sin_a]
        if dim == 3:
            planes += [state.lam_cos_b, state.lam_sin_b]
        lam = np.stack(planes)[:, None]
        alpha = state.alpha[None]
        beta = state.beta[None] if dim == 3 else None
        d = state.d[None]
    else:
        lam = alpha = beta = d = None
    eng.load_state(xi=state.xi[None], alpha=alpha, beta=beta, lam_planes=lam, d=d, rho=[state.rho],
                   rho_o=[state.rho_o], iteration=[state.iteration])


_FSCALARS = ("rho", "rho_o", "res_norm", "res_max")
_ISCALARS = ("status", "level", "n_changes", "iteration", "n_hist", "level_used")


def _host_angles(eng: Alg1Engine, words: np.ndarray, k: int) -> np.ndarray:
    """Angle k (0: alpha, 1: beta) of member 0 from its raw state words (n_o, W, n_p), on the host."""
    if eng.layout == "angle":
        return words[:, k].astype(float)
    if eng.layout == "unit":
        return np.arctan2(words[:, 2 * k + 1].astype(float), words[:, 2 * k].astype(float))
    w = words[:, k].astype(float)  # folded half-angle tangent (half_decode in alg1_elem.cuh)
    inner = np.abs(w) <= 1
    sg = np.where(np.signbit(w), -1.0, 1.0)
    ang = 2.0 * np.arctan(np.where(inner, w, w - 3.0 * sg))
    return np.where(inner, ang, ang + np.pi * sg)


def _snapshot(eng: Alg1Engine) -> dict:
    """Member 0's state, bookkeeping scalars and residual history in TWO device-to-host copies (float64 and
    int32 groups, raw state words: the angles are decoded on the host), instead of one small kernel per
    field."""
    fparts = [("xi", eng.xi[0])]
    if eng.n_o:
        fparts += [("words", eng.state[0]), ("d", eng.d[0] if eng.d is not None else None),
                   ("copies", eng.copies[:, 0] if eng.copies is not None else None)]
    fparts += [(k, getattr(eng, k)[:1]) for k in _FSCALARS]
    if eng.hist is not None:
        fparts.append(("hist", eng.hist[0]))
    fparts = [(k, t) for k, t in fparts if t is not None]
    flat = torch.cat([t.reshape(-1).to(torch.float64) for _, t in fparts]).cpu().numpy()
    ints = torch.cat([getattr(eng, k)[:1] for k in _ISCALARS]).cpu().numpy()
    out, o = {}, 0
    for k, t in fparts:
        out[k] = flat[o:o + t.numel()].reshape(tuple(t.shape))
        o += t.numel()
    for k in _FSCALARS:
        out[k] = float(out[k][0])
    for j, k in enumerate(_ISCALARS):
        out[k] = int(ints[j])
    if eng.n_o:
        words = out.pop("words")  # (n_o, W, n_p)
        out["lam"] = np.ascontiguousarray(np.transpose(words[:, eng.NV:], (1, 0, 2)))
        out["alpha"] = _host_angles(eng, words, 0)
        if eng.dim == 3:
            out["beta"] = _host_angles(eng, words, 1)
    return out


def _download(eng: Alg1Engine, into: SingleState | None = None, snap: dict | None = None) -> SingleState:
    """Member 0 of a device engine -> numpy SingleState (copies exported by the last iteration)."""
    dim, n_o, n_p = eng.dim, eng.n_o, eng.n_p
    snap = snap if snap is not None else _snapshot(eng)
    f = lambda k: snap[k].copy() if k in snap else None  # noqa: E731
    xi = f("xi")
    if n_o:
        lam = snap["lam"]
        alpha = f("alpha")
        beta = f("beta") if dim == 3 else None
        d = f("d")
        cop = snap["copies"]
        lam_pos = lam[:dim].copy()
        lca, lsa = lam[dim].copy(), lam[dim + 1].copy()
        lcb = lam[dim + 2].copy() if dim == 3 else None
        lsb = lam[dim + 3].copy() if dim == 3 else None
        ca, sa = cop[0].copy(), cop[1].copy()
        cb = cop[2].copy() if dim == 3 else None
        sb = cop[3].copy() if dim == 3 else None
    else:
        z = np.zeros((0, n_p))
        lam_pos = np.zeros((dim, 0, n_p))
        alpha = d = ca = sa = lca = lsa = z.copy()
        beta = cb = sb = lcb = lsb = (z.copy() if dim == 3 else None)
    st = into if into is not None else SingleState(xi=xi, d=d, alpha=alpha, beta=beta, cos_a=ca, sin_a=sa,
                                                   cos_b=cb, sin_b=sb, lam_pos=lam_pos, lam_cos_a=lca,
                                                   lam_sin_a=lsa, lam_cos_b=lcb, lam_sin_b=lsb, rho=1.0, rho_o=1.0)
    st.xi, st.d, st.alpha, st.beta = xi, d, alpha, beta
    st.cos_a, st.sin_a, st.cos_b, st.sin_b = ca, sa, cb, sb
    st.lam_pos, st.lam_cos_a, st.lam_sin_a, st.lam_cos_b, st.lam_sin_b = lam_pos, lca, lsa, lcb, lsb
    st.rho = snap["rho"]
    st.rho_o = snap["rho_o"]
    st.iteration = int(snap["iteration"])
    return st


def _raise_if_failed(eng: Alg1Engine, snap: dict | None = None):
    if snap is not None and eng.B == 1:  # member 0 is the batch
        if int(snap["status"]) & _lib.TRO_FACTOR_FAILED:
            raise eng.table.error_for(int(snap["level"]))
        return
    st = eng.status.cpu().numpy()
    bad = np.nonzero(st & _lib.TRO_FACTOR_FAILED)[0]
    if bad.size:
        raise eng.table.error_for(int(eng.level[int(bad[0])].item()))


# ---------------------------------------------------------------- public API
def init_state(problem: SingleProblem, seed: int | None = None, params: SingleParams | None = None) -> SingleState:
    """Initial AM state on device (solver_single.py:115-166), returned as a numpy SingleState."""
    params = params or SingleParams()
    eng = _engine_for(problem, params)
    eng.cold_init()
    st = _download(eng)
    st.rho = st.rho_o = float(params.rho_start)
    st.iteration = 0
    if eng.n_o:  # init_state's copies are cos/sin of the initial angles (exported by the init kernel)
        pass
    return st


def _factor_bookkeeping(state: SingleState, eng: Alg1Engine, snap: dict | None = None) -> int:
    """New factorizations the reference would have performed in this call (solver_single.py:198-202)."""
    fresh = 1 if (state._factor is None or state._factor_rho_o != state.rho_o) else 0
    return fresh + int(snap["n_changes"] if snap is not None else eng.n_changes[0].item())


def am_iteration(state: SingleState, problem: SingleProblem) -> SingleState:
    """One AM sweep (solver_single.py:373-389) on device; mutates and returns the state."""
    params = SingleParams(rho_start=state.rho_o)
    eng = _engine_for(problem, params, rho0=[state.rho_o])
    _upload(eng, state)
    eng.prime(1)
    eng.iterate(1, flags=_lib.TRO_FLAG_NO_SCHEDULE)
    _raise_if_failed(eng)
    new = _factor_bookkeeping(state, eng)
    rho_o_before = state.rho_o
    _download(eng, into=state)
    if new:
        qpcore._bump(new)
        state.n_factorizations += new
    level = eng._level_for(rho_o_before)
    state._factor = eng.table.factors[level]
    state._factor_rho_o = rho_o_before
    return state


def solve_single(problem: SingleProblem, params: SingleParams | None = None,
                 state: SingleState | None = None) -> SingleSolution:
    """AM loop until max_abs <= tol or max_iter (solver_single.py:407-450), fully on device."""
    params = params or SingleParams()
    if state is None:
        eng = _cached_engine(problem, params, max_hist=max(params.max_iter, 1))
        eng.cold_init()  # complete cold start: penalties, counters and schedule back to rho_start
        level_start = int(eng.table.level_of(params.rho_start))
        state = SingleState(xi=None, d=None, alpha=None, beta=None, cos_a=None, sin_a=None, cos_b=None,
                            sin_b=None, lam_pos=None, lam_cos_a=None, lam_sin_a=None, lam_cos_b=None,
                            lam_sin_b=None, rho=params.rho_start, rho_o=params.rho_start)
    else:
        eng = _engine_for(problem, params, rho0=[state.rho_o], max_hist=max(params.max_iter, 1))
        _upload(eng, state)
        eng.prime(1)
        level_start = eng._level_for(state.rho_o)
    ran = eng.run(params.max_iter, use_graph=params.max_iter > 50, chunk=25,
                  check_every=50 if params.max_iter > 50 else 0)
    snap = _snapshot(eng)
    _raise_if_failed(eng, snap)
    # the reference factorizes at a position step whose rho_o differs from the cached factor's
    # (solver_single.py:198-202): levels level_start .. level_used, the first only if not already cached; a
    # growth on the final iteration is not followed by a position step
    fresh = 1 if (state._factor is None or state._factor_rho_o != state.rho_o) else 0
    lv = int(snap["level_used"]) if ran > 0 else level_start
    new = fresh + (lv - level_start) if ran > 0 else 0
    if ran > 0 or state.xi is None:
        _download(eng, into=state, snap=snap)
    if new:
        qpcore._bump(new)
    state.n_factorizations += new
    if ran > 0:
        state._factor = eng.table.factors[lv]
        state._factor_rho_o = eng.table.rhos[lv]

    nh = int(snap["n_hist"])
    hist = snap["hist"][:nh] if "hist" in snap else np.zeros((0, 3))
    history = [{"norm": float(h[0]), "max_abs": float(h[1]), "rho_o": float(h[2])} for h in hist]
    converged = bool(int(snap["status"]) & _lib.TRO_CONVERGED)
    basis = problem.basis
    traj = Trajectory(t=basis.grid.timestamps, pos=basis.P @ state.xi.T, vel=basis.Pdot @ state.xi.T,
                      acc=basis.Pddot @ state.xi.T)
    return SingleSolution(
        trajectory=traj,
        converged=converged,
        iterations=state.iteration,
        residual_norm=snap["res_norm"],
        residual_max=snap["res_max"],
        residual_history=history,
        smoothness_cost=float(np.sum(traj.acc**2)),
        tracking_cost=float(np.sum((traj.pos - problem.desired) ** 2)),
        n_factorizations=state.n_factorizations,
        state=state,
    )


# ---------------------------------------------------------------- batched entry point
@dataclass
class SingleBatch:
    """B members sharing basis + obstacles (each member = one SingleProblem).

    bvals: (B, dim, 6) boundary values (AxisBoundary.values order); desired: (B, n_p, dim)
    or None for each member's straight start->goal line.
    """

    basis: BasisSet
    bvals: np.ndarray
    obstacles: list
    desired: np.ndarray | None = None
    w_smooth: float = 1.0
    w_track: float = 1.0

    @property
    def B(self) -> int:
        return int(self.bvals.shape[0])

    @property
    def dim(self) -> int:
        return int(self.bvals.shape[1])

    @classmethod
    def from_problems(cls, problems: list) -> "SingleBatch":
        p0 = problems[0]
        for p in problems[1:]:
            if p.basis is not p0.basis and not np.array_equal(p.basis.P, p0.basis.P):
                raise ValueError("batched members must share one basis")
            if len(p.obstacles) != len(p0.obstacles) or any(
                    not np.array_equal(a.centers, b.centers) or a.shape != b.shape
                    for a, b in zip(p.obstacles, p0.obstacles)):
                raise ValueError("batched members must share one obstacle set")
            if (p.w_smooth, p.w_track) != (p0.w_smooth, p0.w_track):
                raise ValueError("batched members must share the cost weights")
        bvals = np.stack([np.stack([bc.values() for bc in p.boundary]) for p in problems])
        desired = np.stack([p.desired for p in problems])
        return cls(p0.basis, bvals, list(p0.obstacles), desired, p0.w_smooth, p0.w_track)

    def desired_paths(self) -> np.ndarray:
        """(B, n_p, dim): the given desired paths, or each member's straight start->goal line
        (bench/runner.py:88-94 formula)."""
        if self.desired is not None:
            return np.asarray(self.desired, dtype=float)
        frac = np.linspace(0.0, 1.0, self.basis.n_p)[None, :, None]
        p0, p1 = self.bvals[:, None, :, 0], self.bvals[:, None, :, 3]
        return p0 + frac * (p1 - p0)

    def linear_terms(self) -> np.ndarray:
        """(B, dim, m) = -2 w_track (P' desired_i)' (solver_single.py:173), member by member."""
        return _linear_term(self.basis, self.desired_paths(), self.w_track)

    def problem(self, i: int) -> SingleProblem:
        bnd = tuple(AxisBoundary(*self.bvals[i, k]) for k in range(self.dim))
        return SingleProblem(self.basis, bnd, self.desired_paths()[i], list(self.obstacles), self.w_smooth,
                             self.w_track)


@dataclass
class BatchSolution:
    """Device-resident results of solve_single_batch (torch tensors on the solve device).

    The tensors alias the engine's buffers: the next solve on the same engine overwrites them
    (use ``numpy()`` / ``clone`` to keep a result)."""

    xi: torch.Tensor
    converged: torch.Tensor
    iterations: torch.Tensor
    residual_norm: torch.Tensor
    residual_max: torch.Tensor
    rho_o: torch.Tensor
    n_factorizations: torch.Tensor
    history: torch.Tensor | None
    engine: Alg1Engine

    def trajectory(self, i: int) -> Trajectory:
        b = self.engine.basis
        xi = self.xi[i].cpu().numpy()
        return Trajectory(t=b.grid.timestamps, pos=b.P @ xi.T, vel=b.Pdot @ xi.T, acc=b.Pddot @ xi.T)

    def numpy(self) -> "BatchResult":
        """Every per-member result in ONE device-to-host copy (integers travel as exact fp64)."""
        B = int(self.xi.shape[0])
        parts = [self.xi.reshape(B, -1), self.residual_norm[:, None], self.residual_max[:, None],
                 self.rho_o[:, None], self.converged[:, None].double(), self.iterations[:, None].double(),
                 self.n_factorizations[:, None].double()]
        flat = torch.cat(parts, dim=1).cpu().numpy()
        k = self.xi[0].numel()
        return BatchResult(xi=flat[:, :k].reshape(tuple(self.xi.shape)), residual_norm=flat[:, k],
                           residual_max=flat[:, k + 1], rho_o=flat[:, k + 2], converged=flat[:, k + 3] != 0,
                           iterations=flat[:, k + 4].astype(np.int64),
                           n_factorizations=flat[:, k + 5].astype(np.int64),
                           history=None if self.history is None else self.history.cpu().numpy())


@dataclass
class BatchResult:
    """Host (numpy) copy of a BatchSolution."""

    xi: np.ndarray
    residual_norm: np.ndarray
    residual_max: np.ndarray
    rho_o: np.ndarray
    converged: np.ndarray
    iterations: np.ndarray
    n_factorizations: np.ndarray
    history: np.ndarray | None


def _obstacle_key(batch: SingleBatch) -> bytes:
    h = hashlib.blake2b(digest_size=20)
    b = batch.basis
    h.update(np.asarray([batch.B, batch.dim, len(batch.obstacles), batch.w_smooth, batch.w_track]).tobytes())
    for arr in (b.P, b.Pdot, b.Pddot):
        h.update(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
    if batch.obstacles:
        h.update(np.ascontiguousarray(np.stack([o.centers for o in batch.obstacles]), dtype=np.float64).tobytes())
        h.update(np.array([[o.shape.a, o.shape.b] for o in batch.obstacles], dtype=np.float64).tobytes())
    return h.digest()


def make_batch_engine(batch: SingleBatch, params: SingleParams, *, dtype=torch.float64, device=None,
                      history: bool = False, groups: int = 0, export: bool = False, layout: str = "angle",
                      use_tma: bool = True, tail_split: bool = True) -> Alg1Engine:
    """An Alg. 1 engine for the batch; the linear terms are computed on the device from the members' boundary
    values (straight-line desired paths) or from the given desired paths."""
    a = np.array([o.shape.a for o in batch.obstacles], dtype=float)
    b = np.array([o.shape.b for o in batch.obstacles], dtype=float)
    tracks = (np.stack([o.centers for o in batch.obstacles]) if batch.obstacles
              else np.zeros((0, batch.basis.n_p, batch.dim)))
    eng = Alg1Engine(batch.basis, tracks, a, b, batch.bvals, desired=batch.desired, params=params,
                     w_smooth=batch.w_smooth, w_track=batch.w_track, dtype=dtype, device=device, groups=groups,
                     max_hist=params.max_iter if history else 0, export=export, layout=layout, use_tma=use_tma,
                     tail_split=tail_split)
    eng.obstacle_key = _obstacle_key(batch)
    eng.solve_params = dataclasses.astuple(params)
    return eng


_BATCH_CACHE: dict = {}


def _batch_engine(batch: SingleBatch, params: SingleParams, **kw) -> Alg1Engine:
    """Engines reused across solve_single_batch calls with the same shape, obstacles and parameters (one per
    thread / device / stream: cached engines are single-owner)."""
    key = (_obstacle_key(batch), dataclasses.astuple(params), tuple(sorted(kw.items())), _owner_key())
    eng = _BATCH_CACHE.get(key)
    if eng is None:
        if len(_BATCH_CACHE) >= 4:  # batch engines can hold tens of GB: keep few alive
            _BATCH_CACHE.clear()
            torch.cuda.empty_cache()
        eng = _BATCH_CACHE[key] = make_batch_engine(batch, params, **kw)
    return eng


def solve_single_batch(batch: SingleBatch | list, params: SingleParams | None = None, *, dtype=torch.float64,
                       device=None, history: bool = False, groups: int = 0, use_graph: bool = True,
                       engine: Alg1Engine | None = None, layout: str = "angle", cache: bool = False) -> BatchSolution:
    """Solve B independent members (each = solve_single of its problem, cold start) in one device pass.

    dtype: storage of the per-element state (float64, or float32 with the QP step and all
    per-member reductions kept in fp64).
    layout: "angle" keeps the reference's angle variables (9 words / element in 3-D); "unit"
    keeps each angle as its unit vector (11 words) and skips the atan2/sincos round trip; "half" keeps the
    reference's 9 words with each angle as a folded half-angle tangent.
    engine: reuse this engine (built by make_batch_engine for a batch with the same size, obstacles and
    basis; ValueError otherwise): the new batch's boundary values and desired paths are uploaded and the
    linear terms recomputed on the device before the cold start.
    cache: reuse an engine cached by shape, obstacles and parameters (per thread and stream)."""
    params = params or SingleParams()
    if isinstance(batch, list):
        batch = SingleBatch.from_problems(batch)
    if engine is not None:
        if getattr(engine, "obstacle_key", None) != _obstacle_key(batch):
            raise ValueError("engine was built for a different batch size, basis or obstacle set")
        if getattr(engine, "solve_params", None) not in (None, dataclasses.astuple(params)):
            raise ValueError("engine was built with different SingleParams")
        eng = engine
        eng.set_members(batch.bvals, batch.desired)
    elif cache:
        eng = _batch_engine(batch, params, dtype=dtype, device=device, history=history, groups=groups,
                            layout=layout)
        eng.set_members(batch.bvals, batch.desired)
    else:
        eng = make_batch_engine(batch, params, dtype=dtype, device=device, history=history, groups=groups,
                                layout=layout)
    eng.cold_init()  # complete cold start (rho, rho_o, level, iteration, schedule reset on the device)
    eng.run(params.max_iter, use_graph=use_graph, check_every=50 if params.tol > 0 else 0)
    _raise_if_failed(eng)
    # one shared factorization per distinct rho_o level any member's position steps used
    # (levels level0 .. level_used: a growth on a member's final iteration is not followed by one)
    nf = (eng.level_used - eng.level0 + 1) if params.max_iter > 0 else torch.zeros_like(eng.level0)
    qpcore._bump(int(nf.max().item()) if params.max_iter > 0 else 0)
    return BatchSolution(xi=eng.xi, converged=(eng.status & _lib.TRO_CONVERGED) != 0, iterations=eng.iteration,
                         residual_norm=eng.res_norm, residual_max=eng.res_max, rho_o=eng.rho_o,
                         n_factorizations=nf, history=eng.hist, engine=eng)


# ---------------------------------------------------------------- diagnostics (host, small arrays)
def _deltas(problem: SingleProblem, positions: np.ndarray) -> np.ndarray:
    return positions[None, :, :] - _tracks(problem)


def equality_residuals(state: SingleState, problem: SingleProblem) -> dict:
    """Residual arrays of every relaxed equality family (solver_single.py:294-313).

    Host-side diagnostic on the numpy view of a state (tests / reports)."""
    out: dict[str, np.ndarray] = {}
    if not problem.n_o:
        return out
    dl = _deltas(problem, problem.basis.P @ state.xi.T)
    a, b = (v[:, None] for v in _shapes(problem))
    if problem.dim == 3:
        out["coll_x"] = dl[:, :, 0] - a * state.d * state.cos_a * state.sin_b
        out["coll_y"] = dl[:, :, 1] - a * state.d * state.sin_a * state.sin_b
        out["coll_z"] = dl[:, :, 2] - b * state.d * state.cos_b
        out["copy_cos_b"] = state.cos_b - np.cos(state.beta)
        out["copy_sin_b"] = state.sin_b - np.sin(state.beta)
    else:
        out["coll_x"] = dl[:, :, 0] - a * state.d * state.cos_a
        out["coll_y"] = dl[:, :, 1] - b * state.d * state.sin_a
    out["copy_cos_a"] = state.cos_a - np.cos(state.alpha)
    out["copy_sin_a"] = state.sin_a - np.sin(state.alpha)
    return out


def residual_report(state: SingleState, problem: SingleProblem) -> dict:
    return {k: {"norm": float(np.linalg.norm(r)), "max_abs": float(np.max(np.abs(r))) if r.size else 0.0}
            for k, r in equality_residuals(state, problem).items()}


def augmented_lagrangian(state: SingleState, problem: SingleProblem) -> float:
    """Objective + multiplier + penalty terms at fixed multipliers (solver_single.py:346-370)."""
    b = problem.basis
    acc = b.Pddot @ state.xi.T
    pos = b.P @ state.xi.T
    val = problem.w_smooth * float(np.sum(acc**2)) + problem.w_track * float(np.sum((pos - problem.desired) ** 2))
    res = equality_residuals(state, problem)
    if not res:
        return val
    for k, name in enumerate(("coll_x", "coll_y", "coll_z")[: problem.dim]):
        r = res[name]
        val += float(np.sum(state.lam_pos[k] * r)) + 0.5 * state.rho_o * float(np.sum(r**2))
    pairs = [("copy_cos_a", state.lam_cos_a), ("copy_sin_a", state.lam_sin_a)]
    if problem.dim == 3:
        pairs += [("copy_cos_b", state.lam_cos_b), ("copy_sin_b", state.lam_sin_b)]
    for name, lam in pairs:
        val += 0.5 * state.rho * float(np.sum((res[name] + lam / state.rho) ** 2))
    return val
