"""PRIEST projection-guided sampling and the CEM baseline on B200 (drop-in for ``trajopt.solver_priest``).

Same public surface as the reference module (solver_priest.py:35-498):
``PriestParams``, ``CemParams``, ``SamplingDistribution``, ``ProjectedSample``,
``ProjectionSetup``, ``project``, ``residual_scores``, ``residual_score``,
``PriestResult``, ``update_distribution``, ``priest_optimize``, ``CemResult``,
``cem_optimize``, ``flatness_car``, ``barn_cost`` — plus ``BarnCost``, a c1
cost object that ``priest_optimize`` / ``cem_optimize`` evaluate on the GPU
(any other Python callable is evaluated per sample, as the reference does).

Device path per round: standard normals z from the same numpy Generator
stream (so samples are those of ``multivariate_normal(method="svd")``), the
projection kernel (all inner iterations on chip, ``tro_priest_project_f64``),
stable top-k elites (``tro_topk_stable_f64``), batched costs
(``tro_priest_cost_f64``) and the weighted refit (``tro_elite_update_f64``).
Only the 33x33 SVD of the covariance runs on the host (numpy's LAPACK, exactly
the factor numpy's sampler uses).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, qpcore
from .basis import AxisBoundary, BasisSet, Trajectory, boundary_matrix  # noqa: F401
from .geometry import ObstacleTrack  # noqa: F401

_SPEED_EPS = 1e-6

__all__ = [
    "PriestParams",
    "CemParams",
    "SamplingDistribution",
    "ProjectedSample",
    "ProjectionSetup",
    "project",
    "residual_scores",
    "residual_score",
    "PriestResult",
    "update_distribution",
    "priest_optimize",
    "CemResult",
    "cem_optimize",
    "flatness_car",
    "barn_cost",
    "BarnCost",
]


@dataclass
class PriestParams:
    n_outer: int = 13
    n_batch: int = 110
    n_constraint_elite: int = 80
    n_elite: int = 20
    n_inner: int = 30
    sigma: float = 0.7
    gamma: float = -1.0
    residual_weight: float = 1.0
    seed: int | None = 0

    def __post_init__(self):
        if not (self.n_elite <= self.n_constraint_elite <= self.n_batch):
            raise ValueError("need n_elite <= n_constraint_elite <= n_batch")
        if not (0.0 < self.sigma <= 1.0):
            raise ValueError("learning rate sigma must lie in (0, 1]")
        if self.gamma == 0.0:
            raise ValueError("gamma must be nonzero")


@dataclass
class CemParams:
    n_batch: int = 110
    n_elite: int = 20
    iterations: int = 13
    seed: int | None = 0
    penalty_weight: float = 1.0

    def __post_init__(self):
        if self.n_elite > self.n_batch:
            raise ValueError("need n_elite <= n_batch")


@dataclass
class SamplingDistribution:
    mu: np.ndarray
    sigma_mat: np.ndarray

    def __post_init__(self):
        self.mu = np.asarray(self.mu, dtype=float)
        self.sigma_mat = np.asarray(self.sigma_mat, dtype=float)
        if not np.allclose(self.sigma_mat, self.sigma_mat.T, atol=1e-10):
            raise ValueError("covariance must be symmetric")

    def draw(self, n: int, rng) -> np.ndarray:
        return rng.multivariate_normal(self.mu, self.sigma_mat, size=n, method="svd")


@dataclass
class ProjectedSample:
    original: np.ndarray
    projected: np.ndarray
    residual: float
    trajectory: Trajectory
    aug_cost: float | None = None


def _draw_factor(sigma_mat: np.ndarray) -> np.ndarray:
    """numpy multivariate_normal(method='svd'): samples = mean + z @ (u sqrt(s)).T."""
    u, s, _ = np.linalg.svd(sigma_mat)
    return u * np.sqrt(s)


class ProjectionSetup:
    """Constant matrices of one scene (solver_priest.py:93-168), resident on the GPU.

    The dense F~, G, F, A are kept on the host for API compatibility; the device
    path needs only the basis, F'F's per-axis block, the saddle inverse and the
    obstacle / limit data.
    """

    def __init__(self, basis: BasisSet, boundary: tuple, obstacles: list | None = None, v_max: float | None = None,
                 a_max: float | None = None, s_min=None, s_max=None, rho: float = 1.0, start_orders=(0, 1, 2),
                 end_orders=(0,)):
        self.basis = basis
        self.boundary = boundary
        self.dim = len(boundary)
        self.obstacles = obstacles or []
        self.v_max = v_max
        self.a_max = a_max
        self.s_min = None if s_min is None else np.asarray(s_min, dtype=float)
        self.s_max = None if s_max is None else np.asarray(s_max, dtype=float)
        self.rho = rho
        m, n_p, dim = basis.n_var, basis.n_p, self.dim
        self.m = m
        self.n_o = len(self.obstacles)
        blocks = []
        if self.n_o:
            blocks.append(np.tile(basis.P, (self.n_o, 1)))
        if v_max is not None:
            blocks.append(basis.Pdot)
        if a_max is not None:
            blocks.append(basis.Pddot)
        axis_block = np.vstack(blocks) if blocks else np.zeros((0, m))
        rows = axis_block.shape[0]
        self.F_tilde = np.zeros((dim * rows, dim * m))
        for k in range(dim):
            self.F_tilde[k * rows:(k + 1) * rows, k * m:(k + 1) * m] = axis_block
        self.has_bounds = self.s_min is not None and self.s_max is not None
        if self.has_bounds:
            bound_block = np.vstack([-basis.P, basis.P])
            self.G = np.zeros((dim * 2 * n_p, dim * m))
            self.tau = np.zeros(dim * 2 * n_p)
            for k in range(dim):
                self.G[k * 2 * n_p:(k + 1) * 2 * n_p, k * m:(k + 1) * m] = bound_block
                self.tau[k * 2 * n_p:k * 2 * n_p + n_p] = -self.s_min[k]
                self.tau[k * 2 * n_p + n_p:(k + 1) * 2 * n_p] = self.s_max[k]
        else:
            self.G = np.zeros((0, dim * m))
            self.tau = np.zeros(0)
        self.F = np.vstack([self.F_tilde, self.G])
        B = boundary_matrix(basis, start_orders, end_orders)
        self.A = np.zeros((dim * B.shape[0], dim * m))
        for k in range(dim):
            self.A[k * B.shape[0]:(k + 1) * B.shape[0], k * m:(k + 1) * m] = B
        self.b_eq = np.concatenate([bc.values(start_orders, end_orders) for bc in boundary])
        self.static_tracks = False
        if self.n_o:
            self.obs_pos = np.stack([o.centers for o in self.obstacles])  # (n_o, n_p, dim)
            self.static_tracks = bool(np.all(self.obs_pos == self.obs_pos[:, :1, :]))
            self.obs_a = np.array([o.shape.a for o in self.obstacles])
            self.obs_b = np.array([o.shape.b for o in self.obstacles])
        FtF = self.F.T @ self.F
        self.factor = qpcore.factorize(np.eye(dim * m) + rho * FtF, self.A)  # solver_priest.py:167
        self.n_factorizations = 1
        self._FtF_block = np.ascontiguousarray(FtF[:m, :m])
        self._dev = {}

    # -- device constants -------------------------------------------------------------
    def device(self, dev=None) -> dict:
        _lib.require_cuda()
        dev = torch.device(dev) if dev is not None else torch.device("cuda", torch.cuda.current_device())
        key = str(dev)
        if key in self._dev:
            return self._dev[key]
        f = dict(dtype=torch.float64, device=dev)
        b = self.basis
        tracks = (np.ascontiguousarray(np.transpose(self.obs_pos, (0, 2, 1))) if self.n_o
                  else np.zeros((0, self.dim, b.n_p)))
        start = np.array([bc.p0 for bc in self.boundary], dtype=float)
        goal = np.array([bc.p1 for bc in self.boundary], dtype=float)
        d = {
            "P": torch.as_tensor(np.array(b.P), **f), "Pd": torch.as_tensor(np.array(b.Pdot), **f),
            "Pdd": torch.as_tensor(np.array(b.Pddot), **f), "tracks": torch.as_tensor(tracks, **f),
            "a": torch.as_tensor(self.obs_a if self.n_o else np.ones(1), **f),
            "b": torch.as_tensor(self.obs_b if self.n_o else np.ones(1), **f),
            "kinv": self.factor.kinv_on(dev), "FtF": torch.as_tensor(self._FtF_block, **f),
            "b_eq": torch.as_tensor(self.b_eq, **f),
            "s_min": torch.as_tensor(self.s_min if self.has_bounds else np.zeros(self.dim), **f),
            "s_max": torch.as_tensor(self.s_max if self.has_bounds else np.zeros(self.dim), **f),
            "mu": torch.zeros(self.dim * self.m, **f), "L": torch.zeros((self.dim * self.m,) * 2, **f),
            "line": torch.as_tensor(np.concatenate([start[:2], goal[:2]]), **f), "device": dev,
        }
        self._dev[key] = d
        return d

    def _dims(self, n: int, n_inner: int) -> _lib.PriestDims:
        return _lib.PriestDims(int(n), self.basis.n_p, self.m, self.dim, self.n_o, int(self.A.shape[0]),
                               int(n_inner))

    def _consts(self, d: dict, line=None) -> _lib.PriestConsts:
        return _lib.PriestConsts(
            d["P"].data_ptr(), d["Pd"].data_ptr(), d["Pdd"].data_ptr(), d["tracks"].data_ptr(), d["a"].data_ptr(),
            d["b"].data_ptr(), d["kinv"].data_ptr(), d["FtF"].data_ptr(), d["b_eq"].data_ptr(),
            d["s_min"].data_ptr(), d["s_max"].data_ptr(), d["mu"].data_ptr(), d["L"].data_ptr(),
            (line if line is not None else d["line"]).data_ptr(),
            float(self.v_max) if self.v_max is not None else -1.0,
            float(self.a_max) if self.a_max is not None else -1.0, float(self.rho), int(self.has_bounds),
            int(self.static_tracks), int(self.n_o > 0 and bool(np.array_equal(self.obs_a, self.obs_b))), 0)

    # -- host helpers (reference API) -----------------------------------------------
    def axis_samples(self, xis: np.ndarray, mat: np.ndarray) -> np.ndarray:
        xis = np.atleast_2d(xis)
        out = np.empty((xis.shape[0], self.dim, mat.shape[0]))
        for k in range(self.dim):
            out[:, k, :] = xis[:, k * self.m:(k + 1) * self.m] @ mat.T
        return out

    def trajectory_of(self, xi: np.ndarray) -> Trajectory:
        xi = np.asarray(xi)
        return Trajectory(t=self.basis.grid.timestamps, pos=self.axis_samples(xi, self.basis.P)[0].T,
                          vel=self.axis_samples(xi, self.basis.Pdot)[0].T,
                          acc=self.axis_samples(xi, self.basis.Pddot)[0].T)


# ---------------------------------------------------------------- device primitives
def _stream():
    return ctypes.c_void_p(_lib.stream_handle())


def _run_project(setup: ProjectionSetup, *, samples=None, z=None, n_inner=30, history=False, keep_samples=False):
    """Launch the projection kernel; returns device tensors (xi, scores, history, samples)."""
    d = setup.device()
    dev = d["device"]
    src = z if z is not None else samples
    n = int(src.shape[0])
    dm = setup.dim * setup.m
    xi = torch.empty((n, dm), dtype=torch.float64, device=dev)
    scores = torch.empty(n, dtype=torch.float64, device=dev)
    hist = torch.empty((max(n_inner, 1), n), dtype=torch.float64, device=dev) if history else None
    smp_out = torch.empty((n, dm), dtype=torch.float64, device=dev) if keep_samples else None
    io = _lib.PriestIO(_lib.ptr(z), _lib.ptr(samples), _lib.ptr(smp_out), xi.data_ptr(), scores.data_ptr(),
                       _lib.ptr(hist))
    rc = _lib.load().tro_priest_project_f64(ctypes.byref(setup._dims(n, n_inner)), ctypes.byref(setup._consts(d)),
                                           ctypes.byref(io), _stream())
    _lib.check(rc, "tro_priest_project_f64")
    return xi, scores, hist, smp_out


def _run_cost(setup: ProjectionSetup, xi, index, scores, w_barn, w_score, w_penalty, line):
    d = setup.device()
    count = int(index.numel()) if index is not None else int(xi.shape[0])
    out = torch.empty(count, dtype=torch.float64, device=d["device"])
    rc = _lib.load().tro_priest_cost_f64(ctypes.byref(setup._dims(xi.shape[0], 0)),
                                        ctypes.byref(setup._consts(d, line)), xi.data_ptr(), _lib.ptr(index), count,
                                        _lib.ptr(scores), float(w_barn), float(w_score), float(w_penalty),
                                        out.data_ptr(), _stream())
    _lib.check(rc, "tro_priest_cost_f64")
    return out


def _topk(keys: torch.Tensor, k: int) -> torch.Tensor:
    """np.argsort(keys, kind="stable")[:k] on the device (bit-exact rank select)."""
    lib = _lib.load()
    n = int(keys.numel())
    out = torch.empty(max(k, 1), dtype=torch.int64, device=keys.device)
    ws = torch.empty(max(int(lib.tro_topk_workspace_bytes(n, k)), 8), dtype=torch.uint8, device=keys.device)
    rc = lib.tro_topk_stable_f64(keys.data_ptr(), n, int(k), out.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "tro_topk_stable_f64")
    return out[:k]


def _refit(xi, rows, costs, sigma, gamma, mu, cov, mode=_lib.TRO_REFIT_PRIEST):
    rc = _lib.load().tro_elite_update_f64(xi.data_ptr(), int(xi.shape[1]), rows.data_ptr(), int(rows.numel()),
                                         costs.data_ptr(), float(sigma), float(gamma), int(mode), mu.data_ptr(),
                                         cov.data_ptr(), _stream())
    _lib.check(rc, "tro_elite_update_f64")


# ---------------------------------------------------------------- reference API
def project(setup: ProjectionSetup, samples: np.ndarray, n_inner: int = 30,
            residual_history: list | None = None) -> list[ProjectedSample]:
    """Project every sample toward the feasible set (solver_priest.py:242-287), on the GPU."""
    if n_inner < 1:
        raise ValueError("n_inner must be at least 1")
    samples = np.atleast_2d(np.asarray(samples, dtype=float))
    d = setup.device()
    s_dev = torch.as_tensor(samples, device=d["device"]).contiguous()
    xi, scores, hist, _ = _run_project(setup, samples=s_dev, n_inner=n_inner, history=residual_history is not None)
    xi_h, sc_h = xi.cpu().numpy(), scores.cpu().numpy()
    if residual_history is not None:
        residual_history.extend(list(hist.cpu().numpy()))
    return [ProjectedSample(original=samples[i], projected=xi_h[i], residual=float(sc_h[i]),
                            trajectory=setup.trajectory_of(xi_h[i])) for i in range(samples.shape[0])]


def residual_scores(setup: ProjectionSetup, xis: np.ndarray) -> np.ndarray:
    """Constraint-violation score per sample (solver_priest.py:290-301), on the GPU."""
    xis = np.atleast_2d(np.asarray(xis, dtype=float))
    d = setup.device()
    x_dev = torch.as_tensor(xis, device=d["device"]).contiguous()
    _, scores, _, _ = _run_project(setup, samples=x_dev, n_inner=0)
    return scores.cpu().numpy()


def residual_score(setup: ProjectionSetup, xi_bar: np.ndarray) -> float:
    return float(residual_scores(setup, xi_bar)[0])


@dataclass
class PriestResult:
    best: ProjectedSample
    mu: np.ndarray
    sigma_mat: np.ndarray
    history: list
    params: PriestParams


def update_distribution(mu, sigma_mat, elite_xi, elite_costs, sigma, gamma):
    """Exponentially weighted mean / covariance refit with learning rate (solver_priest.py:317-333)."""
    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.as_tensor(np.atleast_2d(np.asarray(elite_xi, dtype=float)), device=dev).contiguous()
    c = torch.as_tensor(np.asarray(elite_costs, dtype=float), device=dev).contiguous()
    m = torch.as_tensor(np.array(mu, dtype=float), device=dev)
    S = torch.as_tensor(np.array(sigma_mat, dtype=float), device=dev)
    rows = torch.arange(x.shape[0], device=dev, dtype=torch.int64)
    _refit(x, rows, c, sigma, gamma, m, S)
    return m.cpu().numpy(), S.cpu().numpy()


class BarnCost:
    """The benchmark's clutter-navigation c1 (solver_priest.py:475-498, runner._barn_c1) as an
    object: callable on a Trajectory like any c1, and evaluated on the GPU by priest_optimize /
    cem_optimize."""

    def __init__(self, line_start, line_end):
        self.start = np.asarray(line_start, dtype=float)
        self.end = np.asarray(line_end, dtype=float)

    def __call__(self, traj: Trajectory) -> float:
        return barn_cost(traj.pos, traj.vel, traj.acc, self.start, self.end)

    def line(self, dev) -> torch.Tensor:
        return torch.as_tensor(np.concatenate([self.start[:2], self.end[:2]]), dtype=torch.float64, device=dev)


def _draw_z(rng, n: int, d: int) -> np.ndarray:
    """The standard normals multivariate_normal(size=n, method='svd') consumes."""
    return rng.standard_normal((n, d))


SAMPLERS = ("numpy", "philox")


class _DeviceSampler:
    """Throughput-mode draws, all on the device: the draw factor is the Cholesky factor of the current
    covariance (tro_cholesky_f64) and the standard normals come from Philox4x32-10 keyed by the seed with
    the round as the stream id (tro_normal_philox_f64), so a round needs no host round trip.  Parity mode
    ("numpy") keeps numpy's Generator stream and svd factor, which reproduce the reference's samples."""

    def __init__(self, seed: int, n: int, dm: int, dev, first: int = 0):
        self.seed, self.n, self.dm, self.first = int(seed) & (2**64 - 1), int(n), int(dm), int(first)
        self.z = torch.empty((n, dm), dtype=torch.float64, device=dev)

    def factor(self, sig: torch.Tensor, L: torch.Tensor):
        rc = _lib.load().tro_cholesky_f64(sig.data_ptr(), self.dm, L.data_ptr(), _stream())
        _lib.check(rc, "tro_cholesky_f64")

    def normals(self, round_index: int) -> torch.Tensor:
        rc = _lib.load().tro_normal_philox_f64(self.seed, int(round_index), self.first, self.n, self.dm,
                                               self.z.data_ptr(), _stream())
        _lib.check(rc, "tro_normal_philox_f64")
        return self.z


def device_normals(seed: int, round_index: int, n: int, dm: int, first: int = 0, device=None) -> torch.Tensor:
    """(n, dm) throughput-mode standard normals of samples first .. first + n - 1 (see _DeviceSampler)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return _DeviceSampler(seed, n, dm, dev, first).normals(round_index).clone()


def _z_round(z, dev):
    """One round's standard normals on the device: pinned host rows upload asynchronously (the host does
    not wait for the previous round's kernels before queueing this round)."""
    if isinstance(z, torch.Tensor) and z.device.type == "cpu" and z.is_pinned():
        return z.to(device=dev, dtype=torch.float64, non_blocking=True).contiguous()
    return torch.as_tensor(z, device=dev).contiguous()


def priest_optimize(setup: ProjectionSetup, c1, distribution: SamplingDistribution,
                    params: PriestParams | None = None, *, z_rounds=None, sampler: str = "numpy") -> PriestResult:
    """Projection-guided sampling loop (solver_priest.py:336-382), one device pass per round.

    z_rounds: optional pre-drawn standard normals (n_outer, n_batch, d), device or host, in
    place of drawing them from default_rng(params.seed) round by round.
    sampler: "numpy" (parity mode: the reference's Generator stream and svd factor, host draws) or "philox"
    (throughput mode: Cholesky factor and Philox normals on the device; with a BarnCost c1 the rounds run
    without a host synchronisation until the result is read)."""
    params = params or PriestParams()
    if sampler not in SAMPLERS:
        raise ValueError(f"sampler must be one of {SAMPLERS}")
    if sampler == "philox" and z_rounds is None and isinstance(c1, BarnCost):
        return _priest_device_rounds(setup, c1, distribution, params)
    d = setup.device()
    dev = d["device"]
    rng = np.random.default_rng(params.seed)
    mu = torch.as_tensor(distribution.mu.copy(), device=dev)
    sig = torch.as_tensor(distribution.sigma_mat.copy(), device=dev)
    sig_h = distribution.sigma_mat.copy()
    dm = mu.numel()
    device_cost = isinstance(c1, BarnCost)
    line = c1.line(dev) if device_cost else None
    history = []
    best = None
    for r in range(params.n_outer):
        d["L"].copy_(torch.as_tensor(_draw_factor(sig_h)))
        d["mu"].copy_(mu)
        if z_rounds is not None:
            z = _z_round(z_rounds[r], dev)
        else:
            z = torch.as_tensor(_draw_z(rng, params.n_batch, dm), device=dev)
        xi, scores, _, smp = _run_project(setup, z=z, n_inner=params.n_inner, keep_samples=True)
        keep = _topk(scores, params.n_constraint_elite)  # :358
        if device_cost:
            aug = _run_cost(setup, xi, keep, scores, 1.0, params.residual_weight, 0.0, line)  # :359-361
        else:
            xk, sk = xi[keep].cpu().numpy(), scores[keep].cpu().numpy()
            aug = torch.as_tensor(np.array([float(c1(setup.trajectory_of(xk[i]))) + params.residual_weight * sk[i]
                                            for i in range(xk.shape[0])]), device=dev)
        erank = _topk(aug, params.n_elite)  # :362-363 (stable: residual-rank order on ties)
        rows = keep[erank].contiguous()
        ecost = aug[erank].contiguous()
        _refit(xi, rows, ecost, params.sigma, params.gamma, mu, sig)  # :365-372
        sig_h = sig.cpu().numpy()
        b = int(rows[0].item())
        entry = torch.stack([ecost[0], scores[b], scores.min()]).cpu().numpy()
        history.append({"best_aug_cost": float(entry[0]), "best_residual": float(entry[1]),
                        "min_residual": float(entry[2])})
        if r == params.n_outer - 1:
            bx = xi[b].cpu().numpy()
            best = ProjectedSample(original=smp[b].cpu().numpy(), projected=bx, residual=float(entry[1]),
                                   trajectory=setup.trajectory_of(bx), aug_cost=float(entry[0]))
    return PriestResult(best=best, mu=mu.cpu().numpy(), sigma_mat=sig_h, history=history, params=params)


@dataclass
class CemResult:
    best_xi: np.ndarray
    best_cost: float
    best_trajectory: Trajectory
    mu: np.ndarray
    sigma_mat: np.ndarray
    history: list
    params: CemParams


def _priest_device_rounds(setup: ProjectionSetup, c1, distribution: SamplingDistribution,
                          params: PriestParams) -> PriestResult:
    """priest_optimize in throughput mode: every round (factor, draw, projection, scores, stable top-k,
    aug costs, elite top-k, refit, history entry) is enqueued on the device; one host read at the end."""
    d = setup.device()
    dev = d["device"]
    mu = torch.as_tensor(distribution.mu.copy(), device=dev)
    sig = torch.as_tensor(distribution.sigma_mat.copy(), device=dev)
    dm = mu.numel()
    sampler = _DeviceSampler(params.seed, params.n_batch, dm, dev)
    line = c1.line(dev)
    hist = torch.empty((params.n_outer, 3), dtype=torch.float64, device=dev)
    best_row = None
    xi = smp = scores = None
    for r in range(params.n_outer):
        sampler.factor(sig, d["L"])
        d["mu"].copy_(mu)
        xi, scores, _, smp = _run_project(setup, z=sampler.normals(r), n_inner=params.n_inner, keep_samples=True)
        keep = _topk(scores, params.n_constraint_elite)  # :358
        aug = _run_cost(setup, xi, keep, scores, 1.0, params.residual_weight, 0.0, line)  # :359-361
        erank = _topk(aug, params.n_elite)  # :362-363
        rows = keep[erank].contiguous()
        ecost = aug[erank].contiguous()
        _refit(xi, rows, ecost, params.sigma, params.gamma, mu, sig)  # :365-372
        best_row = rows[0]
        hist[r, 0] = ecost[0]
        hist[r, 1] = scores[best_row]
        hist[r, 2] = scores.min()
    h = hist.cpu().numpy()
    b = int(best_row.item())
    bx = xi[b].cpu().numpy()
    best = ProjectedSample(original=smp[b].cpu().numpy(), projected=bx, residual=float(h[-1, 1]),
                           trajectory=setup.trajectory_of(bx), aug_cost=float(h[-1, 0]))
    history = [{"best_aug_cost": float(e[0]), "best_residual": float(e[1]), "min_residual": float(e[2])} for e in h]
    return PriestResult(best=best, mu=mu.cpu().numpy(), sigma_mat=sig.cpu().numpy(), history=history, params=params)


def cem_optimize(setup: ProjectionSetup, c1, distribution: SamplingDistribution,
                 params: CemParams | None = None, *, sampler: str = "numpy") -> CemResult:
    """Plain cross-entropy baseline (solver_priest.py:422-457): no projection, penalty costs,
    unweighted elite refit — costs, top-k and refit on the GPU.  sampler: see priest_optimize."""
    params = params or CemParams()
    if sampler not in SAMPLERS:
        raise ValueError(f"sampler must be one of {SAMPLERS}")
    d = setup.device()
    dev = d["device"]
    rng = np.random.default_rng(params.seed)
    mu = torch.as_tensor(distribution.mu.copy(), device=dev)
    sig = torch.as_tensor(distribution.sigma_mat.copy(), device=dev)
    sig_h = distribution.sigma_mat.copy()
    dm = mu.numel()
    device_cost = isinstance(c1, BarnCost)
    line = c1.line(dev) if device_cost else None
    history = []
    best_xi, best_cost = None, np.inf
    dsamp = _DeviceSampler(params.seed, params.n_batch, dm, dev) if sampler == "philox" else None
    for it in range(params.iterations):
        if dsamp is not None:
            dsamp.factor(sig, d["L"])
            d["mu"].copy_(mu)
            z = dsamp.normals(it)
        else:
            d["L"].copy_(torch.as_tensor(_draw_factor(sig_h)))
            d["mu"].copy_(mu)
            z = torch.as_tensor(_draw_z(rng, params.n_batch, dm), device=dev)
        smp, _, _, _ = _run_project(setup, z=z, n_inner=-1)  # draw only
        if device_cost:
            costs = _run_cost(setup, smp, None, None, 1.0, 0.0, params.penalty_weight, line)
        else:
            sh = smp.cpu().numpy()
            base = torch.as_tensor(np.array([float(c1(setup.trajectory_of(x))) for x in sh]), device=dev)
            costs = base + params.penalty_weight * _run_cost(setup, smp, None, None, 0.0, 0.0, 1.0, d["line"])
        order = _topk(costs, params.n_elite)  # :440
        _refit(smp, order, costs[order].contiguous(), 1.0, 0.0, mu, sig, _lib.TRO_REFIT_CEM)  # :442-444
        if dsamp is None:
            sig_h = sig.cpu().numpy()
        c0 = float(costs[order[0]].item())
        if c0 < best_cost:
            best_cost = c0
            best_xi = smp[order[0]].cpu().numpy()
        history.append({"best_cost": c0, "mean_cost": float(costs.mean().item())})
    return CemResult(best_xi=best_xi, best_cost=best_cost, best_trajectory=setup.trajectory_of(best_xi),
                     mu=mu.cpu().numpy(), sigma_mat=sig.cpu().numpy(), history=history, params=params)


# ---------------------------------------------------------------- cost helpers (host, per trajectory)
def flatness_car(vel: np.ndarray, acc: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Forward speed and curvature of a planar trajectory (NaN below the speed threshold)."""
    vel = np.asarray(vel, dtype=float)
    acc = np.asarray(acc, dtype=float)
    speed = np.hypot(vel[:, 0], vel[:, 1])
    kappa = np.full_like(speed, np.nan)
    ok = speed > _SPEED_EPS
    kappa[ok] = (acc[ok, 1] * vel[ok, 0] - acc[ok, 0] * vel[ok, 1]) / speed[ok] ** 3
    return speed, kappa


def barn_cost(pos: np.ndarray, vel: np.ndarray, acc: np.ndarray, line_start, line_end) -> float:
    """Squared planar accelerations + squared curvature + squared distance to the start-goal line."""
    pos = np.asarray(pos, dtype=float)
    acc = np.asarray(acc, dtype=float)
    smooth = float(np.sum(acc[:, 0] ** 2 + acc[:, 1] ** 2))
    _, kappa = flatness_car(vel, acc)
    c_kappa = float(np.nansum(kappa**2))
    start = np.asarray(line_start, dtype=float)[:2]
    end = np.asarray(line_end, dtype=float)[:2]
    axis = end - start
    length = np.linalg.norm(axis)
    rel = pos[:, :2] - start
    if length < 1e-12:
        dist2 = (rel**2).sum(axis=1)
    else:
        along = rel @ (axis / length)
        dist2 = (rel**2).sum(axis=1) - along**2
    return smooth + c_kappa + float(np.sum(np.maximum(dist2, 0.0)))


# ---------------------------------------------------------------- multi-GPU (sample sharding)
class ShardedRound:
    """One priest_optimize round split into a per-rank LOCAL phase and a replicated GLOBAL phase.

    local(z_shard, lo): project this rank's samples [lo, hi), keep its stable top-min(N_ce, n) by score and
    pack (score, global index, xi, sample) rows.  The rank-ordered all-gather of those rows lists equal
    scores in ascending global index (ranks own contiguous ranges and each block is in stable order), so a
    stable top-k over the gathered scores IS the global np.argsort(scores, kind="stable")[:N_ce]
    (solver_priest.py:358).  global_(rows) then runs the costs, the elite top-k and the refit on the
    gathered rows; every rank computes it identically, so mu / Sigma stay replicated with no broadcast and
    the result is bitwise the single-GPU round."""

    def __init__(self, setup: ProjectionSetup, c1, params: PriestParams):
        self.setup, self.c1, self.params = setup, c1, params
        d = setup.device()
        self.dev = d["device"]
        self.dm = setup.dim * setup.m
        self.line = c1.line(self.dev) if isinstance(c1, BarnCost) else None

    def local(self, z_shard: torch.Tensor, lo: int) -> torch.Tensor:
        p = self.params
        xi, scores, _, smp = _run_project(self.setup, z=z_shard, n_inner=p.n_inner, keep_samples=True)
        k = min(p.n_constraint_elite, int(scores.numel()))
        cand = _topk(scores, k)
        return torch.cat([scores[cand, None], (cand + lo).double()[:, None], xi[cand], smp[cand]], dim=1)

    def global_(self, rows: torch.Tensor, mu: torch.Tensor, sig: torch.Tensor) -> dict:
        p, dm = self.params, self.dm
        g_scores = rows[:, 0].contiguous()
        g_xi = rows[:, 2:2 + dm].contiguous()
        keep = _topk(g_scores, min(p.n_constraint_elite, int(g_scores.numel())))
        if self.line is not None:
            aug = _run_cost(self.setup, g_xi, keep, g_scores, 1.0, p.residual_weight, 0.0, self.line)
        else:
            xk, sk = g_xi[keep].cpu().numpy(), g_scores[keep].cpu().numpy()
            aug = torch.as_tensor(np.array([float(self.c1(self.setup.trajectory_of(xk[i]))) + p.residual_weight
                                            * sk[i] for i in range(xk.shape[0])]), device=self.dev)
        erank = _topk(aug, p.n_elite)
        sel = keep[erank].contiguous()
        ecost = aug[erank].contiguous()
        _refit(g_xi, sel, ecost, p.sigma, p.gamma, mu, sig)
        b = int(sel[0].item())
        entry = torch.stack([ecost[0], g_scores[b], g_scores.min()]).cpu().numpy()
        return {"entry": entry, "best_row": rows[b]}


def priest_optimize_sharded(setup: ProjectionSetup, c1, distribution: SamplingDistribution,
                            params: PriestParams | None = None, *, z_rounds=None, group=None) -> PriestResult:
    """priest_optimize over the ranks of a torch.distributed group: samples shard into contiguous ranges
    (n_batch % world == 0), one all-gather of the candidate rows per round (see ShardedRound)."""
    import torch.distributed as dist

    from .distributed import shard_range

    params = params or PriestParams()
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if params.n_batch % world:
        raise ValueError("n_batch must be a multiple of the world size")
    lo, hi = shard_range(params.n_batch, rank, world)
    d = setup.device()
    dev = d["device"]
    rng = np.random.default_rng(params.seed)
    mu = torch.as_tensor(distribution.mu.copy(), device=dev)
    sig = torch.as_tensor(distribution.sigma_mat.copy(), device=dev)
    sig_h = distribution.sigma_mat.copy()
    rnd = ShardedRound(setup, c1, params)
    history, best = [], None
    for r in range(params.n_outer):
        d["L"].copy_(torch.as_tensor(_draw_factor(sig_h)))
        d["mu"].copy_(mu)
        if z_rounds is not None:
            z = _z_round(z_rounds[r][lo:hi], dev)
        else:  # every rank draws the whole round (the shared stream) and keeps its rows
            z = torch.as_tensor(_draw_z(rng, params.n_batch, mu.numel())[lo:hi], device=dev).contiguous()
        mine = rnd.local(z, lo)
        if world > 1:
            rows = torch.empty((world * mine.shape[0], mine.shape[1]), dtype=torch.float64, device=dev)
            dist.all_gather_into_tensor(rows, mine, group=group)
        else:
            rows = mine
        out = rnd.global_(rows, mu, sig)
        sig_h = sig.cpu().numpy()
        e = out["entry"]
        history.append({"best_aug_cost": float(e[0]), "best_residual": float(e[1]), "min_residual": float(e[2])})
        if r == params.n_outer - 1:
            row = out["best_row"].cpu().numpy()
            dm = rnd.dm
            bx = row[2:2 + dm]
            best = ProjectedSample(original=row[2 + dm:2 + 2 * dm], projected=bx, residual=float(e[1]),
                                   trajectory=setup.trajectory_of(bx), aug_cost=float(e[0]))
    return PriestResult(best=best, mu=mu.cpu().numpy(), sigma_mat=sig_h, history=history, params=params)
