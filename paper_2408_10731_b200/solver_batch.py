"""Batch 2-D trajectory optimization with a multi-circle footprint and heading (Alg. 2).

Drop-in for the reference ``trajopt.solver_batch`` (arXiv 2408.10731,
pkg/src/trajopt/solver_batch.py): same dataclasses, same functions, same
argument meaning and error behaviour.  The iterations run on the B200 through
``tro_b2_run`` (csrc/batch2d.cu, one CTA per member, one launch per
batch_iteration, replayed from CUDA graphs); numpy is only the interchange
format at the API boundary.

Device path per solve_batch_opt call (solver_batch.py:409-498):
  upload xi / xi_psi / psi / multipliers -> prime F'g (mode 1) -> max_iter fused
  iterations (mode 0, the batch-global stall rule runs on the device in the last CTA
  of each launch) -> ranking quantities (mode 3) -> download.
alpha_coll / d_coll / alpha_v / alpha_a / d_v / d_a are pure functions of (xi, psi)
after every step that writes them (:318-344); BatchState keeps them implied by a
snapshot of (xi, psi) and materialises them on the device (mode 2) when read.
"""

from __future__ import annotations

import ctypes
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch


def _graphs_allowed() -> bool:
    """CUDA-graph capture only on the main thread: a capture is invalidated by launches other threads make on
    the legacy default stream at the same time, so solver instances running in other threads launch their
    iterations directly (same kernels, same results)."""
    import threading

    return threading.current_thread() is threading.main_thread()

from . import _lib, qpcore
from ._alg1 import rho_chain
from .basis import AxisBoundary, BasisSet, Trajectory, boundary_matrix
from .geometry import D_CAP, ObstacleTrack  # noqa: F401  (re-exported like the reference module)

__all__ = [
    "FootprintSpec", "BatchProblem", "BatchParams", "BatchState", "RankedSolutions", "sample_initializations",
    "init_state", "batch_xi_step", "heading_step", "alpha_step", "d_step", "batch_iteration",
    "check_raw_feasibility", "solve_batch_opt",
]

_GEO = ("alpha_coll", "alpha_v", "alpha_a", "d_coll", "d_v", "d_a")


@dataclass(frozen=True)
class FootprintSpec:
    """Signed circle offsets along the body x-axis (meters) (solver_batch.py:27-39)."""

    offsets: tuple

    def __post_init__(self):
        if len(self.offsets) < 1:
            raise ValueError("footprint needs at least one circle")

    @property
    def n_c(self) -> int:
        return len(self.offsets)


@dataclass
class BatchProblem:
    """solver_batch.py:42-67."""

    basis: BasisSet
    boundary: tuple[AxisBoundary, AxisBoundary]  # x, y
    psi_boundary: tuple[float, float]
    desired: np.ndarray  # (n_p, 2)
    obstacles: list[ObstacleTrack]
    footprint: FootprintSpec
    v_max: float
    a_max: float
    n_batch: int
    w_smooth: float = 1.0
    w_track: float = 1.0

    def __post_init__(self):
        self.desired = np.asarray(self.desired, dtype=float)
        if self.v_max <= 0 or self.a_max <= 0:
            raise ValueError("v_max and a_max must be positive")
        if self.n_batch < 1:
            raise ValueError("batch size must be at least 1")
        if self.desired.shape != (self.basis.n_p, 2):
            raise ValueError("desired trajectory must be (n_p, 2)")

    @property
    def n_o(self) -> int:
        return len(self.obstacles)


@dataclass
class BatchParams:
    """solver_batch.py:70-81."""

    max_iter: int = 100
    tol: float = 1e-2
    rho_start: float = 1.0
    rho_growth: float = 1.4
    # cap keeps the shared saddle within the qp-core conditioning guard
    rho_cap: float = 1e3
    stall_window: int = 5
    stall_improvement: float = 0.01
    d_margin: float = 1e-2
    kin_margin: float = 1e-2


class BatchState:
    """solver_batch.py:84-104.  xi / xi_psi / psi / lam / lam_psi are numpy arrays owned by the
    caller (mutations are honoured).  The six alpha / d arrays are implied by the (xi, psi)
    snapshot of the last step that wrote them and materialised on the device when read;
    assigning one makes all six explicit."""

    def __init__(self, xi, xi_psi, psi, lam, lam_psi, rho, rho_psi, iteration=0, n_factorizations=0, **geo):
        self.xi = xi
        self.xi_psi = xi_psi
        self.psi = psi
        self.lam = lam
        self.lam_psi = lam_psi
        self.rho = rho
        self.rho_psi = rho_psi
        self.iteration = iteration
        self.n_factorizations = n_factorizations
        self._factor_rho = None
        self._psi_targets = None
        self._geo: dict | None = None  # explicit arrays
        self._implied: tuple | None = None  # (xi, psi, struct) snapshot the arrays are functions of
        if geo:
            missing = [k for k in _GEO if k not in geo]
            if missing:
                raise TypeError(f"missing state arrays {missing}")
            self._geo = {k: np.asarray(geo[k], dtype=float) for k in _GEO}

    # ---- lazily materialised alpha / d arrays
    def _imply(self, struct):
        """alpha / d are now alpha_step + d_step of the current (xi, psi) for struct's problem."""
        self._geo = None
        self._implied = (self.xi.copy(), self.psi.copy(), struct)

    def _implied_now(self, struct) -> bool:
        return (self._geo is None and self._implied is not None and self._implied[2].key == struct.key
                and np.array_equal(self._implied[0], self.xi) and np.array_equal(self._implied[1], self.psi))

    def _materialise(self) -> dict:
        if self._geo is None:
            if self._implied is None:
                raise AttributeError("state has no alpha / d arrays")
            xi, psi, struct = self._implied
            self._geo = _device_geometry(struct, xi, psi)
        return self._geo

    def __repr__(self):
        return f"BatchState(n_b={self.xi.shape[0]}, rho={self.rho!r}, iteration={self.iteration})"


def _geo_property(name):
    def get(self):
        return self._materialise()[name]

    def set_(self, value):
        self._materialise()[name] = np.asarray(value, dtype=float)

    return property(get, set_)


for _name in _GEO:
    setattr(BatchState, _name, _geo_property(_name))


class _TrajectoryList(Sequence):
    """RankedSolutions.trajectories: one Trajectory per member, built on access (:473-485)."""

    def __init__(self, basis, xi, psi, m):
        self._basis, self._xi, self._psi, self._m = basis, xi, psi, m

    def __len__(self):
        return self._xi.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        b, m = self._basis, self._m
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        coeffs = np.column_stack([self._xi[i, :m], self._xi[i, 2 * m:3 * m]])
        return Trajectory(t=b.grid.timestamps, pos=b.P @ coeffs, vel=b.Pdot @ coeffs, acc=b.Pddot @ coeffs,
                          psi=self._psi[i])


@dataclass
class RankedSolutions:
    """solver_batch.py:107-123."""

    trajectories: Sequence
    costs: np.ndarray
    aug_costs: np.ndarray
    residual_max: np.ndarray
    residual_norm: np.ndarray
    feasible: np.ndarray
    best_index: int | None
    best_history: list
    iterations: int
    n_factorizations: int
    state: BatchState

    @property
    def best(self) -> Trajectory | None:
        return self.trajectories[self.best_index] if self.best_index is not None else None


def sample_initializations(mean: np.ndarray, covariance: np.ndarray, n_batch: int, seed) -> np.ndarray:
    """Draw coefficient samples from N(mean, covariance), deterministic per seed (:126-138).

    The host numpy Generator is kept so the stream matches the reference draw for draw."""
    mean = np.asarray(mean, dtype=float)
    covariance = np.asarray(covariance, dtype=float)
    if covariance.shape != (mean.size, mean.size):
        raise ValueError("covariance shape does not match mean")
    if not np.allclose(covariance, covariance.T, atol=1e-10):
        raise ValueError("covariance must be symmetric")
    eigs = np.linalg.eigvalsh(covariance)
    if eigs.min() < -1e-10 * max(1.0, abs(eigs.max())):
        raise ValueError("covariance must be positive semi-definite")
    rng = np.random.default_rng(seed)
    return rng.multivariate_normal(mean, covariance, size=n_batch, method="svd")


def _fingerprint(problem: BatchProblem) -> bytes:
    """Content key of everything _Structure depends on (problems are mutable dataclasses)."""
    import hashlib

    h = hashlib.blake2b(digest_size=20)
    b = problem.basis
    for a in (b.P, b.Pdot, b.Pddot, problem.desired):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    for o in problem.obstacles:
        h.update(np.ascontiguousarray(o.centers, dtype=np.float64).tobytes())
        h.update(np.array([o.shape.a, o.shape.b], dtype=np.float64).tobytes())
    h.update(np.array([v for bc in problem.boundary for v in bc.values()] + list(problem.psi_boundary)
                      + list(problem.footprint.offsets)
                      + [problem.v_max, problem.a_max, problem.w_smooth, problem.w_track, problem.n_o],
                      dtype=np.float64).tobytes())
    return h.digest()


_STRUCT_CACHE: dict = {}


def _structure_for(problem: BatchProblem) -> "_Structure":
    key = _fingerprint(problem)
    st = _STRUCT_CACHE.get(key)
    if st is None:
        if len(_STRUCT_CACHE) > 16:
            _STRUCT_CACHE.clear()
            _ENGINE_CACHE.clear()
        st = _STRUCT_CACHE[key] = _Structure(problem, key=key)
    return st


class _Structure:
    """Constant matrices of one BatchProblem (solver_batch.py:141-193) plus their device copies."""

    def __init__(self, problem: BatchProblem, key: bytes | None = None):
        self.key = key if key is not None else _fingerprint(problem)
        basis = problem.basis
        m, n_p = basis.n_var, basis.n_p
        self.problem = problem
        self.m = m
        P, Pdot, Pddot = basis.P, basis.Pdot, basis.Pddot
        zeros = np.zeros((n_p, m))
        half_rows = [np.hstack([Pdot, zeros]), np.hstack([Pddot, zeros])]
        for r_c in problem.footprint.offsets:
            for _ in range(problem.n_o):
                half_rows.append(np.hstack([P, r_c * P]))
        half_rows.append(np.hstack([zeros, P]))
        F_half = np.vstack(half_rows)
        self._F_half = F_half
        Fh = F_half.T @ F_half
        self.FtF = np.zeros((4 * m, 4 * m))
        self.FtF[: 2 * m, : 2 * m] = Fh
        self.FtF[2 * m:, 2 * m:] = Fh
        cost_xx = problem.w_smooth * Pddot.T @ Pddot + problem.w_track * P.T @ P
        self.Q = np.zeros((4 * m, 4 * m))
        self.Q[:m, :m] = cost_xx
        self.Q[2 * m:3 * m, 2 * m:3 * m] = cost_xx
        self.q = np.concatenate([-problem.w_track * P.T @ problem.desired[:, 0], np.zeros(m),
                                 -problem.w_track * P.T @ problem.desired[:, 1], np.zeros(m)])
        B = boundary_matrix(basis)
        self.A = np.zeros((12, 4 * m))
        self.A[:6, :m] = B
        self.A[6:, 2 * m:3 * m] = B
        self.b = np.concatenate([problem.boundary[0].values(), problem.boundary[1].values()])
        self.A_psi = np.vstack([P[0], P[-1]])
        self.b_psi = np.asarray(problem.psi_boundary, dtype=float)
        self.Q_psi_smooth = Pddot.T @ Pddot
        self.obs_x = np.stack([o.centers[:, 0] for o in problem.obstacles]) if problem.n_o else np.zeros((0, n_p))
        self.obs_y = np.stack([o.centers[:, 1] for o in problem.obstacles]) if problem.n_o else np.zeros((0, n_p))
        self.obs_a = np.array([o.shape.a for o in problem.obstacles])
        self.obs_b = np.array([o.shape.b for o in problem.obstacles])
        self.r = np.asarray(problem.footprint.offsets, dtype=float)
        self._dev = {}

    @property
    def F(self) -> np.ndarray:
        """The stacked constraint matrix (never used by the device path, which contracts by blocks)."""
        Fh = self._F_half
        z = np.zeros_like(Fh)
        return np.block([[Fh, z], [z, Fh]])

    def device(self, dev) -> dict:
        key = str(dev)
        c = self._dev.get(key)
        if c is None:
            pb, basis = self.problem, self.problem.basis
            f64 = dict(dtype=torch.float64, device=dev)
            mats = (basis.P, basis.Pdot, basis.Pddot)
            obs = np.zeros((max(pb.n_o, 1), 2, basis.n_p))
            if pb.n_o:
                obs[:, 0], obs[:, 1] = self.obs_x, self.obs_y
            ab = np.zeros((max(pb.n_o, 1), 2))
            if pb.n_o:
                ab[:, 0], ab[:, 1] = self.obs_a, self.obs_b
            c = dict(
                PT=torch.as_tensor(np.stack([M.T for M in mats]), **f64).contiguous(),
                Pr=torch.as_tensor(np.stack(mats), **f64).contiguous(),
                obs=torch.as_tensor(obs, **f64).contiguous(),
                obs_ab=torch.as_tensor(ab, **f64).contiguous(),
                offsets=torch.as_tensor(self.r, **f64),
                q=torch.as_tensor(self.q, **f64),
                b=torch.as_tensor(self.b, **f64),
                b_psi=torch.as_tensor(self.b_psi, **f64),
                desired=torch.as_tensor(pb.desired, **f64).contiguous(),
            )
            self._dev[key] = c
        return c


# ------------------------------------------------------------------ rho levels (K^-1 tables)
_LEVEL_CACHE: dict = {}


class _Levels:
    """K_xi^-1 / K_psi^-1 for every rho on the min(rho * growth, cap) chains (_ensure_factors, :281-289)."""

    def __init__(self, struct: _Structure, rho0: float, rho_psi0: float, growth: float, cap: float):
        basis = struct.problem.basis
        m = struct.m
        chain = rho_chain(rho0, growth, cap)
        chain_p = rho_chain(rho_psi0, growth, cap)
        n = max(len(chain), len(chain_p))
        chain += [chain[-1]] * (n - len(chain))
        chain_p += [chain_p[-1]] * (n - len(chain_p))
        self.rho, self.rho_psi = chain, chain_p
        nv, nk = 4 * m, 4 * m + 12
        self.kinvT_xi = np.zeros((n, nk, nk))
        self.k_xi = np.zeros((n, nk, nk))
        self.kinvT_psi = np.zeros((n, m + 2, m))
        PtP = basis.P.T @ basis.P
        self.error: list = [None] * n
        for k in range(n):
            try:
                fx = qpcore._build(struct.Q + chain[k] * struct.FtF, struct.A, 1e12)
                fp = qpcore._build(struct.Q_psi_smooth + chain_p[k] * PtP, struct.A_psi, 1e12)
            except qpcore.FactorizationError as exc:
                if k == 0 or "rank-deficient" in str(exc):
                    raise
                self.error[k] = exc  # a level the schedule may never reach: fail when it does
                continue
            self.kinvT_xi[k] = fx.kinv.T
            self.k_xi[k] = qpcore.saddle_matrix(struct.Q + chain[k] * struct.FtF, struct.A)
            self.kinvT_psi[k] = fp.kinv[:m, :].T
        self._dev = {}

    def device(self, dev):
        key = str(dev)
        t = self._dev.get(key)
        if t is None:
            f64 = dict(dtype=torch.float64, device=dev)
            t = dict(kinvT_xi=torch.as_tensor(self.kinvT_xi, **f64).contiguous(),
                     k_xi=torch.as_tensor(self.k_xi, **f64).contiguous(),
                     kinvT_psi=torch.as_tensor(self.kinvT_psi, **f64).contiguous(),
                     rho=torch.as_tensor(self.rho, **f64), rho_psi=torch.as_tensor(self.rho_psi, **f64))
            self._dev[key] = t
        return t


def _levels(struct: _Structure, rho0: float, rho_psi0: float, growth: float, cap: float) -> _Levels:
    pb, basis = struct.problem, struct.problem.basis
    key = (basis.P.tobytes(), basis.Pdot.tobytes(), basis.Pddot.tobytes(), pb.n_o, tuple(map(float, struct.r)),
           float(pb.w_smooth), float(pb.w_track), float(rho0), float(rho_psi0), float(growth), float(cap))
    lv = _LEVEL_CACHE.get(key)
    if lv is None:
        if len(_LEVEL_CACHE) > 32:
            _LEVEL_CACHE.clear()
        lv = _LEVEL_CACHE[key] = _Levels(struct, rho0, rho_psi0, growth, cap)
    return lv


# ------------------------------------------------------------------ device engine
class _Engine:
    """Device-resident state of one batch and the tro_b2_run launch sequence."""

    def __init__(self, struct: _Structure, n_b: int, levels: _Levels, *, params: BatchParams | None = None,
                 max_hist: int = 0, geo: bool = False, device=None, member_offset: int | None = None):
        _lib.require_cuda()
        self.lib = _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.struct, self.levels = struct, levels
        pb = struct.problem
        m, n_p, n_o, n_c = struct.m, pb.basis.n_p, pb.n_o, pb.footprint.n_c
        self.B, self.m, self.n_p, self.n_o, self.n_c = int(n_b), m, n_p, n_o, n_c
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.xi = torch.zeros((n_b, 4 * m), **f64)
        self.xi_psi = torch.zeros((n_b, m), **f64)
        self.lam = torch.zeros((n_b, 4 * m), **f64)
        self.lam_psi = torch.zeros((n_b, m), **f64)
        self.sums = torch.zeros((n_b, 4 * m), **f64)
        self.psi = torch.zeros((n_b, n_p), **f64)
        self.res_max = torch.zeros(n_b, **f64)
        self.res_norm = torch.zeros(n_b, **f64)
        self.rank = torch.zeros((n_b, 6), **f64)
        self.psi_targets = None
        p = params or BatchParams()
        self.ring = torch.zeros(max(2 * p.stall_window, 1), **f64)
        self.max_hist = int(max_hist)
        self.hist = torch.zeros((max(self.max_hist, 1), 4), **f64)
        self.ints = torch.zeros(5, **i32)  # level, iteration, last_change, n_hist, n_changes
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        # sharded batch (multi-GPU Alg. 2): mode 0 writes this shard's summary; mode 6 merges them
        self.member_offset = member_offset
        self.shard = torch.zeros(4, **f64) if member_offset is not None else None
        self.shards_in = None
        self.geo = {}
        if geo:
            self._alloc_geo()
        self.params = p
        self.flags = _lib.TRO_B2_PSI_IN
        if n_o and np.array_equal(struct.obs_a, struct.obs_b):
            self.flags |= _lib.TRO_B2_CIRCLES  # circle fast path (the benchmark recipes)
        self._graph = None
        self._graph_n = 0
        self._pin = {}
        self.h2d_bytes = self.d2h_bytes = 0
        c = struct.device(dev)
        lv = levels.device(dev)
        self._keep = (c, lv)
        self.dims = _lib.B2Dims(n_members=n_b, n_obs=n_o, n_c=n_c, n_p=n_p, m=m, n_levels=len(levels.rho),
                                max_hist=self.max_hist)
        P = _lib.ptr
        self.consts = _lib.B2Consts(
            PT=P(c["PT"]), Pr=P(c["Pr"]), obs=P(c["obs"]), obs_ab=P(c["obs_ab"]), offsets=P(c["offsets"]),
            q=P(c["q"]), b=P(c["b"]), b_psi=P(c["b_psi"]), kinvT_xi=P(lv["kinvT_xi"]),
            kinvT_psi=P(lv["kinvT_psi"]), rho_chain=P(lv["rho"]), rho_psi_chain=P(lv["rho_psi"]),
            desired=P(c["desired"]), v_max=float(pb.v_max), a_max=float(pb.a_max), w_smooth=float(pb.w_smooth),
            w_track=float(pb.w_track), k_xi=P(lv["k_xi"]))
        self._state_struct()

    def _alloc_geo(self):
        f64 = dict(dtype=torch.float64, device=self.device)
        B, n_c, n_o, n_p = self.B, self.n_c, self.n_o, self.n_p
        self.geo = dict(alpha_coll=torch.zeros((B, n_c, n_o, n_p), **f64), d_coll=torch.zeros((B, n_c, n_o, n_p), **f64),
                        alpha_v=torch.zeros((B, n_p), **f64), alpha_a=torch.zeros((B, n_p), **f64),
                        d_v=torch.zeros((B, n_p), **f64), d_a=torch.zeros((B, n_p), **f64))
        self._state_struct()

    def _state_struct(self, geo_out: tuple = _GEO):
        P = _lib.ptr
        ints = self.ints
        base = ints.data_ptr()
        g = {k: (P(self.geo[k]) if (k in self.geo and k in geo_out) else None) for k in _GEO}
        self.state = _lib.B2State(
            xi=P(self.xi), xi_psi=P(self.xi_psi), lam=P(self.lam), lam_psi=P(self.lam_psi), sums=P(self.sums),
            res_max=P(self.res_max), res_norm=P(self.res_norm), ring=P(self.ring), hist=P(self.hist),
            level=base, iteration=base + 4, last_change=base + 8, n_hist=base + 12, n_changes=base + 16,
            counter=P(self.counter), psi=P(self.psi), rank=P(self.rank),
            psi_targets=P(self.psi_targets) if self.psi_targets is not None else None,
            shard=P(self.shard), shards_in=P(self.shards_in), **g)

    # ---- host <-> device
    def _pinned(self, name, like):
        buf = self._pin.get(name)
        if buf is None or buf.shape != like.shape or buf.dtype != like.dtype:
            buf = torch.empty(like.shape, dtype=like.dtype, pin_memory=True)
            self._pin[name] = buf
        return buf

    def load(self, state: BatchState, level: int = 0):
        """Upload the state through pinned staging buffers (asynchronous H2D on the current stream)."""
        for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
            dst = getattr(self, name)
            pin = self._pinned(name, dst)
            pin.numpy()[...] = getattr(state, name)
            dst.copy_(pin, non_blocking=True)
        ints = self._pinned("ints", self.ints)
        ints.numpy()[...] = (level, int(state.iteration), 0, 0, 0)
        self.ints.copy_(ints, non_blocking=True)
        self.counter.zero_()
        self.ring.zero_()
        self.h2d_bytes = sum(getattr(self, n).numel() * 8 for n in ("xi", "xi_psi", "psi", "lam", "lam_psi")) + 20

    def fetch(self, names) -> dict:
        """Download device tensors through pinned buffers with one synchronisation."""
        out = {}
        for name in names:
            src = getattr(self, name)
            pin = self._pinned("out_" + name, src)
            pin.copy_(src, non_blocking=True)
            out[name] = pin
        torch.cuda.current_stream(self.device).synchronize()
        self.d2h_bytes = sum(v.numel() * v.element_size() for v in out.values())
        return {k: v.numpy().copy() for k, v in out.items()}

    def load_geo(self, geo: dict):
        if not self.geo:
            self._alloc_geo()
        for k in _GEO:
            self.geo[k].copy_(torch.as_tensor(np.ascontiguousarray(geo[k], dtype=np.float64)))

    def run_mode(self, mode: int, flags: int | None = None, n_shards: int = 0):
        fl = int(self.flags if flags is None else flags)
        if self.member_offset is not None and mode == 0:
            fl |= _lib.TRO_B2_SHARD
        prm = _lib.B2Params(tol=float(self.params.tol), stall_improvement=float(self.params.stall_improvement),
                            stall_window=int(self.params.stall_window), flags=fl,
                            member_offset=int(self.member_offset or 0), n_shards=int(n_shards))
        with torch.cuda.device(self.device):
            rc = self.lib.tro_b2_run(mode, ctypes.byref(self.dims), ctypes.byref(self.consts),
                                     ctypes.byref(self.state), ctypes.byref(prm), _lib.stream_handle())
        _lib.check(rc, f"tro_b2_run(mode={mode})")

    def prime(self, given: bool = False):
        self.run_mode(1, self.flags | (_lib.TRO_B2_GIVEN_AD if given else 0))

    def iterate(self, schedule: bool = True):
        self.run_mode(0, self.flags | (0 if schedule else _lib.TRO_FLAG_NO_SCHEDULE))

    def merge(self, gathered: torch.Tensor):
        """Mode 6: merge the all-gathered shard summaries (world x 4, rank order), apply the schedule."""
        if self.shards_in is None or self.shards_in.data_ptr() != gathered.data_ptr():
            self.shards_in = gathered
            self._state_struct()
        self.run_mode(6, n_shards=int(gathered.shape[0]))

    def _capture(self, n: int):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            for _ in range(n):
                self.iterate()
        self._graph, self._graph_n = g, n

    def run(self, n_iter: int, *, use_graph: bool = True, chunk: int = 25):
        done = 0
        while done < n_iter:
            n = min(chunk, n_iter - done)
            if use_graph and n == chunk and _graphs_allowed():
                if self._graph is None or self._graph_n != chunk:
                    self._capture(chunk)
                self._graph.replay()
            else:
                for _ in range(n):
                    self.iterate()
            done += n
        return done

    def ints_host(self):
        v = self.ints.cpu().numpy()
        return dict(level=int(v[0]), iteration=int(v[1]), last_change=int(v[2]), n_hist=int(v[3]),
                    n_changes=int(v[4]))


def _rho_level(levels: _Levels, rho: float, rho_psi: float) -> int:
    for k, (r, rp) in enumerate(zip(levels.rho, levels.rho_psi)):
        if r == rho and rp == rho_psi:
            return k
    raise ValueError(f"rho {rho!r} is not on the level chain")


def _device_geometry(struct: _Structure, xi, psi, alpha=None) -> dict:
    """alpha_step + d_step of (xi, psi) on the device (mode 2); alpha given -> d_step alone."""
    lv = _levels(struct, 1.0, 1.0, 1.4, 1e3)
    n_b = xi.shape[0]
    eng = _Engine(struct, n_b, lv, geo=True)
    st = BatchState(xi=xi, xi_psi=np.zeros((n_b, struct.m)), psi=psi, lam=np.zeros_like(xi),
                    lam_psi=np.zeros((n_b, struct.m)), rho=1.0, rho_psi=1.0)
    eng.load(st)
    flags = _lib.TRO_B2_PSI_IN
    if alpha is not None:
        for k in ("alpha_coll", "alpha_v", "alpha_a"):
            eng.geo[k].copy_(torch.as_tensor(np.ascontiguousarray(alpha[k], dtype=np.float64)))
        flags |= _lib.TRO_B2_GIVEN_ALPHA
    eng.run_mode(2, flags)
    out = {k: v.cpu().numpy() for k, v in eng.geo.items()}
    if alpha is not None:
        out.update({k: np.array(alpha[k], dtype=float) for k in ("alpha_coll", "alpha_v", "alpha_a")})
    return out


# ------------------------------------------------------------------ reference API
def init_state(problem: BatchProblem, samples: np.ndarray, params: BatchParams | None = None, *,
               _struct: "_Structure | None" = None) -> BatchState:
    """State from position-coefficient samples (N_b, 2m): [xi_x | xi_y] (solver_batch.py:234-278).

    The heading is seeded from the desired-path direction; copies, angles and scales are made
    consistent with the sampled geometry (implied, materialised on the device when read);
    multipliers start at zero."""
    params = params or BatchParams()
    struct = _struct if _struct is not None else _structure_for(problem)  # solve_batch_opt passes its own
    basis, m = problem.basis, struct.m
    samples = np.asarray(samples, dtype=float)
    n_b = samples.shape[0]
    if samples.shape != (n_b, 2 * m):
        raise ValueError(f"expected samples of shape (N_b, {2 * m})")
    path_dir = np.gradient(problem.desired, axis=0)
    psi_des = np.unwrap(np.arctan2(path_dir[:, 1], path_dir[:, 0]))
    xi_psi_one, *_ = np.linalg.lstsq(basis.P, psi_des, rcond=None)
    xi_psi = np.tile(xi_psi_one, (n_b, 1))
    psi = xi_psi @ basis.P.T
    xi_c_one, *_ = np.linalg.lstsq(basis.P, np.cos(psi_des), rcond=None)
    xi_s_one, *_ = np.linalg.lstsq(basis.P, np.sin(psi_des), rcond=None)
    xi = np.hstack([samples[:, :m], np.tile(xi_c_one, (n_b, 1)), samples[:, m:], np.tile(xi_s_one, (n_b, 1))])
    state = BatchState(xi=xi, xi_psi=xi_psi, psi=psi, lam=np.zeros((n_b, 4 * m)), lam_psi=np.zeros((n_b, m)),
                       rho=params.rho_start, rho_psi=params.rho_start)
    state._imply(struct)  # alpha_step + d_step (:276-277) of the initial (xi, psi)
    return state


def _ensure_factors(state: BatchState, levels: _Levels, level: int) -> None:
    """_ensure_factors bookkeeping (:281-289): two factorizations per new rho value."""
    if levels.error[level] is not None:
        raise levels.error[level]
    rho = levels.rho[level]
    if state._factor_rho is not None and state._factor_rho == rho:
        return
    state._factor_rho = rho
    state.n_factorizations += 2
    qpcore._bump(2)


_ENGINE_CACHE: dict = {}


def _owner_key():
    """Cached engines are single-owner: one per (thread, device, stream), so concurrent calls
    never share device buffers, the captured graph or the grid ticket."""
    import threading

    dev = torch.cuda.current_device()
    return (threading.get_ident(), dev, torch.cuda.current_stream(dev).cuda_stream)


def _engine_for(state: BatchState, problem: BatchProblem, struct: _Structure, params: BatchParams | None = None,
                max_hist: int = 0, cached: bool = False):
    """Engine loaded with the state; `given` = alpha / d must be read from explicit arrays.

    cached=True reuses the device buffers and the captured CUDA graph of an earlier call with the
    same problem content, batch size and parameters (one solver per stream)."""
    p = params or BatchParams()
    lv = _levels(struct, float(state.rho), float(state.rho_psi), p.rho_growth, p.rho_cap)
    n_b = state.xi.shape[0]
    eng = None
    if cached:
        key = (struct.key, n_b, float(state.rho), float(state.rho_psi), float(p.rho_growth), float(p.rho_cap),
               float(p.tol), float(p.stall_improvement), int(p.stall_window), int(max_hist), _owner_key())
        eng = _ENGINE_CACHE.get(key)
        if eng is None:
            if len(_ENGINE_CACHE) > 8:
                _ENGINE_CACHE.clear()
            eng = _ENGINE_CACHE[key] = _Engine(struct, n_b, lv, params=p, max_hist=max_hist)
    if eng is None:
        eng = _Engine(struct, n_b, lv, params=p, max_hist=max_hist)
    eng.load(state, 0)
    given = not state._implied_now(struct)
    if given:
        eng.load_geo(state._materialise())
    return eng, lv, given


def _download(eng: _Engine, state: BatchState, *, xi=True, xi_psi=True, psi=True, lam=True):
    if xi:
        state.xi = eng.xi.cpu().numpy()
    if xi_psi:
        state.xi_psi = eng.xi_psi.cpu().numpy()
    if psi:
        state.psi = eng.psi.cpu().numpy()
    if lam:
        state.lam = eng.lam.cpu().numpy()
        state.lam_psi = eng.lam_psi.cpu().numpy()


def batch_xi_step(state: BatchState, problem: BatchProblem, struct: _Structure | None = None) -> None:
    """Shared-factor QP update of every member's stacked coefficients (:292-299)."""
    struct = struct or _structure_for(problem)
    eng, lv, given = _engine_for(state, problem, struct)
    _ensure_factors(state, lv, 0)
    eng.prime(given)  # F'g of the state's alpha / d / psi (:296)
    eng.run_mode(4)
    _download(eng, state, xi_psi=False, psi=False, lam=False)


def heading_step(state: BatchState, problem: BatchProblem, struct: _Structure | None = None) -> None:
    """Fit the heading block to unwrapped arctan2 targets from the copies (:302-315)."""
    struct = struct or _structure_for(problem)
    lv = _levels(struct, float(state.rho), float(state.rho_psi), BatchParams.rho_growth, BatchParams.rho_cap)
    eng = _Engine(struct, state.xi.shape[0], lv)
    eng.load(state, 0)
    _ensure_factors(state, lv, 0)
    eng.psi_targets = torch.zeros((eng.B, eng.n_p), dtype=torch.float64, device=eng.device)
    eng._state_struct()
    eng.run_mode(5)
    _download(eng, state, xi=False, lam=False)
    state._psi_targets = eng.psi_targets.cpu().numpy()


def alpha_step(state: BatchState, problem: BatchProblem, struct: _Structure | None = None) -> None:
    """alpha_coll / alpha_v / alpha_a of the current (xi, psi) (:318-326); d unchanged."""
    struct = struct or _structure_for(problem)
    if state._implied_now(struct):
        return  # already functions of this (xi, psi)
    geo = dict(state._materialise())
    fresh = _device_geometry(struct, state.xi, state.psi)
    for k in ("alpha_coll", "alpha_v", "alpha_a"):
        geo[k] = fresh[k]
    state._geo = geo


def d_step(state: BatchState, problem: BatchProblem, struct: _Structure | None = None) -> None:
    """Clamped scales of the current (xi, psi) and the state's alpha (:329-344)."""
    struct = struct or _structure_for(problem)
    if state._implied_now(struct):
        return
    geo = state._materialise()
    fresh = _device_geometry(struct, state.xi, state.psi, alpha=geo)
    for k in ("d_coll", "d_v", "d_a"):
        geo[k] = fresh[k]


def batch_iteration(state: BatchState, problem: BatchProblem, struct: _Structure | None = None) -> BatchState:
    """One fused device iteration (:352-363): xi step, heading step, alpha, d, multipliers."""
    struct = struct or _structure_for(problem)
    eng, lv, given = _engine_for(state, problem, struct)
    _ensure_factors(state, lv, 0)
    eng.prime(given)
    eng.iterate(schedule=False)
    _download(eng, state)
    state.iteration += 1
    state._imply(struct)
    return state


def check_raw_feasibility(state, problem, struct, d_margin, kin_margin):
    """Direct evaluation of the original quadratic constraints per member (:377-393), on the device."""
    struct = struct or _structure_for(problem)
    rank = _rank(state, problem, struct)
    return _feasible_from_rank(rank, problem, d_margin, kin_margin)


def _feasible_from_rank(rank, problem, d_margin, kin_margin):
    ok = np.ones(rank.shape[0], dtype=bool)
    if problem.n_o:
        ok &= rank[:, 2] >= 1.0 - d_margin
    ok &= rank[:, 3] <= problem.v_max * (1.0 + kin_margin)
    ok &= rank[:, 4] <= problem.a_max * (1.0 + kin_margin)
    return ok


def _rank(state, problem, struct):
    eng, _, given = _engine_for(state, problem, struct)
    eng.run_mode(3, eng.flags | (_lib.TRO_B2_GIVEN_AD if given else 0))
    return eng.rank.cpu().numpy()


def _default_samples(problem: BatchProblem, m: int, mean, covariance, seed):
    """solver_batch.py:430-445."""
    basis = problem.basis
    if mean is None:
        bx, by = problem.boundary
        line = np.linalg.lstsq(
            basis.P,
            np.column_stack([np.linspace(bx.p0, bx.p1, basis.n_p), np.linspace(by.p0, by.p1, basis.n_p)]),
            rcond=None,
        )[0]
        mean = np.concatenate([line[:, 0], line[:, 1]])
    if covariance is None:
        bx, by = problem.boundary
        scale = max(np.hypot(bx.p1 - bx.p0, by.p1 - by.p0) / 10.0, 0.5)
        covariance = np.eye(2 * m) * scale**2
    return sample_initializations(mean, covariance, problem.n_batch, seed)


def solve_batch_opt(
    problem: BatchProblem,
    params: BatchParams | None = None,
    *,
    samples: np.ndarray | None = None,
    mean: np.ndarray | None = None,
    covariance: np.ndarray | None = None,
    seed=0,
    state: BatchState | None = None,
    use_graph: bool = True,
) -> RankedSolutions:
    """Run the batch optimizer and rank members (solver_batch.py:409-498).

    Members are initialized from explicit coefficient samples, or drawn from N(mean,
    covariance) (defaults: straight-line mean, diagonal covariance scaled to the start-goal
    distance).  Passing state warm-starts.  All iterations run on the device."""
    params = params or BatchParams()
    struct = _structure_for(problem)
    m = struct.m
    if state is None:
        if samples is None:
            samples = _default_samples(problem, m, mean, covariance, seed)
        state = init_state(problem, samples, params, _struct=struct)  # one content fingerprint per call
        state._implied = (state._implied[0], state._implied[1], struct)

    eng, lv, given = _engine_for(state, problem, struct, params, max_hist=params.max_iter, cached=True)
    n_iter = int(params.max_iter)
    if n_iter > 0:
        _ensure_factors(state, lv, 0)
        eng.prime(given)
        eng.run(n_iter, use_graph=use_graph)
    eng.run_mode(3, eng.flags | (_lib.TRO_B2_GIVEN_AD if (given and n_iter == 0) else 0))
    got = eng.fetch(("ints", "hist", "rank") + (("xi", "xi_psi", "psi", "lam", "lam_psi") if n_iter > 0 else ()))
    v = got["ints"]
    ints = dict(level=int(v[0]), iteration=int(v[1]), last_change=int(v[2]), n_hist=int(v[3]), n_changes=int(v[4]))
    hist = got["hist"][: ints["n_hist"]] if n_iter > 0 else np.zeros((0, 4))
    rank = got["rank"]
    if n_iter > 0:
        for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
            setattr(state, name, got[name])
        state.iteration += n_iter
        level = ints["level"]
        # a factor pair is built by the first batch_xi_step at each new rho (:282-289); a growth decided
        # after the last iteration is never factorized.  Levels are visited in order.
        used = _rho_level(lv, float(hist[-1, 2]), lv.rho_psi[lv.rho.index(float(hist[-1, 2]))])
        for k in range(1, used + 1):
            _ensure_factors(state, lv, k)
        state.rho, state.rho_psi = lv.rho[level], lv.rho_psi[level]
        state._imply(struct)
    best_history = [{"norm": float(h[0]), "max_abs": float(h[1]), "rho": float(h[2])} for h in hist]

    residual_max, residual_norm = rank[:, 0].copy(), rank[:, 1].copy()
    feasible = (residual_max <= params.tol) & _feasible_from_rank(rank, problem, params.d_margin,
                                                                  params.kin_margin)
    costs = rank[:, 5].copy()
    aug_costs = costs + state.rho * residual_norm
    best_index = int(np.argmin(np.where(feasible, aug_costs, np.inf))) if feasible.any() else None
    return RankedSolutions(
        trajectories=_TrajectoryList(problem.basis, state.xi, state.psi, m),
        costs=costs,
        aug_costs=aug_costs,
        residual_max=residual_max,
        residual_norm=residual_norm,
        feasible=feasible,
        best_index=best_index,
        best_history=best_history,
        iterations=state.iteration,
        n_factorizations=state.n_factorizations,
        state=state,
    )
