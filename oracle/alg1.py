"""CPU ORACLE for the batched Alg. 1 AM/AL iteration — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker /
the reference CPU arm.  The product path (``paper_2408_10731_b200``) never
imports it and has no CPU fallback.

This is a numpy restatement of the reference ``trajopt.solver_single``
(arXiv 2408.10731, Alg. 1) vectorised over a batch of independent members that
share one basis and one obstacle set.  Every block cites the reference line it
restates.  Arithmetic is written in the reference's operation order so a
single-member run reproduces the reference to rounding (pinned against golden
vectors generated from the live reference, see ``tests/golden/make_golden.py``
and ``tests/test_oracle_golden.py``).

Parity status: PINNED (golden fixtures from the live reference, committed).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import comb

import numpy as np
from scipy.linalg import lu_factor, lu_solve

D_CAP = 1e6  # geometry.py:23


# ---------------------------------------------------------------- basis (basis.py:132-217)
def bernstein(tau: np.ndarray, n: int) -> np.ndarray:
    """basis.py:132-136."""
    return np.stack([comb(n, j) * tau**j * (1.0 - tau) ** (n - j) for j in range(n + 1)], axis=1)


def build_basis(t0: float, tf: float, n_p: int, degree: int):
    """basis.py:143-177 -> (timestamps, P, Pdot, Pddot)."""
    ts = np.linspace(t0, tf, n_p)
    T = tf - t0
    tau = (ts - t0) / T
    n = degree
    P = bernstein(tau, n)
    Pd = np.zeros_like(P)
    Pdd = np.zeros_like(P)

    def col(M, j):
        return M[:, j] if 0 <= j < M.shape[1] else np.zeros(M.shape[0])

    if n >= 1:
        L1 = bernstein(tau, n - 1)
        for j in range(n + 1):
            Pd[:, j] = n * (col(L1, j - 1) - col(L1, j)) / T
    if n >= 2:
        L2 = bernstein(tau, n - 2)
        for j in range(n + 1):
            Pdd[:, j] = n * (n - 1) * (col(L2, j - 2) - 2.0 * col(L2, j - 1) + col(L2, j)) / T**2
    return ts, P, Pd, Pdd


def boundary_matrix(P, Pd, Pdd):
    """basis.py:197-204 with start/end orders (0,1,2)."""
    return np.vstack([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])


# ---------------------------------------------------------------- problem / state containers
@dataclass
class Problem:
    """B members sharing basis + obstacle tracks (solver_single.py:30-55, batched).

    bvals: (B, dim, 6) boundary values per axis (basis.py:126-129 order p0,v0,a0,p1,v1,a1)
    desired: (B, n_p, dim); tracks: (n_o, n_p, dim); a, b: (n_o,)
    """

    P: np.ndarray
    Pd: np.ndarray
    Pdd: np.ndarray
    bvals: np.ndarray
    desired: np.ndarray
    tracks: np.ndarray
    a: np.ndarray
    b: np.ndarray
    w_smooth: float = 1.0
    w_track: float = 1.0

    @property
    def B(self):
        return self.bvals.shape[0]

    @property
    def dim(self):
        return self.bvals.shape[1]

    @property
    def n_o(self):
        return self.tracks.shape[0]

    @property
    def n_p(self):
        return self.P.shape[0]

    @property
    def m(self):
        return self.P.shape[1]


@dataclass
class Params:
    """solver_single.py:58-68."""

    max_iter: int = 300
    tol: float = 1e-3
    rho_start: float = 1.0
    rho_growth: float = 1.4
    rho_cap: float = 1e3
    stall_window: int = 5
    stall_improvement: float = 0.01


@dataclass
class State:
    """solver_single.py:71-92, batched over the leading axis."""

    xi: np.ndarray  # (B, dim, m)
    d: np.ndarray  # (B, n_o, n_p)
    alpha: np.ndarray
    beta: np.ndarray | None
    cos_a: np.ndarray
    sin_a: np.ndarray
    cos_b: np.ndarray | None
    sin_b: np.ndarray | None
    lam_pos: np.ndarray  # (B, dim, n_o, n_p)
    lam_cos_a: np.ndarray
    lam_sin_a: np.ndarray
    lam_cos_b: np.ndarray | None
    lam_sin_b: np.ndarray | None
    rho: np.ndarray  # (B,)
    rho_o: np.ndarray  # (B,)
    iteration: np.ndarray  # (B,) int
    factor_rho_o: list = field(default_factory=list)
    n_factorizations: np.ndarray | None = None

    def copy(self):
        out = State(**{k: (v.copy() if isinstance(v, np.ndarray) else (list(v) if isinstance(v, list) else v))
                       for k, v in self.__dict__.items()})
        return out


def angle2d(dx, dy):
    """geometry.py:96-99."""
    alpha = np.arctan2(dy, dx)
    return np.where(alpha == -np.pi, np.pi, alpha)


def angles3d(dx, dy, dz, a, b):
    """geometry.py:102-114 (a, b broadcast)."""
    alpha = angle2d(dx, dy)
    planar = np.hypot(dx / a, dy / a)
    beta = np.arctan2(planar, dz / b)
    return alpha, beta


def straight_line_coeffs(P, start, goal):
    """basis.py:207-217: (dim, m)."""
    n_p = P.shape[0]
    line = start[None, :] + (goal - start)[None, :] * np.linspace(0.0, 1.0, n_p)[:, None]
    sol, *_ = np.linalg.lstsq(P, line, rcond=None)
    return sol.T


def init_state(prob: Problem, params: Params | None = None) -> State:
    """solver_single.py:115-166, one member at a time (bit-faithful)."""
    params = params or Params()
    B, dim, n_o, n_p, m = prob.B, prob.dim, prob.n_o, prob.n_p, prob.m
    xi = np.empty((B, dim, m))
    alpha = np.zeros((B, n_o, n_p))
    beta = np.zeros((B, n_o, n_p)) if dim == 3 else None
    for i in range(B):
        start = prob.bvals[i, :, 0].copy()
        goal = prob.bvals[i, :, 3].copy()
        xi[i] = straight_line_coeffs(prob.P, start, goal)
        line = prob.P @ xi[i].T
        if n_o:
            deltas = line[None, :, :] - prob.tracks
            if dim == 3:
                for j in range(n_o):
                    al, be = angles3d(deltas[j, :, 0], deltas[j, :, 1], deltas[j, :, 2], prob.a[j], prob.b[j])
                    alpha[i, j] = al
                    beta[i, j] = be
            else:
                for j in range(n_o):
                    alpha[i, j] = angle2d(deltas[j, :, 0] / prob.a[j], deltas[j, :, 1] / prob.b[j])
    z = np.zeros((B, n_o, n_p))
    return State(
        xi=xi,
        d=np.ones((B, n_o, n_p)),
        alpha=alpha,
        beta=beta,
        cos_a=np.cos(alpha),
        sin_a=np.sin(alpha),
        cos_b=np.cos(beta) if beta is not None else None,
        sin_b=np.sin(beta) if beta is not None else None,
        lam_pos=np.zeros((B, dim, n_o, n_p)),
        lam_cos_a=z.copy(),
        lam_sin_a=z.copy(),
        lam_cos_b=z.copy() if dim == 3 else None,
        lam_sin_b=z.copy() if dim == 3 else None,
        rho=np.full(B, params.rho_start),
        rho_o=np.full(B, params.rho_start),
        iteration=np.zeros(B, dtype=np.int64),
        factor_rho_o=[None] * B,
        n_factorizations=np.zeros(B, dtype=np.int64),
    )


# ---------------------------------------------------------------- qp-core (qpcore.py:80-143)
class KKTCache:
    """Per-rho_o factor cache: factorize (qpcore.py:80-114) + lu_solve (qpcore.py:130-143).

    mode "lu" is the reference's LU path; mode "kinv" applies the explicit
    inverse K^-1 = lu_solve(lu, I) as a GEMM (what the device does).
    """

    def __init__(self, prob: Problem, mode: str = "lu", cond_limit: float = 1e12):
        self.prob = prob
        self.mode = mode
        self.cond_limit = cond_limit
        P, Pdd = prob.P, prob.Pdd
        self.Q = 2.0 * (prob.w_smooth * Pdd.T @ Pdd + prob.w_track * P.T @ P)  # solver_single.py:172
        self.PtP = P.T @ P
        self.A = boundary_matrix(prob.P, prob.Pd, prob.Pdd)
        self._lu = {}
        self._kinv = {}

    def saddle(self, rho_o: float) -> np.ndarray:
        """solver_single.py:199 + qpcore.py:102-106."""
        n_o = self.prob.n_o
        D = self.Q + rho_o * n_o * self.PtP if n_o else self.Q
        m, ne = D.shape[0], self.A.shape[0]
        K = np.zeros((m + ne, m + ne))
        K[:m, :m] = D
        K[:m, m:] = self.A.T
        K[m:, :m] = self.A
        return K

    def factor(self, rho_o: float):
        key = float(rho_o)
        if key not in self._lu:
            K = self.saddle(key)
            cond = float(np.linalg.cond(K))
            if not np.isfinite(cond) or cond > self.cond_limit:  # qpcore.py:108-110
                raise ValueError(f"saddle matrix is near-singular (cond estimate {cond:.3e})")
            self._lu[key] = lu_factor(K)
            self._kinv[key] = lu_solve(self._lu[key], np.eye(K.shape[0]))
        return self._lu[key]

    def kinv(self, rho_o: float) -> np.ndarray:
        self.factor(rho_o)
        return self._kinv[float(rho_o)]

    def solve(self, rho_o: float, qs: np.ndarray, bs: np.ndarray) -> np.ndarray:
        """qpcore.solve_batch: rows of qs (N, m), bs (N, 6) -> xi (N, m)."""
        block = np.hstack([-qs, bs]).T
        if self.mode == "lu":
            sol = lu_solve(self.factor(rho_o), block)
        else:
            sol = self.kinv(rho_o) @ block
        return sol[: qs.shape[1]].T


# ---------------------------------------------------------------- AM blocks (solver_single.py:169-343)
def _positions(prob, xi):
    """P @ xi.T per member -> (B, n_p, dim)."""
    return np.matmul(prob.P[None], np.transpose(xi, (0, 2, 1)))


def _deltas(prob, positions):
    """solver_single.py:109-112 -> (B, n_o, n_p, dim)."""
    return positions[:, None, :, :] - prob.tracks[None]


def position_targets(prob, st):
    """solver_single.py:177-189 -> (B, dim, n_o, n_p)."""
    a = prob.a[None, :, None]
    b = prob.b[None, :, None]
    tr = prob.tracks
    if prob.dim == 3:
        tx = tr[None, :, :, 0] + a * st.d * st.cos_a * st.sin_b
        ty = tr[None, :, :, 1] + a * st.d * st.sin_a * st.sin_b
        tz = tr[None, :, :, 2] + b * st.d * st.cos_b
        return np.stack([tx, ty, tz], axis=1)
    tx = tr[None, :, :, 0] + a * st.d * st.cos_a
    ty = tr[None, :, :, 1] + b * st.d * st.sin_a
    return np.stack([tx, ty], axis=1)


def position_step(st, prob, kkt: KKTCache):
    """solver_single.py:192-211 (per-member factor keyed by rho_o)."""
    P = prob.P
    q = -2.0 * prob.w_track * np.transpose(np.matmul(P.T[None], prob.desired), (0, 2, 1))  # :173 (B, dim, m)
    for i in range(prob.B):
        if st.factor_rho_o[i] is None or st.factor_rho_o[i] != st.rho_o[i]:
            kkt.factor(st.rho_o[i])
            st.factor_rho_o[i] = st.rho_o[i]
            st.n_factorizations[i] += 1
    if prob.n_o:
        targets = position_targets(prob, st)
        lam_sum = st.lam_pos.sum(axis=2)  # :206
        q_lin = q + lam_sum @ P - st.rho_o[:, None, None] * targets.sum(axis=2) @ P  # :207
    else:
        q_lin = q
    xi = np.empty_like(st.xi)
    for i in range(prob.B):
        xi[i] = kkt.solve(st.rho_o[i], q_lin[i], prob.bvals[i])  # :210
    st.xi = xi


def alpha_copy_step(st, prob):
    """solver_single.py:214-237."""
    if prob.n_o == 0:
        return
    deltas = _deltas(prob, _positions(prob, st.xi))
    a = prob.a[None, :, None]
    b = prob.b[None, :, None]
    rho = st.rho[:, None, None]
    rho_o = st.rho_o[:, None, None]
    dx, dy = deltas[..., 0], deltas[..., 1]
    if prob.dim == 3:
        coef = a * st.d * st.sin_b
        den = rho + rho_o * coef**2
        st.cos_a = (rho * np.cos(st.alpha) - st.lam_cos_a + coef * (st.lam_pos[:, 0] + rho_o * dx)) / den
        st.sin_a = (rho * np.sin(st.alpha) - st.lam_sin_a + coef * (st.lam_pos[:, 1] + rho_o * dy)) / den
    else:
        cx = a * st.d
        cy = b * st.d
        st.cos_a = (rho * np.cos(st.alpha) - st.lam_cos_a + cx * (st.lam_pos[:, 0] + rho_o * dx)) / (rho + rho_o * cx**2)
        st.sin_a = (rho * np.sin(st.alpha) - st.lam_sin_a + cy * (st.lam_pos[:, 1] + rho_o * dy)) / (rho + rho_o * cy**2)


def alpha_extract(st, prob):
    """solver_single.py:240-242 (raw arctan2, no -pi remap)."""
    if prob.n_o:
        st.alpha = np.arctan2(st.sin_a, st.cos_a)


def beta_copy_step(st, prob):
    """solver_single.py:245-266 (uses the NEW alpha copies)."""
    if prob.n_o == 0 or prob.dim != 3:
        return
    deltas = _deltas(prob, _positions(prob, st.xi))
    a = prob.a[None, :, None]
    b = prob.b[None, :, None]
    rho = st.rho[:, None, None]
    rho_o = st.rho_o[:, None, None]
    dx, dy, dz = deltas[..., 0], deltas[..., 1], deltas[..., 2]
    ccb = b * st.d
    st.cos_b = (rho * np.cos(st.beta) - st.lam_cos_b + ccb * (st.lam_pos[:, 2] + rho_o * dz)) / (rho + rho_o * ccb**2)
    csb = a * st.d
    num = rho * np.sin(st.beta) - st.lam_sin_b + csb * (
        st.cos_a * (st.lam_pos[:, 0] + rho_o * dx) + st.sin_a * (st.lam_pos[:, 1] + rho_o * dy)
    )
    den = rho + rho_o * csb**2 * (st.cos_a**2 + st.sin_a**2)
    st.sin_b = num / den


def beta_extract(st, prob):
    """solver_single.py:269-271."""
    if prob.n_o and prob.dim == 3:
        st.beta = np.arctan2(st.sin_b, st.cos_b)


def d_step(st, prob):
    """solver_single.py:274-291 (new positions only)."""
    if prob.n_o == 0:
        return
    deltas = _deltas(prob, _positions(prob, st.xi))
    a = prob.a[None, :, None]
    b = prob.b[None, :, None]
    if prob.dim == 3:
        quad = deltas[..., 0] ** 2 / a**2 + deltas[..., 1] ** 2 / a**2 + deltas[..., 2] ** 2 / b**2
    else:
        quad = deltas[..., 0] ** 2 / a**2 + deltas[..., 1] ** 2 / b**2
    st.d = np.minimum(np.maximum(1.0, np.sqrt(quad)), D_CAP)


def equality_residuals(st, prob) -> dict:
    """solver_single.py:294-313 -> dict of (B, n_o, n_p) in the reference's key order."""
    res = {}
    if not prob.n_o:
        return res
    deltas = _deltas(prob, _positions(prob, st.xi))
    a = prob.a[None, :, None]
    b = prob.b[None, :, None]
    if prob.dim == 3:
        res["coll_x"] = deltas[..., 0] - a * st.d * st.cos_a * st.sin_b
        res["coll_y"] = deltas[..., 1] - a * st.d * st.sin_a * st.sin_b
        res["coll_z"] = deltas[..., 2] - b * st.d * st.cos_b
        res["copy_cos_b"] = st.cos_b - np.cos(st.beta)
        res["copy_sin_b"] = st.sin_b - np.sin(st.beta)
    else:
        res["coll_x"] = deltas[..., 0] - a * st.d * st.cos_a
        res["coll_y"] = deltas[..., 1] - b * st.d * st.sin_a
    res["copy_cos_a"] = st.cos_a - np.cos(st.alpha)
    res["copy_sin_a"] = st.sin_a - np.sin(st.alpha)
    return res


def residual_extremes(st, prob):
    """solver_single.py:324-329 per member -> (norm (B,), max_abs (B,))."""
    res = equality_residuals(st, prob)
    B = prob.B
    if not res:
        return np.zeros(B), np.zeros(B)
    norms = np.empty(B)
    maxs = np.empty(B)
    for i in range(B):
        stacked = np.concatenate([r[i].ravel() for r in res.values()])
        norms[i] = float(np.linalg.norm(stacked))
        maxs[i] = float(np.max(np.abs(stacked)))
    return norms, maxs


def multiplier_step(st, prob):
    """solver_single.py:332-343."""
    res = equality_residuals(st, prob)
    if not res:
        return
    ro = st.rho_o[:, None, None]
    r = st.rho[:, None, None]
    st.lam_pos[:, 0] += ro * res["coll_x"]
    st.lam_pos[:, 1] += ro * res["coll_y"]
    st.lam_cos_a += r * res["copy_cos_a"]
    st.lam_sin_a += r * res["copy_sin_a"]
    if prob.dim == 3:
        st.lam_pos[:, 2] += ro * res["coll_z"]
        st.lam_cos_b += r * res["copy_cos_b"]
        st.lam_sin_b += r * res["copy_sin_b"]


def am_iteration(st, prob, kkt):
    """solver_single.py:373-389 (mutates and returns st)."""
    if prob.n_o:
        st.cos_a = np.cos(st.alpha)
        st.sin_a = np.sin(st.alpha)
        if prob.dim == 3:
            st.cos_b = np.cos(st.beta)
            st.sin_b = np.sin(st.beta)
    position_step(st, prob, kkt)
    alpha_copy_step(st, prob)
    alpha_extract(st, prob)
    beta_copy_step(st, prob)
    beta_extract(st, prob)
    d_step(st, prob)
    multiplier_step(st, prob)
    st.iteration += 1
    return st


def maybe_grow(rho, rho_o, iteration, params, hist, last_change):
    """solver_single.py:392-404 for one member -> (rho, rho_o, last_change)."""
    w = params.stall_window
    if len(hist) < 2 * w or iteration - last_change < w:
        return rho, rho_o, last_change
    recent = np.mean(hist[-w:])
    previous = np.mean(hist[-2 * w : -w])
    if previous <= max(params.tol, 0.0):
        return rho, rho_o, last_change
    if (previous - recent) / previous < params.stall_improvement:
        rho = min(rho * params.rho_growth, params.rho_cap)
        rho_o = min(rho_o * params.rho_growth, params.rho_cap)
        return rho, rho_o, iteration
    return rho, rho_o, last_change


@dataclass
class Result:
    state: State
    converged: np.ndarray
    iterations: np.ndarray
    norm_hist: list  # per member list of floats
    max_hist: list
    rho_hist: list


def solve(prob: Problem, params: Params | None = None, state: State | None = None, kkt: KKTCache | None = None,
          snapshot_at=(), snapshots: dict | None = None) -> Result:
    """solve_single (solver_single.py:407-450) for every member; members are independent.

    Converged members stop iterating (the reference breaks out of its loop).
    ``snapshot_at``: iteration numbers after which a copy of the state is stored
    in ``snapshots[k]`` (teacher-forcing fixtures).
    """
    params = params or Params()
    state = state if state is not None else init_state(prob, params)
    kkt = kkt or KKTCache(prob)
    B = prob.B
    norm_hist = [[] for _ in range(B)]
    max_hist = [[] for _ in range(B)]
    rho_hist = [[] for _ in range(B)]
    last_change = np.zeros(B, dtype=np.int64)
    active = np.ones(B, dtype=bool)
    converged = np.zeros(B, dtype=bool)
    if snapshots is not None and 0 in snapshot_at:
        snapshots[0] = state.copy()
    for k in range(params.max_iter):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        sub_prob, sub = _subset(prob, state, idx)
        am_iteration(sub, sub_prob, kkt)
        norms, maxs = residual_extremes(sub, sub_prob)
        for n, i in enumerate(idx):
            norm_hist[i].append(norms[n])
            max_hist[i].append(maxs[n])
            rho_hist[i].append(sub.rho_o[n])
            if maxs[n] <= params.tol:
                converged[i] = True
                active[i] = False
                continue
            sub.rho[n], sub.rho_o[n], last_change[i] = maybe_grow(
                sub.rho[n], sub.rho_o[n], sub.iteration[n], params, max_hist[i], last_change[i])
        _scatter(state, sub, idx)
        if snapshots is not None and (k + 1) in snapshot_at:
            snapshots[k + 1] = state.copy()
    return Result(state=state, converged=converged, iterations=state.iteration.copy(),
                  norm_hist=norm_hist, max_hist=max_hist, rho_hist=rho_hist)


_ARRAYS = ("xi", "d", "alpha", "beta", "cos_a", "sin_a", "cos_b", "sin_b", "lam_pos", "lam_cos_a", "lam_sin_a",
           "lam_cos_b", "lam_sin_b", "rho", "rho_o", "iteration", "n_factorizations")


def _subset(prob, st, idx):
    if idx.size == prob.B:
        return prob, st
    sp = Problem(P=prob.P, Pd=prob.Pd, Pdd=prob.Pdd, bvals=prob.bvals[idx], desired=prob.desired[idx],
                 tracks=prob.tracks, a=prob.a, b=prob.b, w_smooth=prob.w_smooth, w_track=prob.w_track)
    kw = {k: (getattr(st, k)[idx] if getattr(st, k) is not None else None) for k in _ARRAYS}
    ss = State(**kw, factor_rho_o=[st.factor_rho_o[i] for i in idx])
    return sp, ss


def _scatter(st, sub, idx):
    if sub is st:
        return
    for k in _ARRAYS:
        v = getattr(sub, k)
        if v is not None:
            getattr(st, k)[idx] = v
    for n, i in enumerate(idx):
        st.factor_rho_o[i] = sub.factor_rho_o[n]


def rho_levels(params: Params) -> np.ndarray:
    """Distinct penalty values reachable by solver_single.py:401-402 (repeated products, capped)."""
    vals = [params.rho_start]
    while True:
        nxt = min(vals[-1] * params.rho_growth, params.rho_cap)
        if nxt == vals[-1]:
            break
        vals.append(nxt)
    return np.array(vals)
