"""CPU ORACLE for the 2-D batch optimizer (Alg. 2, footprint + heading) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this module.
numpy restatement of the reference ``trajopt.solver_batch`` (arXiv 2408.10731)
citing the reference line of every block; pinned bit-exactly against golden
vectors of the live reference (tests/golden/batch2d.npz, tests/test_oracle_batch2d.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from .alg1 import D_CAP, boundary_matrix


@dataclass
class Structure:
    """_Structure (solver_batch.py:141-193) as arrays."""

    P: np.ndarray
    Pd: np.ndarray
    Pdd: np.ndarray
    m: int
    F: np.ndarray
    FtF: np.ndarray
    Q: np.ndarray
    q: np.ndarray
    A: np.ndarray
    b: np.ndarray
    A_psi: np.ndarray
    b_psi: np.ndarray
    Q_psi_smooth: np.ndarray
    obs_x: np.ndarray
    obs_y: np.ndarray
    obs_a: np.ndarray
    obs_b: np.ndarray
    r: np.ndarray
    v_max: float
    a_max: float
    w_smooth: float
    w_track: float
    desired: np.ndarray


def make_structure(P, Pd, Pdd, bvals, psi_boundary, desired, tracks, a, b, offsets, v_max, a_max, w_smooth=1.0,
                   w_track=1.0):
    """bvals (2, 6); tracks (n_o, n_p, 2)."""
    n_p, m = P.shape
    n_o = tracks.shape[0]
    zeros = np.zeros((n_p, m))
    half = [np.hstack([Pd, zeros]), np.hstack([Pdd, zeros])]
    for r_c in offsets:
        for _ in range(n_o):
            half.append(np.hstack([P, r_c * P]))
    half.append(np.hstack([zeros, P]))
    F_half = np.vstack(half)
    F = np.block([[F_half, np.zeros((F_half.shape[0], 2 * m))], [np.zeros((F_half.shape[0], 2 * m)), F_half]])
    cost_xx = w_smooth * Pdd.T @ Pdd + w_track * P.T @ P
    Q = np.zeros((4 * m, 4 * m))
    Q[:m, :m] = cost_xx
    Q[2 * m:3 * m, 2 * m:3 * m] = cost_xx
    q = np.concatenate([-w_track * P.T @ desired[:, 0], np.zeros(m), -w_track * P.T @ desired[:, 1], np.zeros(m)])
    B = boundary_matrix(P, Pd, Pdd)
    A = np.zeros((12, 4 * m))
    A[:6, :m] = B
    A[6:, 2 * m:3 * m] = B
    return Structure(P=P, Pd=Pd, Pdd=Pdd, m=m, F=F, FtF=F.T @ F, Q=Q, q=q, A=A, b=np.concatenate([bvals[0], bvals[1]]),
                     A_psi=np.vstack([P[0], P[-1]]), b_psi=np.asarray(psi_boundary, float),
                     Q_psi_smooth=Pdd.T @ Pdd,
                     obs_x=tracks[:, :, 0] if n_o else np.zeros((0, n_p)),
                     obs_y=tracks[:, :, 1] if n_o else np.zeros((0, n_p)),
                     obs_a=np.asarray(a, float), obs_b=np.asarray(b, float), r=np.asarray(offsets, float),
                     v_max=v_max, a_max=a_max, w_smooth=w_smooth, w_track=w_track, desired=desired)


@dataclass
class State:
    xi: np.ndarray
    xi_psi: np.ndarray
    psi: np.ndarray
    alpha_coll: np.ndarray
    alpha_v: np.ndarray
    alpha_a: np.ndarray
    d_coll: np.ndarray
    d_v: np.ndarray
    d_a: np.ndarray
    lam: np.ndarray
    lam_psi: np.ndarray
    rho: float
    rho_psi: float
    iteration: int = 0
    psi_targets: np.ndarray | None = None


def footprint_deltas(st, x, y, psi):
    """solver_batch.py:196-204."""
    cp, sp = np.cos(psi), np.sin(psi)
    r = st.r[None, :, None, None]
    cx = x[:, None, None, :] + r * cp[:, None, None, :]
    cy = y[:, None, None, :] + r * sp[:, None, None, :]
    return cx - st.obs_x[None, None, :, :], cy - st.obs_y[None, None, :, :]


def build_g(st, s: State):
    """solver_batch.py:207-227."""
    n_b = s.xi.shape[0]
    px = [st.v_max * s.d_v * np.cos(s.alpha_v), st.a_max * s.d_a * np.cos(s.alpha_a)]
    py = [st.v_max * s.d_v * np.sin(s.alpha_v), st.a_max * s.d_a * np.sin(s.alpha_a)]
    if st.obs_x.shape[0]:
        a = st.obs_a[None, None, :, None]
        b = st.obs_b[None, None, :, None]
        px.append((st.obs_x[None, None] + a * s.d_coll * np.cos(s.alpha_coll)).reshape(n_b, -1))
        py.append((st.obs_y[None, None] + b * s.d_coll * np.sin(s.alpha_coll)).reshape(n_b, -1))
    px.append(np.cos(s.psi))
    py.append(np.sin(s.psi))
    return np.hstack(px + py)


def split(xi, m):
    return xi[:, :m], xi[:, m:2 * m], xi[:, 2 * m:3 * m], xi[:, 3 * m:]


def alpha_step(st, s):
    """solver_batch.py:318-326."""
    xx, _, xy, _ = split(s.xi, st.m)
    if st.obs_x.shape[0]:
        dx, dy = footprint_deltas(st, xx @ st.P.T, xy @ st.P.T, s.psi)
        s.alpha_coll = np.arctan2(dy, dx)
    s.alpha_v = np.arctan2(xy @ st.Pd.T, xx @ st.Pd.T)
    s.alpha_a = np.arctan2(xy @ st.Pdd.T, xx @ st.Pdd.T)


def d_step(st, s):
    """solver_batch.py:329-344."""
    xx, _, xy, _ = split(s.xi, st.m)
    if st.obs_x.shape[0]:
        dx, dy = footprint_deltas(st, xx @ st.P.T, xy @ st.P.T, s.psi)
        a = st.obs_a[None, None, :, None]
        b = st.obs_b[None, None, :, None]
        ca, sa = np.cos(s.alpha_coll), np.sin(s.alpha_coll)
        s.d_coll = np.clip((a * dx * ca + b * dy * sa) / (a**2 * ca**2 + b**2 * sa**2), 1.0, D_CAP)
    vx, vy = xx @ st.Pd.T, xy @ st.Pd.T
    s.d_v = np.clip((vx * np.cos(s.alpha_v) + vy * np.sin(s.alpha_v)) / st.v_max, 0.0, 1.0)
    ax, ay = xx @ st.Pdd.T, xy @ st.Pdd.T
    s.d_a = np.clip((ax * np.cos(s.alpha_a) + ay * np.sin(s.alpha_a)) / st.a_max, 0.0, 1.0)


def init_state(st, samples, n_c, rho_start=1.0):
    """solver_batch.py:234-278."""
    m, n_p = st.m, st.P.shape[0]
    n_b = samples.shape[0]
    path_dir = np.gradient(st.desired, axis=0)
    psi_des = np.unwrap(np.arctan2(path_dir[:, 1], path_dir[:, 0]))
    xi_psi_one, *_ = np.linalg.lstsq(st.P, psi_des, rcond=None)
    xi_psi = np.tile(xi_psi_one, (n_b, 1))
    psi = xi_psi @ st.P.T
    xi_c_one, *_ = np.linalg.lstsq(st.P, np.cos(psi_des), rcond=None)
    xi_s_one, *_ = np.linalg.lstsq(st.P, np.sin(psi_des), rcond=None)
    xi = np.hstack([samples[:, :m], np.tile(xi_c_one, (n_b, 1)), samples[:, m:], np.tile(xi_s_one, (n_b, 1))])
    n_o = st.obs_x.shape[0]
    s = State(xi=xi, xi_psi=xi_psi, psi=psi, alpha_coll=np.zeros((n_b, n_c, n_o, n_p)), alpha_v=np.zeros((n_b, n_p)),
              alpha_a=np.zeros((n_b, n_p)), d_coll=np.ones((n_b, n_c, n_o, n_p)), d_v=np.ones((n_b, n_p)),
              d_a=np.ones((n_b, n_p)), lam=np.zeros((n_b, 4 * m)), lam_psi=np.zeros((n_b, m)), rho=rho_start,
              rho_psi=rho_start)
    alpha_step(st, s)
    d_step(st, s)
    return s


class Factors:
    """_ensure_factors (solver_batch.py:281-289) cache keyed by rho."""

    def __init__(self, st, mode="lu"):
        self.st, self.mode, self.cache = st, mode, {}

    def get(self, rho, rho_psi):
        key = (float(rho), float(rho_psi))
        if key not in self.cache:
            st = self.st
            out = []
            for Qb, A in ((st.Q + rho * st.FtF, st.A),
                          (st.Q_psi_smooth + rho_psi * st.P.T @ st.P, st.A_psi)):
                n_v, n_eq = Qb.shape[0], A.shape[0]
                K = np.zeros((n_v + n_eq, n_v + n_eq))
                K[:n_v, :n_v] = Qb
                K[:n_v, n_v:] = A.T
                K[n_v:, :n_v] = A
                lu = lu_factor(K)
                out.append((lu, lu_solve(lu, np.eye(K.shape[0])) if self.mode == "kinv" else None, n_v))
            self.cache[key] = out
        return self.cache[key]

    @staticmethod
    def solve(f, qs, bs):
        lu, kinv, n_v = f
        block = np.hstack([-qs, bs]).T
        sol = lu_solve(lu, block) if kinv is None else kinv @ block
        return sol[:n_v].T


def batch_iteration(st, s: State, fac: Factors):
    """solver_batch.py:352-363 (xi step :292-299, heading :302-315, alpha/d, multipliers)."""
    fx, fp = fac.get(s.rho, s.rho_psi)
    g = build_g(st, s)
    q_lin = st.q[None, :] - s.lam - s.rho * (g @ st.F)
    s.xi = Factors.solve(fx, q_lin, np.tile(st.b, (s.xi.shape[0], 1)))
    _, xc, _, xs = split(s.xi, st.m)
    raw = np.arctan2(xs @ st.P.T, xc @ st.P.T)
    targets = raw + 2.0 * np.pi * np.round((s.psi - raw) / (2.0 * np.pi))
    q_psi = -s.lam_psi - s.rho_psi * (targets @ st.P)
    s.xi_psi = Factors.solve(fp, q_psi, np.tile(st.b_psi, (s.xi.shape[0], 1)))
    s.psi = s.xi_psi @ st.P.T
    s.psi_targets = targets
    alpha_step(st, s)
    d_step(st, s)
    res = s.xi @ st.F.T - build_g(st, s)
    s.lam = s.lam - s.rho * (res @ st.F)
    s.lam_psi = s.lam_psi - s.rho_psi * ((s.psi - s.psi_targets) @ st.P)
    s.iteration += 1


def member_costs(st, s):
    """solver_batch.py:366-374."""
    xx, _, xy, _ = split(s.xi, st.m)
    ax, ay = xx @ st.Pdd.T, xy @ st.Pdd.T
    x, y = xx @ st.P.T, xy @ st.P.T
    smooth = np.sum(ax**2 + ay**2, axis=1) + np.sum((s.xi_psi @ st.Pdd.T) ** 2, axis=1)
    track = np.sum((x - st.desired[:, 0]) ** 2 + (y - st.desired[:, 1]) ** 2, axis=1)
    return st.w_smooth * smooth + st.w_track * track


def raw_feasible(st, s, d_margin, kin_margin):
    """solver_batch.py:377-393."""
    xx, _, xy, _ = split(s.xi, st.m)
    x, y = xx @ st.P.T, xy @ st.P.T
    ok = np.ones(x.shape[0], dtype=bool)
    if st.obs_x.shape[0]:
        dx, dy = footprint_deltas(st, x, y, s.psi)
        dist = np.hypot(dx / st.obs_a[None, None, :, None], dy / st.obs_b[None, None, :, None])
        ok &= dist.min(axis=(1, 2, 3)) >= 1.0 - d_margin
    ok &= np.hypot(xx @ st.Pd.T, xy @ st.Pd.T).max(axis=1) <= st.v_max * (1.0 + kin_margin)
    ok &= np.hypot(xx @ st.Pdd.T, xy @ st.Pdd.T).max(axis=1) <= st.a_max * (1.0 + kin_margin)
    return ok


def solve(st, samples, n_c, max_iter=100, tol=1e-2, rho_start=1.0, rho_growth=1.4, rho_cap=1e3, stall_window=5,
          stall_improvement=0.01, d_margin=1e-2, kin_margin=1e-2, mode="lu"):
    """solve_batch_opt's loop and ranking (solver_batch.py:448-471)."""
    s = init_state(st, samples, n_c, rho_start)
    fac = Factors(st, mode)
    best_hist, maxabs, rho_hist = [], [], []
    last_change = 0
    for _ in range(max_iter):
        batch_iteration(st, s, fac)
        res = s.xi @ st.F.T - build_g(st, s)
        pm_max = np.max(np.abs(res), axis=1)
        pm_norm = np.linalg.norm(res, axis=1)
        bi = int(np.argmin(pm_norm))
        best_hist.append((pm_norm[bi], pm_max[bi], s.rho, bi))
        maxabs.append(float(pm_max.min()))
        w = stall_window
        if not (len(maxabs) < 2 * w or s.iteration - last_change < w):  # :396-406
            recent = np.mean(maxabs[-w:])
            previous = np.mean(maxabs[-2 * w:-w])
            if previous > max(tol, 0.0) and (previous - recent) / previous < stall_improvement:
                s.rho = min(s.rho * rho_growth, rho_cap)
                s.rho_psi = min(s.rho_psi * rho_growth, rho_cap)
                last_change = s.iteration
    res = s.xi @ st.F.T - build_g(st, s)
    rmax = np.max(np.abs(res), axis=1)
    rnorm = np.linalg.norm(res, axis=1)
    feasible = (rmax <= tol) & raw_feasible(st, s, d_margin, kin_margin)
    costs = member_costs(st, s)
    aug = costs + s.rho * rnorm
    best = int(np.argmin(np.where(feasible, aug, np.inf))) if feasible.any() else None
    return dict(state=s, best_hist=np.array(best_hist), maxabs=np.array(maxabs), rmax=rmax, rnorm=rnorm,
                feasible=feasible, costs=costs, aug=aug, best=best)
