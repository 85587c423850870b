"""CPU ORACLE for PRIEST projection-guided sampling and the CEM baseline — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this module.
numpy restatement of the reference ``trajopt.solver_priest`` (arXiv 2408.10731,
Alg. 3 + CEM), with every block citing the reference line it restates, written
in the reference's operation order so it reproduces the reference's numbers.
Pinned against golden vectors from the live reference (tests/golden/priest.npz,
tests/test_oracle_priest.py).

The sampling draw is split exactly like numpy's
``Generator.multivariate_normal(method="svd")``: z = standard_normal((N, d)),
samples = mean + z @ (u * sqrt(s)).T with u, s from svd(cov),
so a test can feed the same z to the oracle and to the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from .alg1 import D_CAP

_SPEED_EPS = 1e-6  # solver_priest.py:32


@dataclass
class Setup:
    """ProjectionSetup (solver_priest.py:93-168) as plain arrays."""

    P: np.ndarray
    Pd: np.ndarray
    Pdd: np.ndarray
    dim: int
    m: int
    n_o: int
    tracks: np.ndarray  # (n_o, n_p, dim)
    a: np.ndarray
    b: np.ndarray
    v_max: float | None
    a_max: float | None
    F_tilde: np.ndarray
    G: np.ndarray
    tau: np.ndarray
    F: np.ndarray
    A: np.ndarray
    b_eq: np.ndarray
    rho: float
    K: np.ndarray
    lu: tuple


def make_setup(P, Pd, Pdd, bvals, tracks=None, a=None, b=None, v_max=None, a_max=None, s_min=None, s_max=None,
               rho=1.0, start_orders=(0, 1, 2), end_orders=(0,)):
    """bvals: (dim, 6) AxisBoundary.values() order (p0 v0 a0 p1 v1 a1)."""
    dim = bvals.shape[0]
    n_p, m = P.shape
    tracks = np.zeros((0, n_p, dim)) if tracks is None else np.asarray(tracks, float)
    n_o = tracks.shape[0]
    blocks = []
    if n_o:
        blocks.append(np.tile(P, (n_o, 1)))  # :130-131
    if v_max is not None:
        blocks.append(Pd)
    if a_max is not None:
        blocks.append(Pdd)
    axis_block = np.vstack(blocks) if blocks else np.zeros((0, m))
    F_tilde = np.zeros((dim * axis_block.shape[0], dim * m))
    for k in range(dim):
        F_tilde[k * axis_block.shape[0]:(k + 1) * axis_block.shape[0], k * m:(k + 1) * m] = axis_block
    if s_min is not None and s_max is not None:  # :142-150
        bound_block = np.vstack([-P, P])
        G = np.zeros((dim * 2 * n_p, dim * m))
        tau = np.zeros(dim * 2 * n_p)
        for k in range(dim):
            G[k * 2 * n_p:(k + 1) * 2 * n_p, k * m:(k + 1) * m] = bound_block
            tau[k * 2 * n_p:k * 2 * n_p + n_p] = -s_min[k]
            tau[k * 2 * n_p + n_p:(k + 1) * 2 * n_p] = s_max[k]
    else:
        G = np.zeros((0, dim * m))
        tau = np.zeros(0)
    F = np.vstack([F_tilde, G])
    full = {0: P, 1: Pd, 2: Pdd}
    Bm = np.vstack([full[o][0] for o in start_orders] + [full[o][-1] for o in end_orders])
    A = np.zeros((dim * Bm.shape[0], dim * m))
    for k in range(dim):
        A[k * Bm.shape[0]:(k + 1) * Bm.shape[0], k * m:(k + 1) * m] = Bm
    order_idx = {0: 0, 1: 1, 2: 2}
    b_eq = np.concatenate([[bvals[k][order_idx[o]] for o in start_orders] + [bvals[k][3 + o] for o in end_orders]
                           for k in range(dim)])
    Q = np.eye(dim * m) + rho * F.T @ F  # :167
    n_v, n_eq = Q.shape[0], A.shape[0]
    K = np.zeros((n_v + n_eq, n_v + n_eq))
    K[:n_v, :n_v] = Q
    K[:n_v, n_v:] = A.T
    K[n_v:, :n_v] = A
    return Setup(P=P, Pd=Pd, Pdd=Pdd, dim=dim, m=m, n_o=n_o, tracks=tracks,
                 a=np.asarray(a, float) if a is not None else np.zeros(0),
                 b=np.asarray(b, float) if b is not None else np.zeros(0), v_max=v_max, a_max=a_max,
                 F_tilde=F_tilde, G=G, tau=tau, F=F, A=A, b_eq=b_eq, rho=rho, K=K, lu=lu_factor(K))


def axis_samples(st: Setup, xis, mat):
    """solver_priest.py:172-178: (N, dim*m) -> (N, dim, rows)."""
    xis = np.atleast_2d(xis)
    out = np.empty((xis.shape[0], st.dim, mat.shape[0]))
    for k in range(st.dim):
        out[:, k, :] = xis[:, k * st.m:(k + 1) * st.m] @ mat.T
    return out


def polar_targets(st: Setup, xis):
    """solver_priest.py:189-239 (trigonometric form, bit-faithful)."""
    n = xis.shape[0]
    pos = axis_samples(st, xis, st.P)
    vel = axis_samples(st, xis, st.Pd)
    acc = axis_samples(st, xis, st.Pdd)
    per_axis = [[] for _ in range(st.dim)]
    if st.n_o:
        obs_pos = st.tracks
        deltas = pos[:, None, :, :] - obs_pos.transpose(0, 2, 1)[None, :, :, :]
        a = st.a[None, :, None]
        b = st.b[None, :, None]
        dx, dy = deltas[:, :, 0], deltas[:, :, 1]
        if st.dim == 3:
            dz = deltas[:, :, 2]
            alpha = np.arctan2(dy, dx)
            beta = np.arctan2(np.hypot(dx / a, dy / a), dz / b)
            d = np.clip(np.sqrt(dx**2 / a**2 + dy**2 / a**2 + dz**2 / b**2), 1.0, D_CAP)
            obs_xyz = obs_pos.transpose(0, 2, 1)[None]
            per_axis[0].append((obs_xyz[:, :, 0] + a * d * np.cos(alpha) * np.sin(beta)).reshape(n, -1))
            per_axis[1].append((obs_xyz[:, :, 1] + a * d * np.sin(alpha) * np.sin(beta)).reshape(n, -1))
            per_axis[2].append((obs_xyz[:, :, 2] + b * d * np.cos(beta)).reshape(n, -1))
        else:
            alpha = np.arctan2(dy / b, dx / a)
            d = np.clip(np.hypot(dx / a, dy / b), 1.0, D_CAP)
            obs_xy = obs_pos.transpose(0, 2, 1)[None]
            per_axis[0].append((obs_xy[:, :, 0] + a * d * np.cos(alpha)).reshape(n, -1))
            per_axis[1].append((obs_xy[:, :, 1] + b * d * np.sin(alpha)).reshape(n, -1))
    for limit, smp in ((st.v_max, vel), (st.a_max, acc)):
        if limit is None:
            continue
        if st.dim == 3:
            vx, vy, vz = smp[:, 0], smp[:, 1], smp[:, 2]
            alpha = np.arctan2(vy, vx)
            beta = np.arctan2(np.hypot(vx, vy), vz)
            d = np.clip(np.sqrt(vx**2 + vy**2 + vz**2) / limit, 0.0, 1.0)
            per_axis[0].append(limit * d * np.cos(alpha) * np.sin(beta))
            per_axis[1].append(limit * d * np.sin(alpha) * np.sin(beta))
            per_axis[2].append(limit * d * np.cos(beta))
        else:
            vx, vy = smp[:, 0], smp[:, 1]
            alpha = np.arctan2(vy, vx)
            d = np.clip(np.hypot(vx, vy) / limit, 0.0, 1.0)
            per_axis[0].append(limit * d * np.cos(alpha))
            per_axis[1].append(limit * d * np.sin(alpha))
    if st.F_tilde.shape[0] == 0:
        return np.zeros((n, 0))
    return np.hstack([np.hstack(parts) for parts in per_axis])


def residual_scores(st: Setup, xis):
    """solver_priest.py:290-301."""
    xis = np.atleast_2d(xis)
    parts = []
    if st.F_tilde.shape[0]:
        parts.append(xis @ st.F_tilde.T - polar_targets(st, xis))
    if st.G.shape[0]:
        parts.append(np.maximum(0.0, xis @ st.G.T - st.tau[None, :]))
    if not parts:
        return np.zeros(xis.shape[0])
    return np.linalg.norm(np.hstack(parts), axis=1)


def project(st: Setup, samples, n_inner=30, history=None, mode="lu"):
    """solver_priest.py:242-287 -> (xi_bar (N, dim*m), scores (N,))."""
    samples = np.atleast_2d(np.asarray(samples, float))
    n = samples.shape[0]
    xi_bar = samples.copy()
    lam = np.zeros_like(samples)
    bs = np.tile(st.b_eq, (n, 1))
    rho = st.rho
    kinv = lu_solve(st.lu, np.eye(st.K.shape[0])) if mode == "kinv" else None
    for _ in range(n_inner):
        e_tilde = polar_targets(st, xi_bar)
        if st.G.shape[0]:
            Gx = xi_bar @ st.G.T
            slack = np.maximum(0.0, st.tau[None, :] - Gx)
            e = np.hstack([e_tilde, st.tau[None, :] - slack])
        else:
            e = e_tilde
        residual = xi_bar @ st.F.T - e
        lam = lam - rho * (residual @ st.F)
        q_lin = -(samples + lam + rho * (e @ st.F))
        block = np.hstack([-q_lin, bs]).T
        sol = lu_solve(st.lu, block) if kinv is None else kinv @ block
        xi_bar = sol[: samples.shape[1]].T
        if history is not None:
            history.append(residual_scores(st, xi_bar))
    return xi_bar, residual_scores(st, xi_bar)


def draw_transform(mu, sigma_mat):
    """numpy multivariate_normal(method='svd') factor: samples = mu + z @ factor.T."""
    u, s, _ = np.linalg.svd(sigma_mat)
    return u * np.sqrt(s)


def update_distribution(mu, sigma_mat, elite_xi, elite_costs, sigma, gamma):
    """solver_priest.py:317-333."""
    elite_xi = np.asarray(elite_xi, float)
    costs = np.asarray(elite_costs, float)
    weights = np.exp((costs - costs.min()) / gamma)
    wsum = weights.sum()
    weighted_mean = (weights[:, None] * elite_xi).sum(axis=0) / wsum
    new_mu = (1.0 - sigma) * mu + sigma * weighted_mean
    centered = elite_xi - new_mu[None, :]
    weighted_cov = (weights[:, None, None] * (centered[:, :, None] * centered[:, None, :])).sum(axis=0) / wsum
    new_sigma = (1.0 - sigma) * sigma_mat + sigma * weighted_cov
    return new_mu, new_sigma


def flatness_car(vel, acc):
    """solver_priest.py:460-472."""
    speed = np.hypot(vel[:, 0], vel[:, 1])
    kappa = np.full_like(speed, np.nan)
    ok = speed > _SPEED_EPS
    kappa[ok] = (acc[ok, 1] * vel[ok, 0] - acc[ok, 0] * vel[ok, 1]) / speed[ok] ** 3
    return speed, kappa


def barn_cost(pos, vel, acc, line_start, line_end):
    """solver_priest.py:475-498."""
    smooth = float(np.sum(acc[:, 0] ** 2 + acc[:, 1] ** 2))
    _, kappa = flatness_car(vel, acc)
    c_kappa = float(np.nansum(kappa**2))
    start = np.asarray(line_start, float)[:2]
    end = np.asarray(line_end, float)[:2]
    axis = end - start
    length = np.linalg.norm(axis)
    rel = pos[:, :2] - start
    if length < 1e-12:
        dist2 = (rel**2).sum(axis=1)
    else:
        u = axis / length
        along = rel @ u
        dist2 = (rel**2).sum(axis=1) - along**2
    return smooth + c_kappa + float(np.sum(np.maximum(dist2, 0.0)))


def trajectory_of(st: Setup, xi):
    """solver_priest.py:180-187 -> (pos, vel, acc) each (n_p, dim)."""
    return (axis_samples(st, xi, st.P)[0].T, axis_samples(st, xi, st.Pd)[0].T, axis_samples(st, xi, st.Pdd)[0].T)


def priest_round(st: Setup, z, mu, sigma_mat, n_constraint_elite, n_elite, n_inner, sigma, gamma,
                 residual_weight, c1):
    """One trip of priest_optimize's loop (solver_priest.py:354-381) given the round's standard normals z."""
    samples = mu + z @ draw_transform(mu, sigma_mat).T
    xi_bar, scores = project(st, samples, n_inner)
    keep = np.argsort(scores, kind="stable")[:n_constraint_elite]  # :358
    aug = np.array([float(c1(*trajectory_of(st, xi_bar[i]))) + residual_weight * float(scores[i]) for i in keep])
    order = sorted(range(len(keep)), key=lambda r: aug[r])  # :362 (stable, residual-rank order)
    elite_rows = np.array(order[:n_elite])
    elites = keep[elite_rows]
    new_mu, new_sigma = update_distribution(mu, sigma_mat, xi_bar[elites], aug[elite_rows], sigma, gamma)
    return dict(samples=samples, xi_bar=xi_bar, scores=scores, keep=keep, aug=aug, elites=elites, mu=new_mu,
                sigma_mat=new_sigma)


def cem_penalty(st: Setup, xis):
    """solver_priest.py:396-419."""
    xis = np.atleast_2d(xis)
    total = np.zeros(xis.shape[0])
    pos = axis_samples(st, xis, st.P)
    if st.n_o:
        deltas = pos[:, None, :, :] - st.tracks.transpose(0, 2, 1)[None, :, :, :]
        a = st.a[None, :, None]
        b = st.b[None, :, None]
        if st.dim == 3:
            quad = deltas[:, :, 0] ** 2 / a**2 + deltas[:, :, 1] ** 2 / a**2 + deltas[:, :, 2] ** 2 / b**2
        else:
            quad = deltas[:, :, 0] ** 2 / a**2 + deltas[:, :, 1] ** 2 / b**2
        total += np.maximum(0.0, 1.0 - quad).sum(axis=(1, 2))
    if st.v_max is not None:
        vel = axis_samples(st, xis, st.Pd)
        total += np.maximum(0.0, (vel**2).sum(axis=1) - st.v_max**2).sum(axis=1)
    if st.a_max is not None:
        acc = axis_samples(st, xis, st.Pdd)
        total += np.maximum(0.0, (acc**2).sum(axis=1) - st.a_max**2).sum(axis=1)
    if st.G.shape[0]:
        total += np.maximum(0.0, xis @ st.G.T - st.tau[None, :]).sum(axis=1)
    return total
