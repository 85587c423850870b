"""CPU ORACLE for the joint multi-agent solver (Alg. 5) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this module.
numpy restatement of the reference ``trajopt.solver_multiagent`` (arXiv
2408.10731), batched over independent problems that share the agent count,
pair structure and rho levels; every block cites the reference line it
restates.  Pinned bit-exactly against golden vectors of the live reference
(tests/golden/multiagent.npz, tests/test_oracle_multiagent.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from .alg1 import D_CAP, boundary_matrix


@dataclass
class Structure:
    """_JointStructure (solver_multiagent.py:100-165) for one agent count."""

    P: np.ndarray
    m: int
    n_a: int
    pair_i: np.ndarray
    pair_j: np.ndarray  # -1: static partner
    pair_s: np.ndarray  # static sphere index of the pair, -1 for agent-agent pairs
    pa: np.ndarray  # (n_pairs, 1)
    pb: np.ndarray
    A_fo: np.ndarray
    Q: np.ndarray
    A_eq: np.ndarray
    rho_levels: list
    lus: list
    inflated: tuple


def make_structure(P, Pd, Pdd, n_a, a, b, n_static=0, static_radii=(), rho_start=1.0, rho_final=1e4, rho_levels=10,
                   inflation_factor=4.0, typical_residual=0.01):
    """solver_multiagent.py:100-165 (pairs: agent-agent i<j first, then agent-static)."""
    n_p, m = P.shape
    a_inf = a + inflation_factor * typical_residual  # :93-97, :108-109
    b_inf = b + inflation_factor * typical_residual
    pi, pj, ps, pa, pb = [], [], [], [], []
    for i in range(n_a):
        for j in range(i + 1, n_a):
            pi.append(i), pj.append(j), ps.append(-1), pa.append(2.0 * a_inf), pb.append(2.0 * b_inf)
    for s in range(n_static):
        for i in range(n_a):
            pi.append(i), pj.append(-1), ps.append(s)
            pa.append(a_inf + static_radii[s]), pb.append(b_inf + static_radii[s])
    n_pairs = len(pi)
    A_fo = np.zeros((n_pairs * n_p, n_a * m))
    for p in range(n_pairs):
        rows = slice(p * n_p, (p + 1) * n_p)
        A_fo[rows, pi[p] * m:(pi[p] + 1) * m] = P
        if pj[p] >= 0:
            A_fo[rows, pj[p] * m:(pj[p] + 1) * m] = -P
    Q = np.kron(np.eye(n_a), Pdd.T @ Pdd)
    A_eq = np.kron(np.eye(n_a), boundary_matrix(P, Pd, Pdd))
    if n_pairs:
        AtA = A_fo.T @ A_fo
        ratio = (rho_final / rho_start) ** (1.0 / max(rho_levels - 1, 1))
        levels = [rho_start * ratio**k for k in range(rho_levels)]
        mats = [Q + r * AtA for r in levels]
    else:
        levels = [rho_start]
        mats = [Q]
    lus = []
    for M in mats:
        n_v, n_eq = M.shape[0], A_eq.shape[0]
        K = np.zeros((n_v + n_eq, n_v + n_eq))
        K[:n_v, :n_v] = M
        K[:n_v, n_v:] = A_eq.T
        K[n_v:, :n_v] = A_eq
        lus.append(lu_factor(K))
    return Structure(P=P, m=m, n_a=n_a, pair_i=np.array(pi), pair_j=np.array(pj), pair_s=np.array(ps),
                     pa=np.asarray(pa)[:, None], pb=np.asarray(pb)[:, None], A_fo=A_fo, Q=Q, A_eq=A_eq,
                     rho_levels=levels, lus=lus, inflated=(a_inf, b_inf))


@dataclass
class Problem:
    """One joint problem: b_eq (3, 6 n_a) per axis (solver_multiagent.py:149-154), static sphere centres (n_static, 3)."""

    b_eq: np.ndarray
    statics: np.ndarray


@dataclass
class State:
    xi: np.ndarray  # (3, n_a m)
    d: np.ndarray  # (n_pairs, n_p)
    alpha: np.ndarray
    beta: np.ndarray
    lam: np.ndarray  # (3, n_pairs, n_p)
    level: int = 0
    iteration: int = 0


def agent_positions(st: Structure, xi):
    """solver_multiagent.py:167-173 -> (n_a, n_p, 3)."""
    out = np.empty((st.n_a, st.P.shape[0], 3))
    for k in range(3):
        out[:, :, k] = xi[k].reshape(st.n_a, st.m) @ st.P.T
    return out


def pair_deltas(st: Structure, prob: Problem, positions):
    """solver_multiagent.py:175-186."""
    out = np.empty((len(st.pair_i), st.P.shape[0], 3))
    for p in range(len(st.pair_i)):
        i, j = st.pair_i[p], st.pair_j[p]
        if j >= 0:
            out[p] = positions[i] - positions[j]
        else:
            out[p] = positions[i] - prob.statics[st.pair_s[p]][None, :]
    return out


def reconstruction(st: Structure, state: State):
    """solver_multiagent.py:189-200."""
    sb, cb = np.sin(state.beta), np.cos(state.beta)
    sa, ca = np.sin(state.alpha), np.cos(state.alpha)
    return np.stack([st.pa * state.d * sb * ca, st.pa * state.d * sb * sa, st.pb * state.d * cb], axis=-1)


def residuals(st: Structure, prob: Problem, state: State):
    """solver_multiagent.py:203-208 -> (3, n_pairs, n_p)."""
    deltas = pair_deltas(st, prob, agent_positions(st, state.xi))
    return np.transpose(deltas - reconstruction(st, state), (2, 0, 1))


def init_state(st: Structure, prob: Problem, P):
    """solver_multiagent.py:228-249 (bvals rows per agent: [p0 v0 a0 p1 v1 a1])."""
    n_p = P.shape[0]
    n_pairs = len(st.pair_i)
    xi = np.empty((3, st.n_a * st.m))
    for k in range(3):
        for i in range(st.n_a):
            p0, p1 = prob.b_eq[k][6 * i + 0], prob.b_eq[k][6 * i + 3]
            line = np.linspace(p0, p1, n_p)
            coeffs, *_ = np.linalg.lstsq(P, line, rcond=None)
            xi[k, i * st.m:(i + 1) * st.m] = coeffs
    state = State(xi=xi, d=np.ones((n_pairs, n_p)), alpha=np.zeros((n_pairs, n_p)),
                  beta=np.full((n_pairs, n_p), np.pi / 2), lam=np.zeros((3, n_pairs, n_p)))
    if n_pairs:
        deltas = pair_deltas(st, prob, agent_positions(st, xi))
        state.alpha = np.arctan2(deltas[:, :, 1], deltas[:, :, 0])
        planar = np.hypot(deltas[:, :, 0] / st.pa, deltas[:, :, 1] / st.pa)
        state.beta = np.arctan2(planar, deltas[:, :, 2] / st.pb)
    return state


def iterate(state: State, st: Structure, prob: Problem, kinv=None):
    """solver_multiagent.py:252-297 (kinv: optional per-level explicit inverses, the device's contraction)."""
    rho = st.rho_levels[state.level]
    n_p = st.P.shape[0]
    n_pairs = len(st.pair_i)
    if n_pairs:
        recon = reconstruction(st, state)
        qs = np.empty((3, st.n_a * st.m))
        statics = np.zeros((n_pairs, n_p, 3))
        for p in range(n_pairs):
            if st.pair_j[p] < 0:
                statics[p] = prob.statics[st.pair_s[p]][None, :]
        for k in range(3):
            b_fo = recon[:, :, k] - state.lam[k] / rho + statics[:, :, k]
            qs[k] = -rho * (st.A_fo.T @ b_fo.ravel())
    else:
        qs = np.zeros((3, st.n_a * st.m))
    block = np.hstack([-qs, prob.b_eq]).T
    sol = lu_solve(st.lus[state.level], block) if kinv is None else kinv[state.level] @ block
    state.xi = sol[: st.n_a * st.m].T
    if not n_pairs:
        state.iteration += 1
        return
    deltas = pair_deltas(st, prob, agent_positions(st, state.xi))
    dx, dy, dz = deltas[:, :, 0], deltas[:, :, 1], deltas[:, :, 2]
    state.alpha = np.arctan2(dy, dx)
    planar = np.hypot(dx / st.pa, dy / st.pa)
    state.beta = np.arctan2(planar, dz / st.pb)
    sb, cb = np.sin(state.beta), np.cos(state.beta)
    sa, ca = np.sin(state.alpha), np.cos(state.alpha)
    shift = state.lam / rho
    num = st.pa * sb * (ca * (dx + shift[0]) + sa * (dy + shift[1])) + st.pb * cb * (dz + shift[2])
    den = st.pa**2 * sb**2 + st.pb**2 * cb**2
    state.d = np.clip(num / den, 1.0, D_CAP)
    res = residuals(st, prob, state)
    state.lam = state.lam + rho * res
    state.iteration += 1


def solve(st: Structure, prob: Problem, P, max_iter=200, tol_norm=0.01, stall_window=5, stall_improvement=0.01,
          kinv=None, state=None):
    """solve_joint's loop (solver_multiagent.py:306-335) -> (state, history [(norm, max, rho)], converged)."""
    state = state or init_state(st, prob, P)
    history = []
    last_change = 0
    converged = False
    n_levels = len(st.rho_levels)
    for _ in range(max_iter):
        iterate(state, st, prob, kinv)
        res = residuals(st, prob, state)
        norm = float(np.linalg.norm(res))
        mx = float(np.max(np.abs(res))) if res.size else 0.0
        history.append((norm, mx, st.rho_levels[state.level]))
        if norm <= tol_norm:
            converged = True
            break
        scheduled = min(int(state.iteration * n_levels / max(max_iter, 1)), n_levels - 1)
        w = stall_window
        stalled = False
        if len(history) >= 2 * w and state.iteration - last_change >= w:
            recent = np.mean([h[0] for h in history[-w:]])
            previous = np.mean([h[0] for h in history[-2 * w:-w]])
            stalled = previous > 0 and (previous - recent) / previous < stall_improvement
        target = max(scheduled, state.level + 1 if stalled else state.level)
        if target > state.level and state.level < n_levels - 1:
            state.level = min(target, n_levels - 1)
            last_change = state.iteration
    return state, np.array(history), converged
