"""CPU ORACLE for receding-horizon driving (single solver) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may use this module.
numpy restatement of the reference ``trajopt.bench.runner.receding_horizon_run`` (bench/runner.py:326-439)
for the single solver, over a fleet of robots that share one scenario (each robot's loop is independent;
they advance in lockstep, so they share t_abs and the predicted tracks), on top of ``oracle.alg1`` (the
pinned restatement of ``solve_single``).  A robot's numbers equal the reference's own run from its start
and goal: pinned against ``tests/golden/mpc.npz`` (the live reference's ``receding_horizon_run``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import alg1
from . import metrics as om


def predict(centers, velocities, timestamps, t_now):
    """bench/scenarios.py:118-127 -> (n_o, n_p, dim)."""
    rel = (t_now + timestamps - timestamps[0])[:, None]
    return np.stack([centers[j][None, :] + velocities[j][None, :] * rel for j in range(len(centers))]) \
        if len(centers) else np.zeros((0, timestamps.size, centers.shape[1] if centers.ndim == 2 else 2))


def in_collision(pos, t_abs, centers, velocities, a, b, dim) -> bool:
    """runner.py:307-323."""
    for j in range(len(a)):
        delta = pos - (centers[j] + velocities[j] * t_abs)
        if dim == 3:
            quad = delta[0] ** 2 / a[j] ** 2 + delta[1] ** 2 / a[j] ** 2 + delta[2] ** 2 / b[j] ** 2
        else:
            quad = delta[0] ** 2 / a[j] ** 2 + delta[1] ** 2 / b[j] ** 2
        if quad < 1.0:
            return True
    return False


@dataclass
class MpcOut:
    flags: np.ndarray          # (B,) 1 collided, 2 reached
    traces: list               # per robot (n, dim) executed positions
    times: list                # per robot (n,) sample times
    metrics: list              # per robot list of (smoothness, tracking, arc, worst, clearance) per step
    residuals: list            # per robot list of residual norms per step


def run(P, Pd, Pdd, timestamps, centers, velocities, a, b, starts, goals, *, step_budget=40, n_steps=30,
        goal_radius=0.5, exec_fraction=0.1, plan_margin=0.05, params: alg1.Params | None = None) -> MpcOut:
    """receding_horizon_run(scenario, "single", ...) for every robot (starts / goals (B, dim))."""
    starts = np.atleast_2d(np.asarray(starts, float))
    goals = np.atleast_2d(np.asarray(goals, float))
    B, dim = starts.shape
    n_p = P.shape[0]
    n_exec = max(1, int(round(exec_fraction * n_p)))  # runner.py:346
    params = params or alg1.Params(max_iter=step_budget)
    pa = a + plan_margin if plan_margin != 0.0 else a
    pb = b + plan_margin if plan_margin != 0.0 else b
    frac = np.linspace(0.0, 1.0, n_p)[:, None]
    pos = starts.copy()
    vel = np.zeros((B, dim))
    acc = np.zeros((B, dim))
    t_abs = 0.0
    traces = [[starts[i].copy()] for i in range(B)]
    times = [[0.0] for _ in range(B)]
    mets = [[] for _ in range(B)]
    ress = [[] for _ in range(B)]
    flags = np.array([1 if in_collision(starts[i], 0.0, centers, velocities, a, b, dim) else 0 for i in range(B)])
    state = None
    kkt = None
    dt = _dt(timestamps)
    for _ in range(n_steps):
        act = np.nonzero(flags == 0)[0]
        if act.size == 0:
            break
        tracks = predict(centers, velocities, timestamps, t_abs)
        bvals = np.zeros((act.size, dim, 6))
        bvals[:, :, 0] = pos[act]
        bvals[:, :, 1] = vel[act]
        bvals[:, :, 2] = acc[act]
        bvals[:, :, 3] = goals[act]
        desired = np.stack([pos[i][None, :] + frac * (goals[i] - pos[i])[None, :] for i in act])  # runner.py:369-370
        prob = alg1.Problem(P=P, Pd=Pd, Pdd=Pdd, bvals=bvals, desired=desired, tracks=tracks, a=pa, b=pb)
        if kkt is None:
            kkt = alg1.KKTCache(prob)
        kkt.prob = prob
        sub = None
        if state is not None:
            sub = state if act.size == B else alg1._subset(_full_problem_like(prob, B), state, act)[1]
            sub.iteration[:] = 0  # runner.py:376-377
        st = alg1.solve(prob, params, state=sub, kkt=kkt).state
        norms, _ = alg1.residual_extremes(st, prob)
        if state is None:
            state = _expand(st, act, B)
        elif st is not state:
            alg1._scatter(state, st, act)
        t_step = t_abs
        for n, i in enumerate(act):
            xi = st.xi[n]
            tp, tv, ta = P @ xi.T, Pd @ xi.T, Pdd @ xi.T  # solver_single.py:429-434
            t_abs_i = t_step
            for k in range(1, n_exec + 1):  # runner.py:407-419
                pos[i], vel[i], acc[i] = tp[k].copy(), tv[k].copy(), ta[k].copy()
                t_abs_i += dt
                traces[i].append(pos[i].copy())
                times[i].append(t_abs_i)
                if in_collision(pos[i], t_abs_i, centers, velocities, a, b, dim):
                    flags[i] = 1
                    break
                if np.linalg.norm(pos[i] - goals[i]) <= goal_radius:
                    flags[i] = 2
                    break
            mets[i].append(om.metrics(tp, ta, timestamps, centers, velocities, a, b, dim, desired=desired[n]))
            ress[i].append(float(norms[n]))
        for k in range(n_exec):  # the lockstep clock (members that stopped no longer use it)
            t_abs += dt
    return MpcOut(flags=flags, traces=[np.array(t) for t in traces], times=[np.array(t) for t in times],
                  metrics=mets, residuals=ress)


def _dt(timestamps):
    """basis.py TimeGrid.dt: (tf - t0) / (n_p - 1)."""
    return (timestamps[-1] - timestamps[0]) / (timestamps.size - 1)


def _full_problem_like(prob, B):
    return alg1.Problem(P=prob.P, Pd=prob.Pd, Pdd=prob.Pdd, bvals=np.zeros((B,) + prob.bvals.shape[1:]),
                        desired=np.zeros((B,) + prob.desired.shape[1:]), tracks=prob.tracks, a=prob.a, b=prob.b)


def _expand(st, act, B):
    """A full-fleet state holding st's members at rows act (the others are never read again)."""
    if act.size == B:
        return st
    kw = {}
    for k in alg1._ARRAYS:
        v = getattr(st, k)
        if v is None:
            kw[k] = None
            continue
        full = np.zeros((B,) + v.shape[1:], dtype=v.dtype)
        full[act] = v
        kw[k] = full
    out = alg1.State(**kw, factor_rho_o=[None] * B)
    for n, i in enumerate(act):
        out.factor_rho_o[i] = st.factor_rho_o[n]
    return out
