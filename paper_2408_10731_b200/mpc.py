"""Receding-horizon driving with device-resident warm state.

The reference drives ONE robot at a time (bench/runner.py:326-439): every control step it re-predicts the
obstacle tracks, rebuilds the problem from the executed state, warm-starts ``solve_single`` from the previous
state (``iteration = 0``), executes the first ``n_exec`` samples against the true obstacle motion and stops on
collision or goal proximity.  ``MpcFleet`` runs that loop for B robots in one scenario at once on an Alg. 1
engine whose state (xi, multipliers, angles, penalties, d) never leaves the GPU:

    per control step  predict tracks (tro_predict_tracks_f64, bit-exact with predict_obstacles)
                      warm prime (d_mode 1)  ->  step_budget fused AM iterations (CUDA graph)
                      per-step metrics (tro_validate_f64, the reference's eval_metrics per record)
                      tro_mpc_advance_f64: execute, collide / goal tests, next boundary + desired + q,
                      warm d of the final iterate, solve-local bookkeeping reset

The host only uploads the time tables once and reads the results at the end.  ``receding_horizon_run``
(bench/runner.py) is a fleet of one for the single solver.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._alg1 import LOOP_MAX_MEMBERS, Alg1Engine
from .basis import Trajectory, build_basis
from .metrics import RunMetrics

__all__ = ["MpcFleet", "FleetResult", "control_times"]


def control_times(dt: float, n_steps: int, n_exec: int):
    """(t_now per control step (n_steps,), executed sample times (n_steps, n_exec)) by the reference's own
    accumulation ``t_abs += dt`` (runner.py:411), so the tables hold the identical floats."""
    t_now = np.empty(n_steps)
    t_exec = np.empty((n_steps, n_exec))
    t_abs = 0.0
    for k in range(n_steps):
        t_now[k] = t_abs
        for s in range(n_exec):
            t_abs += dt
            t_exec[k, s] = t_abs
    return t_now, t_exec


@dataclass
class FleetResult:
    """Per-robot outcome of a fleet run (arrays over robots; steps = control steps actually solved)."""

    n_steps: int
    n_exec: int
    step_budget: int
    flags: np.ndarray       # (B,) 1 collided, 2 reached, 0 still driving
    trace: np.ndarray       # (B, cap, dim) executed positions (first n_trace valid)
    n_trace: np.ndarray     # (B,)
    metrics: np.ndarray     # (n_steps, B, 5) smoothness, tracking, arc length, worst, clearance bound
    residual: np.ndarray    # (n_steps, B) residual norm of each step's final iterate
    step_ms: np.ndarray     # (n_steps,) device time of each control step's solve (prime + iterations)
    exec_times: np.ndarray  # (1 + n_steps * n_exec,) time of each trace sample
    scenario_id: str
    solver: str = "single"
    seed: int = 0

    @property
    def collided(self) -> np.ndarray:
        return self.flags == _lib.TRO_MPC_COLLIDED

    @property
    def reached(self) -> np.ndarray:
        return self.flags == _lib.TRO_MPC_REACHED

    def steps_of(self, i: int) -> int:
        """Control steps robot i was solved for (the reference's record count)."""
        n = int(self.n_trace[i]) - 1
        return min(self.n_steps, -(-n // self.n_exec)) if n > 0 else 0

    def member(self, i: int):
        """Robot i as the reference's MpcResult (runner.py:50-56, 421-439)."""
        from .bench.runner import MpcResult, RunRecord

        steps = self.steps_of(i)
        reached, collided = bool(self.reached[i]), bool(self.collided[i])
        success = reached and not collided
        records = []
        for k in range(steps):
            mt = self.metrics[k, i]
            m = RunMetrics(smoothness=float(mt[0]), tracking=float(mt[1]), arc_length=float(mt[2]),
                           success=success if k == steps - 1 else False, iters=self.step_budget,
                           residual_final=float(self.residual[k, i]), min_clearance=float(mt[4]),
                           wall_time_ms=float(self.step_ms[k]))
            records.append(RunRecord(scenario_id=f"{self.scenario_id}#step{k}", solver=self.solver, seed=self.seed,
                                     metrics=m))
        n = int(self.n_trace[i])
        executed = None
        if n > 1:
            p = self.trace[i, :n].copy()
            t = self.exec_times[:n].copy()
            v = np.gradient(p, t, axis=0)
            executed = Trajectory(t=t, pos=p, vel=v, acc=np.gradient(v, t, axis=0))
        return MpcResult(records=records, success=success, reached_goal=reached, collided=collided, executed=executed)


class MpcFleet:
    """B robots (starts / goals (B, dim)) driving through ``scenario`` with the single-robot solver.

    Defaults follow receding_horizon_run (runner.py:326-334): step_budget 40, exec_fraction 0.1,
    goal_radius 0.5, plan margin 0.05; the basis is the scenario horizon's degree-10 Bernstein basis.
    ``layout`` selects the engine's word layout ("half": the reference's 9 words, the fastest)."""

    def __init__(self, scenario, starts=None, goals=None, *, step_budget: int = 40, exec_fraction: float = 0.1,
                 goal_radius: float = 0.5, plan_margin: float = 0.05, params=None, layout: str = "half",
                 record_metrics: bool = True, device=None, solver_label: str = "single", seed: int = 0):
        from .bench.scenarios import obstacle_arrays, predict_obstacles
        from .solver_single import SingleParams

        _lib.require_cuda()
        self.lib = _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.scenario = scenario
        h = scenario.horizon
        self.basis = basis = build_basis(h.t0, h.tf, h.n_p, degree=10)
        self.dim = dim = int(scenario.dim)
        self.n_p, self.m = basis.n_p, basis.n_var
        self.n_exec = max(1, int(round(exec_fraction * basis.n_p)))
        self.dt = basis.grid.dt
        self.step_budget = int(step_budget)
        self.goal_radius = float(goal_radius)
        self.record_metrics = record_metrics
        self.solver_label, self.seed = solver_label, int(seed)
        starts = np.atleast_2d(np.asarray(scenario.boundary.start if starts is None else starts, dtype=float))
        goals = np.atleast_2d(np.asarray(scenario.boundary.goal if goals is None else goals, dtype=float))
        if starts.shape[1] != dim or goals.shape != starts.shape:
            raise ValueError("starts / goals must be (B, dim) and match")
        self.B = B = starts.shape[0]
        c, v, a, b = obstacle_arrays(scenario)
        self.n_o = n_o = a.size
        pa, pb = (a + plan_margin, b + plan_margin) if plan_margin != 0.0 else (a, b)
        tracks0 = (np.stack([t.centers for t in predict_obstacles(scenario, basis.grid.timestamps)])
                   if n_o else np.zeros((0, basis.n_p, dim)))
        bvals = np.zeros((B, dim, 6))
        bvals[:, :, 0] = starts
        bvals[:, :, 3] = goals
        self.params = params or SingleParams(max_iter=self.step_budget)
        self.eng = Alg1Engine(basis, tracks0, pa, pb, bvals, np.zeros((B, dim, self.m)), params=self.params,
                              layout=layout, device=dev)
        # the fleet owns its solve-local bookkeeping (tro_mpc_advance resets it per control step and freezes
        # finished robots through status): the init launch must not reset it
        self.eng._consts.level0 = None
        # the fleet re-predicts the tracks into eng.tracks every control step: stream them (no register tracks)
        self.eng._consts.track_lin = None
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        up = lambda x: torch.as_tensor(np.array(x, dtype=float, copy=True), **f64)  # noqa: E731
        self.Pdot, self.Pddot = up(basis.Pdot), up(basis.Pddot)
        self.frac = up(np.linspace(0.0, 1.0, basis.n_p))
        self.ts = up(basis.grid.timestamps)
        self.goal = up(goals)
        self.centers, self.velocities = up(c.reshape(-1) if n_o else np.zeros(1)), up(v.reshape(-1) if n_o else np.zeros(1))
        self.raw_a, self.raw_b = up(a if n_o else np.ones(1)), up(b if n_o else np.ones(1))
        self.d = torch.ones((B, max(n_o, 1), basis.n_p), **f64)
        self.desired = torch.empty((B, basis.n_p, dim), **f64)
        self.flags = torch.zeros(B, **i32)
        self.n_trace = torch.zeros(B, **i32)
        # the robots still driving, compacted on the device after every control step: the persistent
        # iteration kernel works through this list only (frozen robots cost nothing, the rest stay balanced)
        self.order = torch.arange(B, **i32)
        self.n_order = torch.full((1,), B, **i32)
        self.eng._state.order = self.order.data_ptr()
        self.eng._state.n_order = self.n_order.data_ptr()
        self._i32 = i32
        self._f64 = f64
        self._mdims = None

    # ------------------------------------------------------------ launches
    def _advance(self, mode: int, k: int, t_exec_dev, res_out):
        e = self.eng
        self._mdims.n_exec = self.n_exec
        consts = _lib.MpcConsts(
            P=e.P.data_ptr(), Pdot=self.Pdot.data_ptr(), Pddot=self.Pddot.data_ptr(), frac=self.frac.data_ptr(),
            goal=self.goal.data_ptr(), centers=self.centers.data_ptr() if self.n_o else None,
            velocities=self.velocities.data_ptr() if self.n_o else None,
            shape_a=self.raw_a.data_ptr() if self.n_o else None, shape_b=self.raw_b.data_ptr() if self.n_o else None,
            plan_a=e.shape_a.data_ptr(), plan_b=e.shape_b.data_ptr(), tracks=e.tracks.data_ptr() if self.n_o else None,
            t_exec=t_exec_dev[k].data_ptr() if mode else None, goal_radius=self.goal_radius,
            w_track=1.0)
        io = _lib.MpcIO(bvals=e.bvals.data_ptr(), q=e.q.data_ptr(), desired=self.desired.data_ptr(),
                        d=self.d.data_ptr() if (mode and self.n_o) else None, trace=self.trace.data_ptr(),
                        n_trace=self.n_trace.data_ptr(), flags=self.flags.data_ptr(),
                        res_out=res_out[k].data_ptr() if (mode and res_out is not None) else None)
        with torch.cuda.device(self.device):
            rc = self.lib.tro_mpc_advance_f64(int(mode), ctypes.byref(self._mdims), ctypes.byref(consts),
                                              ctypes.byref(e._state), ctypes.byref(io), _lib.stream_handle())
        _lib.check(rc, "tro_mpc_advance_f64")
        self._compact()

    def _compact(self):
        with torch.cuda.device(self.device):
            rc = self.lib.tro_mpc_compact(self.B, self.flags.data_ptr(), self.order.data_ptr(),
                                          self.n_order.data_ptr(), _lib.stream_handle())
        _lib.check(rc, "tro_mpc_compact")

    def _predict(self, t_now_dev, k: int):
        if not self.n_o:
            return
        dims = _lib.TrackDims(n_scen=1, n_obs=self.n_o, n_p=self.n_p, dim=self.dim, layout=1, shared_obstacles=0)
        with torch.cuda.device(self.device):
            rc = self.lib.tro_predict_tracks_f64(ctypes.byref(dims), self.centers.data_ptr(),
                                                 self.velocities.data_ptr(), self.ts.data_ptr(),
                                                 t_now_dev[k:k + 1].data_ptr(), self.eng.tracks.data_ptr(),
                                                 _lib.stream_handle())
        _lib.check(rc, "tro_predict_tracks_f64")

    def _validate(self, out_row):
        e = self.eng
        dims = _lib.ValDims(n_members=self.B, n_obs=self.n_o, n_p=self.n_p, m=self.m, dim=self.dim,
                            per_member_desired=1, reserved=0)
        consts = _lib.ValConsts(P=e.P.data_ptr(), Pdd=self.Pddot.data_ptr(), t=self.ts.data_ptr(),
                                centers=self.centers.data_ptr() if self.n_o else None,
                                velocities=self.velocities.data_ptr() if self.n_o else None,
                                shape_a=self.raw_a.data_ptr() if self.n_o else None,
                                shape_b=self.raw_b.data_ptr() if self.n_o else None,
                                desired=self.desired.data_ptr(), margin=0.0)
        io = _lib.ValIO(xi=e.xi.data_ptr(), pos=None, acc=None, out=out_row.data_ptr())
        with torch.cuda.device(self.device):
            rc = self.lib.tro_validate_f64(ctypes.byref(dims), ctypes.byref(consts), ctypes.byref(io),
                                           _lib.stream_handle())
        _lib.check(rc, "tro_validate_f64")

    def _solve(self, first: bool):
        """One control step's solve_single: prime (cold or warm), then step_budget AM iterations; only the
        first iteration reads d (d_mode 1), the rest recompute it, so the graph runs with d = NULL."""
        e = self.eng
        n = self.step_budget
        if first:
            e.cold_init()
            d_mode = 0
        else:
            e._state.d = self.d.data_ptr()
            e.prime(1)
            d_mode = 1
        if n > 0:
            e.iterate(d_mode)
        e._state.d = None
        rest = n - 1
        if rest <= 0:
            return
        if self.B <= LOOP_MAX_MEMBERS:
            e.iterate_n(rest)
            return
        if e._graph is None or e._graph_n != rest:
            e._capture(rest)
        e._graph.replay()

    # ------------------------------------------------------------ driver
    def run(self, n_steps: int = 30, *, early_exit: bool = True, check_every: int = 1) -> FleetResult:
        """Drive every robot for up to n_steps control steps (runner.py:362-428)."""
        B, dim = self.B, self.dim
        t_now, t_exec = control_times(self.dt, n_steps, self.n_exec)
        t_now_dev = torch.as_tensor(t_now, **self._f64)
        t_exec_dev = torch.as_tensor(t_exec, **self._f64)
        cap = 1 + n_steps * self.n_exec
        self.trace = torch.zeros((B, cap, dim), **self._f64)
        self.n_trace.zero_()
        self.flags.zero_()
        metrics = torch.full((max(n_steps, 1), B, 5), float("nan"), **self._f64)
        res = torch.full((max(n_steps, 1), B), float("nan"), **self._f64)
        self._mdims = _lib.MpcDims(n_members=B, n_obs=self.n_o, n_p=self.n_p, m=self.m, dim=dim, n_exec=self.n_exec,
                                   trace_cap=cap, ring_len=2 * self.params.stall_window)
        e = self.eng
        e.reset_cold()
        if n_steps:
            self._predict(t_now_dev, 0)
        self._advance(0, 0, t_exec_dev, None)  # start: collision at t = 0, first problem
        events = []
        ran = 0
        for k in range(n_steps):
            if early_exit and k % max(check_every, 1) == 0 and bool((self.flags != 0).all().item()):
                break
            if k > 0:
                self._predict(t_now_dev, k)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            self._solve(first=(k == 0))
            ev1.record()
            events.append((ev0, ev1))
            if self.record_metrics:
                self._validate(metrics[k])
            self._advance(1, k, t_exec_dev, res)
            ran += 1
        torch.cuda.synchronize(self.device)
        step_ms = np.array([a.elapsed_time(b) for a, b in events])
        exec_times = np.concatenate([[0.0], t_exec.reshape(-1)])
        return FleetResult(n_steps=ran, n_exec=self.n_exec, step_budget=self.step_budget,
                           flags=self.flags.cpu().numpy(), trace=self.trace.cpu().numpy(),
                           n_trace=self.n_trace.cpu().numpy(), metrics=metrics[:ran].cpu().numpy(),
                           residual=res[:ran].cpu().numpy(), step_ms=step_ms, exec_times=exec_times,
                           scenario_id=self.scenario.scenario_id, solver=self.solver_label, seed=self.seed)
