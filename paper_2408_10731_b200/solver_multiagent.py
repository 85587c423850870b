"""Joint multi-agent trajectory optimization on B200 (drop-in for ``trajopt.solver_multiagent``).

Same public surface as the reference module (solver_multiagent.py:32-368):
``StaticSphere``, ``MultiAgentProblem``, ``JointParams``, ``JointState``,
``JointSolution``, ``inflate_radius``, ``pairwise_residuals``,
``pairwise_residuals_arrays``, ``solve_joint`` — plus ``solve_joint_batch``
for B independent problems that share the agent count, agent shape, basis and
static-sphere radii (the C3 configuration: 4096 sixteen-agent problems).

Every iteration of every problem is one CTA of the fused ``tro_ma_run`` kernel
(QP contraction with the level's K^-1, trig-free polar updates, multiplier
ascent, fixed-order agent sums, residual norm and the staged level schedule).
Host work: the one-off structure (pairs, A_fo, 10 saddle factorizations, exactly
as the reference builds them) and result formatting.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch


def _graphs_allowed() -> bool:
    """CUDA-graph capture only on the main thread: a capture is invalidated by launches other threads make on
    the legacy default stream at the same time, so solver instances running in other threads launch their
    iterations directly (same kernels, same results)."""
    import threading

    return threading.current_thread() is threading.main_thread()

from . import _lib, qpcore
from .basis import AxisBoundary, BasisSet, Trajectory, boundary_matrix, line_basis_vectors  # noqa: F401
from .geometry import D_CAP, EllipsoidShape  # noqa: F401

__all__ = [
    "StaticSphere",
    "MultiAgentProblem",
    "JointParams",
    "JointState",
    "JointSolution",
    "inflate_radius",
    "pairwise_residuals",
    "pairwise_residuals_arrays",
    "solve_joint",
    "solve_joint_batch",
]


@dataclass(frozen=True)
class StaticSphere:
    center: np.ndarray
    radius: float


@dataclass
class MultiAgentProblem:
    basis: BasisSet
    boundaries: list
    agent_shape: EllipsoidShape
    static_obstacles: list = field(default_factory=list)

    @property
    def n_agents(self) -> int:
        return len(self.boundaries)

    def __post_init__(self):
        if self.n_agents < 1:
            raise ValueError("need at least one agent")


@dataclass
class JointParams:
    max_iter: int = 200
    tol_norm: float = 0.01
    tol_max: float = 1e-3
    rho_start: float = 1.0
    rho_final: float = 1e4
    rho_levels: int = 10
    stall_window: int = 5
    stall_improvement: float = 0.01
    inflation_factor: float = 4.0
    typical_residual: float = 0.01


@dataclass
class JointState:
    xi: np.ndarray
    d: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    lam: np.ndarray
    level: int = 0
    iteration: int = 0


@dataclass
class JointSolution:
    trajectories: list
    converged: bool
    iterations: int
    residual_norm: float
    residual_max: float
    residual_history: list
    min_pair_distance: float
    inflated_radius: tuple
    n_factorizations: int
    state: JointState


def inflate_radius(radius: float, typical_residual: float, factor: float) -> float:
    """Planning radius absorbing the expected terminal residual (solver_multiagent.py:93-97)."""
    if radius < 0 or typical_residual < 0 or factor < 0:
        raise ValueError("inflation inputs must be non-negative")
    return radius + factor * typical_residual


def _colour_order(n_a: int, pi, pj, ps) -> np.ndarray:
    """Reference pair indices in colour-major order: the agent pairs by the circle method (n_a - 1 perfect
    matchings for even n_a, n_a near-perfect ones for odd), then one colour per static sphere."""
    index = {(i, j): p for p, (i, j) in enumerate(zip(pi, pj)) if j >= 0}
    order = []
    n = n_a + (n_a & 1)  # a dummy agent for odd n_a
    ring = list(range(n))
    for _ in range(n - 1):
        rnd = []
        for k in range(n // 2):
            a, b = ring[k], ring[n - 1 - k]
            if a < n_a and b < n_a:
                rnd.append(index[(min(a, b), max(a, b))])
        order.extend(sorted(rnd, key=lambda p: pi[p]))
        ring = [ring[0]] + [ring[-1]] + ring[1:-1]
    statics = sorted((p for p in range(len(pi)) if pj[p] < 0), key=lambda p: (ps[p], pi[p]))
    order.extend(statics)
    assert sorted(order) == list(range(len(pi)))
    return np.asarray(order, np.int64)


class _Structure:
    """Pairs, A_fo, and the level factorizations (solver_multiagent.py:100-165)."""

    def __init__(self, problem: MultiAgentProblem, params: JointParams):
        basis = problem.basis
        self.basis = basis
        m, n_p, n_a = basis.n_var, basis.n_p, problem.n_agents
        self.m, self.n_a, self.n_p = m, n_a, n_p
        a_inf = inflate_radius(problem.agent_shape.a, params.typical_residual, params.inflation_factor)
        b_inf = inflate_radius(problem.agent_shape.b, params.typical_residual, params.inflation_factor)
        self.inflated = (a_inf, b_inf)
        pi, pj, ps, pa, pb = [], [], [], [], []
        for i in range(n_a):
            for j in range(i + 1, n_a):
                pi.append(i), pj.append(j), ps.append(-1), pa.append(2.0 * a_inf), pb.append(2.0 * b_inf)
        for s, sphere in enumerate(problem.static_obstacles):
            for i in range(n_a):
                pi.append(i), pj.append(-1), ps.append(s)
                pa.append(a_inf + sphere.radius), pb.append(b_inf + sphere.radius)
        self.pair_i, self.pair_j, self.pair_s = np.array(pi), np.array(pj), np.array(ps)
        self.pa, self.pb = np.asarray(pa, float), np.asarray(pb, float)
        self.n_pairs = len(pi)
        self.n_static = len(problem.static_obstacles)
        A_fo = np.zeros((self.n_pairs * n_p, n_a * m))
        for p in range(self.n_pairs):
            rows = slice(p * n_p, (p + 1) * n_p)
            A_fo[rows, pi[p] * m:(pi[p] + 1) * m] = basis.P
            if pj[p] >= 0:
                A_fo[rows, pj[p] * m:(pj[p] + 1) * m] = -basis.P
        Q = np.kron(np.eye(n_a), basis.Pddot.T @ basis.Pddot)
        self.A_eq = np.kron(np.eye(n_a), boundary_matrix(basis))
        if self.n_pairs:
            AtA = A_fo.T @ A_fo
            ratio = (params.rho_final / params.rho_start) ** (1.0 / max(params.rho_levels - 1, 1))
            self.rho_levels = [params.rho_start * ratio**k for k in range(params.rho_levels)]
            self.factors = [qpcore.factorize(Q + r * AtA, self.A_eq) for r in self.rho_levels]
        else:
            self.rho_levels = [params.rho_start]
            self.factors = [qpcore.factorize(Q, self.A_eq)]
        self.n_factorizations = len(self.factors)
        # Device pair order: colour-major (a proper edge colouring, round-robin for the agent pairs, one colour
        # per static sphere), so that at step q of the per-agent scatter every agent reads a pair of colour q,
        # and the pairs of one colour sit in consecutive scratch records (conflict-free shared-memory reads).
        # dev_perm[d] = the reference index of device pair d; the engine's pair planes use the device order.
        self.dev_perm = _colour_order(n_a, pi, pj, ps)
        dpi, dpj = self.pair_i[self.dev_perm], self.pair_j[self.dev_perm]
        # CSR incidence over device pairs: per agent, the pairs it is first (+) / second (-) member of, in
        # device (= colour) order
        inc_ptr, inc = [0], []
        for a in range(n_a):
            for p in range(self.n_pairs):
                if dpi[p] == a:
                    inc.append(p)
                elif dpj[p] == a:
                    inc.append(-p - 1)
            inc_ptr.append(len(inc))
        self.inc_ptr, self.inc_pair = np.array(inc_ptr, np.int32), np.array(inc, np.int32)

    def key(self):
        return (self.n_a, self.m, self.n_p, self.n_pairs, tuple(self.pa), tuple(self.pb), tuple(self.rho_levels))


def _b_eq(problem: MultiAgentProblem) -> np.ndarray:
    """(3, 6 n_a) boundary values per axis (solver_multiagent.py:149-154)."""
    return np.stack([np.concatenate([problem.boundaries[i][k].values() for i in range(problem.n_agents)])
                     for k in range(3)])


class MaEngine:
    """B problems sharing one _Structure, resident on one device."""

    def __init__(self, struct: _Structure, b_eq: np.ndarray, statics: np.ndarray | None, params: JointParams, *,
                 device=None, max_hist: int = 0, export: bool = False, split_qp: bool = True, qp: str = "dmma",
                 ozaki_slices: int = 8):
        # the QP step: "dmma" (tro_ma_run mode 3, fp64 mma.sync), "ozaki" (tro_ma_qp_ozaki: exact int8 GEMM on
        # tcgen05 / TMEM), each followed by the element pass (mode 4); split_qp=False: the fused mode 0
        self.split_qp = split_qp
        if qp not in ("dmma", "ozaki"):
            raise ValueError("qp must be 'dmma' or 'ozaki'")
        self.qp = qp
        _lib.require_cuda()
        self.lib = _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device, self.struct, self.params = dev, struct, params
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        B = int(b_eq.shape[0])
        self.B = B
        n_a, m, n_p, npairs = struct.n_a, struct.m, struct.n_p, struct.n_pairs
        nk = n_a * m + struct.A_eq.shape[0]
        self.P = torch.as_tensor(np.array(struct.basis.P), **f64)
        self.kinv = torch.as_tensor(np.stack([f.kinv for f in struct.factors]), **f64).contiguous()
        assert self.kinv.shape[1] == nk
        self.level_rho = torch.as_tensor(np.asarray(struct.rho_levels), **f64)
        perm = struct.dev_perm  # device pair d = reference pair perm[d]
        self._perm = torch.as_tensor(perm, dtype=torch.long, device=self.device)
        self._inv = torch.as_tensor(np.argsort(perm), dtype=torch.long, device=self.device)
        self.pair_i = torch.as_tensor(struct.pair_i[perm].astype(np.int32), **i32)
        self.pair_j = torch.as_tensor(struct.pair_j[perm].astype(np.int32), **i32)
        self.pair_s = torch.as_tensor(struct.pair_s[perm].astype(np.int32), **i32)
        self.pair_a = torch.as_tensor(struct.pa[perm], **f64)
        self.pair_b = torch.as_tensor(struct.pb[perm], **f64)
        self.inc_ptr = torch.as_tensor(struct.inc_ptr, **i32)
        self.inc_pair = torch.as_tensor(struct.inc_pair, **i32)
        self.b_eq = torch.as_tensor(np.ascontiguousarray(b_eq), **f64)
        self.statics = (torch.as_tensor(np.ascontiguousarray(statics), **f64)
                        if struct.n_static else None)
        u, v = line_basis_vectors(struct.basis)
        self.line_u, self.line_v = torch.as_tensor(u, **f64), torch.as_tensor(v, **f64)
        # one agent's boundary rows and their pseudo-inverse: the boundary projection after each QP step
        Ab = boundary_matrix(struct.basis)
        self.bnd = torch.as_tensor(np.concatenate([Ab.ravel(), np.linalg.pinv(Ab).ravel()]), **f64)
        self.state = torch.zeros((B, n_p, 3, npairs), **f64)
        self.xi = torch.zeros((B, 3, n_a * m), **f64)
        self.sums = torch.zeros((B, 2, n_a, 3, m), **f64)
        self.ring = torch.zeros((B, 2 * params.stall_window), **f64)
        self.res_norm = torch.zeros(B, **f64)
        self.res_max = torch.zeros(B, **f64)
        self.max_hist = int(max_hist)
        self.hist = torch.zeros((B, max(self.max_hist, 1), 3), **f64) if self.max_hist else None
        self.level = torch.zeros(B, **i32)
        self.iteration = torch.zeros(B, **i32)
        self.last_change = torch.zeros(B, **i32)
        self.n_hist = torch.zeros(B, **i32)
        self.status = torch.zeros(B, **i32)
        self.export_d = torch.zeros((B, n_p, npairs), **f64) if export else None
        self.export_ab = torch.zeros((2, B, n_p, npairs), **f64) if export else None
        p = _lib.ptr
        self._dims = _lib.MaDims(B, n_a, npairs, struct.n_static, n_p, m, struct.A_eq.shape[0],
                                 len(struct.rho_levels))
        self._consts = _lib.MaConsts(p(self.P), p(self.kinv), p(self.level_rho), p(self.pair_i), p(self.pair_j),
                                     p(self.pair_s), p(self.pair_a), p(self.pair_b), p(self.inc_ptr),
                                     p(self.inc_pair), p(self.b_eq), p(self.statics), p(self.line_u),
                                     p(self.line_v), p(self.bnd))
        self._state = _lib.MaState(p(self.state), p(self.xi), p(self.sums), p(self.ring), p(self.res_norm),
                                   p(self.res_max), p(self.hist), p(self.level), p(self.iteration),
                                   p(self.last_change), p(self.n_hist), p(self.status), p(self.export_d),
                                   p(self.export_ab))
        self._graph, self._graph_n = None, 0
        self._ozaki = None
        if qp == "ozaki":
            from . import ozaki

            nv, nk = n_a * m, self.kinv.shape[1]
            sl, ea = ozaki.split_blocks(np.stack([f.kinv for f in struct.factors])[:, :nv, :nk], nv, ozaki_slices)
            mt, ks0, ks1 = ozaki.block_tiles(nv, nk - nv)
            ks = ks0 + ks1
            nt = -(-3 * B // ozaki.BN)
            self.oz_a = torch.as_tensor(sl.reshape(-1), device=dev)
            self.oz_ea = torch.as_tensor(ea.reshape(-1), **i32)
            self.oz_b = torch.zeros(ozaki_slices * nt * ks * ozaki.BN * ozaki.BK, dtype=torch.int8, device=dev)
            self.oz_eb = torch.zeros(2 * nt * ozaki.BN, **i32)
            self._ozaki = _lib.OzakiWs(p(self.oz_a), p(self.oz_ea), p(self.oz_b), p(self.oz_eb), int(ozaki_slices), nt)

    def qp_ozaki(self):
        """The QP step of every non-converged problem on the int8 tensor cores (writes xi, like mode 3)."""
        with torch.cuda.device(self.device):
            rc = self.lib.tro_ma_qp_ozaki(ctypes.byref(self._dims), ctypes.byref(self._consts),
                                          ctypes.byref(self._state), ctypes.byref(self._ozaki),
                                          ctypes.c_void_p(_lib.stream_handle()))
        _lib.check(rc, "tro_ma_qp_ozaki")

    def _call(self, mode: int):
        pr = self.params
        prm = _lib.MaParams(float(pr.tol_norm), float(pr.stall_improvement), int(pr.stall_window),
                            int(pr.max_iter), self.max_hist, 0)
        with torch.cuda.device(self.device):
            rc = self.lib.tro_ma_run(int(mode), ctypes.byref(self._dims), ctypes.byref(self._consts),
                                     ctypes.byref(self._state), ctypes.byref(prm),
                                     ctypes.c_void_p(_lib.stream_handle()))
        _lib.check(rc, "tro_ma_run")

    def lam_ref(self, b: int = 0) -> np.ndarray:
        """Problem b's multipliers in the reference layout (3, n_pairs, n_p) and pair order."""
        return self.state[b].permute(1, 2, 0)[:, self._inv].cpu().numpy()

    def export_ref(self, b: int = 0):
        """Problem b's exported d, alpha, beta as (n_pairs, n_p) arrays in the reference pair order."""
        return tuple(x.T[self._inv].cpu().numpy() for x in (self.export_d[b], self.export_ab[0, b],
                                                              self.export_ab[1, b]))

    def load_state(self, xi, lam, d, alpha, beta, level, iteration):
        """Warm state per problem (host arrays, leading batch axis): xi (B, 3, n_a m), lam (B, 3, n_pairs,
        n_p), d / alpha / beta (B, n_pairs, n_p); then prime() computes the first RHS sums."""
        dev = self.device
        self.xi.copy_(torch.as_tensor(np.asarray(xi, float)).reshape(self.xi.shape))
        pc = self._perm.cpu()  # reference pair order -> device pair order
        self.state.copy_(torch.as_tensor(np.asarray(lam, float))[:, :, pc].permute(0, 3, 1, 2))
        self.export_d.copy_(torch.as_tensor(np.asarray(d, float))[:, pc].permute(0, 2, 1))
        self.export_ab[0].copy_(torch.as_tensor(np.asarray(alpha, float))[:, pc].permute(0, 2, 1))
        self.export_ab[1].copy_(torch.as_tensor(np.asarray(beta, float))[:, pc].permute(0, 2, 1))
        self.level.copy_(torch.as_tensor(np.asarray(level).reshape(self.B).astype(np.int32)))
        self.iteration.copy_(torch.as_tensor(np.asarray(iteration).reshape(self.B).astype(np.int32)))
        del dev

    def prime(self):
        self._call(1)

    def reset(self):
        for t in (self.level, self.iteration, self.last_change, self.n_hist, self.status):
            t.zero_()
        self.ring.zero_()

    def init(self):
        self._call(2)

    def iterate(self):
        if self.qp == "ozaki":  # exact int8 GEMM on tcgen05, then the element pass
            self.qp_ozaki()
            self._call(4)
        elif self.split_qp:  # QP step batched on the fp64 tensor cores (DMMA), then the element pass
            self._call(3)
            self._call(4)
        else:  # one fused launch (per-problem QP in the kernel prologue)
            self._call(0)

    def run(self, n_iter: int, *, use_graph: bool = True, chunk: int = 25, check_every: int = 50) -> int:
        done = 0
        since = 0
        while done < n_iter:
            if check_every and since >= check_every:
                since = 0
                if bool((self.status == 0).sum().item() == 0):
                    break
            n = min(chunk, n_iter - done)
            if use_graph and n == chunk and _graphs_allowed():
                if self._graph is None:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, capture_error_mode="thread_local"):
                        for _ in range(chunk):
                            self.iterate()
                    self._graph = g
                self._graph.replay()
            else:
                for _ in range(n):
                    self.iterate()
            done += n
            since += n
        return done


def pairwise_residuals_arrays(struct: _Structure, state: JointState, problem: MultiAgentProblem | None = None):
    """(3, n_pairs, n_p) separation-equality residuals (solver_multiagent.py:203-208), host diagnostic."""
    P = struct.basis.P
    pos = np.stack([np.stack([state.xi[k].reshape(struct.n_a, struct.m) @ P.T for k in range(3)], -1)])[0]
    deltas = np.empty((struct.n_pairs, struct.n_p, 3))
    for p in range(struct.n_pairs):
        i, j = struct.pair_i[p], struct.pair_j[p]
        deltas[p] = pos[i] - (pos[j] if j >= 0 else
                              np.asarray(problem.static_obstacles[struct.pair_s[p]].center, float)[None, :])
    sb, cb, sa, ca = np.sin(state.beta), np.cos(state.beta), np.sin(state.alpha), np.cos(state.alpha)
    pa, pb = struct.pa[:, None], struct.pb[:, None]
    recon = np.stack([pa * state.d * sb * ca, pa * state.d * sb * sa, pb * state.d * cb], axis=-1)
    return np.transpose(deltas - recon, (2, 0, 1))


def pairwise_residuals(state: JointState, problem: MultiAgentProblem, params: JointParams | None = None,
                       struct=None) -> dict:
    struct = struct or _Structure(problem, params or JointParams())
    res = pairwise_residuals_arrays(struct, state, problem)
    rep = {}
    for k, name in enumerate("xyz"):
        rep[name] = {"norm": float(np.linalg.norm(res[k])), "max_abs": float(np.max(np.abs(res[k]))) if res[k].size
                     else 0.0}
    rep["all"] = {"norm": float(np.linalg.norm(res)), "max_abs": float(np.max(np.abs(res))) if res.size else 0.0}
    return rep


def _statics(problem: MultiAgentProblem) -> np.ndarray:
    return np.array([np.asarray(s.center, float) for s in problem.static_obstacles]).reshape(-1, 3)


def solve_joint_batch(problems: list, params: JointParams | None = None, *, history: bool = False,
                      use_graph: bool = True, device=None, engine: MaEngine | None = None,
                      qp: str = "dmma") -> MaEngine:
    """Solve B independent joint problems in one device pass; returns the engine (device tensors:
    xi, res_norm, res_max, status, iteration, level, hist)."""
    params = params or JointParams()
    struct = _Structure(problems[0], params)
    for p in problems[1:]:
        if p.n_agents != struct.n_a or p.agent_shape != problems[0].agent_shape or len(p.static_obstacles) != \
                struct.n_static or [s.radius for s in p.static_obstacles] != \
                [s.radius for s in problems[0].static_obstacles]:
            raise ValueError("batched problems must share agent count, agent shape and static radii")
    b_eq = np.stack([_b_eq(p) for p in problems])
    statics = np.stack([_statics(p) for p in problems]) if struct.n_static else None
    eng = engine or MaEngine(struct, b_eq, statics, params, device=device,
                             max_hist=params.max_iter if history else 0, qp=qp)
    if struct.n_pairs == 0:
        raise ValueError("the device path needs at least one constraint pair")
    eng.reset()
    eng.init()
    eng.run(params.max_iter, use_graph=use_graph, check_every=50)
    return eng


def solve_joint(problem: MultiAgentProblem, params: JointParams | None = None) -> JointSolution:
    """Joint AM loop over the staged penalty schedule (solver_multiagent.py:300-368), on device."""
    params = params or JointParams()
    struct = _Structure(problem, params)
    if struct.n_pairs == 0:
        raise ValueError("solve_joint without pairs is a plain QP; use qpcore directly")
    eng = MaEngine(struct, _b_eq(problem)[None], _statics(problem)[None] if struct.n_static else None, params,
                   max_hist=max(params.max_iter, 1), export=True)
    eng.init()
    eng.run(params.max_iter, use_graph=params.max_iter > 50)
    nh = int(eng.n_hist[0].item())
    hist = eng.hist[0, :nh].cpu().numpy()
    xi = eng.xi[0].cpu().numpy()
    lam = eng.lam_ref(0)  # (3, n_pairs, n_p)
    d, alpha, beta = eng.export_ref(0)
    state = JointState(xi=xi, d=d, alpha=alpha, beta=beta, lam=lam, level=int(eng.level[0].item()),
                       iteration=int(eng.iteration[0].item()))
    basis = problem.basis
    trajs, positions = [], []
    for i in range(struct.n_a):
        coeffs = xi[:, i * struct.m:(i + 1) * struct.m].T
        positions.append(basis.P @ coeffs)
        trajs.append(Trajectory(t=basis.grid.timestamps, pos=basis.P @ coeffs, vel=basis.Pdot @ coeffs,
                                acc=basis.Pddot @ coeffs))
    min_dist = np.inf
    for i in range(struct.n_a):
        for j in range(i + 1, struct.n_a):
            min_dist = min(min_dist, float(np.linalg.norm(positions[i] - positions[j], axis=1).min()))
    return JointSolution(
        trajectories=trajs,
        converged=bool(eng.status[0].item() & _lib.TRO_CONVERGED),
        iterations=state.iteration,
        residual_norm=float(eng.res_norm[0].item()),
        residual_max=float(eng.res_max[0].item()),
        residual_history=[{"norm": float(h[0]), "max_abs": float(h[1]), "rho": float(h[2])} for h in hist],
        min_pair_distance=min_dist,
        inflated_radius=struct.inflated,
        n_factorizations=struct.n_factorizations,
        state=state,
    )
