"""Device engine for batched Alg. 1 (single-robot AM/AL, arXiv 2408.10731).

Owns the device-resident SoA state of B independent members that share one
basis and one obstacle set, the per-rho_o-level K^-1 table, and the launch
sequence (one fused kernel launch per AM iteration, optionally replayed from a
CUDA graph).  Host <-> device traffic happens only at solve boundaries.

HBM layout: one storage-dtype tensor state[i][j][w][t] (member, obstacle, word, sample),
W = 9 words in 3-D [alpha beta lx ly lz lca lsa lcb lsb], 5 in 2-D [alpha lx ly lca lsa],
so one sample's words sit n_p elements apart (one base register + immediate offsets in the
kernel) and the n_p samples of a word are contiguous (coalesced).  Obstacle tracks are
tracks[j][axis][t] (fp64).  Per member (fp64): xi (dim, m), pos (dim, n_p), sums
(2, dim, n_p), rho, rho_o, stall ring, status / level / iteration counters.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch


def _graphs_allowed() -> bool:
    """CUDA-graph capture only on the main thread: a capture is invalidated by launches other threads make on
    the legacy default stream at the same time, so solver instances running in other threads launch their
    iterations directly (same kernels, same results)."""
    import threading

    return threading.current_thread() is threading.main_thread()

from . import _lib, qpcore
from .basis import BasisSet, boundary_matrix, line_basis_vectors


LOOP_MAX_MEMBERS = 64  # batches up to this size run all iterations in one launch (tro_alg1_iterate_n)


def rho_chain(r0: float, growth: float, cap: float) -> list[float]:
    """Distinct penalty values reached from r0 by repeated min(r * growth, cap) (solver_single.py:401-402)."""
    vals = [float(r0)]
    while True:
        nxt = min(vals[-1] * growth, cap)
        if nxt == vals[-1] or len(vals) > 10000:
            return vals
        vals.append(nxt)


def linear_track_record(tracks: np.ndarray, timestamps: np.ndarray) -> np.ndarray | None:
    """Constant-velocity description of obstacle tracks (n_o, n_p, dim), or None.

    Returns [c_j (dim), v_j (dim) padded to 6 doubles per obstacle ..., rel (n_p)] with rel = t - t[0] when
    every sample equals numpy's c + v * rel BITWISE (bench/scenarios.py:118-127, scenarios.tracks_on_grid):
    the velocity is recovered from the end points and its neighbouring doubles are tried until one
    reproduces every sample exactly.  The iteration kernel then generates the tracks in registers
    (tro_alg1_consts.track_lin) instead of streaming them; anything else keeps the streamed tracks."""
    n_o, n_p, dim = tracks.shape
    if n_o == 0 or n_p < 2:
        return None
    rel = np.asarray(timestamps, dtype=float) - float(timestamps[0])
    if rel[0] != 0.0 or rel[-1] == 0.0:
        return None
    c = tracks[:, 0, :]
    # least-squares slope over every sample (the end-point quotient alone can be hundreds of ulps off
    # when |v rel| << |c|); the search below then finds an exactly reproducing double nearby
    v0 = np.einsum("t,jtk->jk", rel, tracks - c[:, None, :]) / float(rel @ rel)
    best = np.full(v0.shape, np.nan)
    steps = [v0]  # v0, then up to 64 doubles either side (the end-point quotient loses ~|c| / |v rel| ulps)
    up, dn = v0, v0
    for _ in range(64):
        up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
        steps += [up, dn]
    for v in steps:
        ok = np.all(c[:, None, :] + v[:, None, :] * rel[None, :, None] == tracks, axis=1)
        best = np.where(np.isnan(best) & ok, v, best)
        if not np.isnan(best).any():
            break
    if np.isnan(best).any():
        return None
    rec = np.zeros((n_o, 6))
    rec[:, :dim] = c
    rec[:, dim:2 * dim] = best
    return np.concatenate([rec.reshape(-1), rel])


_TABLE_CACHE: dict = {}


def level_table(basis: BasisSet, n_o: int, w_smooth: float, w_track: float, starts, growth: float, cap: float,
                cond_limit: float = 1e12) -> "LevelTable":
    """LevelTable cached by content (22 saddle factorizations + inverses cost milliseconds on the host)."""
    key = (basis.P.tobytes(), basis.Pddot.tobytes(), int(n_o), float(w_smooth), float(w_track),
           tuple(sorted(set(float(r) for r in starts))), float(growth), float(cap), float(cond_limit))
    t = _TABLE_CACHE.get(key)
    if t is None:
        if len(_TABLE_CACHE) > 64:
            _TABLE_CACHE.clear()
        t = _TABLE_CACHE[key] = LevelTable(basis, n_o, w_smooth, w_track, starts, growth, cap, cond_limit)
    return t


class LevelTable:
    """K^-1 per rho_o level for the position-step saddle (solver_single.py:198-202)."""

    def __init__(self, basis: BasisSet, n_o: int, w_smooth: float, w_track: float, starts, growth: float,
                 cap: float, cond_limit: float = 1e12):
        P, Pdd = basis.P, basis.Pddot
        Q = 2.0 * (w_smooth * Pdd.T @ Pdd + w_track * P.T @ P)  # solver_single.py:172
        PtP = P.T @ P
        A = boundary_matrix(basis)
        self.m = basis.n_var
        self.n_eq = A.shape[0]
        nk = self.m + self.n_eq
        self.rhos: list[float] = []
        self.factors: list[qpcore.KKTFactor | None] = []
        self.offsets: dict[float, int] = {}
        for r0 in sorted(set(float(r) for r in starts)):
            self.offsets[r0] = len(self.rhos)
            for r in rho_chain(r0, growth, cap):
                D = Q + r * n_o * PtP if n_o else Q  # solver_single.py:199
                try:
                    f = qpcore._build(D, A, cond_limit)
                except qpcore.FactorizationError as exc:
                    if "rank-deficient" in str(exc):
                        raise
                    f = None
                self.rhos.append(r)
                self.factors.append(f)
        self.kinv = np.zeros((len(self.rhos), nk, nk))
        for k, f in enumerate(self.factors):
            if f is not None:
                self.kinv[k] = f.kinv
        self.ok = np.array([f is not None for f in self.factors], dtype=np.int32)

    def level_of(self, r0: float) -> int:
        return self.offsets[float(r0)]

    def error_for(self, level: int) -> qpcore.FactorizationError:
        return qpcore.FactorizationError(
            f"saddle matrix is near-singular at rho_o={self.rhos[level]!r} (cond guard 1e12)")


class Alg1Engine:
    """B members on one device.  All per-member inputs may be numpy or torch."""

    def __init__(self, basis: BasisSet, tracks, shape_a, shape_b, bvals, q=None, *, params, desired=None, rho0=None,
                 w_smooth: float = 1.0, w_track: float = 1.0, dtype=torch.float64, device=None, groups: int = 0,
                 max_hist: int = 0, export: bool = False, keep_d: bool = False, cond_limit: float = 1e12,
                 use_tma: bool = True, layout: str = "angle", tail_split: bool = True):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        self.dtype = dtype
        self.code = _lib.TRO_F64 if dtype == torch.float64 else _lib.TRO_F32
        if dtype not in (torch.float64, torch.float32):
            raise ValueError("storage dtype must be float64 or float32")
        self.params = params
        tracks = np.asarray(tracks, dtype=float)
        n_o, n_p, dim = tracks.shape if tracks.size else (int(tracks.shape[0]), basis.n_p, int(bvals.shape[1]))
        self.n_o, self.n_p, self.dim, self.m = int(n_o), int(n_p), int(dim), basis.n_var
        self.B = int(bvals.shape[0])
        if self.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        B, n_o, n_p, dim, m = self.B, self.n_o, self.n_p, self.dim, self.m

        # ---- constants
        rho0 = np.full(B, params.rho_start) if rho0 is None else np.broadcast_to(np.asarray(rho0, float), (B,))
        self.table = level_table(basis, n_o, w_smooth, w_track, np.unique(rho0), params.rho_growth, params.rho_cap,
                                 cond_limit)
        self.basis = basis
        self.P = torch.as_tensor(np.array(basis.P, dtype=float, copy=True), **f64)
        self.tracks = torch.as_tensor(np.ascontiguousarray(np.transpose(tracks, (0, 2, 1))) if n_o else
                                      np.zeros((0, dim, n_p)), **f64).contiguous()
        self.shape_a = torch.as_tensor(np.asarray(shape_a, dtype=float).reshape(-1), **f64)
        self.shape_b = torch.as_tensor(np.asarray(shape_b, dtype=float).reshape(-1), **f64)
        if n_o == 0:
            self.shape_a = torch.ones(1, **f64)
            self.shape_b = torch.ones(1, **f64)
        lin = linear_track_record(tracks, basis.grid.timestamps) if n_o and tracks.shape[1] == n_p else None
        self.track_lin = torch.as_tensor(lin, **f64) if lin is not None else None
        self.kinv = torch.as_tensor(self.table.kinv, **f64).contiguous()
        self.level_rho = torch.as_tensor(np.asarray(self.table.rhos), **f64)
        self.level_ok = torch.as_tensor(self.table.ok, **i32)
        self.bvals = torch.as_tensor(bvals, **f64).reshape(B, dim, -1).contiguous()
        self.n_eq = int(self.bvals.shape[2])
        self.w_track = float(w_track)
        self.frac = torch.as_tensor(np.linspace(0.0, 1.0, n_p), **f64)
        self.q = torch.empty((B, dim, m), **f64)
        if q is not None:
            self.q.copy_(torch.as_tensor(q, **f64).reshape(B, dim, m))
        else:
            self.compute_linear_terms(desired)
        u, v = line_basis_vectors(basis)
        self.line_u = torch.as_tensor(u, **f64)
        self.line_v = torch.as_tensor(v, **f64)

        # ---- state
        T = dict(dtype=dtype, device=dev)
        if layout not in ("angle", "unit", "half"):
            raise ValueError("layout must be 'angle', 'unit' or 'half'")
        self.layout = layout
        n_ang = 2 if dim == 3 else 1
        self.NV = n_ang * (2 if layout == "unit" else 1)
        W = self.NV + (7 if dim == 3 else 4)
        self.W = W
        self.state = torch.empty((B, n_o, W, n_p), **T)
        # multiplier planes as a (plane, member, obstacle, sample) view
        self.lam = self.state[:, :, self.NV:].permute(2, 0, 1, 3)
        self.d = torch.empty((B, n_o, n_p), **T) if (keep_d or export) else None
        self.copies = torch.empty((4 if dim == 3 else 2, B, n_o, n_p), **T) if export else None
        self.xi = torch.zeros((B, dim, m), **f64)
        self.pos = torch.zeros((B, dim, n_p), **f64)
        self.sums = torch.zeros((B, 2, dim, n_p), **f64)
        self.rho0_dev = torch.as_tensor(rho0.copy(), **f64)
        self.rho = torch.as_tensor(rho0.copy(), **f64)
        self.rho_o = torch.as_tensor(rho0.copy(), **f64)
        self.ring = torch.zeros((B, 2 * params.stall_window), **f64)
        self.res_norm = torch.zeros(B, **f64)
        self.res_max = torch.zeros(B, **f64)
        self.max_hist = int(max_hist)
        self.hist = torch.zeros((B, max(self.max_hist, 1), 3), **f64) if self.max_hist else None
        levels0 = np.array([self.table.level_of(r) for r in rho0], dtype=np.int32)
        self.level0 = torch.as_tensor(levels0, **i32)
        self.level = self.level0.clone()
        self.iteration = torch.zeros(B, **i32)
        self.last_change = torch.zeros(B, **i32)
        self.n_hist = torch.zeros(B, **i32)
        self.status = torch.zeros(B, **i32)
        self.n_changes = torch.zeros(B, **i32)
        self.level_used = torch.zeros(B, **i32)
        # tail balancing of the persistent kernel: per grid slot two halves' partial sums + a ticket
        slots = 2 * torch.cuda.get_device_properties(dev).multi_processor_count
        self.split_scratch = torch.zeros((slots, 2, 2 * dim * n_p + 2), **f64) if tail_split else None
        self.split_ticket = torch.zeros(slots, **i32) if tail_split else None

        self._dims = _lib.Alg1Dims(B, n_o, n_p, m, dim, self.n_eq, len(self.table.rhos), int(groups),
                                   {"unit": _lib.TRO_LAYOUT_UNIT, "half": _lib.TRO_LAYOUT_HALF}.get(
                                       layout, _lib.TRO_LAYOUT_ANGLE), 0)
        self._consts = _lib.Alg1Consts(
            self.P.data_ptr(), self.tracks.data_ptr(), self.shape_a.data_ptr(), self.shape_b.data_ptr(),
            self.kinv.data_ptr(), self.level_rho.data_ptr(), self.level_ok.data_ptr(), self.q.data_ptr(),
            self.bvals.data_ptr(), self.line_u.data_ptr(), self.line_v.data_ptr(), self.level0.data_ptr(),
            _lib.ptr(self.track_lin))
        p = _lib.ptr
        self._state = _lib.Alg1State(
            p(self.state), p(self.d), p(self.copies), p(self.xi), p(self.pos),
            p(self.sums), p(self.rho), p(self.rho_o), p(self.ring), p(self.res_norm), p(self.res_max), p(self.hist),
            p(self.level), p(self.iteration), p(self.last_change), p(self.n_hist), p(self.status),
            p(self.n_changes), p(self.split_scratch), p(self.split_ticket), None, None, p(self.level_used))
        # the persistent kernel's work list (batches above the in-kernel-loop size): run() compacts it to the
        # members still iterating before every chunk, so converged members cost nothing and the rest stay
        # balanced over the CTAs; outside run() it is the identity
        self.order = self.n_order = None
        if B > LOOP_MAX_MEMBERS:
            self._identity = torch.arange(B, **i32)
            self.order = self._identity.clone()
            self.n_order = torch.full((1,), B, **i32)
            self._state.order = self.order.data_ptr()
            self._state.n_order = self.n_order.data_ptr()
        self._graph = None
        self._graph_n = 0
        # TMA-pipelined persistent kernel for the iteration unless disabled (flags bit 2)
        self.base_flags = 0 if use_tma else _lib.TRO_FLAG_NO_TMA

    def compute_linear_terms(self, desired=None):
        """q = -2 w_track (P' desired_i)' on the device (tro_alg1_linear_terms, solver_single.py:173);
        desired None: each member's straight start -> goal line from the current bvals."""
        des = None
        if desired is not None:
            des = torch.as_tensor(desired, dtype=torch.float64, device=self.device).reshape(
                self.B, self.n_p, self.dim).contiguous()
        with torch.cuda.device(self.device):
            rc = self.lib.tro_alg1_linear_terms(self.B, self.n_p, self.m, self.dim, self.n_eq, self.P.data_ptr(),
                                                self.frac.data_ptr(), self.bvals.data_ptr(), _lib.ptr(des),
                                                self.w_track, self.q.data_ptr(), _lib.stream_handle())
        _lib.check(rc, "tro_alg1_linear_terms")

    def set_members(self, bvals, desired=None):
        """New members' boundary values (and desired paths; None = straight lines) for the next cold solve on
        this engine (same obstacles, basis and batch size)."""
        bv = torch.as_tensor(bvals, dtype=torch.float64)
        if tuple(bv.shape) != tuple(self.bvals.shape):
            raise ValueError(f"boundary values must be {tuple(self.bvals.shape)}, got {tuple(bv.shape)}")
        self.bvals.copy_(bv, non_blocking=bv.is_pinned())
        self.compute_linear_terms(desired)

    # ------------------------------------------------------------ angle views
    @staticmethod
    def _half_angle(w: torch.Tensor) -> torch.Tensor:
        """Angle of a folded half-angle tangent (half_decode in alg1_elem.cuh), in (-pi, pi]."""
        w = w.double()
        inner = w.abs() <= 1
        sg = torch.where(torch.signbit(w), -1.0, 1.0).to(w)
        t = torch.where(inner, w, w - 3.0 * sg)
        ang = 2.0 * torch.atan(t)
        return torch.where(inner, ang, ang + math.pi * sg)

    @staticmethod
    def _half_of(a: torch.Tensor) -> torch.Tensor:
        c, s = torch.cos(a), torch.sin(a)
        pos = c >= 0
        sg = torch.where(torch.signbit(s), -1.0, 1.0).to(a)
        t = s / torch.where(pos, 1.0 + c, 1.0 - c)
        return torch.where(pos, t, 3.0 * sg - t)

    @property
    def alpha(self) -> torch.Tensor:
        """(B, n_o, n_p) alpha (a view in the angle layout, decoded from the stored words otherwise)."""
        if self.layout == "angle":
            return self.state[:, :, 0]
        if self.layout == "half":
            return self._half_angle(self.state[:, :, 0])
        return torch.atan2(self.state[:, :, 1], self.state[:, :, 0])

    @property
    def beta(self) -> torch.Tensor | None:
        if self.dim != 3:
            return None
        if self.layout == "angle":
            return self.state[:, :, 1]
        if self.layout == "half":
            return self._half_angle(self.state[:, :, 1])
        return torch.atan2(self.state[:, :, 3], self.state[:, :, 2])

    def _set_angles(self, alpha, beta):
        T = self.dtype
        a = torch.as_tensor(np.asarray(alpha), dtype=torch.float64, device=self.device)
        if self.layout == "angle":
            self.state[:, :, 0].copy_(a.to(T))
            if self.dim == 3:
                self.state[:, :, 1].copy_(torch.as_tensor(np.asarray(beta), device=self.device).to(T))
            return
        if self.layout == "half":
            self.state[:, :, 0].copy_(self._half_of(a).to(T))
            if self.dim == 3:
                b = torch.as_tensor(np.asarray(beta), dtype=torch.float64, device=self.device)
                self.state[:, :, 1].copy_(self._half_of(b).to(T))
            return
        self.state[:, :, 0].copy_(torch.cos(a).to(T))
        self.state[:, :, 1].copy_(torch.sin(a).to(T))
        if self.dim == 3:
            b = torch.as_tensor(np.asarray(beta), dtype=torch.float64, device=self.device)
            self.state[:, :, 2].copy_(torch.cos(b).to(T))
            self.state[:, :, 3].copy_(torch.sin(b).to(T))

    # ------------------------------------------------------------ launches
    def _params(self, d_mode: int, flags: int = 0) -> _lib.Alg1Params:
        pr = self.params
        return _lib.Alg1Params(float(pr.tol), float(pr.rho_growth), float(pr.rho_cap), float(pr.stall_improvement),
                               int(pr.stall_window), int(d_mode), self.max_hist, int(flags))

    def _call(self, name: str, d_mode: int, flags: int = 0):
        fn = getattr(self.lib, name)
        prm = self._params(d_mode, flags | self.base_flags)
        with torch.cuda.device(self.device):
            rc = fn(self.code, ctypes.byref(self._dims), ctypes.byref(self._consts), ctypes.byref(self._state),
                    ctypes.byref(prm), ctypes.c_void_p(_lib.stream_handle()))
        _lib.check(rc, name)

    def cold_init(self):
        """init_state (solver_single.py:115-166) for every member, on device; d == 1.  A complete cold start:
        the launch also resets rho, rho_o, level, iteration and the solve-local schedule to rho_start
        (unless the engine's consts.level0 is NULL, as in the MPC fleet)."""
        self._call("tro_alg1_init", 0)
        self.first_d_mode = 0

    def prime(self, d_mode: int):
        self._call("tro_alg1_prime", d_mode)
        self.first_d_mode = d_mode

    def iterate(self, d_mode: int = 2, flags: int = 0):
        self._call("tro_alg1_iterate", d_mode, flags)

    def iterate_n(self, n: int, d_mode: int = 2):
        """n AM iterations in ONE launch (each CTA loops its member until converged / n)."""
        prm = self._params(d_mode, self.base_flags)
        with torch.cuda.device(self.device):
            rc = self.lib.tro_alg1_iterate_n(self.code, ctypes.byref(self._dims), ctypes.byref(self._consts),
                                             ctypes.byref(self._state), ctypes.byref(prm), int(n),
                                             ctypes.c_void_p(_lib.stream_handle()))
        _lib.check(rc, "tro_alg1_iterate_n")

    def reset_cold(self):
        """Reuse this engine for a new cold-start solve of the same problem (penalties back to rho0)."""
        self.rho.copy_(self.rho0_dev)
        self.rho_o.copy_(self.rho0_dev)
        self.level.copy_(self.level0)
        self.iteration.zero_()
        self.reset_schedule()

    def reset_schedule(self):
        """Solve-local bookkeeping of solve_single (history, last_change) restarts per call."""
        self.last_change.zero_()
        self.n_hist.zero_()
        self.n_changes.zero_()
        self.ring.zero_()
        self.status.zero_()

    def compact_active(self):
        """Work list = the members whose status is 0 (not converged / failed), on the device."""
        if not self._state.order:
            return
        with torch.cuda.device(self.device):
            rc = self.lib.tro_mpc_compact(self.B, self.status.data_ptr(), self._state.order, self._state.n_order,
                                          _lib.stream_handle())
        _lib.check(rc, "tro_mpc_compact")

    def _restore_order(self):
        if self.order is not None and self._state.order == self.order.data_ptr():
            self.order.copy_(self._identity)
            self.n_order.fill_(self.B)

    def _capture(self, n: int):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            # warm-up launch outside capture is not needed: launches are plain kernels
            pass
        torch.cuda.current_stream(self.device).wait_stream(s)
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            self.compact_active()
            for _ in range(n):
                self.iterate(2)
        self._graph, self._graph_n = g, n

    def launches_per_run(self, n_iter: int, chunk: int = 25, loop: bool | None = None) -> int:
        """Kernel launches of run(n_iter) without early exit (iterations + work-list compactions)."""
        if n_iter <= 0:
            return 0
        if (self.B <= LOOP_MAX_MEMBERS) if loop is None else loop:
            return 1 + (1 if n_iter > 1 else 0)
        rest = n_iter - 1
        compactions = -(-rest // chunk) if self._state.order else 0
        return n_iter + compactions

    def run(self, n_iter: int, *, use_graph: bool = True, chunk: int = 25, check_every: int = 0,
            loop: bool | None = None) -> int:
        """n_iter AM iterations (the first with the primed d_mode).  Returns iterations launched.

        check_every > 0 stops early (host sync every `check_every` iterations) once every
        member is frozen (converged or failed)."""
        done = 0
        if n_iter <= 0:
            return 0
        if loop is None:
            loop = self.B <= LOOP_MAX_MEMBERS
        if loop:  # small batches: one launch for all iterations (members stop at convergence on device)
            self.iterate(self.first_d_mode)
            if n_iter > 1:
                self.iterate_n(n_iter - 1)
            return n_iter
        self.iterate(self.first_d_mode)
        done = 1
        since_check = 1
        while done < n_iter:
            if check_every and since_check >= check_every:
                since_check = 0
                if bool((self.status == 0).sum().item() == 0):
                    break
            n = min(chunk, n_iter - done)
            if check_every:
                n = min(n, check_every - since_check)
            if use_graph and n == chunk and _graphs_allowed():
                if self._graph is None or self._graph_n != chunk:
                    self._capture(chunk)
                self._graph.replay()  # compacts the work list, then n iterations
            else:
                self.compact_active()
                for _ in range(n):
                    self.iterate(2)
            done += n
            since_check += n
        self._restore_order()
        return done

    # ------------------------------------------------------------ host transfer
    def load_state(self, *, xi, alpha, beta, lam_planes, d, rho, rho_o, iteration):
        """Upload a warm state (numpy, member-major)."""
        dev, T = self.device, self.dtype
        self.xi.copy_(torch.as_tensor(np.asarray(xi, float).reshape(self.B, self.dim, self.m)))
        if self.n_o:
            self._set_angles(alpha, beta)
            self.lam.copy_(torch.as_tensor(np.asarray(lam_planes)).to(T))
            if d is not None:
                if self.d is None:
                    self.d = torch.empty((self.B, self.n_o, self.n_p), dtype=T, device=dev)
                    self._state.d = self.d.data_ptr()
                self.d.copy_(torch.as_tensor(np.asarray(d)).to(T))
        self.rho.copy_(torch.as_tensor(np.asarray(rho, float).reshape(self.B)))
        self.rho_o.copy_(torch.as_tensor(np.asarray(rho_o, float).reshape(self.B)))
        self.iteration.copy_(torch.as_tensor(np.asarray(iteration).reshape(self.B).astype(np.int32)))
        lv = np.array([self._level_for(r) for r in np.asarray(rho_o, float).reshape(self.B)], dtype=np.int32)
        self.level.copy_(torch.as_tensor(lv))

    def load_schedule(self, max_hist_lists, last_change):
        """Restore solve-local stall bookkeeping (history of max_abs, last_change) per member."""
        w2 = 2 * self.params.stall_window
        ring = np.zeros((self.B, w2))
        n = np.zeros(self.B, dtype=np.int32)
        for i, h in enumerate(max_hist_lists):
            h = list(h)
            n[i] = len(h)
            for k in range(max(0, len(h) - w2), len(h)):
                ring[i, k % w2] = h[k]
        self.ring.copy_(torch.as_tensor(ring))
        self.n_hist.copy_(torch.as_tensor(n))
        self.last_change.copy_(torch.as_tensor(np.asarray(last_change).reshape(self.B).astype(np.int32)))

    def _level_for(self, r: float) -> int:
        for k, v in enumerate(self.table.rhos):
            if v == float(r):
                return k
        raise ValueError(f"rho_o={r!r} is not in this engine's level table")
