"""Saddle-point QP core (drop-in for ``trajopt.qpcore``).

min 0.5 xi'Q xi + q'xi  s.t.  A xi = b  is solved through
K [xi; nu] = [-q; b] with K = [[Q, A'], [A, 0]]  (qpcore.py:1-14).

B200 design: ``factorize`` runs once per saddle on the host in fp64 — same
guards as the reference (symmetry, row rank of A, cond(K) <= 1e12,
qpcore.py:80-114) — and additionally forms the explicit inverse
K^-1 = LU \\ I.  Every solve is then a batched fp64 contraction
``[xi; nu] = K^-1 [-q; b]`` on the GPU (``tro_kkt_apply_f64``), which is what
the fused solver kernels also do in their prologue.  fp64 is kept on purpose:
these saddles reach cond ~1e12.

``solve``/``solve_batch`` accept numpy arrays (returned as numpy, like the
reference) or CUDA tensors (returned as CUDA tensors, no host round trip).
"""

from __future__ import annotations

from dataclasses import field, make_dataclass

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from . import _lib

_factorization_count = 0

__all__ = [
    "factorization_count",
    "FactorizationError",
    "EqQP",
    "BatchRHS",
    "KKTFactor",
    "factorize",
    "solve",
    "solve_batch",
    "kkt_residuals",
]


def factorization_count() -> int:
    """Saddle factorizations performed in this process (qpcore.py:26-31)."""
    return _factorization_count


def _bump(n: int = 1) -> None:
    global _factorization_count
    _factorization_count += int(n)


class FactorizationError(ValueError):
    """Saddle matrix is rank-deficient or too ill-conditioned to trust."""


def _frozen(name, fields, **ns):
    return make_dataclass(name, fields, frozen=True, namespace={"__module__": __name__, **ns})


# min 0.5 xi'Q xi + q'xi s.t. A xi = b
EqQP = _frozen("EqQP", [(k, np.ndarray) for k in ("Q", "q", "A", "b")])


def _check_rhs(self):
    if self.qs.ndim != 2 or self.bs.ndim != 2:
        raise ValueError("batch right-hand sides must be 2-D arrays")
    if self.qs.shape[0] != self.bs.shape[0]:
        raise ValueError("qs and bs must have the same batch size")
    if self.qs.shape[0] < 1:
        raise ValueError("empty batch")


# stacked right-hand sides: qs (N, n_v), bs (N, n_eq); numpy arrays or CUDA tensors
BatchRHS = _frozen("BatchRHS", [("qs", object), ("bs", object)], __post_init__=_check_rhs,
                   size=property(lambda r: int(r.qs.shape[0])))


def _kinv_on(self, device):
    """fp64 K^-1 resident on `device` (uploaded once per device)."""
    import torch

    cache = self._device
    key = str(device)
    if key not in cache:
        cache[key] = torch.as_tensor(self._kinv, dtype=torch.float64, device=device).contiguous()
    return cache[key]


# one saddle's LU (host) and explicit inverse (host + per-device copies)
KKTFactor = _frozen("KKTFactor", [("n_v", int), ("n_eq", int), ("cond_estimate", float),
                                  ("_lu", tuple, field(repr=False)),
                                  ("_kinv", np.ndarray, field(repr=False, default=None)),
                                  ("_device", dict, field(repr=False, default_factory=dict, compare=False))],
                    size=property(lambda f: f.n_v + f.n_eq), kinv=property(lambda f: f._kinv), kinv_on=_kinv_on)


def saddle_matrix(Q: np.ndarray, A: np.ndarray) -> np.ndarray:
    n_v, n_eq = Q.shape[0], A.shape[0]
    K = np.zeros((n_v + n_eq, n_v + n_eq))
    K[:n_v, :n_v] = Q
    if n_eq:
        K[:n_v, n_v:] = A.T
        K[n_v:, :n_v] = A
    return K


def _build(Q, A, cond_limit: float) -> KKTFactor:
    """factorize without touching the process-wide counter (engines count the levels they use)."""
    Q = np.asarray(Q, dtype=float)
    A = np.atleast_2d(np.asarray(A, dtype=float))
    n_v, n_eq = Q.shape[0], A.shape[0]
    if Q.shape != (n_v, n_v):
        raise ValueError(f"Q must be square, got {Q.shape}")
    if not np.allclose(Q, Q.T, rtol=1e-10, atol=1e-12):
        raise ValueError("Q must be symmetric")
    if A.shape[1] != n_v:
        raise ValueError(f"A has {A.shape[1]} columns, expected {n_v}")
    if n_eq and np.linalg.matrix_rank(A) < n_eq:  # qpcore.py:98-100
        raise FactorizationError(f"equality matrix A is rank-deficient (rank < {n_eq})")
    K = saddle_matrix(Q, A)
    cond = float(np.linalg.cond(K))  # qpcore.py:108-110
    if not (np.isfinite(cond) and cond <= cond_limit):
        raise FactorizationError(f"saddle matrix is near-singular (cond estimate {cond:.3e})")
    lu = lu_factor(K)
    return KKTFactor(n_v=n_v, n_eq=n_eq, cond_estimate=cond, _lu=lu, _kinv=lu_solve(lu, np.eye(K.shape[0])))


def factorize(Q: np.ndarray, A: np.ndarray, *, cond_limit: float = 1e12) -> KKTFactor:
    """Factorize the saddle once for repeated solves (qpcore.py:80-114)."""
    f = _build(Q, A, cond_limit)
    _bump(1)
    return f


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _apply(factor: KKTFactor, block):
    """rows of `block` (N, n) -> rows of K^-1 applied (N, n), on the GPU."""
    import torch

    _lib.require_cuda()
    lib = _lib.load()
    on_host = not _is_torch(block)
    if on_host:
        dev = torch.device("cuda", torch.cuda.current_device())
        rhs = torch.as_tensor(np.ascontiguousarray(block, dtype=np.float64)).to(dev, non_blocking=False)
    else:
        rhs = block.to(torch.float64).contiguous()
        dev = rhs.device
    out = torch.empty_like(rhs)
    kinv = factor.kinv_on(dev)
    with torch.cuda.device(dev):
        rc = lib.tro_kkt_apply_f64(kinv.data_ptr(), factor.size, rhs.data_ptr(), rhs.shape[0], out.data_ptr(),
                                   _lib.stream_handle())
    _lib.check(rc, "tro_kkt_apply_f64")
    return out.cpu().numpy() if on_host else out


def solve(factor: KKTFactor, q, b):
    """One instance -> (xi, nu) (qpcore.py:117-127)."""
    if _is_torch(q):
        import torch

        qv, bv = q.to(torch.float64), b.to(torch.float64)
        if tuple(qv.shape) != (factor.n_v,) or tuple(bv.shape) != (factor.n_eq,):
            raise ValueError("q/b shapes do not match the factor")
        sol = _apply(factor, torch.cat([-qv, bv])[None, :])[0]
        return sol[: factor.n_v], sol[factor.n_v :]
    q = np.asarray(q, dtype=float)
    b = np.asarray(b, dtype=float)
    if q.shape != (factor.n_v,):
        raise ValueError(f"q has shape {q.shape}, expected ({factor.n_v},)")
    if b.shape != (factor.n_eq,):
        raise ValueError(f"b has shape {b.shape}, expected ({factor.n_eq},)")
    sol = _apply(factor, np.concatenate([-q, b])[None, :])[0]
    return sol[: factor.n_v], sol[factor.n_v :]


def solve_batch(factor: KKTFactor, rhs: BatchRHS):
    """All instances in one contraction -> (xis (N, n_v), nus (N, n_eq)) (qpcore.py:130-143)."""
    if rhs.qs.shape[1] != factor.n_v:
        raise ValueError(f"qs have length {rhs.qs.shape[1]}, expected {factor.n_v}")
    if rhs.bs.shape[1] != factor.n_eq:
        raise ValueError(f"bs have length {rhs.bs.shape[1]}, expected {factor.n_eq}")
    if _is_torch(rhs.qs):
        import torch

        block = torch.cat([-rhs.qs.to(torch.float64), rhs.bs.to(torch.float64)], dim=1)
    else:
        block = np.hstack([-np.asarray(rhs.qs, dtype=float), np.asarray(rhs.bs, dtype=float)])
    sol = _apply(factor, block)
    return sol[:, : factor.n_v], sol[:, factor.n_v :]


def kkt_residuals(Q, A, q, b, xi, nu) -> tuple[float, float]:
    """Stationarity / feasibility residual norms (test helper, qpcore.py:146-150)."""
    return float(np.linalg.norm(Q @ xi + A.T @ nu + q)), float(np.linalg.norm(A @ xi - b))
