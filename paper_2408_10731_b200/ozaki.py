"""Host side of the Ozaki int8 tensor-core QP backend (csrc/ozaki.cu, tro_ma_qp_ozaki).

The level inverses' rows are split ONCE per engine into 7-bit int8 slices with one power-of-two exponent per
row, exactly in fp64 (SURVEY.md §2 K1 "Ozaki int8 slices on kind::i8"):

    A[r][k] = 2^ea(r) * sum_i a_i[r][k] * 128^-(i+1),   |a_i| <= 127,

and laid out as the canonical no-swizzle K-major core-matrix blocks the tcgen05 MMA reads (one 128 x 32 block
of 4096 bytes per (level, slice, m-tile, k-step)); the kernel's tensor maps bring each block in with one TMA.
"""

from __future__ import annotations

import numpy as np

BM, BN, BK = 128, 32, 32


def tiles(nv: int, nk: int) -> tuple[int, int]:
    """(m_tiles, k_steps) of an nv x nk operand in one K block."""
    return -(-nv // BM), -(-nk // BK)


def block_tiles(nv: int, n_eq: int) -> tuple[int, int, int]:
    """(m_tiles, k_steps of the primal block [0, nv), k_steps of the boundary block [nv, nv + n_eq)).

    The saddle inverse's columns against the penalised sums (rho B - C, ~rho large) and against the boundary
    values (O(1)) differ by orders of magnitude; one exponent per row over both would cost the small block
    its precision, so each K block gets its own row / column exponents and its own accumulators."""
    return -(-nv // BM), -(-nv // BK), -(-n_eq // BK)


def split_blocks(A: np.ndarray, nv: int, n_slices: int) -> tuple[np.ndarray, np.ndarray]:
    """A (L, nv, nk) -> (slices int8 (L, S, m_tiles, ks0 + ks1, 4096), exponents int32 (L, 2, m_tiles * 128)):
    split_rows of the primal columns [0, nv) and of the boundary columns [nv, nk), k-steps concatenated."""
    s0, e0 = split_rows(A[:, :, :nv], n_slices)
    s1, e1 = split_rows(A[:, :, nv:], n_slices)
    return np.ascontiguousarray(np.concatenate([s0, s1], axis=3)), np.ascontiguousarray(np.stack([e0, e1], axis=1))


def split_rows(A: np.ndarray, n_slices: int) -> tuple[np.ndarray, np.ndarray]:
    """A (L, nv, nk) fp64 -> (slices int8 (L, S, m_tiles, k_steps, 4096), exponents int32 (L, m_tiles * 128)).

    Row r of level L: ea = the exponent with max_k |A[r][k]| < 2^ea (0 for a zero row); x = A 2^-ea in (-1, 1);
    slice i = trunc(128 x), x <- 128 x - slice (both exact)."""
    A = np.asarray(A, dtype=np.float64)
    L, nv, nk = A.shape
    mt, ks = tiles(nv, nk)
    pad = np.zeros((L, mt * BM, ks * BK))
    pad[:, :nv, :nk] = A
    mx = np.max(np.abs(pad), axis=2)
    _, ea = np.frexp(mx)
    ea = np.where(mx > 0, ea, 0).astype(np.int32)
    x = np.ldexp(pad, -ea[:, :, None])
    sl = np.empty((L, n_slices, mt * BM, ks * BK), dtype=np.int8)
    for i in range(n_slices):
        y = x * 128.0
        t = np.trunc(y)
        sl[:, i] = t.astype(np.int8)
        x = y - t
    # (L, S, [mt, rg 16, r8 8], [ks, kc 2, kb 16]) -> (L, S, mt, ks, rg, kc, r8, kb)
    sl = sl.reshape(L, n_slices, mt, 16, 8, ks, 2, 16).transpose(0, 1, 2, 5, 3, 6, 4, 7)
    return np.ascontiguousarray(sl).reshape(L, n_slices, mt, ks, BM * BK), ea


def reconstruct(slices: np.ndarray, ea: np.ndarray, nv: int, nk: int) -> np.ndarray:
    """Inverse of split_rows (test helper): the fp64 rows the slices represent."""
    L, S, mt, ks, _ = slices.shape
    t = slices.reshape(L, S, mt, ks, 16, 2, 8, 16).transpose(0, 1, 2, 4, 6, 3, 5, 7).reshape(L, S, mt * BM, ks * BK)
    acc = np.zeros((L, mt * BM, ks * BK))
    for i in range(S - 1, -1, -1):
        acc = (acc + t[:, i].astype(np.float64)) / 128.0
    return np.ldexp(acc, ea[:, :, None])[:, :nv, :nk]
