"""Joint multi-agent device kernel (tro_ma_run) vs golden vectors of the live reference / the oracle."""

import numpy as np
import pytest
import torch

from oracle import multiagent as OM
from paper_2408_10731_b200 import scenarios
from paper_2408_10731_b200 import solver_multiagent as MA
from paper_2408_10731_b200.basis import AxisBoundary, BasisSet, TimeGrid
from paper_2408_10731_b200.geometry import EllipsoidShape

pytestmark = pytest.mark.gpu


def basis_from(g):
    P = g["P"]
    ts = np.linspace(0.0, 10.0, P.shape[0])
    return BasisSet(grid=TimeGrid(0.0, 10.0, P.shape[0], ts), degree=P.shape[1] - 1, P=P, Pdot=g["Pd"],
                    Pddot=g["Pdd"])


def problem(g, key, statics=None):
    bv = g[f"{key}_bvals"]
    bnds = [tuple(AxisBoundary(*bv[i, k]) for k in range(3)) for i in range(bv.shape[0])]
    st = [] if statics is None else [MA.StaticSphere(center=s[:3], radius=float(s[3])) for s in statics]
    return MA.MultiAgentProblem(basis=basis_from(g), boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45),
                                static_obstacles=st)


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def test_random_roster_solve(golden):
    g = golden("multiagent.npz")
    sol = MA.solve_joint(problem(g, "r6", g["r6_static"]), MA.JointParams(max_iter=60, rho_final=1e3))
    h = np.array([[x["norm"], x["max_abs"], x["rho"]] for x in sol.residual_history])
    ref = g["r6_hist"]
    n = min(len(h), len(ref))
    # this roster is contractive: histories agree over the whole run
    np.testing.assert_allclose(h[:n, :2], ref[:n, :2], rtol=1e-9)
    np.testing.assert_array_equal(h[:n, 2], ref[:n, 2])
    assert sol.converged and sol.iterations == int(g["r6_meta"][0])
    assert rel(sol.state.xi, g["r6_xi"]) < 1e-9
    assert abs(sol.min_pair_distance - g["r6_meta"][4]) < 1e-8


@pytest.mark.parametrize("k", [0, 12])
def test_teacher_forced_step(golden, k):
    g = golden("multiagent.npz")
    prob = problem(g, "r6", g["r6_static"])
    params = MA.JointParams(max_iter=60, rho_final=1e3)
    struct = MA._Structure(prob, params)
    eng = MA.MaEngine(struct, MA._b_eq(prob)[None], MA._statics(prob)[None], params, max_hist=4, export=True)
    lv, it = g[f"r6_k{k}_meta"]
    eng.load_state(g[f"r6_k{k}_xi"][None], g[f"r6_k{k}_lam"][None], g[f"r6_k{k}_d"][None],
                   g[f"r6_k{k}_alpha"][None], g[f"r6_k{k}_beta"][None], [lv], [it])
    eng.prime()
    eng.iterate()
    torch.cuda.synchronize()
    assert rel(eng.xi[0].cpu().numpy(), g[f"r6_k{k + 1}_xi"]) < 1e-10
    d, alpha, beta = eng.export_ref(0)  # the engine's colour-major pair order mapped back
    np.testing.assert_allclose(d, g[f"r6_k{k + 1}_d"], atol=1e-9)
    np.testing.assert_allclose(alpha, g[f"r6_k{k + 1}_alpha"], atol=1e-9)
    np.testing.assert_allclose(beta, g[f"r6_k{k + 1}_beta"], atol=1e-9)
    lam = eng.lam_ref(0)
    ref = g[f"r6_k{k + 1}_lam"]
    assert np.max(np.abs(lam - ref)) <= 1e-8 * max(1.0, np.abs(ref).max())


def test_c3_recipe_window(golden):
    """16 agents, square-antipodal (chaotic): 1e-9 agreement over the first iterations."""
    g = golden("multiagent.npz")
    sol = MA.solve_joint(problem(g, "a16"), MA.JointParams(max_iter=25, rho_final=1e3))
    h = np.array([[x["norm"], x["max_abs"], x["rho"]] for x in sol.residual_history])
    np.testing.assert_allclose(h[:6, :2], g["a16_hist"][:6, :2], rtol=1e-9)
    np.testing.assert_array_equal(h[:12, 2], g["a16_hist"][:12, 2])


def test_batch_equals_single_and_oracle_step():
    basis = MA.BasisSet if False else None  # noqa: F841
    from paper_2408_10731_b200.basis import build_basis

    b = build_basis(0.0, 10.0, 100, 10)
    probs = []
    for s in range(3):
        starts, goals = scenarios.square_antipodal(8, 6.0, 0.4, seed=s)
        bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
                for i in range(8)]
        probs.append(MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45)))
    params = MA.JointParams(max_iter=12, rho_final=1e3)
    eng = MA.solve_joint_batch(probs, params, history=True)
    xi_b = eng.xi.cpu().numpy()
    for s in range(3):
        one = MA.solve_joint(probs[s], params)
        np.testing.assert_array_equal(one.state.xi, xi_b[s])
    # oracle (explicit-inverse contraction, like the device) over the same 12 iterations
    st = OM.make_structure(b.P, b.Pdot, b.Pddot, 8, 0.3, 0.45, rho_final=1e3)
    kinv = [f.kinv for f in MA._Structure(probs[0], params).factors]
    for s in range(3):
        prob = OM.Problem(b_eq=MA._b_eq(probs[s]), statics=np.zeros((0, 3)))
        _, hist, _ = OM.solve(st, prob, b.P, max_iter=12, kinv=kinv)
        np.testing.assert_allclose(eng.hist[s, :4, 0].cpu().numpy(), hist[:4, 0], rtol=1e-9)
