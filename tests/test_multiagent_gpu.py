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


@pytest.mark.parametrize("n_agents,n_static", [(5, 1), (7, 0)])
def test_odd_roster_colour_order_matches_oracle(n_agents, n_static):
    """Odd agent counts: the round-robin colouring leaves every agent one bye, so the incidence steps are not
    aligned across lanes (conflicting, still correct) -- the device run must match the oracle step for step,
    and the multipliers must come back in the reference pair order."""
    from paper_2408_10731_b200.basis import build_basis

    b = build_basis(0.0, 10.0, 100, 10)
    starts, goals = scenarios.square_antipodal(n_agents, 6.0, 0.4, seed=3)
    bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
            for i in range(n_agents)]
    statics = [MA.StaticSphere(center=np.array([0.3, -0.2, 1.0]), radius=0.5)][:n_static]
    prob = MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45),
                                static_obstacles=statics)
    params = MA.JointParams(max_iter=8, rho_final=1e3)
    struct = MA._Structure(prob, params)
    assert sorted(struct.dev_perm.tolist()) == list(range(struct.n_pairs))
    assert not np.array_equal(struct.dev_perm, np.arange(struct.n_pairs))  # the order really is permuted
    sol = MA.solve_joint(prob, params)
    st = OM.make_structure(b.P, b.Pdot, b.Pddot, n_agents, 0.3, 0.45, n_static=n_static,
                           static_radii=[s.radius for s in statics], rho_final=1e3)
    oprob = OM.Problem(b_eq=MA._b_eq(prob), statics=np.array([s.center for s in statics]).reshape(-1, 3))
    kinv = [f.kinv for f in struct.factors]
    ostate, hist, _ = OM.solve(st, oprob, b.P, max_iter=8, kinv=kinv)
    h = np.array([[x["norm"], x["max_abs"]] for x in sol.residual_history])
    np.testing.assert_allclose(h[:4], hist[:4, :2], rtol=1e-9)
    # multipliers in the reference pair order (lam_ref / JointState.lam): a wrong pair mapping would be O(1) off
    assert sol.state.lam.shape == ostate.lam.shape
    assert np.max(np.abs(sol.state.lam - ostate.lam)) <= 1e-6 * max(1.0, np.abs(ostate.lam).max())


@pytest.mark.parametrize("n_p,degree", [(37, 8), (10, 10), (131, 8), (37, 10), (100, 8), (40, 10), (100, 10)])
def test_sample_rounds_and_basis_sizes_match_oracle(n_p, degree):
    """The element pass runs in rounds of 10 samples: sample counts that leave a partial last round (37, 131)
    or a single round (10), and both compiled basis sizes (m = 9, 11), step for step against the oracle."""
    from paper_2408_10731_b200.basis import build_basis

    b = build_basis(0.0, 10.0, n_p, degree)
    n_agents = 6
    # random endpoints: antipodal rosters put every agent at the layout centre at the middle sample of an
    # odd grid (all pair offsets exactly zero, alpha = atan2 of rounding noise on either side)
    rng = np.random.default_rng(5)
    starts, goals = rng.uniform(-3.0, 3.0, (n_agents, 3)), rng.uniform(-3.0, 3.0, (n_agents, 3))
    bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
            for i in range(n_agents)]
    prob = MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45))
    params = MA.JointParams(max_iter=6, rho_final=1e3)
    struct = MA._Structure(prob, params)
    sol = MA.solve_joint(prob, params)
    st = OM.make_structure(b.P, b.Pdot, b.Pddot, n_agents, 0.3, 0.45, rho_final=1e3)
    oprob = OM.Problem(b_eq=MA._b_eq(prob), statics=np.zeros((0, 3)))
    ostate, hist, _ = OM.solve(st, oprob, b.P, max_iter=6, kinv=[f.kinv for f in struct.factors])
    h = np.array([[x["norm"], x["max_abs"]] for x in sol.residual_history])
    np.testing.assert_allclose(h[:4], hist[:4, :2], rtol=1e-9)
    assert np.max(np.abs(sol.state.lam - ostate.lam)) <= 1e-6 * max(1.0, np.abs(ostate.lam).max())
