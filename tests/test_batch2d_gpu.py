"""Alg. 2 device kernel (tro_b2_run via solver_batch) vs golden vectors of the live reference,
plus the reference's own solver_batch unit tests (test_solver_batch.py) restated on the device path."""

import numpy as np
import pytest

from oracle import batch2d as OB
from paper_2408_10731_b200 import qpcore, scenarios
from paper_2408_10731_b200 import solver_batch as SB
from paper_2408_10731_b200.basis import AxisBoundary, BasisSet, TimeGrid, boundary_matrix, build_basis, \
    straight_line_coeffs
from paper_2408_10731_b200.geometry import EllipsoidShape, ObstacleTrack

pytestmark = pytest.mark.gpu

GEO = ("alpha_coll", "alpha_v", "alpha_a", "d_coll", "d_v", "d_a")
TOL = 1e-9  # north_star fp64 tolerance, relative to the array's scale


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def geo_err(name, got, ref, ref_state):
    """alpha arrays: wrapped angle difference, ignoring samples whose vector is rounding noise
    (alpha_v / alpha_a at rest, e.g. the zero boundary velocity: atan2 of +-1e-16 flips by 2 pi
    in every implementation, and its g row v_max d_v (cos, sin) is ~0 either way)."""
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    if not name.startswith("alpha"):
        return rel(got, ref)
    diff = np.abs(np.angle(np.exp(1j * (got - ref))))
    if name in ("alpha_v", "alpha_a"):
        diff = np.where(ref_state["d" + name[5:]] > 1e-9, diff, 0.0)
    return float(np.max(diff)) / np.pi


def basis_from(g, tag):
    P = g[f"{tag}_P"]
    ts = np.linspace(0.0, 10.0, P.shape[0])
    return BasisSet(grid=TimeGrid(0.0, 10.0, P.shape[0], ts), degree=P.shape[1] - 1, P=P, Pdot=g[f"{tag}_Pd"],
                    Pddot=g[f"{tag}_Pdd"])


def tracks(g, tag):
    return [ObstacleTrack(centers=c, shape=EllipsoidShape(float(ab[0]), float(ab[1])))
            for c, ab in zip(g[f"{tag}_tracks"], g[f"{tag}_ab"])]


def t50_problem(g):
    basis = basis_from(g, "t50")
    n_p = basis.n_p
    return SB.BatchProblem(basis=basis, boundary=(AxisBoundary(p0=0.0, p1=10.0), AxisBoundary(p0=0.0, p1=0.0)),
                           psi_boundary=(0.0, 0.0),
                           desired=np.column_stack([np.linspace(0.0, 10.0, n_p), np.zeros(n_p)]),
                           obstacles=tracks(g, "t50"), footprint=SB.FootprintSpec(offsets=(0.3, -0.3)), v_max=3.0,
                           a_max=3.0, n_batch=8)


def f10_problem(g):
    bv = g["f10_bvals"]
    return SB.BatchProblem(basis=basis_from(g, "f10"), boundary=(AxisBoundary(*bv[0]), AxisBoundary(*bv[1])),
                           psi_boundary=tuple(g["f10_psib"]), desired=g["f10_desired"], obstacles=tracks(g, "f10"),
                           footprint=SB.FootprintSpec(offsets=(0.0,)), v_max=3.0, a_max=3.0, n_batch=16)


PROBLEMS = {"t50": (t50_problem, 40, (0, 1, 7, 25)), "f10": (f10_problem, 60, (0, 10, 30))}


def golden_state(g, prefix):
    rho, rho_psi, it = g[prefix + "meta"]
    return SB.BatchState(xi=g[prefix + "xi"].copy(), xi_psi=g[prefix + "xi_psi"].copy(), psi=g[prefix + "psi"].copy(),
                         lam=g[prefix + "lam"].copy(), lam_psi=g[prefix + "lam_psi"].copy(), rho=float(rho),
                         rho_psi=float(rho_psi), iteration=int(it), **{k: g[prefix + k] for k in GEO})


# ------------------------------------------------------------------ parity with the reference
@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_init_state_geometry(golden, tag):
    g = golden("batch2d.npz")
    prob = PROBLEMS[tag][0](g)
    st = SB.init_state(prob, g[f"{tag}_samples"])
    for name in ("xi", "xi_psi", "psi"):
        np.testing.assert_array_equal(getattr(st, name), g[f"{tag}_init_{name}"], err_msg=name)
    ref = {name: g[f"{tag}_init_{name}"] for name in GEO}
    for name in GEO:  # materialised on the device (mode 2)
        assert geo_err(name, getattr(st, name), ref[name], ref) <= 1e-12, name


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_teacher_forced_iteration(golden, tag):
    """One device batch_iteration from each reference snapshot lands on the reference's next state."""
    g = golden("batch2d.npz")
    make, _, snaps = PROBLEMS[tag]
    prob = make(g)
    for k in snaps:
        st = golden_state(g, f"{tag}_k{k}_")
        SB.batch_iteration(st, prob)
        nxt = {name: g[f"{tag}_k{k + 1}_{name}"] for name in GEO}
        for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
            err = rel(getattr(st, name), g[f"{tag}_k{k + 1}_{name}"])
            assert err <= TOL, f"k={k} {name}: {err:.3e}"
        for name in GEO:
            err = geo_err(name, getattr(st, name), nxt[name], nxt)
            assert err <= TOL, f"k={k} {name}: {err:.3e}"


def test_teacher_forced_from_implied_state(golden):
    """Same step with alpha / d left implied by (xi, psi) (the solve loop's path, mode 1 without
    GIVEN_AD): the golden alpha / d are functions of the snapshot's xi / psi."""
    g = golden("batch2d.npz")
    prob = f10_problem(g)
    k = 10
    st = golden_state(g, f"f10_k{k}_")
    st._imply(SB._Structure(prob))
    SB.batch_iteration(st, prob)
    for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
        assert rel(getattr(st, name), g[f"f10_k{k + 1}_{name}"]) <= TOL, name


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_free_run_matches_reference(golden, tag):
    """Full solve_batch_opt on the device against the reference's own run: Alg. 2 is not chaotic
    (alpha / d are recomputed each iteration and lambda lives in coefficient space), so
    the final state, the per-iteration best-member history and the ranking match within the fp64
    tolerance, with the identical rho schedule, feasibility mask and best index."""
    g = golden("batch2d.npz")
    make, iters, _ = PROBLEMS[tag]
    prob = make(g)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=iters), samples=g[f"{tag}_samples"])
    h = np.array([[x["norm"], x["max_abs"], x["rho"]] for x in ranked.best_history])
    ref = g[f"{tag}_hist"]
    assert h.shape == ref.shape
    np.testing.assert_array_equal(h[:, 2], ref[:, 2])  # rho schedule
    for c in (0, 1):
        assert rel(h[:, c], ref[:, c]) <= TOL, c
    for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
        assert rel(getattr(ranked.state, name), g[f"{tag}_final_{name}"]) <= TOL, name
    rank = g[f"{tag}_rank"]
    assert rel(ranked.residual_max, rank[:, 0]) <= TOL
    assert rel(ranked.residual_norm, rank[:, 1]) <= TOL
    assert rel(ranked.costs, rank[:, 2]) <= TOL
    assert rel(ranked.aug_costs, rank[:, 3]) <= TOL
    np.testing.assert_array_equal(ranked.feasible, rank[:, 4] > 0)
    best, iters_ref, nfac = g[f"{tag}_meta"]
    assert (-1 if ranked.best_index is None else ranked.best_index) == int(best)
    assert ranked.iterations == int(iters_ref) and ranked.n_factorizations == int(nfac)


def test_final_ranking_quantities_match_state(golden):
    """Mode 3 (ranking) of the device's final state agrees with the oracle evaluated on that state."""
    g = golden("batch2d.npz")
    prob = t50_problem(g)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=40), samples=g["t50_samples"])
    st = OB.make_structure(g["t50_P"], g["t50_Pd"], g["t50_Pdd"], np.stack([b.values() for b in prob.boundary]),
                           prob.psi_boundary, prob.desired, g["t50_tracks"], g["t50_ab"][:, 0], g["t50_ab"][:, 1],
                           (0.3, -0.3), 3.0, 3.0)
    s = ranked.state
    o = OB.State(xi=s.xi, xi_psi=s.xi_psi, psi=s.psi, lam=s.lam, lam_psi=s.lam_psi, rho=s.rho, rho_psi=s.rho_psi,
                 **{k: getattr(s, k) for k in GEO})
    res = s.xi @ st.F.T - OB.build_g(st, o)
    assert rel(ranked.residual_max, np.max(np.abs(res), axis=1)) <= 1e-9
    assert rel(ranked.residual_norm, np.linalg.norm(res, axis=1)) <= 1e-9
    assert rel(ranked.costs, OB.member_costs(st, o)) <= 1e-12
    raw = OB.raw_feasible(st, o, 1e-2, 1e-2)
    assert np.array_equal(ranked.feasible, (np.max(np.abs(res), axis=1) <= 1e-2) & raw)


def test_default_samples_path(golden):
    g = golden("batch2d.npz")
    ranked = SB.solve_batch_opt(f10_problem(g), SB.BatchParams(max_iter=1), seed=3)
    assert rel(ranked.state.xi, g["f10_default_xi1"]) <= TOL


# ------------------------------------------------------------------ the reference's unit tests (test_solver_batch.py)
N_P = 50


def _static_obstacle(center, a, b):
    return ObstacleTrack(centers=np.tile(np.asarray(center, dtype=float), (N_P, 1)), shape=EllipsoidShape(a, b))


def make_problem(obstacles=(), n_batch=8, v_max=3.0, a_max=3.0, offsets=(0.3, -0.3)):
    basis = build_basis(0.0, 10.0, N_P, 10)
    line = np.column_stack([np.linspace(0.0, 10.0, N_P), np.zeros(N_P)])
    return SB.BatchProblem(basis=basis, boundary=(AxisBoundary(p0=0.0, p1=10.0), AxisBoundary(p0=0.0, p1=0.0)),
                           psi_boundary=(0.0, 0.0), desired=line, obstacles=list(obstacles),
                           footprint=SB.FootprintSpec(offsets=offsets), v_max=v_max, a_max=a_max, n_batch=n_batch)


def _sample_state(problem, seed=0, spread=0.5):
    m = problem.basis.n_var
    rng = np.random.default_rng(seed)
    mean = straight_line_coeffs(problem.basis, [0.0, 0.0], [10.0, 0.0]).ravel()
    samples = mean[None, :] + spread * rng.normal(size=(problem.n_batch, 2 * m))
    return SB.init_state(problem, samples)


def test_identical_members_identical_updates():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.2], 0.5, 0.5)], n_batch=4)
    mean = straight_line_coeffs(prob.basis, [0.0, 0.0], [10.0, 0.0]).ravel()
    state = SB.init_state(prob, np.tile(mean, (4, 1)))
    SB.batch_xi_step(state, prob)
    for i in range(1, 4):
        np.testing.assert_array_equal(state.xi[i], state.xi[0])


def test_xi_step_matches_per_member_solve():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.2], 0.5, 0.5)], n_batch=6)
    state = _sample_state(prob, seed=1)
    struct = SB._Structure(prob)
    g = OB.build_g(_oracle_struct(prob), _oracle_state(state))
    q_lin = struct.q[None, :] - state.lam - state.rho * (g @ struct.F)
    K = qpcore.saddle_matrix(struct.Q + state.rho * struct.FtF, struct.A)
    expected = np.stack([np.linalg.solve(K, np.concatenate([-q_lin[i], struct.b]))[:44] for i in range(6)])
    SB.batch_xi_step(state, prob, struct)
    assert np.max(np.abs(state.xi - expected)) <= 1e-10 * max(1.0, np.max(np.abs(expected)))


def test_small_rho_recovers_pure_qp_optimum():
    prob = make_problem(obstacles=[], n_batch=2)
    state = _sample_state(prob, seed=2, spread=0.0)
    state.rho = 1e-4
    SB.batch_xi_step(state, prob)
    m = prob.basis.n_var
    xi_x, xi_y = state.xi[:, :m], state.xi[:, 2 * m:3 * m]
    basis = prob.basis
    Q_axis = basis.Pddot.T @ basis.Pddot + basis.P.T @ basis.P
    factor = qpcore.factorize(Q_axis, boundary_matrix(basis))
    ox, _ = qpcore.solve(factor, -basis.P.T @ prob.desired[:, 0], prob.boundary[0].values())
    oy, _ = qpcore.solve(factor, -basis.P.T @ prob.desired[:, 1], prob.boundary[1].values())
    assert np.max(np.abs(basis.P @ (xi_x[0] - ox))) < 1e-3
    assert np.max(np.abs(basis.P @ (xi_y[0] - oy))) < 1e-3


def test_constant_targets_give_constant_heading():
    psi_bar = 0.35
    prob = make_problem(obstacles=[], n_batch=3)
    prob.psi_boundary = (psi_bar, psi_bar)
    state = _sample_state(prob, seed=3, spread=0.0)
    m = prob.basis.n_var
    state.xi[:, m:2 * m] = np.linalg.lstsq(prob.basis.P, np.full(N_P, np.cos(psi_bar)), rcond=None)[0]
    state.xi[:, 3 * m:] = np.linalg.lstsq(prob.basis.P, np.full(N_P, np.sin(psi_bar)), rcond=None)[0]
    state.psi = np.full((3, N_P), psi_bar)
    SB.heading_step(state, prob)
    np.testing.assert_allclose(state.psi, psi_bar, atol=1e-8)
    assert np.max(np.abs(state.xi_psi @ prob.basis.Pddot.T)) < 1e-6


def test_ramp_targets_fitted_exactly():
    prob = make_problem(obstacles=[], n_batch=2)
    ramp = np.linspace(-0.4, 0.4, N_P)
    prob.psi_boundary = (float(ramp[0]), float(ramp[-1]))
    state = _sample_state(prob, seed=4, spread=0.0)
    m = prob.basis.n_var
    state.xi[:, m:2 * m] = np.linalg.lstsq(prob.basis.P, np.cos(ramp), rcond=None)[0]
    state.xi[:, 3 * m:] = np.linalg.lstsq(prob.basis.P, np.sin(ramp), rcond=None)[0]
    state.psi = np.tile(ramp, (2, 1))
    SB.heading_step(state, prob)
    np.testing.assert_allclose(state.psi[0], ramp, atol=1e-5)


def test_heading_step_matches_per_member_solve():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.0], 0.5, 0.5)], n_batch=5)
    state = _sample_state(prob, seed=5)
    SB.batch_xi_step(state, prob)
    m = prob.basis.n_var
    P = prob.basis.P
    raw = np.arctan2(state.xi[:, 3 * m:] @ P.T, state.xi[:, m:2 * m] @ P.T)
    targets = raw + 2.0 * np.pi * np.round((state.psi - raw) / (2.0 * np.pi))
    Q_psi = prob.basis.Pddot.T @ prob.basis.Pddot + state.rho_psi * P.T @ P
    K = qpcore.saddle_matrix(Q_psi, np.vstack([P[0], P[-1]]))
    expected = np.stack([np.linalg.solve(K, np.concatenate([state.lam_psi[i] + state.rho_psi * P.T @ targets[i],
                                                            np.zeros(2)]))[:m] for i in range(5)])
    SB.heading_step(state, prob)
    assert np.max(np.abs(state.xi_psi - expected)) <= 1e-10
    np.testing.assert_allclose(state._psi_targets, targets, atol=1e-12)


def test_heading_boundary_held():
    prob = make_problem(obstacles=[], n_batch=3)
    state = _sample_state(prob, seed=6)
    SB.batch_iteration(state, prob)
    psi = state.xi_psi @ prob.basis.P.T
    np.testing.assert_allclose(psi[:, 0], 0.0, atol=1e-8)
    np.testing.assert_allclose(psi[:, -1], 0.0, atol=1e-8)


def test_velocity_angle_45_degrees():
    prob = make_problem(obstacles=[], n_batch=1)
    state = _sample_state(prob, seed=8, spread=0.0)
    m = prob.basis.n_var
    diag = straight_line_coeffs(prob.basis, [0.0, 0.0], [10.0, 10.0])
    state.xi[:, :m] = diag[0]
    state.xi[:, 2 * m:3 * m] = diag[1]
    SB.alpha_step(state, prob)
    np.testing.assert_allclose(state.alpha_v[0], np.pi / 4, atol=1e-9)


def test_alpha_update_reduces_collision_residual_term():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.3], 0.6, 0.6)], n_batch=4)
    state = _sample_state(prob, seed=9)
    SB.batch_xi_step(state, prob)
    SB.heading_step(state, prob)
    m = prob.basis.n_var
    P = prob.basis.P
    x, y = state.xi[:, :m] @ P.T, state.xi[:, 2 * m:3 * m] @ P.T
    r = np.array([0.3, -0.3])[None, :, None, None]
    dx = x[:, None, None, :] + r * np.cos(state.psi)[:, None, None, :] - 5.0
    dy = y[:, None, None, :] + r * np.sin(state.psi)[:, None, None, :] - 0.3

    def sq(alpha):
        return (dx - 0.6 * state.d_coll * np.cos(alpha)) ** 2 + (dy - 0.6 * state.d_coll * np.sin(alpha)) ** 2

    before = sq(state.alpha_coll)
    SB.alpha_step(state, prob)
    after = sq(state.alpha_coll)
    assert after.sum() <= before.sum() + 1e-12


def test_velocity_half_of_limit_and_clamp():
    for v_max, expect in ((2.0, 0.5), (0.5, 1.0)):
        prob = make_problem(obstacles=[], n_batch=1, v_max=v_max)
        state = _sample_state(prob, seed=10, spread=0.0)
        m = prob.basis.n_var
        diag = straight_line_coeffs(prob.basis, [0.0, 0.0], [10.0, 0.0])
        state.xi[:, :m] = diag[0]
        state.xi[:, 2 * m:3 * m] = diag[1]
        SB.alpha_step(state, prob)
        SB.d_step(state, prob)
        np.testing.assert_allclose(state.d_v[0], expect, atol=1e-9)


def test_collision_scale_matches_grid_search():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.3], 0.7, 1.1)], n_batch=2)
    state = _sample_state(prob, seed=12)
    SB.batch_iteration(state, prob)
    m = prob.basis.n_var
    P = prob.basis.P
    x, y = state.xi[:, :m] @ P.T, state.xi[:, 2 * m:3 * m] @ P.T
    dx = x[0] + 0.3 * np.cos(state.psi[0]) - 5.0
    dy = y[0] + 0.3 * np.sin(state.psi[0]) - 0.3
    grid = np.linspace(1.0, 20.0, 1_900_001)
    for t in (0, N_P // 2, N_P - 1):
        alpha = state.alpha_coll[0, 0, 0, t]
        cost = (dx[t] - 0.7 * grid * np.cos(alpha)) ** 2 + (dy[t] - 1.1 * grid * np.sin(alpha)) ** 2
        assert abs(state.d_coll[0, 0, 0, t] - grid[np.argmin(cost)]) < 1e-4


def test_d_bounds_hold_after_every_iteration():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.0], 0.8, 0.8)], n_batch=4)
    state = _sample_state(prob, seed=13)
    for _ in range(10):
        SB.batch_iteration(state, prob)
        assert np.all(state.d_coll >= 1.0)
        assert np.all((state.d_v >= 0.0) & (state.d_v <= 1.0))
        assert np.all((state.d_a >= 0.0) & (state.d_a <= 1.0))


def test_obstacle_free_all_feasible_and_near_optimal():
    prob = make_problem(obstacles=[], n_batch=12)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=60), seed=0)
    assert ranked.feasible.all()
    basis = prob.basis
    factor = qpcore.factorize(basis.Pddot.T @ basis.Pddot + basis.P.T @ basis.P, boundary_matrix(basis))
    ox, _ = qpcore.solve(factor, -basis.P.T @ prob.desired[:, 0], prob.boundary[0].values())
    oy, _ = qpcore.solve(factor, -basis.P.T @ prob.desired[:, 1], prob.boundary[1].values())
    cost = float(np.sum((basis.Pddot @ ox) ** 2 + (basis.Pddot @ oy) ** 2)
                 + np.sum((basis.P @ ox - prob.desired[:, 0]) ** 2 + (basis.P @ oy - prob.desired[:, 1]) ** 2))
    assert float(ranked.costs[ranked.best_index]) <= cost + 1e-6


def test_single_member_matches_manual_update_sequence():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.1], 0.5, 0.5)], n_batch=1)
    samples = straight_line_coeffs(prob.basis, [0.0, 0.0], [10.0, 0.0]).ravel()[None, :]
    params = SB.BatchParams(max_iter=7)
    ranked = SB.solve_batch_opt(prob, params, samples=samples)
    state = SB.init_state(prob, samples.copy(), params)
    for _ in range(7):
        SB.batch_iteration(state, prob)
    np.testing.assert_allclose(ranked.state.xi, state.xi, atol=1e-12)


def test_all_infeasible_batch_reports_no_best():
    obstacles = [_static_obstacle([5.0, y], 0.9, 0.9) for y in np.linspace(-6, 6, 11)]
    prob = make_problem(obstacles=obstacles, n_batch=4)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=2), seed=1)
    if ranked.best_index is None:
        assert not ranked.feasible.any()
    else:
        assert ranked.feasible[ranked.best_index]


def test_one_factorization_per_rho_value():
    prob = make_problem(obstacles=[_static_obstacle([5.0, 0.0], 0.8, 0.8)], n_batch=6)
    before = qpcore.factorization_count()
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=40), seed=2)
    distinct_rho = len({h["rho"] for h in ranked.best_history})
    assert ranked.n_factorizations == 2 * distinct_rho
    assert qpcore.factorization_count() - before == 2 * distinct_rho


def test_warm_start_continues_the_run(golden):
    """solve(20) then solve(20, state=...) equals the first 40 iterations up to the stall-rule reset
    of last_change (solver_batch.py:448-449): compare against the oracle doing the same two calls."""
    g = golden("batch2d.npz")
    prob = t50_problem(g)
    r1 = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=3), samples=g["t50_samples"])
    r2 = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=3), state=r1.state)
    assert r2.iterations == 6
    st = golden_state(g, "t50_k0_")
    for _ in range(6):
        SB.batch_iteration(st, prob)
    assert rel(r2.state.xi, st.xi) <= 1e-9


# ------------------------------------------------------------------ helpers
def _oracle_struct(prob):
    return OB.make_structure(prob.basis.P, prob.basis.Pdot, prob.basis.Pddot,
                             np.stack([b.values() for b in prob.boundary]), prob.psi_boundary, prob.desired,
                             np.stack([o.centers for o in prob.obstacles]) if prob.obstacles else np.zeros((0, prob.basis.n_p, 2)),
                             [o.shape.a for o in prob.obstacles], [o.shape.b for o in prob.obstacles],
                             prob.footprint.offsets, prob.v_max, prob.a_max)


def _oracle_state(s):
    return OB.State(xi=s.xi, xi_psi=s.xi_psi, psi=s.psi, lam=s.lam, lam_psi=s.lam_psi, rho=s.rho, rho_psi=s.rho_psi,
                    **{k: getattr(s, k) for k in GEO})


def test_c2alt_recipe_matches_oracle():
    """The C2-alt recipe at full obstacle count and horizon (n_o 50, n_p 100, 200 iterations) on a
    64-member batch (SURVEY.md A.1's probe size): device vs the oracle (bit-exact with the reference)."""
    prob = scenarios.batch2d_problem(n_o=50, n_batch=64)
    assert prob.n_o == 50 and prob.footprint.n_c == 1 and prob.n_batch == 64
    samples = SB._default_samples(prob, prob.basis.n_var, None, None, 0)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=200), samples=samples)
    out = OB.solve(_oracle_struct(prob), samples, 1, max_iter=200)
    np.testing.assert_array_equal(np.array([h["rho"] for h in ranked.best_history]), out["best_hist"][:, 2])
    assert rel(np.array([h["norm"] for h in ranked.best_history]), out["best_hist"][:, 0]) <= TOL
    for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
        assert rel(getattr(ranked.state, name), getattr(out["state"], name)) <= TOL, name
    assert rel(ranked.residual_max, out["rmax"]) <= TOL
    np.testing.assert_array_equal(ranked.feasible, out["feasible"])
    assert ranked.best_index == out["best"]


# ------------------------------------------------------------------ multi-GPU semantics on one GPU
def test_sharded_batch_is_bitwise_the_single_batch():
    """Two member shards, each with its own engine, merged every iteration exactly as the ranks of a
    multi-GPU run do (shard summary -> all-gather -> mode 6): bitwise the single-batch solve."""
    import torch

    prob = scenarios.batch2d_problem(n_o=50, n_batch=64)
    samples = SB._default_samples(prob, prob.basis.n_var, None, None, 0)
    params = SB.BatchParams(max_iter=60)
    ref = SB.solve_batch_opt(prob, params, samples=samples)
    struct = SB._structure_for(prob)
    lv = SB._levels(struct, 1.0, 1.0, params.rho_growth, params.rho_cap)
    engs = []
    for lo, hi in ((0, 27), (27, 64)):
        e = SB._Engine(struct, hi - lo, lv, params=params, max_hist=60, member_offset=lo)
        e.load(SB.init_state(prob, samples[lo:hi], params), 0)
        e.prime(False)
        engs.append(e)
    gathered = torch.zeros((2, 4), dtype=torch.float64, device="cuda")
    for _ in range(60):
        for e in engs:
            e.iterate()
        gathered.copy_(torch.stack([e.shard for e in engs]))
        for e in engs:
            e.merge(gathered)
    np.testing.assert_array_equal(torch.cat([e.xi for e in engs]).cpu().numpy(), ref.state.xi)
    np.testing.assert_array_equal(torch.cat([e.lam for e in engs]).cpu().numpy(), ref.state.lam)
    h = np.array([[x["norm"], x["max_abs"], x["rho"]] for x in ref.best_history])
    for e in engs:
        np.testing.assert_array_equal(e.hist[:60, :3].cpu().numpy(), h)
        assert e.ints_host()["level"] == engs[0].ints_host()["level"]


def test_sharded_entry_point_single_rank():
    from paper_2408_10731_b200.distributed import solve_batch_opt_sharded

    prob = scenarios.batch2d_problem(n_o=50, n_batch=48)
    params = SB.BatchParams(max_iter=40)
    ref = SB.solve_batch_opt(prob, params, seed=5)
    got = solve_batch_opt_sharded(prob, params, seed=5)
    np.testing.assert_array_equal(got.state.xi, ref.state.xi)
    np.testing.assert_array_equal(got.feasible, ref.feasible)
    assert got.best_index == ref.best_index and got.n_factorizations == ref.n_factorizations
    assert [h["rho"] for h in got.best_history] == [h["rho"] for h in ref.best_history]


def test_three_circle_footprint_with_ellipses_matches_oracle():
    """Generic path (n_c = 3 > the compiled specialisations, ellipses a != b, n_p 60): 25 iterations of the
    full solve against the oracle (bit-exact with the reference) within 1e-9."""
    n_p = 60
    basis = build_basis(0.0, 8.0, n_p, 10)
    rng = np.random.default_rng(11)
    obs = []
    for _ in range(6):
        c0 = np.array([rng.uniform(2, 7), rng.uniform(-1.5, 1.5)])
        v = np.array([rng.uniform(-0.3, 0.0), rng.uniform(-0.1, 0.1)])
        cen = c0[None, :] + v[None, :] * basis.grid.timestamps[:, None]
        obs.append(ObstacleTrack(centers=cen, shape=EllipsoidShape(rng.uniform(0.3, 0.6), rng.uniform(0.3, 0.6))))
    prob = SB.BatchProblem(basis=basis, boundary=(AxisBoundary(p0=0.0, p1=9.0), AxisBoundary(p0=0.5, p1=-0.5)),
                           psi_boundary=(0.1, -0.1),
                           desired=np.column_stack([np.linspace(0.0, 9.0, n_p), np.linspace(0.5, -0.5, n_p)]),
                           obstacles=obs, footprint=SB.FootprintSpec(offsets=(0.4, 0.0, -0.4)), v_max=2.5, a_max=2.0,
                           n_batch=12)
    samples = SB._default_samples(prob, basis.n_var, None, None, 4)
    ranked = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=25), samples=samples)
    out = OB.solve(_oracle_struct(prob), samples, 3, max_iter=25)
    for name in ("xi", "xi_psi", "lam", "lam_psi"):
        assert rel(getattr(ranked.state, name), getattr(out["state"], name)) <= TOL, name
    np.testing.assert_array_equal(np.array([h["rho"] for h in ranked.best_history]), out["best_hist"][:, 2])
    np.testing.assert_array_equal(ranked.feasible, out["feasible"])
