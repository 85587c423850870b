"""Host-side logic that needs no GPU: basis, level tables, scenario recipes, API guards."""

import numpy as np
import pytest

from oracle import alg1 as O
from paper_2408_10731_b200 import basis as B
from paper_2408_10731_b200 import qpcore, scenarios
from paper_2408_10731_b200._alg1 import LevelTable, rho_chain
from paper_2408_10731_b200.solver_single import SingleBatch, SingleParams


def test_basis_matches_golden(golden):
    g = golden("c1.npz")
    bs = B.build_basis(0.0, 10.0, 100, 10)
    np.testing.assert_allclose(bs.P, g["P"], atol=1e-15)
    np.testing.assert_allclose(bs.Pdot, g["Pd"], atol=1e-14)
    np.testing.assert_allclose(bs.Pddot, g["Pdd"], atol=1e-13)


def test_basis_guards():
    with pytest.raises(ValueError):
        B.build_basis(1.0, 1.0, 10, 3)
    with pytest.raises(ValueError):
        B.build_basis(0.0, 1.0, 1, 3)
    with pytest.raises(ValueError):
        B.build_basis(0.0, 1.0, 10, -1)


def test_line_vectors_reproduce_lstsq():
    bs = B.build_basis(0.0, 10.0, 100, 10)
    u, v = B.line_basis_vectors(bs)
    p0, p1 = np.array([0.0, -0.3, 0.2]), np.array([12.0, 0.7, -0.1])
    ref = B.straight_line_coeffs(bs, p0, p1)
    got = u[None, :] * p0[:, None] + v[None, :] * (p1 - p0)[:, None]
    np.testing.assert_allclose(got, ref, atol=1e-13)


def test_rho_chain_is_the_reference_schedule():
    chain = rho_chain(1.0, 1.4, 1e3)
    np.testing.assert_array_equal(chain, O.rho_levels(O.Params()))
    assert len(chain) == 22


def test_level_table_matches_oracle_kinv(golden):
    g = golden("c1.npz")
    bs = B.build_basis(0.0, 10.0, 100, 10)
    tab = LevelTable(bs, 10, 1.0, 1.0, [1.0], 1.4, 1e3)
    prob = O.Problem(P=g["P"], Pd=g["Pd"], Pdd=g["Pdd"], bvals=g["bvals"], desired=g["desired"],
                     tracks=g["tracks"], a=g["a"], b=g["b"])
    kkt = O.KKTCache(prob, mode="kinv")
    for lv in (0, 5, 21):
        ref = kkt.kinv(tab.rhos[lv])
        np.testing.assert_allclose(tab.kinv[lv], ref, rtol=0, atol=1e-9 * np.abs(ref).max())
    assert tab.ok.all()


def test_level_table_cond_guard_marks_levels():
    bs = B.build_basis(0.0, 10.0, 100, 10)
    # a tiny cond limit makes every level fail the guard -> marked, not raised
    tab = LevelTable(bs, 10, 1.0, 1.0, [1.0], 1.4, 1e3, cond_limit=10.0)
    assert not tab.ok.any()
    assert isinstance(tab.error_for(0), qpcore.FactorizationError)


def test_factorize_guards_and_count():
    before = qpcore.factorization_count()
    Q = np.eye(3)
    A = np.array([[1.0, 1.0, 1.0]])
    f = qpcore.factorize(Q, A)
    assert f.size == 4 and qpcore.factorization_count() == before + 1
    np.testing.assert_allclose(f.kinv @ qpcore.saddle_matrix(Q, A), np.eye(4), atol=1e-12)
    with pytest.raises(qpcore.FactorizationError):
        qpcore.factorize(Q, np.array([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]]))
    with pytest.raises(ValueError):
        qpcore.factorize(np.array([[1.0, 2.0], [0.0, 1.0]]), np.array([[1.0, 0.0]]))
    with pytest.raises(qpcore.FactorizationError):
        qpcore.factorize(np.diag([1.0, 1e-14, 1.0]), np.array([[1.0, 0.0, 0.0]]))


def test_batch_rhs_guards():
    with pytest.raises(ValueError):
        qpcore.BatchRHS(qs=np.zeros((2, 3)), bs=np.zeros((3, 1)))
    with pytest.raises(ValueError):
        qpcore.BatchRHS(qs=np.zeros((0, 3)), bs=np.zeros((0, 1)))


def test_flow3d_recipe_matches_golden(golden):
    g = golden("flow3d_hist.npz")
    bs = B.build_basis(0.0, 10.0, 100, 10)
    batch = scenarios.flow3d_batch(50, range(8), basis=bs)
    tracks = np.stack([o.centers for o in batch.obstacles])
    np.testing.assert_array_equal(tracks, g["tracks"])
    np.testing.assert_array_equal([o.shape.a for o in batch.obstacles], g["a"])
    np.testing.assert_array_equal(batch.bvals[:, :, 0], g["starts"])
    np.testing.assert_array_equal(batch.bvals[:, :, 3], g["goals"])


def test_c1_scenario_matches_golden(golden):
    g = golden("c1.npz")
    prob = scenarios.c1_problem()
    np.testing.assert_array_equal(np.stack([o.centers for o in prob.obstacles]), g["tracks"])
    np.testing.assert_array_equal(prob.desired, g["desired"][0])


def test_batch_linear_terms_match_single_formula(golden):
    g = golden("flow3d_tf.npz")
    bs = B.build_basis(0.0, 10.0, 100, 10)
    batch = scenarios.flow3d_batch(50, [0, 1], basis=bs)
    q = batch.linear_terms()
    for i in range(2):
        ref = -2.0 * 1.0 * (g["P"].T @ g[f"m{i}_desired"][0]).T
        np.testing.assert_allclose(q[i], ref, atol=1e-12)
    p = batch.problem(1)
    np.testing.assert_allclose(p.desired, g["m1_desired"][0], atol=1e-15)


def test_single_params_defaults_match_reference():
    p = SingleParams()
    assert (p.max_iter, p.tol, p.rho_start, p.rho_growth, p.rho_cap, p.stall_window, p.stall_improvement) == (
        300, 1e-3, 1.0, 1.4, 1e3, 5, 0.01)


def test_from_problems_requires_shared_obstacles():
    bs = B.build_basis(0.0, 10.0, 50, 8)
    b1 = scenarios.flow3d_batch(5, [0], basis=bs).problem(0)
    b2 = scenarios.flow3d_batch(6, [1], basis=bs).problem(0)
    with pytest.raises(ValueError):
        SingleBatch.from_problems([b1, b2])


def test_linear_track_record_reproduces_tracks_bitwise():
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200._alg1 import linear_track_record
    from paper_2408_10731_b200.basis import build_basis

    b = build_basis(0.0, 10.0, 100, 10)
    for n_o in (10, 50, 100):
        tr = np.stack([o.centers for o in scenarios.flow3d_batch(n_o, [0], basis=b).obstacles])
        rec = linear_track_record(tr, b.grid.timestamps)
        assert rec is not None
        cv, rel = rec[: 6 * n_o].reshape(n_o, 6), rec[6 * n_o:]
        np.testing.assert_array_equal(cv[:, None, :3] + cv[:, None, 3:] * rel[None, :, None], tr)
    bad = tr.copy()
    bad[3, 40, 1] = np.nextafter(bad[3, 40, 1], np.inf)  # one sample off by one ulp: not a linear track
    assert linear_track_record(bad, b.grid.timestamps) is None
    p = scenarios.c1_problem()  # static obstacles: v = 0
    tr = np.stack([o.centers for o in p.obstacles])
    rec = linear_track_record(tr, p.basis.grid.timestamps)
    assert rec is not None and not np.any(rec[: 6 * len(tr)].reshape(-1, 6)[:, 3:])


def test_ozaki_row_split_is_exact():
    """The int8 slices of the level inverses reconstruct the fp64 rows to the truncation of S 7-bit slices
    (S = 8: below one ulp of the row maximum), in the tiled canonical layout the tensor-core kernel reads."""
    from paper_2408_10731_b200 import ozaki

    rng = np.random.default_rng(3)
    A = rng.standard_normal((2, 176, 272)) * 10.0 ** rng.uniform(-6, 6, (2, 176, 1))
    A[0, 5] = 0.0  # a zero row
    for S, tol in ((8, 2.0 ** -54), (7, 2.0 ** -47)):
        sl, ea = ozaki.split_rows(A, S)
        assert sl.dtype == np.int8 and sl.shape == (2, S, 2, 9, 4096)
        assert np.abs(sl.astype(int)).max() <= 127
        R = ozaki.reconstruct(sl, ea, 176, 272)
        scale = np.maximum(np.abs(A).max(axis=2, keepdims=True), 1e-300)
        assert np.max(np.abs(R - A) / scale) <= tol
    assert ea[0, 5] == 0 and not sl[0, :, 0].reshape(S, -1)[:, :0].size


@pytest.mark.parametrize("n_a,n_static", [(2, 0), (3, 1), (5, 2), (16, 0), (16, 3)])
def test_multiagent_colour_order(n_a, n_static):
    """The device pair order is a permutation in colour-major order: a proper edge colouring (every agent in at
    most one pair per colour), each colour's pairs contiguous, so step q of every agent's incidence list reads
    one contiguous block of scratch records (conflict-free shared-memory reads in the MA scatter)."""
    from paper_2408_10731_b200.solver_multiagent import _colour_order

    pi, pj, ps = [], [], []
    for i in range(n_a):
        for j in range(i + 1, n_a):
            pi.append(i), pj.append(j), ps.append(-1)
    for s in range(n_static):
        for i in range(n_a):
            pi.append(i), pj.append(-1), ps.append(s)
    pi, pj, ps = np.array(pi), np.array(pj), np.array(ps)
    order = _colour_order(n_a, pi, pj, ps)
    assert sorted(order.tolist()) == list(range(len(pi)))
    # split the order into colours: consecutive blocks where no agent repeats
    colours, cur, seen = [], [], set()
    for p in order:
        members = {pi[p]} | ({pj[p]} if pj[p] >= 0 else set())
        if members & seen:
            colours.append(cur)
            cur, seen = [], set()
        cur.append(p)
        seen |= members
    colours.append(cur)
    n_agent_colours = n_a - 1 + (n_a & 1) if n_a > 1 else 0
    assert len(colours) == n_agent_colours + n_static
    if n_a % 2 == 0:  # perfect matchings: every agent once per colour, so incidence steps stay aligned
        for c in colours[:n_agent_colours]:
            assert len(c) == n_a // 2
