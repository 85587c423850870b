"""Cold solves on reused engines are cold solves (solver_single.py:413-414 -> init_state :115-166).

A solve on an engine that already ran must start from rho = rho_o = rho_start, iteration 0 and an empty
stall schedule, exactly like a fresh engine; new members passed with ``engine=`` must be honoured; and the
linear terms the device computes from the boundary values must be the reference's formula
(-2 w_track P' desired, solver_single.py:173).
"""

import threading

import numpy as np
import pytest
import torch

from paper_2408_10731_b200 import scenarios
from paper_2408_10731_b200.basis import build_basis
from paper_2408_10731_b200.solver_single import (SingleBatch, SingleParams, make_batch_engine, solve_single,
                                                 solve_single_batch)

pytestmark = pytest.mark.gpu

# tol > 0 with a short stall window: members converge at different iterations and penalties grow, so a
# stale rho / schedule / iteration counter would show in every compared field
PARAMS = SingleParams(max_iter=120, tol=2e-3)


def _batch(members, n_o=20):
    return scenarios.flow3d_batch(n_o, members, basis=build_basis(0.0, 10.0, 100, 10))


def _result(sol):
    r = sol.numpy()
    return r.xi.copy(), r.iterations.copy(), r.rho_o.copy(), r.residual_max.copy(), r.history.copy()


def _same(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("layout", ["angle", "half"])
def test_same_batch_twice_on_one_engine_is_bitwise_a_fresh_solve(layout):
    batch = _batch(range(80))  # > LOOP_MAX_MEMBERS: the persistent kernel + graph path
    eng = make_batch_engine(batch, PARAMS, history=True, layout=layout)
    first = _result(solve_single_batch(batch, PARAMS, engine=eng))
    second = _result(solve_single_batch(batch, PARAMS, engine=eng))
    fresh = _result(solve_single_batch(batch, PARAMS, history=True, layout=layout))
    _same(first, second)
    _same(first, fresh)
    assert first[2].max() > 1.0  # penalties grew: a stale rho_o would show in every field


def test_small_batch_in_kernel_loop_reuse():
    batch = _batch(range(5))  # <= LOOP_MAX_MEMBERS: one-launch in-kernel loop
    eng = make_batch_engine(batch, PARAMS, history=True)
    a = _result(solve_single_batch(batch, PARAMS, engine=eng))
    b = _result(solve_single_batch(batch, PARAMS, engine=eng))
    _same(a, b)
    _same(a, _result(solve_single_batch(batch, PARAMS, history=True)))


def test_engine_honours_new_members():
    b1, b2 = _batch(range(80)), _batch(range(1000, 1080))
    eng = make_batch_engine(b1, PARAMS, history=True)
    solve_single_batch(b1, PARAMS, engine=eng)
    got = _result(solve_single_batch(b2, PARAMS, engine=eng))
    _same(got, _result(solve_single_batch(b2, PARAMS, history=True)))


def test_engine_mismatch_raises():
    eng = make_batch_engine(_batch(range(8)), PARAMS)
    with pytest.raises(ValueError):
        solve_single_batch(_batch(range(9)), PARAMS, engine=eng)
    with pytest.raises(ValueError):
        solve_single_batch(_batch(range(8), n_o=21), PARAMS, engine=eng)
    with pytest.raises(ValueError):
        solve_single_batch(_batch(range(8)), SingleParams(max_iter=7), engine=eng)


def test_cached_engine_reuse_and_thread_ownership():
    batch = _batch(range(70))
    ref = _result(solve_single_batch(batch, PARAMS, history=True))
    a = _result(solve_single_batch(batch, PARAMS, history=True, cache=True))
    b = _result(solve_single_batch(batch, PARAMS, history=True, cache=True))
    _same(ref, a)
    _same(ref, b)
    engines = {}

    def worker(k):
        engines[k] = solve_single_batch(batch, PARAMS, history=True, cache=True).engine
        _same(ref, _result(solve_single_batch(batch, PARAMS, history=True, cache=True)))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert engines[0] is not engines[1]  # one cached engine per thread


def test_solve_single_twice_same_solution():
    prob = scenarios.c1_problem()
    s1 = solve_single(prob, SingleParams())
    s2 = solve_single(prob, SingleParams())
    assert s1.iterations == s2.iterations == 261
    assert [h["rho_o"] for h in s1.residual_history] == [h["rho_o"] for h in s2.residual_history]
    np.testing.assert_array_equal(s1.state.xi, s2.state.xi)


def test_device_linear_terms_match_the_reference_formula():
    batch = _batch(range(40))
    eng = make_batch_engine(batch, PARAMS)
    host = batch.linear_terms()  # -2 w_track (P' desired)' with numpy, per member
    dev = eng.q.cpu().numpy()
    assert np.max(np.abs(dev - host)) <= 1e-13 * np.max(np.abs(host))
    # explicit desired paths take the same route
    des = batch.desired_paths() + 0.01 * np.sin(np.arange(100))[None, :, None]
    eng.set_members(batch.bvals, des)
    host2 = -2.0 * np.transpose(np.matmul(batch.basis.P.T[None], des), (0, 2, 1))
    assert np.max(np.abs(eng.q.cpu().numpy() - host2)) <= 1e-13 * np.max(np.abs(host2))
    torch.cuda.synchronize()


def test_from_problems_batch_equals_single_batch_recipe():
    batch = _batch(range(6))
    via_problems = SingleBatch.from_problems([batch.problem(i) for i in range(6)])
    a = _result(solve_single_batch(batch, PARAMS, history=True))
    b = _result(solve_single_batch(via_problems, PARAMS, history=True))
    _same(a, b)


def test_register_tracks_equal_streamed_tracks():
    """Constant-velocity obstacles: the TMA kernel generates c + v rel in registers (track_lin) instead of
    streaming the track rows; the result is bitwise the streamed-track run (the record reproduces every
    sample exactly, tests/test_host_logic.py)."""
    batch = _batch(range(150), n_o=30)
    out = []
    for lin in (True, False):
        eng = make_batch_engine(batch, PARAMS, history=True, layout="half")
        assert eng.track_lin is not None
        if not lin:
            eng._consts.track_lin = None
        out.append(_result(solve_single_batch(batch, PARAMS, engine=eng)))
    _same(out[0], out[1])


def test_factorization_count_when_the_final_iteration_grows_the_penalty():
    """A run that stops right after a penalty growth never factorizes the new level (the reference factorizes
    in the NEXT position step, solver_single.py:198-202): n_factorizations counts the levels used."""
    from oracle import alg1 as O

    prob = scenarios.c1_problem()
    op = O.Problem(P=prob.basis.P, Pd=prob.basis.Pdot, Pdd=prob.basis.Pddot,
                   bvals=np.stack([bc.values() for bc in prob.boundary])[None], desired=prob.desired[None],
                   tracks=np.stack([o.centers for o in prob.obstacles]),
                   a=np.array([o.shape.a for o in prob.obstacles]), b=np.array([o.shape.b for o in prob.obstacles]))
    prm = dict(tol=0.0, stall_improvement=0.5)  # frequent growths
    full = O.solve(op, O.Params(max_iter=120, **prm))
    rho = np.array(full.rho_hist[0])  # rho_o used by each iteration's position step
    grow_after = [k + 1 for k in range(len(rho) - 1) if rho[k + 1] != rho[k]]  # iterations ending in a growth
    assert len(grow_after) >= 2
    for n in (grow_after[0], grow_after[1], grow_after[0] + 1):
        ref = O.solve(op, O.Params(max_iter=n, **prm))
        want = int(ref.state.n_factorizations[0])
        sol = solve_single(prob, SingleParams(max_iter=n, **prm))
        assert sol.n_factorizations == want, (n, sol.n_factorizations, want)
        bs = solve_single_batch(SingleBatch.from_problems([prob] * 70), SingleParams(max_iter=n, **prm))
        assert set(bs.n_factorizations.cpu().numpy().tolist()) == {want}, n
