"""Device obstacle prediction, the receding-horizon fleet and run_scenario against the oracle and the live
reference's fixtures.  B200 only."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import mpc as omp
from paper_2408_10731_b200.basis import build_basis
from paper_2408_10731_b200.bench import runner as RN
from paper_2408_10731_b200.bench import scenarios as SC
from paper_2408_10731_b200.mpc import MpcFleet

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

CASES = {  # as tests/golden/make_golden.py make_mpc
    "s3": ("random-static", {"dim": 3, "n_o": 6}, 2, dict(step_budget=25, n_steps=12)),
    "f2": ("dynamic-flow", {"n_o": 6}, 4, dict(step_budget=20, n_steps=14, exec_fraction=0.3, goal_radius=1.0)),
    "r2": ("random-static", {"n_o": 5}, 1, dict(step_budget=30, n_steps=10, exec_fraction=0.5, goal_radius=3.0)),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_predict_obstacles_device_bitwise():
    with open(os.path.join(GOLD, "scenarios.json")) as fh:
        cases = json.load(fh)
    g = np.load(os.path.join(GOLD, "scenarios.npz"))
    for key, c in sorted(cases.items()):
        sc = SC.from_json(c["json"])
        tn = g[f"{key}_tnow"]
        ref = np.stack([g[f"{key}_t{m}"] for m in range(tn.size)])  # (S, n_o, n_p, dim)
        got = SC.predict_obstacles_device(sc, g[f"{key}_ts"], t_now=tn).cpu().numpy()
        np.testing.assert_array_equal(got, ref, err_msg=key)
        eng = SC.predict_obstacles_device(sc, g[f"{key}_ts"], t_now=tn, layout="engine").cpu().numpy()
        np.testing.assert_array_equal(eng, np.transpose(ref, (0, 1, 3, 2)), err_msg=key)
    # S scenarios with the same obstacle count in one launch
    scs = [SC.gen_scenario("dynamic-flow", {"n_o": 7}, seed=s) for s in range(5)]
    ts = np.linspace(0.0, 10.0, 100)
    got = SC.predict_obstacles_device(scs, ts, t_now=np.arange(5) * 0.7).cpu().numpy()
    for s, sc in enumerate(scs):
        ref = np.stack([t.centers for t in SC.predict_obstacles(sc, ts, t_now=s * 0.7)])
        np.testing.assert_array_equal(got[s], ref)


def _check_member(res, g, tag, pos_tol):
    flags = g[f"{tag}_flags"]
    assert (res.success, res.reached_goal, res.collided) == tuple(bool(x) for x in flags)
    rec = g[f"{tag}_records"]
    assert len(res.records) == rec.shape[0]
    np.testing.assert_allclose(res.executed.pos, g[f"{tag}_pos"], rtol=0, atol=pos_tol)
    np.testing.assert_array_equal(res.executed.t, g[f"{tag}_t"])
    got = np.array([[r.metrics.smoothness, r.metrics.tracking, r.metrics.arc_length, r.metrics.min_clearance,
                     r.metrics.residual_final, float(r.metrics.success), float(r.metrics.iters)] for r in res.records])
    np.testing.assert_allclose(got[:, :4], rec[:, :4], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(got[:, 4], rec[:, 4], rtol=1e-5, atol=1e-9)
    np.testing.assert_array_equal(got[:, 5:], rec[:, 5:])
    for k, r in enumerate(res.records):
        assert r.scenario_id.endswith(f"#step{k}") and r.metrics.wall_time_ms > 0


@pytest.mark.parametrize("tag", sorted(CASES))
def test_receding_horizon_single_matches_reference(tag):
    kind, params, seed, kw = CASES[tag]
    sc = SC.gen_scenario(kind, params, seed=seed)
    res = RN.receding_horizon_run(sc, "single", **kw)
    _check_member(res, np.load(os.path.join(GOLD, "mpc.npz")), tag, pos_tol=1e-8)


@pytest.mark.parametrize("layout,tol", [("unit", 1e-6), ("angle", 1e-6), ("half", 1e-6)])
def test_fleet_matches_oracle_per_robot(layout, tol):
    """B robots with their own starts / goals in one field: each robot equals the oracle's own run (the unit
    layout computes the angle copies as unit vectors: a different rounding path, 12 steps x 25 iterations)."""
    kind, params, seed, kw = CASES["s3"]
    sc = SC.gen_scenario(kind, params, seed=seed)
    rng = np.random.default_rng(7)
    B = 9
    jit = np.array([0.0, 1.0, 1.0])
    starts = np.array(sc.boundary.start)[None] + rng.uniform(-0.6, 0.6, (B, 3)) * jit
    goals = np.array(sc.boundary.goal)[None] + rng.uniform(-0.6, 0.6, (B, 3)) * jit
    fleet = MpcFleet(sc, starts, goals, step_budget=kw["step_budget"], layout=layout)
    fr = fleet.run(kw["n_steps"])
    b = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
    c, v, a, bb = SC.obstacle_arrays(sc)
    ref = omp.run(b.P, b.Pdot, b.Pddot, b.grid.timestamps, c, v, a, bb, starts, goals, **kw)
    for i in range(B):
        n = int(fr.n_trace[i])
        assert n == len(ref.traces[i]) and fr.flags[i] == ref.flags[i]
        np.testing.assert_allclose(fr.trace[i, :n], ref.traces[i], rtol=0, atol=tol)
        m = np.array(ref.metrics[i])
        steps = fr.steps_of(i)
        assert steps == m.shape[0]
        np.testing.assert_allclose(fr.metrics[:steps, i, [0, 1, 2, 4]], m[:, [0, 1, 2, 4]], rtol=10 * tol, atol=1e-9)
        np.testing.assert_allclose(fr.residual[:steps, i], ref.residuals[i], rtol=1e-4, atol=1e-9)


def test_fleet_large_graph_path_and_frozen_members():
    """> LOOP_MAX_MEMBERS robots (CUDA-graph iteration path); a robot starting inside an obstacle is frozen at
    the start with no records; members equal the oracle."""
    sc = SC.gen_scenario("dynamic-flow", {"n_o": 8}, seed=3)
    B = 80
    rng = np.random.default_rng(1)
    starts = np.stack([np.zeros(B), rng.uniform(-1.5, 1.5, B)], axis=1)
    goals = np.stack([np.full(B, 12.0), rng.uniform(-1.5, 1.5, B)], axis=1)
    starts[5] = sc.obstacles[0].center  # in collision at t = 0
    kw = dict(step_budget=15, n_steps=6)
    fr = MpcFleet(sc, starts, goals, step_budget=15).run(6)
    assert fr.flags[5] == 1 and fr.steps_of(5) == 0 and fr.member(5).records == []
    b = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
    c, v, a, bb = SC.obstacle_arrays(sc)
    idx = [0, 5, 17, 42, 79]
    ref = omp.run(b.P, b.Pdot, b.Pddot, b.grid.timestamps, c, v, a, bb, starts[idx], goals[idx], **kw)
    for n, i in enumerate(idx):
        k = int(fr.n_trace[i])
        assert k == len(ref.traces[n]) and fr.flags[i] == ref.flags[n]
        np.testing.assert_allclose(fr.trace[i, :k], ref.traces[n], rtol=0, atol=1e-8)


def test_receding_horizon_batch_matches_reference():
    g = np.load(os.path.join(GOLD, "mpc.npz"))
    sc = SC.gen_scenario("dynamic-flow", {"n_o": 5, "n_p": 60}, seed=1)
    res = RN.receding_horizon_run(sc, "batch", step_budget=15, n_steps=4)
    _check_member(res, g, "b2", pos_tol=1e-7)


@pytest.mark.parametrize("tag,kind,params,solver,iters", [
    ("single", "random-static", {"dim": 3, "n_o": 8}, "single", 120),
    ("batch", "dynamic-flow", {"n_o": 6, "n_p": 60}, "batch", 40),
])
def test_run_scenario_matches_reference(tmp_path, tag, kind, params, solver, iters):
    g = np.load(os.path.join(GOLD, "runs.npz"))[tag]
    sc = SC.gen_scenario(kind, params, seed=1)
    rec = RN.run_scenario(sc, solver, seed=0, iters=iters, out_dir=tmp_path)
    m = rec.metrics
    got = np.array([m.smoothness, m.tracking, m.arc_length, float(m.success), float(m.iters), m.residual_final,
                    m.min_clearance])
    np.testing.assert_allclose(got, g, rtol=1e-6, atol=1e-9)
    assert os.path.exists(rec.trajectory_path)
    back = RN.read_results_csv(tmp_path / "results.csv")
    assert back[0].metrics.smoothness == m.smoothness


def test_run_scenario_other_solvers_structural():
    """multiagent follows the reference within its chaos (compare structure); PRIEST / CEM run."""
    g = np.load(os.path.join(GOLD, "runs.npz"))["multi"]
    rec = RN.run_scenario(SC.gen_scenario("square-antipodal", {"n_agents": 4, "n_p": 40}, seed=1), "multiagent", 0, 25)
    assert rec.metrics.iters == g[4] and np.isfinite(rec.metrics.min_clearance)
    np.testing.assert_allclose(rec.metrics.arc_length, g[2], rtol=0.05)
    for solver in ("priest", "cem"):
        r = RN.run_scenario(SC.gen_scenario("barn-like", {"n_o": 6, "n_p": 40}, seed=2), solver, 0, 2)
        assert r.metrics.iters == 2 and np.isfinite(r.metrics.smoothness) and isinstance(r.metrics.success, bool)


def test_compact_active_members():
    """tro_mpc_compact: the indices with flags == 0, increasing, and their count (several 1024-chunks)."""
    import ctypes  # noqa: F401

    from paper_2408_10731_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    for n in (1, 1023, 1024, 5000):
        flags = rng.integers(0, 3, n).astype(np.int32)
        f = torch.as_tensor(flags, device="cuda")
        order = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.tro_mpc_compact(n, f.data_ptr(), order.data_ptr(), cnt.data_ptr(), _lib.stream_handle()),
                   "tro_mpc_compact")
        ref = np.nonzero(flags == 0)[0]
        assert int(cnt.item()) == ref.size
        np.testing.assert_array_equal(order.cpu().numpy()[:ref.size], ref)
