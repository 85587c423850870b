"""Scenario model, generators, JSON and CSV wire formats, host obstacle prediction
against fixtures written by the live reference (tests/golden/make_golden.py scenarios / wire).  CPU only."""

import json
import os

import numpy as np
import pytest

from paper_2408_10731_b200.basis import Trajectory
from paper_2408_10731_b200.bench import runner as RN
from paper_2408_10731_b200.bench import scenarios as SC
from paper_2408_10731_b200.metrics import RunMetrics

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases():
    with open(os.path.join(GOLD, "scenarios.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("key", sorted(_cases()))
def test_gen_scenario_json_bytes(key):
    c = _cases()[key]
    sc = SC.gen_scenario(c["kind"], c["params"], seed=c["seed"])
    assert SC.to_json(sc) == c["json"]
    back = SC.from_json(c["json"])
    assert SC.to_json(back) == c["json"]
    assert back.scenario_id == f"{c['kind']}-{c['seed']}"


@pytest.mark.parametrize("key", sorted(_cases()))
def test_predict_obstacles_bitwise(key):
    c = _cases()[key]
    g = np.load(os.path.join(GOLD, "scenarios.npz"))
    sc = SC.from_json(c["json"])
    for m, t_now in enumerate(g[f"{key}_tnow"]):
        tr = SC.predict_obstacles(sc, g[f"{key}_ts"], t_now=float(t_now))
        got = np.stack([t.centers for t in tr]) if tr else np.zeros((0, g[f"{key}_ts"].size, sc.dim))
        np.testing.assert_array_equal(got, g[f"{key}_t{m}"])
        for t, o in zip(tr, sc.obstacles):
            assert (t.shape.a, t.shape.b) == (o.a, o.b)
    if c["kind"] == "square-antipodal":
        roster = np.array([np.concatenate([s, gl]) for s, gl in SC.agent_boundaries(sc)])
        np.testing.assert_array_equal(roster, g[f"{key}_roster"])


def test_scenario_file_roundtrip(tmp_path):
    sc = SC.gen_scenario("dynamic-flow", {"n_o": 4}, seed=3)
    p = tmp_path / "s.json"
    SC.save_scenario(sc, p)
    assert p.read_text() == SC.to_json(sc) + "\n"
    assert SC.to_json(SC.load_scenario(p)) == SC.to_json(sc)


def test_scenario_validation():
    with pytest.raises(ValueError):
        SC.gen_scenario("maze")
    sc = SC.gen_scenario("corridor")
    with pytest.raises(ValueError):
        SC.Scenario(kind="maze", dim=2, horizon=sc.horizon, robot=sc.robot, obstacles=[], boundary=sc.boundary, seed=0)
    with pytest.raises(ValueError):
        SC.Scenario(kind="corridor", dim=4, horizon=sc.horizon, robot=sc.robot, obstacles=[], boundary=sc.boundary,
                    seed=0)
    bad = SC.ScenarioObstacle(a=1.0, b=1.0, center=[0.0, 0.0, 0.0], velocity=[0.0, 0.0])
    with pytest.raises(ValueError):
        SC.Scenario(kind="corridor", dim=2, horizon=sc.horizon, robot=sc.robot, obstacles=[bad], boundary=sc.boundary,
                    seed=0)


def _records():
    vals = list(np.load(os.path.join(GOLD, "wire", "values.npy")))
    recs = []
    for k in range(4):
        m = RunMetrics(smoothness=vals[k], tracking=vals[k + 1], arc_length=vals[k + 2], success=bool(k % 2),
                       iters=10 * k + 3, residual_final=vals[k + 3], min_clearance=vals[k + 4], wall_time_ms=vals[k + 1])
        recs.append(RN.RunRecord(scenario_id=f"corridor-{k}", solver=RN.SOLVERS[k], seed=k * 11, metrics=m))
    return recs


def test_results_csv_bytes_and_roundtrip(tmp_path):
    recs = _records()
    p = tmp_path / "results.csv"
    RN.write_results_csv(p, recs[:2])
    RN.write_results_csv(p, recs[2:])
    with open(os.path.join(GOLD, "wire", "results.csv"), "rb") as fh:
        assert p.read_bytes() == fh.read()
    back = RN.read_results_csv(p)
    assert [(r.scenario_id, r.solver, r.seed) for r in back] == [(r.scenario_id, r.solver, r.seed) for r in recs]
    for a, b in zip(back, recs):
        for f in ("smoothness", "tracking", "arc_length", "residual_final", "min_clearance", "wall_time_ms"):
            x, y = getattr(a.metrics, f), getattr(b.metrics, f)
            assert x == y and np.signbit(x) == np.signbit(y)
        assert (a.metrics.success, a.metrics.iters) == (b.metrics.success, b.metrics.iters)
    RN.write_results_csv(p, recs[:1], append=False)  # fresh file: header + one row
    assert p.read_text().count("\n") == 2


@pytest.mark.parametrize("dim", [2, 3])
def test_trajectory_csv_bytes(tmp_path, dim):
    g = np.load(os.path.join(GOLD, "wire", f"traj{dim}d.npz"))
    n = g["t"].size
    tr = Trajectory(t=g["t"], pos=g["pos"], vel=np.zeros((n, dim)), acc=np.zeros((n, dim)))
    p = tmp_path / "t.csv"
    RN.write_trajectory_csv(p, tr, dim=dim, psi=g["psi"] if g["psi"].size else None)
    with open(os.path.join(GOLD, "wire", f"traj{dim}d.csv"), "rb") as fh:
        assert p.read_bytes() == fh.read()


def test_adapters_shapes():
    """The adapters build the same problems as the reference runner (host-side objects; no GPU needed)."""
    from paper_2408_10731_b200.basis import build_basis

    sc = SC.gen_scenario("random-static", {"dim": 3, "n_o": 4}, seed=1)
    basis = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
    pr = RN.single_problem_from_scenario(sc, basis)
    assert len(pr.obstacles) == 4 and pr.obstacles[0].shape.a == sc.obstacles[0].a + 0.05
    np.testing.assert_array_equal(pr.desired[0], sc.boundary.start)
    np.testing.assert_array_equal(pr.desired[-1], sc.boundary.goal)
    fb = RN.fleet_batch_from_scenario(sc, basis, [sc.boundary.start] * 3, [sc.boundary.goal] * 3)
    assert fb.B == 3 and fb.bvals.shape == (3, 3, 6)
    with pytest.raises(ValueError):
        RN.batch_problem_from_scenario(sc, basis)
    with pytest.raises(ValueError):
        RN.multiagent_problem_from_scenario(sc, basis)
    ma = RN.multiagent_problem_from_scenario(SC.gen_scenario("square-antipodal", {"n_agents": 4}), basis)
    assert ma.n_agents == 4
    with pytest.raises(ValueError):
        RN.run_scenario(sc, "nope", 0, 1)
    with pytest.raises(ValueError):
        RN.receding_horizon_run(sc, "priest")
