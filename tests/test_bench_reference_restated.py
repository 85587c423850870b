"""The reference's own bench tests (pkg/tests/test_bench.py) restated against this package: scenario
generation / JSON / prediction / results CSV on the CPU, metrics / collision checks / run_scenario /
receding-horizon driving on the GPU (marked)."""

import json

import numpy as np
import pytest

from paper_2408_10731_b200.basis import Trajectory
from paper_2408_10731_b200.bench import (Boundary, Horizon, RobotSpec, RunMetrics, RunRecord, Scenario,
                                         ScenarioObstacle, agent_boundaries, check_collision_free, eval_metrics,
                                         from_json, gen_scenario, load_scenario, predict_obstacles,
                                         predict_obstacles_device, read_results_csv, receding_horizon_run,
                                         run_scenario, save_scenario, to_json, write_results_csv)


def _traj(t, pos):
    pos = np.asarray(pos, dtype=float)
    vel = np.gradient(pos, t, axis=0)
    return Trajectory(t=np.asarray(t), pos=pos, vel=vel, acc=np.gradient(vel, t, axis=0))


def empty_scenario(dim=2, n_p=50):
    return Scenario(kind="random-static", dim=dim, horizon=Horizon(t0=0.0, tf=5.0, n_p=n_p),
                    robot=RobotSpec(shape=[0.0, 0.0], v_max=3.0, a_max=3.0), obstacles=[],
                    boundary=Boundary(start=[0.0] * dim, goal=[5.0] + [0.0] * (dim - 1)), seed=0)


# ---------------------------------------------------------------- CPU (test_bench.py:48-213)
def test_square_antipodal_goals_are_rotations():
    sc = gen_scenario("square-antipodal", {"n_agents": 4, "jitter": 0.0}, seed=1)
    roster = agent_boundaries(sc)
    assert len(roster) == 4
    centre = 0.5 * (np.asarray(sc.boundary.start) + np.asarray(sc.boundary.goal))
    for s, g in roster:
        np.testing.assert_allclose(g, 2.0 * centre - s, atol=1e-12)


def test_seed_repetition_identical():
    assert to_json(gen_scenario("corridor", seed=5)) == to_json(gen_scenario("corridor", seed=5))


def test_random_static_respects_clearance():
    sc = gen_scenario("random-static", {"n_o": 10, "clearance": 1.5}, seed=2)
    assert len(sc.obstacles) == 10
    for ob in sc.obstacles:
        c = np.asarray(ob.center)
        assert np.linalg.norm(c - np.asarray(sc.boundary.start)) >= 1.5
        assert np.linalg.norm(c - np.asarray(sc.boundary.goal)) >= 1.5


def test_probe_puts_sampling_mean_inside_obstacle():
    sc = gen_scenario("all-infeasible-probe", seed=3)
    s, g = np.asarray(sc.boundary.start), np.asarray(sc.boundary.goal)
    blk = sc.obstacles[0]
    line = s + np.linspace(0, 1, 200)[:, None] * (g - s)
    assert np.hypot(line[:, 0] - blk.center[0], line[:, 1] - blk.center[1]).min() < blk.a


def test_unknown_kind_rejected():
    with pytest.raises(ValueError):
        gen_scenario("no-such-kind", seed=0)


def test_json_round_trips(tmp_path):
    sc = gen_scenario("dynamic-flow", seed=7)
    assert to_json(from_json(to_json(sc))) == to_json(sc)
    sc = gen_scenario("barn-like", seed=9)
    save_scenario(sc, tmp_path / "scn.json")
    assert to_json(load_scenario(tmp_path / "scn.json")) == to_json(sc)


def test_schema_keys_exact():
    raw = json.loads(to_json(gen_scenario("corridor", seed=0)))
    assert set(raw) == {"kind", "dim", "horizon", "robot", "obstacles", "boundary", "seed"}
    assert set(raw["horizon"]) == {"t0", "tf", "n_p"}
    assert set(raw["robot"]) == {"shape", "v_max", "a_max", "footprint_offsets"}
    assert set(raw["boundary"]) == {"start", "goal"}
    for ob in raw["obstacles"]:
        assert set(ob) == {"a", "b", "center", "velocity"}


def test_predict_obstacles_kinematics():
    sc = empty_scenario()
    sc.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=[1.0, 2.0], velocity=[0.0, 0.0])]
    np.testing.assert_array_equal(predict_obstacles(sc, np.linspace(0, 5, 11))[0].centers,
                                  np.tile([1.0, 2.0], (11, 1)))
    sc3 = empty_scenario(dim=3)
    sc3.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=[0.0, 0.0, 0.0], velocity=[1.0, 0.0, 0.0])]
    np.testing.assert_allclose(predict_obstacles(sc3, np.linspace(0, 4, 5))[0].centers[2], [2.0, 0.0, 0.0])
    rng = np.random.default_rng(0)
    v, c = rng.normal(size=2), rng.normal(size=2)
    sc.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=list(c), velocity=list(v))]
    ts = np.linspace(0.0, 5.0, 13)
    tr = predict_obstacles(sc, ts, t_now=1.5)
    for i, t in enumerate(ts):
        np.testing.assert_allclose(tr[0].centers[i], c + v * (1.5 + t), atol=1e-12)


def test_results_csv_round_trip(tmp_path):
    m = RunMetrics(smoothness=1.2345678901234567, tracking=0.1, arc_length=12.0, success=True, iters=42,
                   residual_final=1e-9, min_clearance=0.25, wall_time_ms=17.5)
    rec = RunRecord(scenario_id="corridor-0", solver="single", seed=3, metrics=m)
    write_results_csv(tmp_path / "results.csv", [rec])
    out = read_results_csv(tmp_path / "results.csv")
    assert len(out) == 1 and (out[0].scenario_id, out[0].solver, out[0].seed) == ("corridor-0", "single", 3)
    assert out[0].metrics == m


# ---------------------------------------------------------------- GPU (test_bench.py:111-266)
gpu = pytest.mark.gpu


@gpu
def test_eval_metrics_cases():
    sc = empty_scenario()
    t = np.linspace(0.0, 5.0, 50)
    m = eval_metrics(Trajectory(t=t, pos=np.ones((50, 2)), vel=np.zeros((50, 2)), acc=np.zeros((50, 2))), sc)
    assert m.smoothness == 0.0 and m.arc_length == 0.0
    pos = np.column_stack([t, np.zeros(50)])
    m = eval_metrics(Trajectory(t=t, pos=pos, vel=np.tile([1.0, 0.0], (50, 1)), acc=np.zeros((50, 2))), sc)
    assert m.smoothness == 0.0 and m.arc_length == pytest.approx(5.0)
    th = np.linspace(0.0, 2.0 * np.pi, 2000)
    m = eval_metrics(_traj(th, np.column_stack([np.cos(th), np.sin(th)])), sc)
    assert abs(m.arc_length - 2.0 * np.pi) / (2.0 * np.pi) < 0.01


@gpu
def test_check_collision_free_cases():
    sc = empty_scenario()
    sc.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=[2.5, 0.0], velocity=[0.0, 0.0])]
    t = np.linspace(0.0, 5.0, 50)
    ok, worst = check_collision_free(_traj(t, np.column_stack([t, np.zeros(50)])), sc)
    assert not ok and worst > 0.0
    t10 = np.linspace(0.0, 5.0, 10)
    assert check_collision_free(_traj(t10, np.column_stack([t10, np.zeros(10)])), empty_scenario())[0]
    sc.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=[2.5, -0.5], velocity=[0.0, 0.0])]
    t51 = np.linspace(0.0, 5.0, 51)
    ok, worst = check_collision_free(_traj(t51, np.column_stack([np.linspace(0, 5, 51), np.zeros(51)])), sc,
                                     margin=0.0)
    assert ok and abs(worst) <= 1e-9  # grazes the top at (2.5, 0)


@gpu
def test_predict_obstacles_device_kinematics():
    rng = np.random.default_rng(0)
    v, c = rng.normal(size=2), rng.normal(size=2)
    sc = empty_scenario()
    sc.obstacles = [ScenarioObstacle(a=0.5, b=0.5, center=list(c), velocity=list(v))]
    ts = np.linspace(0.0, 5.0, 13)
    got = predict_obstacles_device(sc, ts, t_now=1.5).cpu().numpy()[0, 0]
    np.testing.assert_array_equal(got, predict_obstacles(sc, ts, t_now=1.5)[0].centers)


@gpu
def test_run_scenario_single_end_to_end(tmp_path):
    sc = gen_scenario("corridor", {"n_o": 4, "n_p": 60}, seed=0)
    rec = run_scenario(sc, solver="single", seed=0, iters=300, out_dir=tmp_path)
    assert rec.metrics.success
    assert (tmp_path / "results.csv").exists() and rec.trajectory_path is not None
    assert open(rec.trajectory_path).readline().strip() == "t,x,y,z,psi"
    with pytest.raises(ValueError):
        run_scenario(gen_scenario("corridor", seed=0), solver="nope", seed=0, iters=5)


@gpu
def test_run_scenario_determinism_modulo_wall_time():
    sc = gen_scenario("random-static", {"n_o": 5, "n_p": 60}, seed=1)
    m1 = run_scenario(sc, solver="priest", seed=4, iters=3).metrics
    m2 = run_scenario(sc, solver="priest", seed=4, iters=3).metrics
    m1.wall_time_ms = m2.wall_time_ms = 0.0
    assert m1 == m2


@gpu
def test_receding_horizon_empty_world_reaches_goal():
    res = receding_horizon_run(empty_scenario(n_p=40), solver="single", step_budget=20, n_steps=25)
    assert res.success and res.reached_goal and not res.collided
    assert len(res.records) >= 1 and res.records[-1].metrics.success


@gpu
def test_receding_horizon_start_in_collision_fails_immediately():
    sc = empty_scenario(n_p=40)
    sc.obstacles = [ScenarioObstacle(a=1.0, b=1.0, center=[0.0, 0.0], velocity=[0.0, 0.0])]
    res = receding_horizon_run(sc, solver="single", step_budget=10, n_steps=5)
    assert not res.success and res.collided and res.records == []


@gpu
def test_receding_horizon_dynamic_flow_success_rate_definition():
    outcomes = []
    for seed in range(3):
        sc = gen_scenario("dynamic-flow", {"n_o": 3, "n_p": 40, "tf": 8.0}, seed=seed)
        outcomes.append(receding_horizon_run(sc, solver="single", step_budget=25, n_steps=25).success)
    rate = sum(outcomes) / len(outcomes)
    assert 0.0 <= rate <= 1.0 and rate == pytest.approx(np.mean(outcomes))
