"""Batched post-solve validation (tro_validate_f64 via metrics.py) vs golden vectors of the live reference."""

import math
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import metrics as OMT
from paper_2408_10731_b200 import metrics as MT
from paper_2408_10731_b200.basis import BasisSet, TimeGrid, Trajectory

pytestmark = pytest.mark.gpu


@dataclass
class Obs:
    a: float
    b: float
    center: list
    velocity: list


@dataclass
class Scene:  # the fields of bench.scenarios.Scenario the metrics read
    dim: int
    obstacles: list


def scene(g, tag, dim):
    o = g[f"{tag}_obs"]
    return Scene(dim, [Obs(float(r[2 * dim]), float(r[2 * dim + 1]), list(r[:dim]), list(r[dim:2 * dim])) for r in o])


def basis_of(g, tag):
    P = g[f"{tag}_P"]
    t = g[f"{tag}_t"]
    return BasisSet(grid=TimeGrid(float(t[0]), float(t[-1]), t.size, t), degree=P.shape[1] - 1, P=P,
                    Pdot=np.zeros_like(P), Pddot=g[f"{tag}_Pdd"])


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


CASES = [("s3", 3), ("f2", 2)]


@pytest.mark.parametrize("tag,dim", CASES)
def test_validate_batch_coefficients(golden, tag, dim):
    g = golden("metrics.npz")
    sc, ref = scene(g, tag, dim), g[f"{tag}_res"]
    r = MT.validate_batch(sc, g[f"{tag}_t"], xi=g[f"{tag}_xi"], basis=basis_of(g, tag), desired=g[f"{tag}_desired"])
    got = np.stack([r["smoothness"], r["tracking"], r["arc_length"], r["min_clearance"], r["worst"]], axis=1)
    assert rel(got, ref[:, [0, 1, 2, 3, 4]]) <= 1e-12
    np.testing.assert_array_equal(r["success"], ref[:, 5] > 0)
    r1 = MT.validate_batch(sc, g[f"{tag}_t"], xi=g[f"{tag}_xi"], basis=basis_of(g, tag), margin=0.1)
    assert rel(r1["worst"], ref[:, 6]) <= 1e-12
    np.testing.assert_array_equal(r1["success"], ref[:, 7] > 0)


@pytest.mark.parametrize("tag,dim", CASES)
def test_reference_api_on_sampled_trajectories(golden, tag, dim):
    g = golden("metrics.npz")
    sc = scene(g, tag, dim)
    for x, ref in zip(g[f"{tag}_xi"], g[f"{tag}_res"]):
        tr = Trajectory(t=g[f"{tag}_t"], pos=g[f"{tag}_P"] @ x.T, vel=np.zeros((g[f"{tag}_t"].size, dim)),
                        acc=g[f"{tag}_Pdd"] @ x.T)
        m = MT.eval_metrics(tr, sc, g[f"{tag}_desired"])
        assert rel([m.smoothness, m.tracking, m.arc_length, m.min_clearance], ref[[0, 1, 2, 3]]) <= 1e-12
        ok, w = MT.check_collision_free(tr, sc, margin=0.1)
        assert ok == bool(ref[7]) and rel(w, ref[6]) <= 1e-12
        assert rel(MT.clearance_lower_bound(tr, sc), ref[8]) <= 1e-12


def test_no_obstacles_semantics():
    t = np.linspace(0.0, 10.0, 50)
    pos = np.stack([t, np.sin(t), np.zeros_like(t)], axis=1)
    tr = Trajectory(t=t, pos=pos, vel=pos, acc=pos)
    sc = Scene(3, [])
    assert MT.check_collision_free(tr, sc) == (True, -math.inf)
    assert MT.clearance_lower_bound(tr, sc) == math.inf
    r = MT.validate_batch(sc, t, pos=pos[None], acc=pos[None])
    assert r["worst"][0] == -math.inf and r["min_clearance"][0] == math.inf and r["success"][0]


def test_large_batch_matches_oracle_on_a_sample():
    rng = np.random.default_rng(3)
    n_o, n_p, B = 100, 100, 4096
    t = np.linspace(0.0, 10.0, n_p)
    obs = [Obs(float(rng.uniform(0.3, 0.6)), float(rng.uniform(0.3, 0.6)), list(rng.uniform(0, 10, 3)),
               list(rng.uniform(-0.3, 0.3, 3))) for _ in range(n_o)]
    sc = Scene(3, obs)
    pos = rng.uniform(0, 10, (B, n_p, 3))
    acc = rng.normal(size=(B, n_p, 3))
    des = rng.uniform(0, 10, (n_p, 3))
    r = MT.validate_batch(sc, t, pos=pos, acc=acc, desired=des, margin=0.05)
    c = np.array([o.center for o in obs]); v = np.array([o.velocity for o in obs])
    a = np.array([o.a for o in obs]); b = np.array([o.b for o in obs])
    for i in rng.choice(B, 16, replace=False):
        ref = OMT.metrics(pos[i], acc[i], t, c, v, a, b, 3, des, 0.05)
        got = [r["smoothness"][i], r["tracking"][i], r["arc_length"][i], r["worst"][i], r["min_clearance"][i]]
        assert rel(got, ref) <= 1e-12, i


@pytest.mark.parametrize("per_member_desired", [False, True])
def test_pinned_host_input_pipelined_matches_one_launch(golden, per_member_desired):
    """Coefficients in pinned host memory take the chunked upload/validate/download path (metrics.py
    _validate_pipelined): bitwise the results of one launch over device-resident coefficients."""
    import torch

    g = golden("metrics.npz")
    sc, bs = scene(g, "s3", 3), basis_of(g, "s3")
    xi0 = g["s3_xi"]
    B = 3 * MT._PIPE_MIN_CHUNK + 17  # 3 ragged chunks
    rng = np.random.default_rng(5)
    xi = xi0[rng.integers(0, xi0.shape[0], B)] + rng.normal(scale=0.05, size=(B,) + xi0.shape[1:])
    des = g["s3_desired"]
    if per_member_desired:
        des = des[None] + rng.normal(scale=0.1, size=(B,) + des.shape)
    xi_pin = torch.as_tensor(xi).pin_memory()
    r = MT.validate_batch(sc, g["s3_t"], xi=xi_pin, basis=bs, desired=des, margin=0.05)
    ref = MT.validate_batch(sc, g["s3_t"], xi=torch.as_tensor(xi, device="cuda"), basis=bs, desired=des,
                            margin=0.05, return_device=True)["out"].cpu().numpy()
    got = np.stack([r["smoothness"], r["tracking"], r["arc_length"], r["worst"], r["min_clearance"]], axis=1)
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(r["success"], ref[:, 3] <= 0.0)


@pytest.mark.parametrize("n_p", [20, 40, 64, 100, 131])
@pytest.mark.parametrize("dim", [2, 3])
def test_coefficient_mode_sample_counts(n_p, dim):
    """Coefficient input across sample counts: no full 32-sample group (20), a group + tail (40, 100, 131),
    groups only (64); positions / accelerations from the tensor-core products, the distance pass's register
    groups and lane-spread tail -- all against the oracle metrics on P xi, Pddot xi."""
    rng = np.random.default_rng(n_p + 10 * dim)
    m, n_o, B = 11, 37, 96
    t = np.linspace(0.0, 10.0, n_p)
    P = rng.normal(size=(n_p, m))
    Pdd = rng.normal(size=(n_p, m))
    basis = BasisSet(grid=TimeGrid(0.0, 10.0, n_p, t), degree=m - 1, P=P, Pdot=np.zeros_like(P), Pddot=Pdd)
    obs = [Obs(float(rng.uniform(0.3, 0.6)), float(rng.uniform(0.3, 0.6)), list(rng.uniform(-2, 2, dim)),
               list(rng.uniform(-0.3, 0.3, dim))) for _ in range(n_o)]
    sc = Scene(dim, obs)
    xi = rng.normal(size=(B, dim, m)) * 0.5
    des = rng.uniform(-2, 2, (n_p, dim))
    r = MT.validate_batch(sc, t, xi=xi, basis=basis, desired=des, margin=0.05)
    c = np.array([o.center for o in obs]); v = np.array([o.velocity for o in obs])
    a = np.array([o.a for o in obs]); b = np.array([o.b for o in obs])
    for i in range(0, B, 7):
        pos = P @ xi[i].T
        acc = Pdd @ xi[i].T
        ref = OMT.metrics(pos, acc, t, c, v, a, b, dim, des, 0.05)
        got = [r["smoothness"][i], r["tracking"][i], r["arc_length"][i], r["worst"][i], r["min_clearance"][i]]
        assert rel(got, ref) <= 1e-12, (i, got, ref)
