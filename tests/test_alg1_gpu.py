"""Parity of the sm_100a Alg. 1 kernels (through the C-ABI) with the reference / oracle.

Tolerances (north_star): fp64 trajectories and residuals within 1e-9 relative; fp32
storage within 1e-4 relative.  The AM map is chaotic in clutter,
so long free-running comparisons are only made where the reference's own LU-vs-K^-1
twin stays within 1e-9 (C1, the 2-D corridor, and per member up to its twin window);
everything else is teacher-forced one-step parity from full reference snapshots.
"""

import numpy as np
import pytest
import torch

from oracle import alg1 as O
from paper_2408_10731_b200 import _lib, qpcore, scenarios
from paper_2408_10731_b200._alg1 import Alg1Engine
from paper_2408_10731_b200.basis import AxisBoundary, BasisSet, TimeGrid
from paper_2408_10731_b200.geometry import EllipsoidShape, ObstacleTrack
from paper_2408_10731_b200.solver_single import (SingleParams, SingleProblem, am_iteration, init_state,
                                                 solve_single, solve_single_batch)

pytestmark = pytest.mark.gpu


def basis_from(g):
    t = g["t"]
    return BasisSet(grid=TimeGrid(float(t[0]), float(t[-1]), len(t), t), degree=g["P"].shape[1] - 1, P=g["P"],
                    Pdot=g["Pd"], Pddot=g["Pdd"])


def problem_from(g, bvals=None, desired=None):
    bvals = g["bvals"][0] if bvals is None else bvals
    desired = g["desired"][0] if desired is None else desired
    dim = bvals.shape[0]
    obs = [ObstacleTrack(g["tracks"][j], EllipsoidShape(float(g["a"][j]), float(g["b"][j])))
           for j in range(g["tracks"].shape[0])]
    bnd = tuple(AxisBoundary(*bvals[k]) for k in range(dim))
    return SingleProblem(basis_from(g), bnd, desired, obs, float(g["w"][0]), float(g["w"][1]))


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


def engine_from(g, bvals, desired, params, *, dtype=torch.float64, rho0=None, max_hist=0, layout="angle",
                use_tma=True):
    basis = basis_from(g)
    q = -2.0 * float(g["w"][1]) * np.einsum("tc,btk->bkc", basis.P, desired)
    return Alg1Engine(basis, g["tracks"], g["a"], g["b"], bvals, q, params=params, rho0=rho0,
                      w_smooth=float(g["w"][0]), w_track=float(g["w"][1]), dtype=dtype, max_hist=max_hist,
                      export=True, keep_d=True, layout=layout, use_tma=use_tma)


KERNELS = [("angle", True), ("angle", False), ("unit", True), ("unit", False), ("half", True), ("half", False)]


def load_snapshot(eng, g, pre, dim):
    planes = [g[pre + "lam_pos"][k] for k in range(dim)] + [g[pre + "lam_cos_a"], g[pre + "lam_sin_a"]]
    if dim == 3:
        planes += [g[pre + "lam_cos_b"], g[pre + "lam_sin_b"]]
    sc = g[pre + "scal"]
    eng.load_state(xi=g[pre + "xi"][None], alpha=g[pre + "alpha"][None],
                   beta=g[pre + "beta"][None] if dim == 3 else None, lam_planes=np.stack(planes)[:, None],
                   d=g[pre + "d"][None], rho=[sc[0]], rho_o=[sc[1]], iteration=[int(sc[2])])


# ------------------------------------------------------------------------ C1 (stable: free-running parity)
def test_c1_init_state(golden):
    g = golden("c1.npz")
    st = init_state(problem_from(g))
    assert rel(st.xi, g["init_xi"]) < 1e-13
    np.testing.assert_allclose(st.alpha, g["init_alpha"], atol=1e-12)
    np.testing.assert_allclose(st.beta, g["init_beta"], atol=1e-12)
    assert np.all(st.d == 1.0) and np.all(st.lam_pos == 0.0)


def test_c1_fixed_100_iterations(golden):
    g = golden("c1.npz")
    sol = solve_single(problem_from(g), SingleParams(max_iter=100, tol=0.0))
    h = np.array([[x["norm"], x["max_abs"], x["rho_o"]] for x in sol.residual_history])
    ref = g["fixed_hist"]
    assert h.shape == ref.shape
    np.testing.assert_array_equal(h[:, 2], ref[:, 2])  # identical rho schedule
    np.testing.assert_allclose(h[:, :2], ref[:, :2], rtol=1e-9, atol=0)
    assert rel(sol.state.xi, g["fixed_xi"]) < 1e-10
    assert rel(sol.state.lam_pos, g["fixed_lam_pos"]) < 1e-8
    assert sol.n_factorizations == int(g["fixed_nfact"][0])


@pytest.mark.parametrize("layout", ["angle", "unit", "half"])
def test_c1_fixed_100_iterations_every_layout(golden, layout):
    """The bench's layouts on the stable C1 problem: the whole 100-iteration history within 1e-9 of the
    reference, identical rho schedule (the batched entry point, one member)."""
    from paper_2408_10731_b200.solver_single import SingleBatch, solve_single_batch

    g = golden("c1.npz")
    prob = problem_from(g)
    sol = solve_single_batch(SingleBatch.from_problems([prob]), SingleParams(max_iter=100, tol=0.0), history=True,
                             layout=layout)
    h = sol.history[0].cpu().numpy()
    ref = g["fixed_hist"]
    np.testing.assert_array_equal(h[:, 2], ref[:, 2])
    np.testing.assert_allclose(h[:, :2], ref[:, :2], rtol=1e-9, atol=0)
    assert rel(sol.xi[0].cpu().numpy(), g["fixed_xi"]) < 1e-10


def test_c1_converged_solve(golden):
    g = golden("c1.npz")
    sol = solve_single(problem_from(g), SingleParams())
    meta = g["conv_meta"]
    assert sol.converged and sol.iterations == int(meta[0]) == 261
    assert sol.n_factorizations == int(meta[2])
    h = np.array([[x["norm"], x["max_abs"], x["rho_o"]] for x in sol.residual_history])
    np.testing.assert_allclose(h[:, :2], g["conv_hist"][:, :2], rtol=1e-9)
    assert rel(sol.state.xi, g["conv_xi"]) < 1e-9
    assert abs(sol.smoothness_cost - meta[5]) <= 1e-9 * abs(meta[5])
    assert abs(sol.tracking_cost - meta[6]) <= 1e-9 * abs(meta[6])


def test_corridor2d_free_run(golden):
    g = golden("corridor2d.npz")
    sol = solve_single(problem_from(g), SingleParams(max_iter=200, tol=0.0))
    h = np.array([[x["norm"], x["max_abs"], x["rho_o"]] for x in sol.residual_history])
    np.testing.assert_array_equal(h[:, 2], g["hist"][:, 2])
    np.testing.assert_allclose(h[:, :2], g["hist"][:, :2], rtol=1e-9)
    assert rel(sol.state.xi, g["final_xi"]) < 1e-9


# ------------------------------------------------------------------------ teacher-forced (chaotic C2 members)
CASES = [(0, 0), (0, 1), (0, 60), (1, 10)]


@pytest.mark.parametrize("layout,tma", KERNELS)
@pytest.mark.parametrize("member,k", CASES)
def test_flow3d_teacher_forced_fp64(golden, member, k, layout, tma):
    g = golden("flow3d_tf.npz")
    gh = golden("flow3d_hist.npz")
    pre, nxt = f"m{member}_k{k}_", f"m{member}_k{k + 1}_"
    bvals, desired = g[f"m{member}_bvals"], g[f"m{member}_desired"]
    sc = g[pre + "scal"]
    eng = engine_from(g, bvals, desired, SingleParams(max_iter=200, tol=0.0), rho0=[sc[1]], max_hist=4,
                      layout=layout, use_tma=tma)
    load_snapshot(eng, g, pre, 3)
    eng.load_schedule([g[pre + "maxhist"]], [int(g[pre + "last_change"][0])])
    eng.prime(0 if k == 0 else 1)
    eng.iterate(0 if k == 0 else 1)
    torch.cuda.synchronize()
    assert rel(eng.xi[0].cpu().numpy(), g[nxt + "xi"]) < 1e-10
    for name, t in (("alpha", eng.alpha), ("beta", eng.beta), ("d", eng.d)):
        ref = g[nxt + name]
        np.testing.assert_allclose(t[0].cpu().numpy(), ref, atol=1e-9, err_msg=name)
    lam = eng.lam[:, 0].cpu().numpy()
    refs = [g[nxt + "lam_pos"][0], g[nxt + "lam_pos"][1], g[nxt + "lam_pos"][2], g[nxt + "lam_cos_a"],
            g[nxt + "lam_sin_a"], g[nxt + "lam_cos_b"], g[nxt + "lam_sin_b"]]
    for w, ref in enumerate(refs):
        assert np.max(np.abs(lam[w] - ref)) <= 1e-8 * max(1.0, np.abs(ref).max()), w
    hist_ref = gh["hist"][member][k]
    assert abs(eng.res_norm[0].item() - hist_ref[0]) <= 1e-9 * hist_ref[0]
    assert abs(eng.res_max[0].item() - hist_ref[1]) <= 1e-9 * hist_ref[1]
    assert eng.rho_o[0].item() == g[nxt + "scal"][1]  # identical penalty decision


@pytest.mark.parametrize("layout,tma", KERNELS)
@pytest.mark.parametrize("member,k", CASES)
def test_flow3d_teacher_forced_fp32(golden, member, k, layout, tma):
    """fp32 per-element storage and arithmetic; QP step and reductions in fp64."""
    g = golden("flow3d_tf.npz")
    gh = golden("flow3d_hist.npz")
    pre, nxt = f"m{member}_k{k}_", f"m{member}_k{k + 1}_"
    sc = g[pre + "scal"]
    eng = engine_from(g, g[f"m{member}_bvals"], g[f"m{member}_desired"], SingleParams(max_iter=200, tol=0.0),
                      dtype=torch.float32, rho0=[sc[1]], layout=layout, use_tma=tma)
    load_snapshot(eng, g, pre, 3)
    eng.prime(0 if k == 0 else 1)
    eng.iterate(0 if k == 0 else 1)
    torch.cuda.synchronize()
    pos_ref = g["P"] @ g[nxt + "xi"].T
    pos = g["P"] @ eng.xi[0].cpu().numpy().T
    assert rel(pos, pos_ref) < 1e-4
    assert rel(eng.xi[0].cpu().numpy(), g[nxt + "xi"]) < 1e-4
    # residuals compared absolutely, normalised by the iteration-0 residual
    r0 = gh["hist"][member][0][0]
    assert abs(eng.res_norm[0].item() - gh["hist"][member][k][0]) <= 1e-4 * r0


def test_flow3d_batch_free_window(golden):
    """8 C2 members batched: histories agree inside each member's LU-vs-K^-1 twin window."""
    gh = golden("flow3d_hist.npz")
    bs = basis_from(gh)
    batch = scenarios.flow3d_batch(50, gh["members"], basis=bs)
    sol = solve_single_batch(batch, SingleParams(max_iter=200, tol=0.0), history=True)
    hist = sol.history.cpu().numpy()
    report = []
    for i, tw in enumerate(gh["twin"]):
        # inside the window where the reference's own LU and K^-1 runs agree to 1e-9, with
        # margin for the ~10x/iteration amplification near its end
        err = np.max(np.abs(hist[i, :, :2] - gh["hist"][i][:, :2]) / np.abs(gh["hist"][i][:, :2]), axis=1)
        bad = np.nonzero(err > 1e-9)[0]
        first = int(bad[0]) if bad.size else 200
        report.append((i, int(tw), first))
        np.testing.assert_array_equal(hist[i, : int(tw) - 4, 2], gh["hist"][i][: int(tw) - 4, 2])
    print("member, twin window, device leaves 1e-9 at:", report)
    # The AM map amplifies rounding ~10x per iteration in clutter: the
    # device (different but equally exact rounding) must hold 1e-9 agreement for as long as
    # the reference's own LU-vs-K^-1 twin does, in distribution.
    firsts = np.array([f for _, _, f in report])
    twins = np.array([int(t) for _, t, _ in report])
    assert firsts.min() >= 8
    assert np.median(firsts) >= np.median(twins) - 3
    # end-state distribution (tier 3): final residual levels of the same order
    fin = hist[:, -1, 1]
    ref = gh["hist"][:, -1, 1]
    assert 0.2 < np.median(fin) / np.median(ref) < 5.0


@pytest.mark.parametrize("layout", ["angle", "unit", "half"])
def test_batch_layouts_agree_over_a_window(golden, layout):
    """The unit-vector layout (11 words) reproduces the angle layout's C2 histories (the AM
    map only sees cos/sin of the angles); chaos bounds the window like the twin test."""
    gh = golden("flow3d_hist.npz")
    bs = basis_from(gh)
    batch = scenarios.flow3d_batch(50, gh["members"], basis=bs)
    p = SingleParams(max_iter=200, tol=0.0)
    h = solve_single_batch(batch, p, history=True, layout=layout).history.cpu().numpy()
    for i in range(len(gh["members"])):
        np.testing.assert_allclose(h[i, :8, :2], gh["hist"][i][:8, :2], rtol=1e-9)
    fin, ref = h[:, -1, 1], gh["hist"][:, -1, 1]
    assert 0.2 < np.median(fin) / np.median(ref) < 5.0


def test_batch_members_equal_single_solves(golden):
    """A member's arithmetic does not depend on the batch it runs in (bitwise)."""
    bs = basis_from(golden("flow3d_hist.npz"))
    batch = scenarios.flow3d_batch(20, range(4), basis=bs)
    params = SingleParams(max_iter=40, tol=0.0)
    sol = solve_single_batch(batch, params)
    xi = sol.xi.cpu().numpy()
    for i in range(4):
        one = solve_single(batch.problem(i), params)
        np.testing.assert_array_equal(one.state.xi, xi[i])


@pytest.mark.parametrize("n_p,layout", [(100, "angle"), (100, "unit"), (100, "half"), (60, "angle"), (60, "unit"), (60, "half"),
                                        (37, "half"), (130, "half")])
def test_oracle_vs_device_step(golden, n_p, layout):
    """C5 shape (n_o 100) and a generic horizon (n_p 60, the non-specialised kernel): device one
    step == oracle one step from an oracle mid-run state."""
    from paper_2408_10731_b200.basis import build_basis

    bs = basis_from(golden("flow3d_hist.npz")) if n_p == 100 else build_basis(0.0, 10.0, n_p, 10)
    batch = scenarios.flow3d_batch(100, [5, 6], basis=bs)
    tracks = np.stack([o.centers for o in batch.obstacles])
    a = np.array([o.shape.a for o in batch.obstacles])
    b = np.array([o.shape.b for o in batch.obstacles])
    des = batch.desired_paths()
    prob = O.Problem(P=bs.P, Pd=bs.Pdot, Pdd=bs.Pddot, bvals=batch.bvals, desired=des, tracks=tracks, a=a, b=b)
    r = O.solve(prob, O.Params(max_iter=25, tol=0.0))
    st = r.state
    kkt = O.KKTCache(prob, mode="kinv")
    eng = Alg1Engine(bs, tracks, a, b, batch.bvals, batch.linear_terms(), params=SingleParams(max_iter=1, tol=0.0),
                     rho0=st.rho_o, export=True, keep_d=True, layout=layout)
    eng.load_state(xi=st.xi, alpha=st.alpha, beta=st.beta,
                   lam_planes=np.stack([st.lam_pos[:, 0], st.lam_pos[:, 1], st.lam_pos[:, 2], st.lam_cos_a,
                                        st.lam_sin_a, st.lam_cos_b, st.lam_sin_b]),
                   d=st.d, rho=st.rho, rho_o=st.rho_o, iteration=st.iteration)
    eng.prime(1)
    eng.iterate(1, flags=_lib.TRO_FLAG_NO_SCHEDULE)
    O.am_iteration(st, prob, kkt)
    torch.cuda.synchronize()
    assert rel(eng.xi.cpu().numpy(), st.xi) < 1e-10
    np.testing.assert_allclose(eng.alpha.cpu().numpy(), st.alpha, atol=1e-9)
    np.testing.assert_allclose(eng.beta.cpu().numpy(), st.beta, atol=1e-9)
    np.testing.assert_allclose(eng.d.cpu().numpy(), st.d, atol=1e-9)
    np.testing.assert_allclose(eng.lam[0].cpu().numpy(), st.lam_pos[:, 0], atol=1e-8 * np.abs(st.lam_pos).max())


def test_am_iteration_api_matches_oracle(golden):
    g = golden("c1.npz")
    prob = problem_from(g)
    st = init_state(prob)
    oprob = O.Problem(P=g["P"], Pd=g["Pd"], Pdd=g["Pdd"], bvals=g["bvals"], desired=g["desired"], tracks=g["tracks"],
                      a=g["a"], b=g["b"])
    ost = O.init_state(oprob)
    kkt = O.KKTCache(oprob)
    before = qpcore.factorization_count()
    for _ in range(3):
        am_iteration(st, prob)
        O.am_iteration(ost, oprob, kkt)
    assert qpcore.factorization_count() == before + 1
    assert st.iteration == 3 and st.n_factorizations == 1 and st._factor.size == 17
    assert rel(st.xi, ost.xi[0]) < 1e-11
    np.testing.assert_allclose(st.cos_a, ost.cos_a[0], atol=1e-10)
    np.testing.assert_allclose(st.d, ost.d[0], atol=1e-10)


def test_no_obstacles_one_iteration():
    from paper_2408_10731_b200.basis import build_basis

    basis = build_basis(0.0, 6.0, 60, 8)
    s = np.linspace(0, 1, 60)[:, None]
    prob = SingleProblem(basis, (AxisBoundary(p0=0.0, p1=8.0), AxisBoundary(p0=0.0, p1=0.0)),
                         np.hstack([8.0 * s, 0.0 * s]))
    sol = solve_single(prob, SingleParams(max_iter=5, tol=0.0))
    assert sol.converged and sol.iterations == 1 and sol.residual_max == 0.0
    pos = sol.trajectory.pos
    assert abs(pos[0, 0]) < 1e-8 and abs(pos[-1, 0] - 8.0) < 1e-8


def test_factorization_guard_raises(golden):
    g = golden("c1.npz")
    eng = engine_from(g, g["bvals"], g["desired"], SingleParams(max_iter=3, tol=0.0))
    eng.level_ok.zero_()
    eng.cold_init()
    eng.run(3, use_graph=False)
    assert int(eng.status[0].item()) & _lib.TRO_FACTOR_FAILED
    assert int(eng.iteration[0].item()) == 0


# ------------------------------------------------------------------------ qp-core and top-k
def test_qpcore_solve_batch_golden(golden):
    g = golden("qp.npz")
    for c in range(6):
        f = qpcore.factorize(g[f"c{c}_Q"], g[f"c{c}_A"])
        xis, nus = qpcore.solve_batch(f, qpcore.BatchRHS(qs=g[f"c{c}_qs"], bs=g[f"c{c}_bs"]))
        np.testing.assert_allclose(xis, g[f"c{c}_xis"], rtol=0, atol=1e-10 * np.abs(g[f"c{c}_xis"]).max())
        np.testing.assert_allclose(nus, g[f"c{c}_nus"], rtol=0, atol=1e-10 * np.abs(g[f"c{c}_nus"]).max())
        xi, nu = qpcore.solve(f, g[f"c{c}_qs"][3], g[f"c{c}_bs"][3])
        np.testing.assert_allclose(xi, g[f"c{c}_xis"][3], atol=1e-10 * np.abs(g[f"c{c}_xis"]).max())
    # device-resident path (torch in -> torch out)
    qs = torch.as_tensor(g["c0_qs"], device="cuda")
    bs_ = torch.as_tensor(g["c0_bs"], device="cuda")
    f = qpcore.factorize(g["c0_Q"], g["c0_A"])
    xis, _ = qpcore.solve_batch(f, qpcore.BatchRHS(qs=qs, bs=bs_))
    assert xis.is_cuda
    np.testing.assert_allclose(xis.cpu().numpy(), g["c0_xis"], atol=1e-10 * np.abs(g["c0_xis"]).max())


def test_kkt_apply_large_n():
    rng = np.random.default_rng(3)
    n_v, n_eq = 176, 96
    M = rng.normal(size=(n_v, n_v))
    Q = M @ M.T + n_v * np.eye(n_v)
    A = rng.normal(size=(n_eq, n_v))
    f = qpcore.factorize(Q, A)
    qs = rng.normal(size=(3, n_v))
    bs = rng.normal(size=(3, n_eq))
    xis, nus = qpcore.solve_batch(f, qpcore.BatchRHS(qs=qs, bs=bs))
    K = qpcore.saddle_matrix(Q, A)
    ref = np.linalg.solve(K, np.hstack([-qs, bs]).T).T
    np.testing.assert_allclose(xis, ref[:, :n_v], atol=1e-9 * np.abs(ref).max())


def _topk(keys, k):
    lib = _lib.load()
    dk = torch.as_tensor(keys, device="cuda", dtype=torch.float64)
    out = torch.full((max(k, 1),), -1, dtype=torch.int64, device="cuda")
    ws = torch.empty(max(lib.tro_topk_workspace_bytes(len(keys), k), 8), dtype=torch.uint8, device="cuda")
    rc = lib.tro_topk_stable_f64(dk.data_ptr(), len(keys), k, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                 _lib.stream_handle())
    _lib.check(rc, "topk")
    return out[:k].cpu().numpy()


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (1000, 1000), (4096, 4096), (4097, 4097), (16384, 8192),
                                 (16384, 256), (50000, 17), (20000, 1), (131072, 65536), (131072, 256),
                                 (131072, 131072), (262144, 5000)])
def test_topk_stable_bitexact(n, k):
    rng = np.random.default_rng(n + k)
    keys = np.round(rng.normal(size=n), 2)  # many exact ties
    if n > 10:
        keys[rng.integers(0, n, size=n // 10)] = np.nan
        keys[rng.integers(0, n, size=5)] = -0.0
        keys[rng.integers(0, n, size=5)] = 0.0
        keys[rng.integers(0, n, size=3)] = np.inf
        keys[rng.integers(0, n, size=3)] = -np.inf
    ref = np.argsort(keys, kind="stable")[:k]
    np.testing.assert_array_equal(_topk(keys, k), ref)


@pytest.mark.parametrize("n,k", [(10000, 5000), (10000, 1), (10000, 10000)])
def test_topk_all_ties_and_sorted_inputs(n, k):
    """Radix select edge cases: every key equal (all ties: index order), ascending and descending inputs."""
    for keys in (np.full(n, 0.25), np.arange(n, dtype=float), -np.arange(n, dtype=float),
                 np.repeat(np.array([3.0, -1.0, 2.0, -1.0]), n // 4)):
        np.testing.assert_array_equal(_topk(keys, k), np.argsort(keys, kind="stable")[:k])


def test_tail_split_matches_unsplit_batch(golden):
    """Tail balancing of the persistent kernel (B not a multiple of the grid: the last round's members run
    as two obstacle halves on two CTAs, combined in a fixed order) vs the same batch without it: equal up to
    the association of the obstacle sums (1e-10 over 20 iterations), identical schedules."""
    bs = basis_from(golden("flow3d_hist.npz"))
    slots = 2 * torch.cuda.get_device_properties(0).multi_processor_count
    B = slots + 5  # 5 tail members -> 10 half-units
    batch = scenarios.flow3d_batch(50, range(B), basis=bs)
    params = SingleParams(max_iter=20, tol=0.0)
    out = {}
    for split in (True, False):
        eng = Alg1Engine(bs, np.stack([o.centers for o in batch.obstacles]), [o.shape.a for o in batch.obstacles],
                         [o.shape.b for o in batch.obstacles], batch.bvals, batch.linear_terms(), params=params,
                         max_hist=20, layout="half", tail_split=split)
        eng.cold_init()
        eng.run(20, use_graph=False, loop=False)
        torch.cuda.synchronize()
        out[split] = (eng.hist.cpu().numpy(), eng.xi.cpu().numpy(), eng.rho_o.cpu().numpy())
    hs, xs, rs = out[True]
    hu, xu, ru = out[False]
    np.testing.assert_array_equal(hs[:, :, 2], hu[:, :, 2])
    np.testing.assert_array_equal(rs, ru)
    assert rel(hs[:, :, :2], hu[:, :, :2]) < 1e-10
    assert rel(xs, xu) < 1e-10
    np.testing.assert_array_equal(xs[:slots], xu[:slots])  # members of the full round: bitwise


def test_converged_members_leave_the_work_list(golden):
    """run() compacts the persistent kernel's work list to the members still iterating: a tol > 0 batch above
    the in-kernel-loop size gives the same results as the same batch run one launch per iteration without
    a work list (members converge at different iterations)."""
    from paper_2408_10731_b200 import _alg1

    bs = basis_from(golden("flow3d_hist.npz"))
    B = 200
    batch = scenarios.flow3d_batch(20, range(B), basis=bs)
    params = SingleParams(max_iter=150, tol=0.1)  # 77 of 200 members converge along the way
    res = {}
    for compact in (True, False):
        eng = Alg1Engine(bs, np.stack([o.centers for o in batch.obstacles]), [o.shape.a for o in batch.obstacles],
                         [o.shape.b for o in batch.obstacles], batch.bvals, batch.linear_terms(), params=params,
                         layout="half", tail_split=False)
        if not compact:
            eng._state.order = None
            eng._state.n_order = None
        eng.cold_init()
        eng.run(150, use_graph=compact, loop=False)
        torch.cuda.synchronize()
        res[compact] = (eng.xi.cpu().numpy(), eng.iteration.cpu().numpy(), eng.status.cpu().numpy())
        if compact:
            assert int(eng.n_order.item()) == B and np.array_equal(eng.order.cpu().numpy(), np.arange(B))
    (xa, ia, sa), (xb, ib, sb) = res[True], res[False]
    n_conv = int(((sa & _lib.TRO_CONVERGED) > 0).sum())
    assert 0 < n_conv < B, n_conv  # some members converged early, some did not
    np.testing.assert_array_equal(ia, ib)
    np.testing.assert_array_equal(sa, sb)
    np.testing.assert_array_equal(xa, xb)  # same kernel arithmetic per member, only the CTA assignment moved
    assert _alg1.LOOP_MAX_MEMBERS < B
