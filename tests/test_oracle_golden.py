"""Pin the CPU oracle (oracle/alg1.py) against golden vectors of the live reference.

The fixtures in tests/golden were produced by tests/golden/make_golden.py from
the unmodified reference package; the oracle must reproduce them before any
device result is checked against it.
"""

import numpy as np
import pytest

from oracle import alg1 as O


def problem_from(g, member_key=None):
    bvals = g["bvals"] if member_key is None else g[f"{member_key}_bvals"]
    desired = g["desired"] if member_key is None else g[f"{member_key}_desired"]
    return O.Problem(P=g["P"], Pd=g["Pd"], Pdd=g["Pdd"], bvals=bvals, desired=desired, tracks=g["tracks"],
                     a=g["a"], b=g["b"], w_smooth=float(g["w"][0]), w_track=float(g["w"][1]))


def state_from(g, prefix, dim):
    sc = g[prefix + "scal"]
    beta = g.get(prefix + "beta")
    st = O.State(
        xi=g[prefix + "xi"][None].copy(), d=g[prefix + "d"][None].copy(), alpha=g[prefix + "alpha"][None].copy(),
        beta=None if beta is None else beta[None].copy(),
        cos_a=g[prefix + "cos_a"][None].copy(), sin_a=g[prefix + "sin_a"][None].copy(),
        cos_b=None if dim == 2 else g[prefix + "cos_b"][None].copy(),
        sin_b=None if dim == 2 else g[prefix + "sin_b"][None].copy(),
        lam_pos=g[prefix + "lam_pos"][None].copy(), lam_cos_a=g[prefix + "lam_cos_a"][None].copy(),
        lam_sin_a=g[prefix + "lam_sin_a"][None].copy(),
        lam_cos_b=None if dim == 2 else g[prefix + "lam_cos_b"][None].copy(),
        lam_sin_b=None if dim == 2 else g[prefix + "lam_sin_b"][None].copy(),
        rho=np.array([sc[0]]), rho_o=np.array([sc[1]]), iteration=np.array([int(sc[2])]),
        factor_rho_o=[sc[1]], n_factorizations=np.zeros(1, dtype=np.int64))
    return st


def test_c1_init_state_bitexact(golden):
    g = golden("c1.npz")
    st = O.init_state(problem_from(g))
    np.testing.assert_array_equal(st.xi[0], g["init_xi"])
    np.testing.assert_array_equal(st.alpha[0], g["init_alpha"])
    np.testing.assert_array_equal(st.beta[0], g["init_beta"])


def test_c1_fixed_run_bitexact(golden):
    g = golden("c1.npz")
    r = O.solve(problem_from(g), O.Params(max_iter=100, tol=0.0))
    h = np.array([r.norm_hist[0], r.max_hist[0], r.rho_hist[0]]).T
    np.testing.assert_array_equal(h, g["fixed_hist"])
    np.testing.assert_array_equal(r.state.xi[0], g["fixed_xi"])
    np.testing.assert_array_equal(r.state.lam_pos[0], g["fixed_lam_pos"])


def test_c1_converged_run(golden):
    g = golden("c1.npz")
    r = O.solve(problem_from(g), O.Params())
    meta = g["conv_meta"]
    assert int(r.iterations[0]) == int(meta[0]) == 261
    assert bool(r.converged[0])
    assert int(r.state.n_factorizations[0]) == int(meta[2])
    np.testing.assert_array_equal(r.state.xi[0], g["conv_xi"])


def test_corridor2d_free_run(golden):
    g = golden("corridor2d.npz")
    r = O.solve(problem_from(g), O.Params(max_iter=200, tol=0.0))
    h = np.array([r.norm_hist[0], r.max_hist[0], r.rho_hist[0]]).T
    np.testing.assert_allclose(h, g["hist"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("member,k", [(0, 0), (0, 1), (0, 60), (1, 10)])
def test_flow3d_teacher_forced_step(golden, member, k):
    g = golden("flow3d_tf.npz")
    prob = problem_from(g, f"m{member}")
    st = state_from(g, f"m{member}_k{k}_", 3)
    kkt = O.KKTCache(prob)
    O.am_iteration(st, prob, kkt)
    pre = f"m{member}_k{k + 1}_"
    np.testing.assert_allclose(st.xi[0], g[pre + "xi"], rtol=0, atol=1e-12 * np.abs(g[pre + "xi"]).max())
    for name in ("alpha", "beta", "d", "lam_pos", "lam_cos_a", "lam_sin_a", "lam_cos_b", "lam_sin_b"):
        ref = g[pre + name]
        got = getattr(st, name)[0]
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-10 * max(1.0, np.abs(ref).max()), err_msg=name)


def test_flow3d_free_window(golden):
    """Oracle (LU, like the reference) reproduces the 200-iteration histories of 8 members."""
    g = golden("flow3d_hist.npz")
    members = g["members"]
    B = len(members)
    bvals = np.zeros((B, 3, 6))
    bvals[:, :, 0] = g["starts"]
    bvals[:, :, 3] = g["goals"]
    s = np.linspace(0.0, 1.0, g["P"].shape[0])
    desired = g["starts"][:, None, :] + s[None, :, None] * (g["goals"] - g["starts"])[:, None, :]
    prob = O.Problem(P=g["P"], Pd=g["Pd"], Pdd=g["Pdd"], bvals=bvals, desired=desired, tracks=g["tracks"],
                     a=g["a"], b=g["b"])
    r = O.solve(prob, O.Params(max_iter=200, tol=0.0))
    for i in range(B):
        h = np.array([r.norm_hist[i], r.max_hist[i], r.rho_hist[i]]).T
        np.testing.assert_allclose(h, g["hist"][i], rtol=1e-12, atol=0)


def test_qp_golden(golden):
    g = golden("qp.npz")
    for c in range(6):
        Q, A = g[f"c{c}_Q"], g[f"c{c}_A"]
        K = np.block([[Q, A.T], [A, np.zeros((A.shape[0], A.shape[0]))]])
        rhs = np.hstack([-g[f"c{c}_qs"], g[f"c{c}_bs"]])
        sol = np.linalg.solve(K, rhs.T).T
        np.testing.assert_allclose(sol[:, : Q.shape[0]], g[f"c{c}_xis"], atol=1e-9)


def test_rho_levels_match_repeated_products():
    lv = O.rho_levels(O.Params())
    assert len(lv) == 22
    assert lv[2] == 1.9599999999999997 and lv[-1] == 1000.0 and lv[-2] == 836.682554252847
