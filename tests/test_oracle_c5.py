"""Pin the oracle's Alg. 1 step in the C5 regime (n_o 100, rho_o up to the 1e3 cap, cond(K) ~1e11-1e12).

tests/golden/c5_tf.npz holds full reference states after iteration k (members of the C5 recipe at
k in {25, 100, 150, 199}) and, for the reference's state after k+1, xi, the penalties, the residual extremes
and a sha256 of every state array.  One oracle step from each snapshot must reproduce all of them bit for
bit: the GPU teacher-forced tests (tests/test_c5_parity_gpu.py) then compare the device with this oracle step.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import alg1 as O

C5_STATE = ("xi", "d", "alpha", "beta", "lam_pos", "lam_cos_a", "lam_sin_a", "lam_cos_b", "lam_sin_b")


def c5_cases():
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5_tf.npz"))
    return [(int(m[1:].split("_")[0]), int(k)) for m in g.files if m.endswith("_ks") for k in g[m]]


def c5_problem(g, member):
    return O.Problem(P=g["P"], Pd=g["Pd"], Pdd=g["Pdd"], bvals=g[f"m{member}_bvals"],
                     desired=g[f"m{member}_desired"], tracks=g["tracks"], a=g["a"], b=g["b"],
                     w_smooth=float(g["w"][0]), w_track=float(g["w"][1]))


def c5_state(g, pre):
    sc = g[pre + "scal"]
    one = lambda k: g[pre + k][None].copy()  # noqa: E731
    return O.State(xi=one("xi"), d=one("d"), alpha=one("alpha"), beta=one("beta"),
                   cos_a=np.cos(one("alpha")), sin_a=np.sin(one("alpha")), cos_b=np.cos(one("beta")),
                   sin_b=np.sin(one("beta")), lam_pos=one("lam_pos"), lam_cos_a=one("lam_cos_a"),
                   lam_sin_a=one("lam_sin_a"), lam_cos_b=one("lam_cos_b"), lam_sin_b=one("lam_sin_b"),
                   rho=np.array([sc[0]]), rho_o=np.array([sc[1]]), iteration=np.array([int(sc[2])]),
                   factor_rho_o=[sc[1]], n_factorizations=np.zeros(1, dtype=np.int64))


def oracle_step(g, member, k, mode="lu"):
    """The reference's loop body at iteration k+1 (solver_single.py:419-427) on the snapshot.
    mode "kinv": the position step applies the explicit K^-1 (the reference's LU-vs-K^-1 twin)."""
    pre = f"m{member}_k{k}_"
    prob = c5_problem(g, member)
    st = c5_state(g, pre)
    O.am_iteration(st, prob, O.KKTCache(prob, mode=mode))
    norm, mx = O.residual_extremes(st, prob)
    hist = list(g[pre + "maxhist"]) + [float(mx[0])]
    rho, rho_o, lc = O.maybe_grow(st.rho[0], st.rho_o[0], int(st.iteration[0]), O.Params(max_iter=200, tol=0.0),
                                  hist, int(g[pre + "last_change"][0]))
    return st, float(norm[0]), float(mx[0]), (rho, rho_o, lc)


@pytest.mark.parametrize("member,k", c5_cases())
def test_oracle_step_reproduces_the_reference_bitwise(golden, member, k):
    g = golden("c5_tf.npz")
    st, norm, mx, (rho, rho_o, lc) = oracle_step(g, member, k)
    nxt = f"m{member}_k{k}_next_"
    np.testing.assert_array_equal(st.xi[0], g[nxt + "xi"])
    assert (norm, mx) == tuple(g[nxt + "res"])
    assert (rho, rho_o, int(st.iteration[0]), lc) == tuple(g[nxt + "scal"])
    for name, sha in zip(C5_STATE, g[nxt + "sha"]):
        got = hashlib.sha256(np.ascontiguousarray(getattr(st, name)[0], dtype=np.float64).tobytes()).hexdigest()
        assert got == str(sha), name


def test_c5_snapshots_cover_the_cap(golden):
    g = golden("c5_tf.npz")
    rho_o = [g[f"m{m}_k{k}_scal"][1] for m, k in c5_cases()]
    assert max(rho_o) == 1000.0 and min(rho_o) < 2.0
