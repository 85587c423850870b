"""Pin the multi-agent oracle (oracle/multiagent.py) against golden vectors of the live reference."""

import numpy as np

from oracle import multiagent as OM
from paper_2408_10731_b200 import scenarios


def r6(g):
    st = OM.make_structure(g["P"], g["Pd"], g["Pdd"], 6, 0.3, 0.45, n_static=1, static_radii=[0.6], rho_final=1e3)
    bv = g["r6_bvals"]  # (n_a, 3, 6)
    b_eq = np.stack([np.concatenate([bv[i, k] for i in range(6)]) for k in range(3)])
    return st, OM.Problem(b_eq=b_eq, statics=g["r6_static"][:, :3])


def test_random_roster_free_run_bitexact(golden):
    g = golden("multiagent.npz")
    st, prob = r6(g)
    state, hist, conv = OM.solve(st, prob, g["P"], max_iter=60)
    np.testing.assert_array_equal(hist, g["r6_hist"])
    np.testing.assert_array_equal(state.xi, g["r6_xi"])
    assert conv and state.iteration == int(g["r6_meta"][0])


def test_teacher_forced_steps_bitexact(golden):
    g = golden("multiagent.npz")
    st, prob = r6(g)
    for k in (0, 12):
        lv, it = g[f"r6_k{k}_meta"]
        s = OM.State(xi=g[f"r6_k{k}_xi"].copy(), d=g[f"r6_k{k}_d"].copy(), alpha=g[f"r6_k{k}_alpha"].copy(),
                     beta=g[f"r6_k{k}_beta"].copy(), lam=g[f"r6_k{k}_lam"].copy(), level=int(lv), iteration=int(it))
        OM.iterate(s, st, prob)
        for name in ("xi", "d", "lam", "alpha", "beta"):
            np.testing.assert_array_equal(getattr(s, name), g[f"r6_k{k + 1}_{name}"], err_msg=name)


def test_c3_recipe_window_bitexact(golden):
    g = golden("multiagent.npz")
    st = OM.make_structure(g["P"], g["Pd"], g["Pdd"], 16, 0.3, 0.45, rho_final=1e3)
    bv = g["a16_bvals"]
    b_eq = np.stack([np.concatenate([bv[i, k] for i in range(16)]) for k in range(3)])
    prob = OM.Problem(b_eq=b_eq, statics=np.zeros((0, 3)))
    state0 = OM.init_state(st, prob, g["P"])
    np.testing.assert_array_equal(state0.alpha, g["a16_init_alpha"])
    state, hist, _ = OM.solve(st, prob, g["P"], max_iter=25)
    np.testing.assert_array_equal(hist, g["a16_hist"])


def test_square_antipodal_roster_matches_reference(golden):
    g = golden("multiagent.npz")
    starts, goals = scenarios.square_antipodal(16, 8.0, 0.3, seed=0)
    bv = g["a16_bvals"]
    np.testing.assert_array_equal(bv[:, :, 0], starts)
    np.testing.assert_array_equal(bv[:, :, 3], goals)
