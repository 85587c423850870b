"""Where does criterion 5's residual noise floor come from? Device state vs host (oracle) residual."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import batch2d as OB  # noqa: E402
from paper_2408_10731_b200 import solver_batch as SB  # noqa: E402
from paper_2408_10731_b200.basis import build_basis  # noqa: E402
from paper_2408_10731_b200.bench import gen_scenario  # noqa: E402
from paper_2408_10731_b200.bench.adapters import batch_problem_from_scenario  # noqa: E402
from test_batch2d_gpu import _oracle_state, _oracle_struct  # noqa: E402

sc = gen_scenario("random-static", {"n_o": 10}, seed=0)
basis = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
prob = batch_problem_from_scenario(sc, basis, n_batch=100)
samples = SB._default_samples(prob, basis.n_var, None, None, 0)
for it in (1, 5, 100):
    r = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=it), samples=samples)
    st = _oracle_struct(prob)
    res = r.state.xi @ st.F.T - OB.build_g(st, _oracle_state(r.state))
    hn = np.linalg.norm(res, axis=1)
    k = int(np.argmin(r.residual_norm))
    print(it, "device best norm", r.residual_norm[k], "host norm of device state", hn[k], "min host", hn.min(),
          "hist", r.best_history[-1]["norm"])
    out = OB.solve(st, samples, 1, max_iter=it)
    print("   oracle best hist", out["best_hist"][-1, 0])
    # residual split by row block: collision, velocity, acceleration
    nF = st.F.shape[0]
    print("   host |res| by block (x-part first):", [float(np.abs(res[k, s]).max()) for s in
                                                    np.array_split(np.arange(res.shape[1]), 6)])
