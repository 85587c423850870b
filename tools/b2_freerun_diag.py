import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_batch2d_gpu as T
from paper_2408_10731_b200 import solver_batch as SB
g = dict(np.load("tests/golden/batch2d.npz"))
for tag in ("t50", "f10"):
    make, iters, _ = T.PROBLEMS[tag]
    prob = make(g)
    r = SB.solve_batch_opt(prob, SB.BatchParams(max_iter=iters), samples=g[f"{tag}_samples"])
    h = np.array([[x["norm"], x["max_abs"], x["rho"]] for x in r.best_history])
    ref = g[f"{tag}_hist"]
    print(tag, "hist rel err per col", [float(np.max(np.abs(h[:, c] - ref[:, c]) / np.abs(ref[:, c]))) for c in range(3)])
    for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
        print("  ", name, T.rel(getattr(r.state, name), g[f"{tag}_final_{name}"]))
    rank = g[f"{tag}_rank"]
    print("   rmax", T.rel(r.residual_max, rank[:, 0]), "rnorm", T.rel(r.residual_norm, rank[:, 1]), "cost", T.rel(r.costs, rank[:, 2]),
          "feasible eq", np.array_equal(r.feasible, rank[:, 4] > 0), "best", r.best_index, g[f"{tag}_meta"])
