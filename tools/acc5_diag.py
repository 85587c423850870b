"""Acceptance criterion 5 on the device vs the reference's best-member histories (tests/golden/acceptance5.npz)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import solver_batch  # noqa: E402
from paper_2408_10731_b200.basis import build_basis  # noqa: E402
from paper_2408_10731_b200.bench import gen_scenario  # noqa: E402
from paper_2408_10731_b200.bench.adapters import batch_problem_from_scenario  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "acceptance5.npz"))
for seed in range(10):
    sc = gen_scenario("random-static", {"n_o": 10}, seed=seed)
    basis = build_basis(sc.horizon.t0, sc.horizon.tf, sc.horizon.n_p, 10)
    r = solver_batch.solve_batch_opt(batch_problem_from_scenario(sc, basis, n_batch=100),
                                     solver_batch.BatchParams(max_iter=100), seed=seed)
    norms = np.array([h["norm"] for h in r.best_history])
    ref = g[f"s{seed}_norm"]
    w, burn = 5, 20
    win = np.array([norms[k:k + w].mean() for k in range(burn, len(norms) - w)])
    d = np.diff(win) - (win[:-1] * 1e-6 + 1e-12)
    rel = np.abs(norms - ref) / np.abs(ref)
    first = int(np.argmax(rel > 1e-9)) if np.any(rel > 1e-9) else -1
    if seed == 0:
        print("ours", norms[:5], norms[20:25], norms[-5:])
    print(seed, "best", r.best_index, int(g[f"s{seed}_best"][0]), "trend", bool(np.all(d <= 0)), "worst", float(d.max()),
          "max rel", float(rel.max()), "first>1e-9 at", first, "len", len(norms), len(ref))
