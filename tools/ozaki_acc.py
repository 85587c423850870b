"""Accuracy of the two QP backends against a long-double reference at the C3 shape (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_ozaki_gpu import _c3  # noqa: E402

from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402

params = MA.JointParams(max_iter=200, rho_final=1e3)
n = 150
probs = _c3(n)
struct = MA._Structure(probs[0], params)
b_eq = np.stack([MA._b_eq(p) for p in probs])
d = MA.MaEngine(struct, b_eq, None, params, qp="dmma")
o = MA.MaEngine(struct, b_eq, None, params, qp="ozaki", ozaki_slices=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
for e in (d, o):
    e.reset()
    e.init()
    e.run(5, use_graph=False, check_every=0)
o.sums.copy_(d.sums)
lv = torch.arange(n, device=d.level.device, dtype=torch.int32) % len(struct.rho_levels)
for e in (d, o):
    e.level.copy_(lv)
    e.status.zero_()
d._call(3)
o.qp_ozaki()
torch.cuda.synchronize()
xd, xo = d.xi.cpu().numpy(), o.xi.cpu().numpy()
sums = d.sums.cpu().numpy()  # (B, 2, n_a, 3, m)
K = np.stack([f.kinv for f in struct.factors]).astype(np.longdouble)
nv = struct.n_a * struct.m
worst_d = worst_o = 0.0
for p in range(n):
    L = int(lv[p])
    for ax in range(3):
        Bv = sums[p, 0, :, ax, :].reshape(-1).astype(np.longdouble)
        Cv = sums[p, 1, :, ax, :].reshape(-1).astype(np.longdouble)
        r = np.concatenate([np.longdouble(struct.rho_levels[L]) * Bv - Cv, b_eq[p, ax].astype(np.longdouble)])
        # the device forms rho * B - C in fp64 first: use that rounding for both
        r64 = np.concatenate([struct.rho_levels[L] * sums[p, 0, :, ax, :].reshape(-1) - sums[p, 1, :, ax, :].reshape(-1),
                              b_eq[p, ax]]).astype(np.longdouble)
        truth = (K[L, :nv, :] @ r64).astype(np.float64)
        sc = np.abs(truth).max()
        worst_d = max(worst_d, np.abs(xd[p, ax] - truth).max() / sc)
        worst_o = max(worst_o, np.abs(xo[p, ax] - truth).max() / sc)
print({"dmma_vs_truth": worst_d, "ozaki_vs_truth": worst_o, "dmma_vs_ozaki":
       float((np.abs(xd - xo).max(axis=2) / np.abs(xd).max(axis=2)).max())})
