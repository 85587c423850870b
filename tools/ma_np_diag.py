"""Diagnostic: MA device vs oracle for a sample count that leaves a partial round (first iterations)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import multiagent as OM  # noqa: E402
from paper_2408_10731_b200 import scenarios  # noqa: E402
from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402
from paper_2408_10731_b200.basis import AxisBoundary, build_basis  # noqa: E402
from paper_2408_10731_b200.geometry import EllipsoidShape  # noqa: E402

n_p = int(sys.argv[1]) if len(sys.argv) > 1 else 37
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b = build_basis(0.0, 10.0, n_p, deg)
n_a = 6
starts, goals = scenarios.square_antipodal(n_a, 6.0, 0.4, seed=5)
bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3)) for i in range(n_a)]
prob = MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45))
params = MA.JointParams(max_iter=6, rho_final=1e3)
struct = MA._Structure(prob, params)
eng = MA.MaEngine(struct, MA._b_eq(prob)[None], None, params, max_hist=6, export=True)
eng.init()
torch.cuda.synchronize()
st = OM.make_structure(b.P, b.Pdot, b.Pddot, n_a, 0.3, 0.45, rho_final=1e3)
oprob = OM.Problem(b_eq=MA._b_eq(prob), statics=np.zeros((0, 3)))
ost = OM.init_state(st, oprob, b.P)
print("init xi diff", np.abs(eng.xi[0].cpu().numpy() - ost.xi).max())
kinv = [f.kinv for f in struct.factors]
for it in range(3):
    eng.iterate()
    torch.cuda.synchronize()
    ost = OM.iterate(ost, st, oprob, kinv=kinv) or ost
    xd = eng.xi[0].cpu().numpy()
    print(it, "xi diff", np.abs(xd - ost.xi).max(), "lam diff", np.abs(eng.lam_ref(0) - ost.lam).max(),
          "norm dev", float(eng.res_norm[0]))

# init sums: device B (which 0) vs the oracle's A_fo' recon
eng2 = MA.MaEngine(struct, MA._b_eq(prob)[None], None, params, max_hist=6, export=True)
eng2.init()
torch.cuda.synchronize()
ost = OM.init_state(st, oprob, b.P)
recon = OM.reconstruction(st, ost)  # (n_pairs, n_p, 3)
B = np.zeros((n_a, 3, struct.m))
for p in range(len(st.pair_i)):
    i, j = st.pair_i[p], st.pair_j[p]
    for k in range(3):
        v = b.P.T @ recon[p, :, k]
        B[i, k] += v
        if j >= 0:
            B[j, k] -= v
dev = eng2.sums[0, 0].cpu().numpy()
print("init B diff", np.abs(dev - B).max(), "scale", np.abs(B).max())
print("per-agent max diff", np.abs(dev - B).reshape(n_a, -1).max(axis=1))
d_dev, a_dev, b_dev = eng2.export_ref(0)
print("alpha diff", np.abs(a_dev - ost.alpha).max(), "beta diff", np.abs(b_dev - ost.beta).max(),
      "d diff", np.abs(d_dev - ost.d).max())
ad = np.abs(a_dev - ost.alpha)
print("alpha diff by t (max over pairs):", np.round(ad.max(axis=0), 3).tolist()[:50])
