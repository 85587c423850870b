"""Small odd-shaped runs of the round-2 kernels (MA with statics on a 37-sample grid, 5 agents; validation on 41
samples): a quick crash / NaN check.  compute-sanitizer is closed on this GPU pool, so bounds are covered by the
odd-shape parity tests instead (tests/test_multiagent_gpu.py, tests/test_metrics_gpu.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import metrics as MT  # noqa: E402
from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402
from paper_2408_10731_b200.basis import AxisBoundary, BasisSet, TimeGrid, build_basis  # noqa: E402
from paper_2408_10731_b200.geometry import EllipsoidShape  # noqa: E402

b = build_basis(0.0, 10.0, 37, 10)
probs = []
for s in range(3):
    rng = np.random.default_rng(s)
    st, go = rng.uniform(-3, 3, (5, 3)), rng.uniform(-3, 3, (5, 3))
    probs.append(MA.MultiAgentProblem(basis=b, boundaries=[tuple(AxisBoundary(p0=float(st[i, k]), p1=float(go[i, k]))
                                                                 for k in range(3)) for i in range(5)],
                                      agent_shape=EllipsoidShape(0.3, 0.45),
                                      static_obstacles=[MA.StaticSphere(center=np.zeros(3), radius=0.4)]))
eng = MA.solve_joint_batch(probs, MA.JointParams(max_iter=6, rho_final=1e3), use_graph=False)
torch.cuda.synchronize()
print("ma ok", float(eng.res_norm.sum()))


class Obs:
    def __init__(self, a, b, c, v):
        self.a, self.b, self.center, self.velocity = a, b, c, v


class Scene:
    def __init__(self, dim, obs):
        self.dim, self.obstacles = dim, obs


rng = np.random.default_rng(1)
t = np.linspace(0, 10, 41)
P = rng.normal(size=(41, 11))
basis = BasisSet(grid=TimeGrid(0.0, 10.0, 41, t), degree=10, P=P, Pdot=np.zeros_like(P), Pddot=P.copy())
sc = Scene(3, [Obs(0.5, 0.4, list(rng.uniform(-2, 2, 3)), list(rng.uniform(-0.2, 0.2, 3))) for _ in range(7)])
r = MT.validate_batch(sc, t, xi=rng.normal(size=(9, 3, 11)), basis=basis, desired=rng.normal(size=(41, 3)))
print("val ok", float(np.sum(r["smoothness"])))
