"""Time / profile the joint multi-agent kernel (C3 shape) with CUDA events."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--problems", type=int, default=1024)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
probs = bench.c3_problems(0, a.problems)
params = MA.JointParams(max_iter=200, rho_final=1e3, tol_norm=0.0)
struct = MA._Structure(probs[0], params)
eng = MA.MaEngine(struct, np.stack([MA._b_eq(p) for p in probs]), None, params)
eng.init()
for _ in range(5):
    eng.iterate()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    eng.iterate()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
gb = 2 * 3 * 120 * 100 * 8 * a.problems / 1e9
print(json.dumps({"problems": a.problems, "ms_per_iter": ms, "GBps_alg": gb / (ms / 1e3)}))
