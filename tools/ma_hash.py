"""C3 multi-agent engine: ms per iteration and a hash of the state after a fixed run (A/B of kernel variants:
TRO_LIB_PATH selects the library)."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
probs = bench.c3_problems(0, n)
params = MA.JointParams(max_iter=200, rho_final=1e3, tol_norm=0.0)
struct = MA._Structure(probs[0], params)
eng = MA.MaEngine(struct, np.stack([MA._b_eq(p) for p in probs]), None, params, max_hist=200)
eng.init()
for _ in range(5):
    eng.iterate()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for rep in range(3):
    e0.record()
    for _ in range(10):
        eng.iterate()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 10)
h = hashlib.sha1()
for t in (eng.xi, eng.state, eng.sums, eng.res_norm, eng.res_max, eng.level):
    h.update(t.cpu().numpy().tobytes())
print(json.dumps({"lib": os.environ.get("TRO_LIB_PATH", "default"), "problems": n, "ms_per_iter": round(best, 4),
                  "problem_it_per_s": round(n / best * 1e3), "hash": h.hexdigest()}))
