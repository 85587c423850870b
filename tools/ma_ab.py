import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2408_10731_b200 import solver_multiagent as MA
probs = bench.c3_problems(0, 4096)
params = MA.JointParams(max_iter=200, rho_final=1e3, tol_norm=0.0)
struct = MA._Structure(probs[0], params)
beq = np.stack([MA._b_eq(p) for p in probs])
res = {}
for split in (False, True):
    eng = MA.MaEngine(struct, beq, None, params, split_qp=split)
    eng.init()
    for _ in range(5): eng.iterate()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): eng.iterate()
    e1.record(); torch.cuda.synchronize()
    res[split] = (e0.elapsed_time(e1) / 10, eng.xi.clone())
    print("split", split, "ms/iter", res[split][0])
d = (res[True][1] - res[False][1]).abs().max().item() / res[False][1].abs().max().item()
print("xi rel diff after 15 its", d)
